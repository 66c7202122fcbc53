"""Device CSR build (ials_build_csr) vs the host build the reference does
(InteractionDataset.__init__ + item_view, NumPy stable argsorts) on the
synthetic configs[1] / configs[4] shapes.  Prints one JSON line per shape:
device milliseconds (CUDA events, inputs resident, median of 10), the same
with the COO upload (pinned host -> device) inside the timed region, host
seconds, and the bit-exactness check."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2110_14044_b200 as ials
from paper_2110_14044_b200 import synthetic
from paper_2110_14044_b200.csr import build_csr_device

for shape in (sys.argv[1:] or ["mid", "msd"]):
    U, I, users, items = synthetic.generate(shape, 0)
    t0 = time.perf_counter()
    ref = ials.InteractionDataset(U, I, users, items)
    iv = ref.item_view()
    host_s = time.perf_counter() - t0
    dev = torch.device("cuda", 0)
    u_d = torch.from_numpy(users.astype(np.int32)).to(dev)
    i_d = torch.from_numpy(items.astype(np.int32)).to(dev)
    u_h = torch.from_numpy(users.astype(np.int32)).pin_memory()
    i_h = torch.from_numpy(items.astype(np.int32)).pin_memory()
    for _ in range(3):
        got = build_csr_device(U, I, u_d, i_d)
    torch.cuda.synchronize()
    ts, te = [], []
    for _ in range(10):
        a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); got = build_csr_device(U, I, u_d, i_d); z.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(z))
        a.record()
        got = build_csr_device(U, I, u_h.to(dev, non_blocking=True), i_h.to(dev, non_blocking=True))
        z.record(); torch.cuda.synchronize()
        te.append(a.elapsed_time(z))
    exact = (np.array_equal(got.user_ptr.cpu().numpy(), ref.user_ptr)
             and np.array_equal(got.user_cols.cpu().numpy(), ref.items)
             and np.array_equal(got.item_ptr.cpu().numpy(), ref.item_ptr)
             and np.array_equal(got.item_pos.cpu().numpy(), iv.cache_pos)
             and np.array_equal(got.item_cols.cpu().numpy(), iv.cols))
    print(json.dumps({"shape": shape, "users": U, "items": I, "nnz": int(users.size),
                      "device_ms": round(float(np.median(ts)), 3),
                      "device_ms_with_upload": round(float(np.median(te)), 3),
                      "host_reference_s": round(host_s, 3),
                      "speedup_vs_host": round(host_s * 1e3 / float(np.median(ts)), 1),
                      "bit_exact": bool(exact),
                      "note": "device_ms includes the host-side range check (torch.aminmax + .item())"}))
