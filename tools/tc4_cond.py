"""Accuracy / redo-rate scan of the fused tensor-core sweep (mode 2) over the
cancellation limit: stress instances vs the f64 oracle, and the full-size
L1 workload's redo fraction.  usage: python tools/tc4_cond.py [--l1]"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2110_14044_b200 as ials  # noqa: E402
from paper_2110_14044_b200 import _lib  # noqa: E402
from paper_2110_14044_b200._runtime import default_engine_session  # noqa: E402
from oracle import ialspp_oracle as orc  # noqa: E402
from conftest import relf, relmax  # noqa: E402
from test_gpu_parity import _heavy_instance  # noqa: E402

lib = _lib.load()
rt = default_engine_session()
CONDS = [1e9, 4096, 1024, 256, 64, 16]

for (d, b, I) in [(128, 128, 60), (128, 128, 600), (128, 96, 60)]:
    U, I, users, items = _heavy_instance(9000, I, 12, 1.2, 3)
    data = ials.InteractionDataset(U, I, users, items)
    cfg = ials.SolverConfig(dim=d, block_size=b, unobserved_weight=0.1, reg=1e-3,
                            reg_exponent=1.0, epochs=1, seed=1)
    init = ials.init_model(cfg, U, I)
    init.user_factors[:] = init.user_factors.astype(np.float32)
    init.item_factors[:] = init.item_factors.astype(np.float32)
    w, h = init.user_factors.copy(), init.item_factors.copy()
    orc.train(w, h, orc.build_csr(U, I, users, items), 0.1, 1e-3, 1.0, b, 1)
    rows = U + I
    for mode, conds in ((0, [None]), (1, [None]), (2, CONDS)):
        for c in conds:
            lib.ials_set_tensor_cores(mode)
            if c is not None:
                lib.ials_set_tc_cond_max(c)
            m = init.copy()
            rt.session.tc_redo_rows(reset=True)
            ials.train(m, data, cfg)
            redo = rt.session.tc_redo_rows()
            print(f"d{d} b{b} I{I} mode {mode} cond {c}: relf U {relf(m.user_factors, w):.2e} "
                  f"I {relf(m.item_factors, h):.2e} relmax I {relmax(m.item_factors, h):.2e} "
                  f"redo {redo}/{rows * (d // b)}", flush=True)
lib.ials_set_tensor_cores(0)

if "--l1" in sys.argv:
    import torch
    import bench
    from paper_2110_14044_b200.engine import DeviceProblem, Engine
    from paper_2110_14044_b200.model import SolverConfig, init_model
    shape, d, b, _ = bench.CONFIGS["L1"]
    ds = bench.dataset(shape)
    U, I = int(ds["U"]), int(ds["I"])
    dev = torch.device("cuda", 0)
    prob = DeviceProblem(dev, U, I, ds["user_ptr"], ds["user_cols"], ds["item_ptr"],
                         ds["item_cols"], ds["item_pos"])
    prob.set_regularizer(bench.ALPHA0, bench.REG, bench.NU)
    eng = Engine(prob)
    cfg = SolverConfig(dim=d, block_size=b, unobserved_weight=bench.ALPHA0, reg=bench.REG,
                       reg_exponent=bench.NU, init_stddev=bench.SIGMA, seed=0)
    m = init_model(cfg, U, I)
    W0 = torch.from_numpy(m.user_factors.astype(np.float32)).to(dev)
    H0 = torch.from_numpy(m.item_factors.astype(np.float32)).to(dev)
    cache = torch.zeros(int(ds["user_ptr"][-1]), dtype=torch.float32, device=dev)
    rows = (U + I) * (d // b)
    print("L1 redo rows per epoch (mode 2):", flush=True)
    for c in (4096, 1024, 256, 64):
        lib.ials_set_tensor_cores(2)
        lib.ials_set_tc_cond_max(c)
        W, H = W0.clone(), H0.clone()
        out = []
        for e in range(6):
            eng.sess.tc_redo_rows(reset=True)
            eng.epoch(W, H, cache, b, bench.ALPHA0)
            out.append(eng.sess.tc_redo_rows())
        loss = eng.loss(W, H, bench.ALPHA0) if hasattr(eng, "loss") else None
        print(f"  cond {c}: redo/epoch {out} of {rows} row-updates; loss {loss}", flush=True)
    lib.ials_set_tensor_cores(0)
