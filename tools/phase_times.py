"""Per-phase cycle counts of k_tc_factor (one row per CTA, via ials_debug_timestamps)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2110_14044_b200 import _lib
from paper_2110_14044_b200.engine import DeviceProblem, Engine
lib = _lib.load()
lib.ials_set_tensor_cores(1)
shape, d, b, _ = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "L1"]
ds = bench.dataset(shape)
U, I, S = int(ds["U"]), int(ds["I"]), int(ds["user_ptr"][-1])
dev = torch.device("cuda", 0)
prob = DeviceProblem(dev, U, I, ds["user_ptr"], ds["user_cols"], ds["item_ptr"], ds["item_cols"], ds["item_pos"])
prob.set_regularizer(0.1, 1e-3, 1.0)
eng = Engine(prob)
W = (torch.randn(U, d, device=dev) * (0.1 / d ** 0.5)).contiguous()
H = (torch.randn(I, d, device=dev) * (0.1 / d ** 0.5)).contiguous()
cache = torch.zeros(S, device=dev)
eng.predictions(W, H, cache)
slab = torch.empty(d, b, device=dev)
dbg = torch.zeros(16 * 1024, dtype=torch.int64, device=dev)
lib.ials_debug_timestamps(ctypes.c_void_p(dbg.data_ptr()))
eng.partial_gramian(H, 0, b, slab)
eng.side_pass("user", H, W, 0, b, slab, 0.1, cache)
torch.cuda.synchronize()
t = dbg.view(-1, 8)[:592].cpu().numpy().astype(np.float64)
t = t[t[:, 0] > 0]
order = [0, 5, 6, 7, 1, 2, 3, 4]
tt = t[:, order]
dif = np.diff(tt, axis=1)
print("rows sampled", len(t))
for name, col in zip(["start->batch0", "batch0", "batch1+wait", "grad+sync", "factor", "backward", "update+sync"], dif.T):
    print(f"{name:14s} median {np.median(col):9.0f}  p90 {np.percentile(col, 90):9.0f} cycles")

h = dbg[8 * 1024:].view(-1, 4)[:444].cpu().numpy().astype(np.float64)
h = h[h[:, 2] > 0]
print("hess slices sampled", len(h), "median entries", np.median(h[:, 2]))
print(f"hess accumulate median {np.median(h[:, 0]):9.0f} p90 {np.percentile(h[:, 0], 90):9.0f}; write {np.median(h[:, 1]):7.0f}")
print("cycles per entry (accumulate)", np.median(h[:, 0] / h[:, 2]))
