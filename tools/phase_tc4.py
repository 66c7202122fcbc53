"""Per-phase cycle counts of k_sweep_tc4 (2nd row of every CTA, via ials_debug_timestamps)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2110_14044_b200 import _lib
from paper_2110_14044_b200.engine import DeviceProblem, Engine
lib = _lib.load()
lib.ials_set_tensor_cores(2)
shape, d, b, _ = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "L1"]
targets = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1, 100]
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
dbg = torch.zeros(32 * 1024, dtype=torch.int64, device=dev)
for side, fixed, own, tgt in [(sd, f, o, t) for (sd, f, o) in (("user", H, W), ("item", W, H))
                              for t in targets]:
    dbg.zero_()
    dbg[32767] = tgt
    lib.ials_debug_timestamps(ctypes.c_void_p(dbg.data_ptr()))
    eng.partial_gramian(fixed, 0, b, slab)
    eng.side_pass(side, fixed, own, 0, b, slab, 0.1, cache)
    torch.cuda.synchronize()
    lib.ials_debug_timestamps(None)
    t = dbg.view(-1, 8)[:592].cpu().numpy().astype(np.float64)
    t = t[t[:, 0] > 0]
    if len(t) == 0:
        print(f"{side} (row #{tgt}): no CTA has that many rows")
        continue
    dif = np.diff(t[:, :7], axis=1)
    n = t[:, 7]
    print(f"{side} (row #{tgt} of each CTA): rows sampled {len(t)}, median entries {np.median(n):.0f}")
    for name, col in zip(["init", "accumulate", "diag+grad", "factor", "copy+backward", "update+cache"], dif.T):
        print(f"  {name:14s} median {np.median(col):9.0f}  p90 {np.percentile(col, 90):9.0f} cycles")
    print(f"  accumulate cycles/entry median {np.median(dif[:, 1] / np.maximum(n, 1)):.1f}")
    a = dbg[16384:16384 + 592 * 16].view(-1, 2, 8).cpu().numpy().astype(np.float64)
    a = a[a[:, 0, 0] > 0]
    if len(a):
        # 0 before cp.async wait, 1 after wait, 2 after barrier, 3 after gradient,
        # 4 after MMA(c-2) wait + operand writes, 5 after barrier + MMA issue, 6 after next gathers
        base = a[:, 0, 0:1]
        print("  accumulate chunk 3 timeline (cycles after thread 0 reached the cp.async wait):")
        for w, wn in enumerate(["thread 0 (MMA issuer)", "thread 64"]):
            t = np.median(a[:, w, :7] - base, axis=0)
            print(f"    {wn:24s} " + "  ".join(f"{int(x):6d}" for x in t))
    f = dbg[8192:8192 + 592 * 24].view(-1, 3, 8).cpu().numpy().astype(np.float64)
    f = f[f[:, 0, 6] > 0]
    if len(f):
        # probes: 6 after ld8, 1 after S2 (block factored), 3 after trsm, 4 after S3, 5 after MMA wait
        order = [6, 1, 3, 4, 5]
        base = f[:, 0, 6:7]
        print("  panel 8 timeline (cycles after thread 0 finished ld8), median over CTAs:")
        for w, wn in enumerate(["thread 0 (rows<c0)", "thread 64 (diag warp)", "thread 96 (trailing)"]):
            t = np.median(f[:, w, order] - base, axis=0)
            print(f"    {wn:24s} " + "  ".join(f"{int(x):6d}" for x in t))
