"""Run a few side passes of one bench config (for ncu / nsight-free profiling).

    python tools/profile_pass.py --config L1 [--passes 2]
Warm-up: one epoch through the C ABI; then `passes` x (slab H, user pass,
slab W, item pass) of block 0, each bracketed by CUDA events (printed)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import bench
from paper_2110_14044_b200.engine import DeviceProblem, Engine

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="L1")
ap.add_argument("--passes", type=int, default=1)
ap.add_argument("--no-warm-epoch", action="store_true")
a = ap.parse_args()
shape, d, b, _ = bench.CONFIGS[a.config]
ds = bench.dataset(shape)
U, I, S = int(ds["U"]), int(ds["I"]), int(ds["user_ptr"][-1])
dev = torch.device("cuda", 0)
prob = DeviceProblem(dev, U, I, ds["user_ptr"], ds["user_cols"], ds["item_ptr"], ds["item_cols"],
                     ds["item_pos"])
prob.set_regularizer(0.1, 1e-3, 1.0)
eng = Engine(prob)
g = torch.Generator(device=dev).manual_seed(0)
W = (torch.randn(U, d, device=dev, generator=g) * (0.1 / d ** 0.5)).contiguous()
H = (torch.randn(I, d, device=dev, generator=g) * (0.1 / d ** 0.5)).contiguous()
cache = torch.zeros(S, device=dev)
if not a.no_warm_epoch:
    eng.epoch(W, H, cache, b, 0.1)
slab = torch.empty(d, b, device=dev)
eng.predictions(W, H, cache)
torch.cuda.synchronize()
for _ in range(a.passes):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    ev[0].record()
    eng.partial_gramian(H, 0, b, slab); ev[1].record()
    eng.side_pass("user", H, W, 0, b, slab, 0.1, cache); ev[2].record()
    eng.partial_gramian(W, 0, b, slab); ev[3].record()
    eng.side_pass("item", W, H, 0, b, slab, 0.1, cache); ev[4].record()
    torch.cuda.synchronize()
    print("slabH %.3f user %.3f slabW %.3f item %.3f ms" % tuple(ev[i].elapsed_time(ev[i + 1]) for i in range(4)))
su, si = prob.users.schedule(b), prob.items.schedule(b)
print("users light/heavy/slices", su.n_light, su.n_heavy, su.n_slices, "items", si.n_light, si.n_heavy, si.n_slices)
