"""Rotated vs unrotated user passes, pass by pass (ials_epoch_range) on the
20k-user subsample of the configs[1] shape: where do they part?"""
import sys
import numpy as np
import torch
sys.path.insert(0, "/root/repo")
from paper_2110_14044_b200 import _lib, synthetic
from paper_2110_14044_b200.data import InteractionDataset
from paper_2110_14044_b200.engine import DeviceProblem, Engine

lib = _lib.load()
d = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
nu = int(sys.argv[2]) if len(sys.argv) > 2 else 20000
U, I, users, items = synthetic.generate("mid", 0)
keep = users < nu
data = InteractionDataset(nu, I, users[keep], items[keep])
prob = DeviceProblem.from_dataset(data, torch.device("cuda", 0))
prob.set_regularizer(0.1, 1e-3, 1.0)
eng = Engine(prob)
g = torch.Generator(device="cuda").manual_seed(0)
W0 = torch.randn(nu, d, device="cuda", generator=g) * (0.1 / d ** 0.5)
H0 = torch.randn(I, d, device="cuda", generator=g) * (0.1 / d ** 0.5)
nb = d // 128
st = {}
for rot in (0, 1):
    lib.ials_set_rotation(rot)
    W, H = W0.clone(), H0.clone()
    c = torch.zeros(data.n_interactions, device="cuda")
    eng.epoch_passes(W, H, c, 128, 0.1, 0, 0, recompute_cache=True)
    snaps = []
    for p in range(2 * nb):
        eng.epoch_passes(W, H, c, 128, 0.1, p, 1)
        snaps.append((W.clone(), H.clone(), c.clone()))
    st[rot] = snaps
e = lambda a, b: float((a - b).norm() / b.norm())
for p in range(2 * nb):
    (w1, h1, c1), (w0, h0, c0) = st[1][p], st[0][p]
    print(f"pass {p:2d}: W {e(w1, w0):.1e} H {e(h1, h0):.1e} cache {e(c1, c0):.1e}", flush=True)
