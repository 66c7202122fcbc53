"""Small epochs through every sweep kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck):  python tools/sanitize_cases.py
b = 8 (SIMT), 32 (packed, 4 rows per tile), 64 (packed, 2 rows), 128 (fused
tc4 + rotated user pass with Woodbury tiles, heavy item slices)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np

import paper_2110_14044_b200 as ials

rng = np.random.default_rng(0)
for d, b, U, I in [(16, 8, 300, 120), (64, 32, 400, 150), (128, 64, 400, 150), (128, 128, 500, 60)]:
    nnz = 12000
    users = rng.integers(0, U, nnz)
    items = np.minimum(rng.zipf(1.15, nnz) - 1, I - 1)
    items[:5000] = 0                      # one heavy item (> 4096 entries: the sliced path)
    data = ials.InteractionDataset(U, I, users, items)
    cfg = ials.SolverConfig(dim=d, block_size=b, unobserved_weight=0.1, reg=1e-3,
                            reg_exponent=1.0, epochs=1, seed=1)
    model = ials.init_model(cfg, U, I)
    ials.train(model, data, cfg)
    print(f"d={d} b={b}: ok", flush=True)
