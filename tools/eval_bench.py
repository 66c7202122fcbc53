"""Fold-in + ranking evaluation timing: the configs[1]
item count (20,108 items, d=128) with held-out folds cut 80/20 from the first
N synthetic users; device evaluate_holdout (fold-in sweep, FP32 score GEMM,
ials_topk) vs the oracle restatement of the reference on a user sample
(scaled).  Prints one JSON line."""
import json
import os
import sys
import time
from types import SimpleNamespace

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2110_14044_b200 as ials
from paper_2110_14044_b200 import synthetic
from oracle import ialspp_oracle as orc

N = int(sys.argv[1]) if len(sys.argv) > 1 else 10000
U, I, users, items = synthetic.generate("mid", 0)
data = ials.InteractionDataset(U, I, users, items)
rng = np.random.default_rng(0)
folds = []
for u in range(N):
    its = data.items[data.user_ptr[u]:data.user_ptr[u + 1]]
    perm = rng.permutation(its.size)
    nt = max(1, int(its.size * 0.2)) if its.size >= 5 else 0
    folds.append(SimpleNamespace(input_items=its[np.sort(perm[nt:])], input_labels=None, input_weights=None,
                                 target_items=its[np.sort(perm[:nt])]))
d = 128
hf = (rng.standard_normal((I, d)) * 0.1).astype(np.float32).astype(np.float64)
cfg = ials.SolverConfig(dim=d, block_size=d, unobserved_weight=0.1, reg=1e-3)
ials.evaluate_holdout(hf, folds[:200], cfg)   # warm-up (sessions, extension)
torch.cuda.synchronize()
t0 = time.perf_counter()
rep = ials.evaluate_holdout(hf, folds, cfg, recall_ks=(20, 50), ndcg_ks=(100,))
torch.cuda.synchronize()
gpu_s = time.perf_counter() - t0
ns = 300
tup = [(f.input_items, None, None, f.target_items) for f in folds[:ns]]
t0 = time.perf_counter()
orc.evaluate(hf, tup, 0.1, 1e-3, 1.0, (20, 50), (100,))
cpu_s = (time.perf_counter() - t0) * N / ns
print(json.dumps({"users": N, "evaluated": rep.num_users_evaluated, "items": I, "d": d,
                  "gpu_seconds_wall": round(gpu_s, 4), "cpu_oracle_seconds_est": round(cpu_s, 2),
                  "cpu_sample_users": ns, "recall@20": round(rep.recall_at[20], 5),
                  "ndcg@100": round(rep.ndcg_at[100], 5),
                  "note": "wall clock of the whole call (host CSR build + metrics included)"}))
