"""Golden vectors at the BASELINE dimensions, made by the UNMODIFIED reference.

Run in the CPU container (needs ``/root/reference``; the GPU box does not
have it, so the outputs are committed):

    python tests/golden/make_golden_scale.py [128 1024 2048]

Full 10-epoch reference runs at the 136,677-user shapes take hours per epoch
at d >= 1024, so -- as SURVEY.md §8c plans -- the 1- and
10-epoch checks run on a user subsample of the configs[1] / configs[3] shape:
the first 20,000 users of the seeded synthetic set (``synthetic.generate("mid",
0)``), all of their interactions (1,464,242 pairs) and all 20,108 items.

Per (d, b) in {(128, 32), (1024, 128), (2048, 128)}: ``init_model(seed=0)``
rounded to fp32 (both sides start from the same values), then the reference's
``ialspp_epoch`` ten times (``train``'s loop, solvers.py:378-413) with
alpha0 = 0.1, reg = 1e-3, nu = 1.  Stored (``scale_d{d}.npz``):

* ``loss`` -- ``compute_loss`` after every epoch (model.py:168-188);
* ``w1``/``h1``, ``w10``/``h10`` -- the rows ``user_rows`` / ``item_rows`` of W
  and H after epochs 1 and 10 (float32: parity is judged at 1e-3), a sample of
  the heaviest, lightest and systematically spaced rows by degree;
* ``wnorm``/``hnorm`` -- Frobenius norms of the full W and H at 1 and 10
  epochs;
* ``digest`` -- sha256 prefix of the subsampled COO arrays (the GPU test
  regenerates the subsample and checks it).
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

import blockals as ref  # noqa: E402  (the reference package)
from paper_2110_14044_b200 import synthetic  # noqa: E402

N_USERS = 20_000


def subsample():
    """The first N_USERS users of the configs[1] shape with all their pairs."""
    U, I, users, items = synthetic.generate("mid", 0)
    keep = users < N_USERS
    return N_USERS, I, users[keep], items[keep]


def sample_rows(counts, n_heavy=48, n_sys=144, n_light=8):
    order = np.argsort(-np.asarray(counts), kind="stable")
    sys_rows = order[n_heavy::max(1, (order.size - n_heavy) // n_sys)]
    return np.unique(np.concatenate([order[:n_heavy], sys_rows, order[-n_light:]]))


def make(d, b):
    U, I, users, items = subsample()
    data = ref.InteractionDataset(U, I, users, items)
    cfg = ref.SolverConfig(dim=d, block_size=b, unobserved_weight=0.1, reg=1e-3,
                           reg_exponent=1.0, init_stddev=0.1, epochs=10, seed=0, threads=0)
    model = ref.init_model(cfg, U, I)
    model.user_factors[:] = model.user_factors.astype(np.float32)
    model.item_factors[:] = model.item_factors.astype(np.float32)
    urows = sample_rows(data.user_counts)
    irows = sample_rows(data.item_counts)
    out = {"d": d, "b": b, "num_users": U, "num_items": I, "nnz": users.size,
           "digest": synthetic.digest(users, items), "user_rows": urows.astype(np.int32),
           "item_rows": irows.astype(np.int32),
           "w0": model.user_factors[urows].astype(np.float32),
           "h0": model.item_factors[irows].astype(np.float32)}
    cache = ref.PredictionCache.zeros(data.n_interactions)
    part = ref.partition_dims(d, b)
    losses, wn, hn = [], [], []
    for e in range(10):
        t = time.time()
        ref.ialspp_epoch(model, data, cache, cfg, part, e)
        losses.append(ref.compute_loss(model, data, cfg))
        if e in (0, 9):
            tag = "1" if e == 0 else "10"
            out["w" + tag] = model.user_factors[urows].astype(np.float32)
            out["h" + tag] = model.item_factors[irows].astype(np.float32)
            wn.append(np.linalg.norm(model.user_factors))
            hn.append(np.linalg.norm(model.item_factors))
        print(f"d={d} b={b} epoch {e + 1}: loss {losses[-1]:.6f} ({time.time() - t:.0f} s)",
              flush=True)
    out["loss"] = np.array(losses)
    out["wnorm"] = np.array(wn)
    out["hnorm"] = np.array(hn)
    np.savez_compressed(os.path.join(HERE, f"scale_d{d}.npz"), **out)


if __name__ == "__main__":
    dims = [int(a) for a in sys.argv[1:]] or [128, 1024, 2048]
    for d in dims:
        make(d, 32 if d == 128 else 128)
