"""Multi-rank path on CPU with the gloo backend: sharded
users/items, replicated tables, all-reduced slabs, all-gathered column blocks
and the dual-cache delta correction must reproduce the single-process oracle
(float64, so the comparison is tight)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import ialspp_oracle as orc
from paper_2110_14044_b200.distributed import ShardedTrainer, shard_bounds


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _instance(seed, U=37, I=23, nnz=420, weighted=True):
    rng = np.random.default_rng(seed)
    users = rng.integers(0, U, nnz)
    items = np.minimum(rng.zipf(1.4, nnz) - 1, I - 1)
    users[users == U - 1] = 0                       # an empty user row
    labels = rng.uniform(0, 2, nnz) if weighted else None
    weights = rng.uniform(0.5, 2, nnz) if weighted else None
    csr = orc.build_csr(U, I, users, items, labels, weights)
    data = {"num_users": U, "num_items": I, "user_ptr": csr["user_ptr"],
            "user_cols": csr["items"], "item_ptr": csr["item_ptr"],
            "item_cols": csr["users"][csr["item_order"]], "item_order": csr["item_order"],
            "labels": csr["labels"] if weighted else None,
            "weights": csr["weights"] if weighted else None}
    return csr, data


def _worker(rank, world, port, seed, d, b, epochs, q, rot=False):
    import sys
    sys.path.insert(0, os.path.dirname(__file__))
    from dist_cpu_ops import CpuOps
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        csr, data = _instance(seed, weighted=not rot)
        w, h = orc.init_factors(data["num_users"], data["num_items"], d, 0.1, seed)
        W, H = torch.from_numpy(w.copy()), torch.from_numpy(h.copy())
        ops = CpuOps()
        ops.enable_rot = rot
        tr = ShardedTrainer(data, W, H, 0.1, 0.01, 1.0, ops)
        for _ in range(epochs):
            tr.epoch(b)
        if rot:   # every user pass of every epoch saw the all-reduced diagonal blocks
            assert ops.rot_checks == epochs * (d // b), ops.rot_checks
        cache = tr.gather_cache()
        if rank == 0:
            q.put((W.numpy().copy(), H.numpy().copy(), cache.numpy().copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,d,b,epochs,rot", [(2, 6, 2, 2, False), (2, 5, 5, 1, False),
                                                   (3, 8, 3, 2, False), (2, 8, 4, 2, True),
                                                   (3, 6, 2, 1, True)])
def test_sharded_epoch_matches_oracle(world, d, b, epochs, rot):
    """rot: the rotated-user-pass protocol (one all-reduce of the stacked
    diagonal Gram blocks at epoch start; unit weights)."""
    seed = 11
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, seed, d, b, epochs, q, rot))
             for r in range(world)]
    for p in procs:
        p.start()
    W, H, cache = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    csr, data = _instance(seed, weighted=not rot)
    w, h = orc.init_factors(data["num_users"], data["num_items"], d, 0.1, seed)
    ref_cache = orc.train(w, h, csr, 0.1, 0.01, 1.0, b, epochs)
    assert np.abs(W - w).max() <= 1e-10 * max(1.0, np.abs(w).max())
    assert np.abs(H - h).max() <= 1e-10 * max(1.0, np.abs(h).max())
    assert np.abs(cache - ref_cache).max() <= 1e-10 * max(1.0, np.abs(ref_cache).max())


def test_shard_bounds_balance_and_cover():
    ptr = np.concatenate([[0], np.cumsum([5, 0, 9, 1, 1, 30, 2, 2, 2, 8])])
    for world in (1, 2, 3, 4, 12):
        b = shard_bounds(ptr, world)
        assert b[0][0] == 0 and b[-1][1] == 10 and len(b) == world
        assert all(b[r][1] == b[r + 1][0] for r in range(world - 1))
        assert all(lo <= hi for lo, hi in b)
