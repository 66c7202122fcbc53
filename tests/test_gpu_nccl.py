"""The sharded epoch over NCCL with two ranks (one process per GPU): W, H and
the gathered canonical cache against the single-process oracle.  Needs two
GPUs; skipped below that (this build's GPU runs have one -- the orchestration
itself is covered at world size 2 and 3 by the gloo tests, and with the real
kernels at world size 1 by test_gpu_parity.py::test_sharded_path_gpu_ops_single_rank)."""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
TOL = 1e-3


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, d, b, q):
    import sys
    import torch.distributed as dist
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import ialspp_oracle as orc
    from paper_2110_14044_b200.distributed import GpuOps, ShardedTrainer
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world,
                            device_id=torch.device("cuda", rank))
    try:
        rng = np.random.default_rng(3)
        U, I, n = 3000, 800, 60000
        users = rng.integers(0, U, n)
        items = np.minimum(rng.zipf(1.2, n) - 1, I - 1)
        csr = orc.build_csr(U, I, users, items)
        data = {"num_users": U, "num_items": I, "user_ptr": csr["user_ptr"], "user_cols": csr["items"],
                "item_ptr": csr["item_ptr"], "item_cols": csr["users"][csr["item_order"]],
                "item_order": csr["item_order"], "labels": None, "weights": None}
        w, h = orc.init_factors(U, I, d, 0.1, 4)
        w, h = w.astype(np.float32).astype(np.float64), h.astype(np.float32).astype(np.float64)
        W = torch.from_numpy(w.astype(np.float32)).cuda()
        H = torch.from_numpy(h.astype(np.float32)).cuda()
        tr = ShardedTrainer(data, W, H, 0.1, 1e-3, 1.0, GpuOps(f"cuda:{rank}"))
        for _ in range(2):
            tr.epoch(b)
        cache = tr.gather_cache().double().cpu().numpy()
        if rank == 0:
            ref_cache = orc.train(w, h, csr, 0.1, 1e-3, 1.0, b, 2)
            q.put((np.linalg.norm(W.double().cpu().numpy() - w) / np.linalg.norm(w),
                   np.linalg.norm(H.double().cpu().numpy() - h) / np.linalg.norm(h),
                   float(np.abs(cache - ref_cache).max() / np.abs(ref_cache).max())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("d,b", [(256, 128), (96, 32)])
def test_two_rank_nccl_epoch_vs_oracle(d, b):
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, d, b, q)) for r in range(2)]
    for p in procs:
        p.start()
    ew, eh, ec = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert ew < TOL and eh < TOL and ec < TOL, (ew, eh, ec)
