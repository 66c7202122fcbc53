"""Full-size parity at the BASELINE shapes (GPU).  The CPU oracle cannot run
whole epochs at these sizes in test time, so this checks, per row, the exact
quantity the reference computes (``_newton_side_pass``, solvers.py:152-186):
from the GPU's pre-pass state (W, H, cache), the f64 Newton step of a sample
of rows (all of the 40 heaviest items, plus systematic samples of users and
items) must match the GPU's update within rel 1e-3, and the cache must stay
consistent with fresh predictions.  Run one user pass and one item pass of
block 0 at the configs[1] (d=128, b=32) and configs[3] (d=1024, b=128) shapes.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _dataset():
    from paper_2110_14044_b200 import synthetic
    from paper_2110_14044_b200.data import InteractionDataset
    U, I, users, items = synthetic.generate("mid", 0)
    return InteractionDataset(U, I, users, items)


def _newton_rows(rows, ptr, cols, pos, fixed, own, cache, b0, b, alpha0, lam):
    """f64 restatement of solvers.py:171-185 for a handful of rows."""
    blk = slice(b0, b0 + b)
    slab = fixed.T @ fixed[:, blk]
    out = np.empty((len(rows), b))
    for n, r in enumerate(rows):
        e = slice(ptr[r], ptr[r + 1])
        x = fixed[cols[e], blk]
        rho = cache[pos[e]] - 1.0
        g = rho @ x + alpha0 * (own[r] @ slab) + lam[r] * own[r, blk]
        hs = x.T @ x + alpha0 * slab[blk] + lam[r] * np.eye(b)
        out[n] = own[r, blk] - np.linalg.solve(hs, g)
    return out


@pytest.mark.parametrize("d,b", [(128, 32), (1024, 128)])
def test_block0_sampled_rows_fullscale(d, b):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2110_14044_b200.engine import DeviceProblem, Engine
    data = _dataset()
    U, I = data.num_users, data.num_items
    prob = DeviceProblem.from_dataset(data, torch.device("cuda", 0))
    alpha0, reg = 0.1, 1e-3
    prob.set_regularizer(alpha0, reg, 1.0)
    eng = Engine(prob)
    rng = np.random.default_rng(0)
    W = torch.from_numpy((rng.standard_normal((U, d)) * 0.1 / np.sqrt(d)).astype(np.float32)).cuda()
    H = torch.from_numpy((rng.standard_normal((I, d)) * 0.1 / np.sqrt(d)).astype(np.float32)).cuda()
    cache = torch.empty(data.n_interactions, device="cuda")
    eng.predictions(W, H, cache)
    slab = torch.empty(d, b, device="cuda")
    lam_u = reg * (data.user_counts + alpha0 * I)
    lam_i = reg * (data.item_counts + alpha0 * U)
    uv, iv = data.user_view(), data.item_view()
    # ---- user pass of block 0
    w0, h0, c0 = (W.double().cpu().numpy(), H.double().cpu().numpy(), cache.double().cpu().numpy())
    eng.partial_gramian(H, 0, b, slab)
    eng.side_pass("user", H, W, 0, b, slab, alpha0, cache)
    eng.sess.raise_if_singular()
    order = np.argsort(-data.user_counts, kind="stable")
    urows = np.concatenate([order[:8], order[:: max(1, U // 120)]])
    want = _newton_rows(urows, uv.ptr, uv.cols, uv.cache_pos, h0, w0, c0, 0, b, alpha0, lam_u)
    got = W.double().cpu().numpy()[urows, :b]
    err_u = np.linalg.norm(got - want) / np.linalg.norm(want)
    # ---- item pass of block 0 (against the GPU's post-user-pass state)
    w1, c1 = W.double().cpu().numpy(), cache.double().cpu().numpy()
    eng.partial_gramian(W, 0, b, slab)
    eng.side_pass("item", W, H, 0, b, slab, alpha0, cache)
    eng.sess.raise_if_singular()
    iorder = np.argsort(-data.item_counts, kind="stable")
    irows = np.concatenate([iorder[:40], iorder[40:: max(1, I // 80)]])
    want_i = _newton_rows(irows, iv.ptr, iv.cols, iv.cache_pos, w1, h0, c1, 0, b, alpha0, lam_i)
    got_i = H.double().cpu().numpy()[irows, :b]
    err_i = np.linalg.norm(got_i - want_i) / np.linalg.norm(want_i)
    rowerr_i = np.linalg.norm(got_i - want_i, axis=1) / np.linalg.norm(want_i, axis=1)
    print(f"d={d} b={b}: user relF {err_u:.2e}, item relF {err_i:.2e}, worst item row {rowerr_i.max():.2e}")
    assert err_u < 1e-3 and err_i < 1e-3 and rowerr_i.max() < 1e-3
    # cache consistent with the updated factors
    fresh = torch.empty_like(cache)
    eng.predictions(W, H, fresh)
    drift = (cache - fresh).abs() / (1 + fresh.abs())
    assert float(drift.max()) < 1e-4
