"""GPU parity of the wide side passes (block widths above 256,
csrc/ials_sweep_wide.cuh): the dedicated iALS epoch at d > 256
(reference solvers.py:216-233, 275-300), iALS++ partitions with blocks wider
than 256 columns (solvers.py:152-186, 340-375) and the direct fold-in
(solvers.py:416-466), against the f64 oracle.  Tolerance: north_star's rel
1e-3 (FP32 build vs float64 reference)."""

import numpy as np
import pytest

from conftest import relf, relmax

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 1e-3


@pytest.fixture(scope="module")
def ials():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2110_14044_b200 as m
    from paper_2110_14044_b200 import _lib
    _lib.load()
    return m


def _instance(U, I, per_user, s, seed):
    rng = np.random.default_rng(seed)
    w = np.arange(1, I + 1, dtype=np.float64) ** -s
    w /= w.sum()
    users, items = [], []
    for u in range(U):
        k = int(rng.integers(0, per_user + 1))   # empty rows included
        its = rng.choice(I, size=min(k, I), replace=False, p=w)
        users.append(np.full(its.size, u))
        items.append(its)
    return np.concatenate(users), np.concatenate(items)


def _f32_model(ials, cfg, U, I):
    m = ials.init_model(cfg, U, I)
    m.user_factors[:] = m.user_factors.astype(np.float32)
    m.item_factors[:] = m.item_factors.astype(np.float32)
    return m


@pytest.mark.parametrize("d", [512, 1024, 320, 301])
def test_dedicated_ials_epoch_wide(ials, d):
    """ials_epoch at d > 256: an exact user pass then an exact item pass (one
    d-wide Newton step each from an exact cache) vs the oracle's b = d epoch;
    d = 320 is not a multiple of the 64-column panels, d = 301 takes the
    unaligned (scalar staging) path."""
    from oracle import ialspp_oracle as orc
    U, I = 500, 260
    users, items = _instance(U, I, 40, 1.0, d)
    data = ials.InteractionDataset(U, I, users, items)
    cfg = ials.SolverConfig(dim=d, block_size=128, unobserved_weight=0.1, reg=1e-3,
                            reg_exponent=1.0, epochs=1, seed=3)
    m = _f32_model(ials, cfg, U, I)
    w, h = m.user_factors.copy(), m.item_factors.copy()
    ials.ials_epoch(m, data, cfg)
    orc.train(w, h, orc.build_csr(U, I, users, items), 0.1, 1e-3, 1.0, d, 1)
    assert relf(m.user_factors, w) < TOL and relf(m.item_factors, h) < TOL
    assert relmax(m.user_factors, w) < TOL and relmax(m.item_factors, h) < TOL


@pytest.mark.parametrize("d,b,epochs", [(640, 320, 1), (640, 320, 3), (768, 512, 2), (600, 300, 2)])
def test_wide_blocks_ialspp(ials, d, b, epochs):
    """iALS++ with blocks wider than 256 columns (the cache is maintained
    across the wide passes; (768, 512) mixes a wide and a 256-wide block)."""
    from oracle import ialspp_oracle as orc
    U, I = 700, 300
    users, items = _instance(U, I, 30, 1.1, 7 * d + b)
    data = ials.InteractionDataset(U, I, users, items)
    cfg = ials.SolverConfig(dim=d, block_size=b, unobserved_weight=0.1, reg=1e-3,
                            reg_exponent=1.0, epochs=epochs, seed=5)
    m = _f32_model(ials, cfg, U, I)
    w, h = m.user_factors.copy(), m.item_factors.copy()
    _, reps = ials.train(m, data, cfg, log_loss=True)
    csr = orc.build_csr(U, I, users, items)
    orc.train(w, h, csr, 0.1, 1e-3, 1.0, b, epochs)
    assert relf(m.user_factors, w) < TOL and relf(m.item_factors, h) < TOL
    assert relmax(m.user_factors, w) < TOL and relmax(m.item_factors, h) < TOL
    want = orc.loss(w, h, csr, 0.1, 1e-3, 1.0)
    assert abs(reps[-1].loss - want) <= TOL * abs(want)


def test_wide_heavy_rows_labels_weights(ials):
    """Items far above the heavy threshold (their Hessian tiles are spread
    over CTAs, no slices) with non-unit labels and weights, d = 384."""
    from oracle import ialspp_oracle as orc
    rng = np.random.default_rng(11)
    U, I, d = 15000, 450, 384
    users, items = _instance(U, I, 8, 1.4, 4)
    n = users.size
    labels = rng.uniform(0.5, 2.0, n)
    weights = rng.uniform(0.2, 3.0, n)
    data = ials.InteractionDataset(U, I, users, items, labels, weights)
    assert data.item_counts.max() > 4096
    cfg = ials.SolverConfig(dim=d, block_size=d, unobserved_weight=0.1, reg=1e-3,
                            reg_exponent=1.0, epochs=1, seed=9)
    m = _f32_model(ials, cfg, U, I)
    w, h = m.user_factors.copy(), m.item_factors.copy()
    ials.train(m, data, cfg)
    csr = orc.build_csr(U, I, users, items, labels, weights)
    orc.train(w, h, csr, 0.1, 1e-3, 1.0, d, 1)
    assert relf(m.user_factors, w) < TOL and relf(m.item_factors, h) < TOL
    assert relmax(m.user_factors, w) < TOL and relmax(m.item_factors, h) < TOL


def test_wide_singular_row_is_named(ials):
    """The reference's singular case (tests/test_solvers.py:82-91: an empty
    row, nu = 1, alpha0 = 0) at a wide block: the failing (side, row, pivot)
    is raised as SingularMatrixError."""
    d = 300
    data = ials.InteractionDataset(2, 2, [0], [0])
    cfg = ials.SolverConfig(dim=d, unobserved_weight=0.0, reg=0.1, reg_exponent=1.0)
    model = ials.init_model(cfg, 2, 2)
    cache = ials.compute_predictions(model, data)
    with pytest.raises(ials.SingularMatrixError) as err:
        ials.block_update(model, data, cache, cfg, np.arange(d), side="user")
    assert err.value.row == 1 and err.value.pivot == 0


@pytest.mark.parametrize("d", [384, 520])
def test_fold_in_wide_direct(ials, d):
    """fold_in_users at d > 256 is one direct solve per history (the wide
    pass from a zero embedding), as the reference's project_user."""
    from oracle import ialspp_oracle as orc
    rng = np.random.default_rng(17)
    I = 900
    hf = (rng.standard_normal((I, d)) * 0.05).astype(np.float32).astype(np.float64)
    hist = [(rng.choice(I, int(rng.integers(0, 60)), replace=False), None, None) for _ in range(300)]
    cfg = ials.SolverConfig(dim=d, block_size=128, unobserved_weight=0.1, reg=1e-3)
    got = ials.fold_in_users(hf, hist, cfg)
    want = orc.fold_in(hf, hist, 0.1, 1e-3, 1.0)
    assert relf(got, want) < TOL and relmax(got, want) < TOL
