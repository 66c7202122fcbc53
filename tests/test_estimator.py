"""ImplicitALS (estimator.py, the reference's estimator.py:17-160): input
conversion and errors on the CPU; fit / transform / recommend on the GPU
against the device solvers, the f64 oracle and the reference's padding rules."""

import numpy as np
import pytest
import scipy.sparse as sp

import paper_2110_14044_b200 as ials
from paper_2110_14044_b200.estimator import _interactions as _as_dataset

from conftest import relf


def _matrix(U=300, I=120, n=4000, seed=0):
    rng = np.random.default_rng(seed)
    u = rng.integers(0, U, n)
    i = np.minimum(rng.zipf(1.3, n) - 1, I - 1)
    m = sp.coo_matrix((np.ones(n), (u, i)), shape=(U, I)).tocsr()
    m.sum_duplicates()
    return m


def test_as_dataset_conversions():
    X = _matrix()
    d_sparse = _as_dataset(X)
    d_dense = _as_dataset(X.toarray())
    assert d_sparse.num_users == 300 and d_sparse.num_items == 120
    assert np.array_equal(d_sparse.user_ptr, d_dense.user_ptr)
    assert np.array_equal(d_sparse.items, d_dense.items)
    assert np.array_equal(d_sparse.weights, d_dense.weights)   # values -> weights
    assert np.all(d_sparse.labels == 1.0)
    assert _as_dataset(d_sparse) is d_sparse


def test_as_dataset_errors():
    X = _matrix()
    with pytest.raises(TypeError):
        _as_dataset([[1, 0], [0, 1]])
    with pytest.raises(ValueError, match="2-d"):
        _as_dataset(np.ones(5))
    with pytest.raises(ValueError, match="item columns"):
        _as_dataset(X, num_items=7)
    with pytest.raises(ValueError, match="items"):
        _as_dataset(_as_dataset(X), num_items=7)


def test_params_and_unfitted():
    from sklearn.base import clone
    est = ials.ImplicitALS(factors=16, solver="icd", epochs=3)
    c = clone(est)
    assert c.get_params()["solver"] == "icd" and c.get_params()["factors"] == 16
    with pytest.raises(RuntimeError, match="not fitted"):
        est.transform(_matrix())


@pytest.mark.gpu
@pytest.mark.parametrize("solver,factors,block", [("ialspp", 32, 8), ("ialspp", 128, 64),
                                                  ("ials", 16, None), ("icd", 8, None)])
def test_fit_matches_train_and_oracle(solver, factors, block):
    from oracle import ialspp_oracle as orc
    X = _matrix()
    est = ials.ImplicitALS(factors=factors, solver=solver, block_size=block, epochs=3,
                           reg=0.003, alpha0=0.1, random_state=5).fit(X)
    data = _as_dataset(X)
    cfg = est._config()
    model = ials.init_model(cfg, data.num_users, data.num_items)
    w0, h0 = model.user_factors.copy(), model.item_factors.copy()
    ials.train(model, data, cfg)
    assert np.array_equal(est.user_factors_, model.user_factors)   # same device path
    assert np.array_equal(est.item_factors_, model.item_factors)
    assert len(est.training_reports_) == 3
    b = {"ialspp": cfg.block_size, "ials": factors, "icd": 1}[solver]
    w, h = w0.astype(np.float32).astype(np.float64), h0.astype(np.float32).astype(np.float64)
    csr = orc.build_csr(data.num_users, data.num_items, data.users, data.items, data.labels,
                        data.weights)
    orc.train(w, h, csr, 0.1, 0.003, 1.0, b, 3)
    assert relf(est.user_factors_, w) < 1e-3 and relf(est.item_factors_, h) < 1e-3


@pytest.mark.gpu
def test_transform_and_recommend():
    from oracle import ialspp_oracle as orc
    X = _matrix()
    est = ials.ImplicitALS(factors=32, block_size=32, epochs=2).fit(X)
    Q = _matrix(U=6, I=120, n=40, seed=3).toarray()
    Q[5, :] = 1.0           # row 5 has seen every item but two
    Q[5, [7, 11]] = 0.0
    emb = est.transform(Q)
    hist = []
    for r in range(Q.shape[0]):
        its = np.nonzero(Q[r])[0]
        hist.append((its, np.ones(its.size), Q[r, its]))
    want = orc.fold_in(est.item_factors_, hist, 0.1, 0.003, 1.0)
    assert relf(emb, want) < 1e-3
    items, scores = est.recommend(Q, k=5)
    assert items.shape == (6, 5) and scores.shape == (6, 5)
    assert set(items[5, :2]) == {7, 11} and np.all(items[5, 2:] == -1)
    assert np.all(np.isnan(scores[5, 2:]))
    for r in range(5):
        assert not set(items[r][items[r] >= 0]) & set(np.nonzero(Q[r])[0])
        assert np.all(np.diff(scores[r]) <= 1e-6)   # descending
    items_all, _ = est.recommend(Q, k=5, exclude_seen=False)
    assert np.all(items_all >= 0)
