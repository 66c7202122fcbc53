"""Fold-in and ranking on the device vs the reference's
own outputs (tests/golden/eval.npz, made by tests/golden/make_golden.py from
the unmodified reference) and the oracle restatement."""

from types import SimpleNamespace

import numpy as np
import pytest

from conftest import load_golden, relf

import paper_2110_14044_b200 as ials

pytestmark = pytest.mark.gpu


def _rag(ptr, flat, i):
    return flat[ptr[i]:ptr[i + 1]]


@pytest.fixture(scope="module")
def eval_golden():
    g = load_golden("eval")
    nf = g["in_ptr"].size - 1
    folds = [SimpleNamespace(input_items=_rag(g["in_ptr"], g["in_items"], i), input_labels=None,
                             input_weights=None, target_items=_rag(g["tg_ptr"], g["tg_items"], i))
             for i in range(nf)]
    return g, folds


CFG = ials.SolverConfig(dim=32, block_size=8, unobserved_weight=0.1, reg=1e-3, reg_exponent=1.0)


def test_top_k_ties_and_exclusion_exact(eval_golden):
    g, _ = eval_golden
    for c in range(g["tk_k"].size):
        s = _rag(g["tk_sptr"], g["tk_scores"], c)
        e = _rag(g["tk_eptr"], g["tk_exclude"], c)
        got = ials.top_k_from_scores(s, int(g["tk_k"][c]), exclude=e)
        assert np.array_equal(got, _rag(g["tk_optr"], g["tk_out"], c)), c


def test_top_k_random_vs_oracle():
    from oracle import ialspp_oracle as orc
    rng = np.random.default_rng(3)
    for n, k in [(20108, 100), (41140, 1024), (5000, 7), (3, 10)]:
        s = rng.standard_normal(n).astype(np.float32)
        s[rng.choice(n, n // 10)] = np.round(s[0], 2)       # ties
        s[rng.choice(n, 3)] = np.nan
        s[rng.choice(n, 3)] = -0.0
        ex = rng.choice(n, n // 5, replace=False)
        want = orc.top_k(s.astype(np.float64), k, ex)
        assert np.array_equal(ials.top_k_from_scores(s, k, exclude=ex), want)
    with pytest.raises(ValueError, match="k must be positive"):
        ials.top_k_from_scores(np.zeros(3), 0)


def test_fold_in_matches_reference(eval_golden):
    g, folds = eval_golden
    ev = [f for f in folds if f.target_items.size > 0]
    emb = ials.fold_in_users(g["item_factors"], [(f.input_items, None, None) for f in ev], CFG)
    assert relf(emb, g["embeddings"]) < 1e-3
    one = ials.project_user(g["item_factors"], ev[0].input_items, config=CFG)
    assert relf(one, g["embeddings"][0]) < 1e-3
    assert np.array_equal(ials.project_user(g["item_factors"], [], config=CFG),
                          np.zeros(g["item_factors"].shape[1]))


def test_ranking_and_metrics_match_reference(eval_golden):
    g, folds = eval_golden
    ev = [f for f in folds if f.target_items.size > 0]
    same = 0
    for r, f in enumerate(ev):
        tk = ials.rank_items(g["embeddings"][r], g["item_factors"], exclude=f.input_items, k=100)
        same += np.array_equal(tk, _rag(g["topk_ptr"], g["topk"], r))
    # FP32 scores vs the reference's f64: only exact near-ties may reorder
    assert same >= len(ev) - 2, (same, len(ev))
    rep = ials.evaluate_holdout(g["item_factors"], folds, CFG, recall_ks=(20, 50), ndcg_ks=(10, 100))
    assert rep.num_users_evaluated == int(g["n_evaluated"])
    for k in (20, 50):
        assert abs(rep.recall_at[k] - float(g[f"recall_{k}"])) < 2e-3, (k, rep.recall_at[k])
    for k in (10, 100):
        assert abs(rep.ndcg_at[k] - float(g[f"ndcg_{k}"])) < 2e-3, (k, rep.ndcg_at[k])
    # batching of the score matrix does not change the result
    rep2 = ials.evaluate_holdout(g["item_factors"], folds, CFG, recall_ks=(20, 50),
                                 ndcg_ks=(10, 100), users_per_batch=7)
    assert rep2 == rep
    with pytest.raises(ValueError, match="no holdout users"):
        ials.evaluate_holdout(g["item_factors"], [f for f in folds if f.target_items.size == 0], CFG)


@pytest.mark.parametrize("d", [32, 128, 200])
def test_fold_in_with_labels_and_weights(d):
    """Non-unit labels / weights reach the device fold-in (the sweep's
    weighted path) exactly as the reference's rhs / Hessian use them."""
    from oracle import ialspp_oracle as orc
    rng = np.random.default_rng(23 + d)
    I = 500
    hf = (rng.standard_normal((I, d)) * 0.1).astype(np.float32).astype(np.float64)
    hist = []
    for _ in range(120):
        n = int(rng.integers(0, 40))
        its = rng.choice(I, n, replace=False)
        hist.append((its, rng.uniform(0.5, 2.0, n), rng.uniform(0.2, 3.0, n)))
    cfg = ials.SolverConfig(dim=d, block_size=8, unobserved_weight=0.1, reg=1e-3, reg_exponent=1.0)
    got = ials.fold_in_users(hf, hist, cfg)
    want = orc.fold_in(hf, hist, 0.1, 1e-3, 1.0)
    assert relf(got, want) < 1e-3


def test_top_k_float64_near_ties_exact():
    """top_k_from_scores ranks the caller's float64 scores as float64: values
    that differ below fp32 resolution keep the reference's order (metrics.py:31-57)."""
    from oracle import ialspp_oracle as orc
    rng = np.random.default_rng(9)
    for n, k in [(20108, 100), (5000, 1024), (64, 10)]:
        base = rng.standard_normal(n // 4 + 1)
        s = np.repeat(base, 4)[:n] + rng.integers(-3, 4, n) * 1e-13   # near-ties within 1 ulp of fp32
        s[rng.choice(n, 5)] = base[0]                                   # exact ties
        s[rng.choice(n, 2)] = np.nan
        ex = rng.choice(n, n // 7, replace=False)
        want = orc.top_k(s, k, ex)
        assert np.array_equal(ials.top_k_from_scores(s, k, exclude=ex), want)


def test_scores_gemm_and_batched_recommend():
    """ials_scores (3xTF32 tensor-core GEMM, 128-item tiles) against f64, and
    ImplicitALS.recommend (one batched device ranking) against per-row
    rank_items with the same exclusions (the reference's loop, estimator.py:135-152)."""
    import torch
    from paper_2110_14044_b200.evaluation import _padded_f32, device_scores
    rng = np.random.default_rng(4)
    for nu, ni, d in [(300, 20108, 64), (1, 1000, 30), (129, 257, 128)]:
        E = rng.standard_normal((nu, d)).astype(np.float32)
        H = rng.standard_normal((ni, d)).astype(np.float32)
        got = device_scores(_padded_f32(E, "cuda"), _padded_f32(H, "cuda"), d).double().cpu().numpy()
        want = E.astype(np.float64) @ H.astype(np.float64).T
        assert np.abs(got - want).max() <= 2e-6 * np.abs(want).max() * np.sqrt(d)
    import scipy.sparse as sp
    X = sp.random(400, 150, density=0.05, random_state=1, format="csr")
    X.data[:] = 1.0
    est = ials.ImplicitALS(factors=16, block_size=8, epochs=2).fit(X)
    Q = sp.random(37, 150, density=0.1, random_state=2, format="csr")
    Q.data[:] = 1.0
    items, scores = est.recommend(Q, k=12)
    emb = est.transform(Q)
    for r in range(Q.shape[0]):
        seen = Q[r].indices
        top = ials.rank_items(emb[r], est.item_factors_, exclude=seen, k=12)
        assert np.array_equal(items[r, :top.size], top)
        np.testing.assert_allclose(scores[r, :top.size], est.item_factors_[top] @ emb[r])
