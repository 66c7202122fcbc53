"""Pin the CPU oracle (oracle/ialspp_oracle.py) against golden vectors that
the unmodified reference produced (tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

from conftest import relf, relmax, small_case
from oracle import ialspp_oracle as orc

SMALL_SEEDS = list(range(1, 11))


def test_csr_bit_exact_tiny(tiny_golden):
    g = tiny_golden
    csr = orc.build_csr(int(g["num_users"]), int(g["num_items"]), g["coo_users"], g["coo_items"])
    assert np.array_equal(csr["users"], g["csr_users"])
    assert np.array_equal(csr["items"], g["csr_items"])
    assert np.array_equal(csr["user_ptr"], g["user_ptr"])
    assert np.array_equal(csr["item_ptr"], g["item_ptr"])
    assert np.array_equal(csr["item_order"], g["item_order"])


def test_init_matches_reference(tiny_golden):
    g = tiny_golden
    w, h = orc.init_factors(int(g["num_users"]), int(g["num_items"]), 32, 0.1, 0)
    assert np.array_equal(w.astype(np.float32), g["w0"])
    assert np.array_equal(h.astype(np.float32), g["h0"])


def _tiny_state(g):
    csr = orc.build_csr(int(g["num_users"]), int(g["num_items"]), g["coo_users"], g["coo_items"])
    return csr, g["w0"].astype(np.float64), g["h0"].astype(np.float64)


def test_predictions_slab_and_block0_passes(tiny_golden):
    g = tiny_golden
    csr, w, h = _tiny_state(g)
    pred = orc.predictions(w, h, csr["users"], csr["items"])
    assert relmax(pred, g["pred0"]) < 1e-6
    blk = np.arange(8)
    assert relmax(orc.partial_gramian(h, blk), g["slab_h_b0"]) < 1e-12
    lu, li = orc.side_regs(csr, 0.1, 1e-3, 1.0)
    cache = pred.copy()
    orc.side_pass(*orc.side_view(csr, "user"), h, w, cache, blk, orc.partial_gramian(h, blk), 0.1, lu)
    assert relmax(w, g["w_user_b0"]) < 1e-6
    assert relmax(cache, g["cache_user_b0"]) < 1e-6
    orc.side_pass(*orc.side_view(csr, "item"), w, h, cache, blk, orc.partial_gramian(w, blk), 0.1, li)
    assert relmax(h, g["h_item_b0"]) < 1e-6
    assert relmax(cache, g["cache_item_b0"]) < 1e-6


def test_tiny_one_and_ten_epochs(tiny_golden):
    g = tiny_golden
    csr, w, h = _tiny_state(g)
    assert orc.loss(w, h, csr, 0.1, 1e-3, 1.0) == pytest.approx(float(g["loss0"]), rel=1e-12)
    cache = np.zeros(csr["users"].size)
    blocks = orc.partition(32, 8)
    losses = []
    for e in range(10):
        orc.ialspp_epoch(w, h, csr, cache, 0.1, 1e-3, 1.0, blocks)
        if e == 0:
            assert relmax(w, g["w1"]) < 1e-6 and relmax(h, g["h1"]) < 1e-6
            assert relmax(cache, g["cache1"]) < 1e-6
            assert orc.loss(w, h, csr, 0.1, 1e-3, 1.0) == pytest.approx(float(g["loss1"]), rel=1e-10)
        losses.append(orc.loss(w, h, csr, 0.1, 1e-3, 1.0))
    assert relmax(w, g["w10"]) < 1e-6 and relmax(h, g["h10"]) < 1e-6
    assert np.allclose(losses, g["losses"], rtol=1e-10)
    assert orc.cache_drift(cache, w, h, csr) < 1e-5


@pytest.mark.parametrize("seed", SMALL_SEEDS)
def test_small_instances(small_golden, seed):
    c = small_case(small_golden, seed)
    csr = orc.build_csr(c["U"], c["I"], c["users"], c["items"], c["labels"], c["weights"])
    assert np.array_equal(csr["user_ptr"], c["user_ptr"])
    assert np.array_equal(csr["item_ptr"], c["item_ptr"])
    assert np.array_equal(csr["item_order"], c["item_order"])
    assert np.array_equal(csr["items"], c["csr_items"])
    w, h = c["w0"].copy(), c["h0"].copy()
    assert np.allclose(orc.predictions(w, h, csr["users"], csr["items"]), c["pred0"], rtol=1e-12, atol=1e-15)
    blocks = c.get("blocks") or orc.partition(c["d"], c["b"])
    assert orc.loss(w, h, csr, c["alpha0"], c["reg"], c["nu"]) == pytest.approx(float(c["loss0"]), rel=1e-12)
    cache = np.zeros(c["nnz"])
    for e in range(3):
        orc.ialspp_epoch(w, h, csr, cache, c["alpha0"], c["reg"], c["nu"], blocks)
        if e == 0:
            assert relmax(w, c["w1"]) < 1e-9 and relmax(h, c["h1"]) < 1e-9
            assert np.allclose(cache, c["cache1"], rtol=1e-9, atol=1e-12)
    assert relmax(w, c["w3"]) < 1e-9 and relmax(h, c["h3"]) < 1e-9
    assert orc.loss(w, h, csr, c["alpha0"], c["reg"], c["nu"]) == pytest.approx(float(c["loss3"]), rel=1e-9)
    # one item-side block_update of the last block from the init
    w, h = c["w0"].copy(), c["h0"].copy()
    cache = orc.predictions(w, h, csr["users"], csr["items"])
    blk = c["bu_block"]
    slab = orc.partial_gramian(w, blk)
    assert relmax(slab, c["slab_w_last"]) < 1e-12
    _, li = orc.side_regs(csr, c["alpha0"], c["reg"], c["nu"])
    orc.side_pass(*orc.side_view(csr, "item"), w, h, cache, blk, slab, c["alpha0"], li)
    assert relmax(h, c["bu_h"]) < 1e-9
    assert np.allclose(cache, c["bu_cache"], rtol=1e-9, atol=1e-12)


def test_singular_row_named():
    # empty user row + nu=1 + alpha0=0 -> zero system for user 1
    # (reference tests/test_solvers.py:82-91)
    csr = orc.build_csr(2, 2, [0], [0])
    w, h = orc.init_factors(2, 2, 2, 0.1, 0)
    lu, _ = orc.side_regs(csr, 0.0, 0.1, 1.0)
    cache = orc.predictions(w, h, csr["users"], csr["items"])
    blk = np.arange(2)
    with pytest.raises(orc.SingularRow) as err:
        orc.side_pass(*orc.side_view(csr, "user"), h, w, cache, blk, orc.partial_gramian(h, blk), 0.0, lu)
    assert err.value.row == 1 and err.value.pivot == 0


# ------------------------------------------------ fold-in / ranking (8f rank 3)
def _rag(ptr, flat, i):
    return flat[ptr[i]:ptr[i + 1]]


def test_oracle_fold_in_and_ranking_match_reference():
    from conftest import load_golden
    from oracle import ialspp_oracle as orc
    g = load_golden("eval")
    nf = g["in_ptr"].size - 1
    folds = [(_rag(g["in_ptr"], g["in_items"], i), None, None, _rag(g["tg_ptr"], g["tg_items"], i))
             for i in range(nf)]
    ev = [f for f in folds if len(f[3]) > 0]
    emb = orc.fold_in(g["item_factors"], [(f[0], None, None) for f in ev], 0.1, 1e-3, 1.0)
    assert np.abs(emb - g["embeddings"]).max() <= 1e-9 * np.abs(g["embeddings"]).max()
    for r, f in enumerate(ev):
        tk = orc.top_k(g["item_factors"] @ g["embeddings"][r], 100, exclude=f[0])
        assert np.array_equal(tk, _rag(g["topk_ptr"], g["topk"], r))
    rec, ndcg, n = orc.evaluate(g["item_factors"], folds, 0.1, 1e-3, 1.0, (20, 50), (10, 100))
    assert n == int(g["n_evaluated"])
    assert abs(rec[20] - float(g["recall_20"])) < 1e-12 and abs(rec[50] - float(g["recall_50"])) < 1e-12
    assert abs(ndcg[10] - float(g["ndcg_10"])) < 1e-12 and abs(ndcg[100] - float(g["ndcg_100"])) < 1e-12


def test_oracle_top_k_ties_and_exclusion_match_reference():
    from conftest import load_golden
    from oracle import ialspp_oracle as orc
    g = load_golden("eval")
    for c in range(g["tk_k"].size):
        s = _rag(g["tk_sptr"], g["tk_scores"], c)
        e = _rag(g["tk_eptr"], g["tk_exclude"], c)
        assert np.array_equal(orc.top_k(s, int(g["tk_k"][c]), e), _rag(g["tk_optr"], g["tk_out"], c))
