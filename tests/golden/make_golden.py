"""Generate the golden fixtures by running the UNMODIFIED reference.

Run in the CPU container (needs ``/root/reference``; the GPU box does not
have it):

    python tests/golden/make_golden.py

It imports ``blockals`` from ``/root/reference/pkg/src`` and records, for a
set of inputs, what the reference's own public API returns:

* ``tiny.npz`` -- BASELINE config 0 (2,000 x 1,000, d=32, b=8, alpha0=0.1,
  reg=1e-3, nu=1, sigma*=0.1, seed 0) on the synthetic generator's data: the
  reference CSR arrays (bit-exact contract), the fp32-rounded init, the
  block-0 slab / user pass / item pass, and W, H, cache and loss after 1 and
  after 10 epochs of ``train``.
* ``small.npz`` -- small random instances in the style of the reference's
  ``random_instance`` fixture (duplicates, empty rows, non-unit labels and
  weights, remainder blocks, b=1 and b=d, a non-contiguous partition), each
  with the state after one and after three epochs.

* ``eval.npz`` -- fold-in and ranking: a holdout split
  of the tiny data (``split_holdout``), three epochs of ``train`` on its
  training part, then ``fold_in_users`` embeddings of the evaluated folds,
  ``rank_items`` top-100 lists, ``evaluate_holdout`` metrics, and
  ``top_k_from_scores`` on tie-heavy score vectors with exclusions.

The COO inputs are stored too, so the fixtures are self-contained.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

import blockals as ref  # noqa: E402  (the reference package)
from paper_2110_14044_b200 import synthetic  # noqa: E402


def fp32_init(config, U, I):
    model = ref.init_model(config, U, I)
    model.user_factors[:] = model.user_factors.astype(np.float32)
    model.item_factors[:] = model.item_factors.astype(np.float32)
    return model


def make_tiny():
    U, I, users, items = synthetic.generate("tiny", 0)
    data = ref.InteractionDataset(U, I, users, items)
    cfg = ref.SolverConfig(dim=32, block_size=8, unobserved_weight=0.1, reg=1e-3,
                           reg_exponent=1.0, init_stddev=0.1, epochs=10, seed=0,
                           threads=1)
    out = {"coo_users": users.astype(np.int32), "coo_items": items.astype(np.int32),
           "num_users": U, "num_items": I, "digest": synthetic.digest(users, items)}
    out["csr_users"] = data.users.astype(np.int32)
    out["csr_items"] = data.items.astype(np.int32)
    out["user_ptr"] = data.user_ptr
    out["item_ptr"] = data.item_ptr
    out["item_order"] = data.item_view().cache_pos.astype(np.int32)
    model = fp32_init(cfg, U, I)
    out["w0"] = model.user_factors.astype(np.float32)
    out["h0"] = model.item_factors.astype(np.float32)
    out["loss0"] = ref.compute_loss(model, data, cfg)
    # block-0 pieces from the fp32 init
    blk = ref.partition_dims(32, 8).blocks[0]
    out["slab_h_b0"] = ref.partial_gramian(model.item_factors, blk)
    m = model.copy()
    cache = ref.compute_predictions(m, data)
    out["pred0"] = cache.scores.copy()
    ref.block_update(m, data, cache, cfg, blk, side="user")
    out["w_user_b0"] = m.user_factors.copy()
    out["cache_user_b0"] = cache.scores.copy()
    ref.block_update(m, data, cache, cfg, blk, side="item")
    out["h_item_b0"] = m.item_factors.copy()
    out["cache_item_b0"] = cache.scores.copy()
    # full training, 1 and 10 epochs
    m = model.copy()
    reports = []
    cache = ref.PredictionCache.zeros(data.n_interactions)
    part = ref.partition_dims(32, 8)
    for e in range(10):
        ref.ialspp_epoch(m, data, cache, cfg, part, e)
        if e == 0:
            out["w1"] = m.user_factors.copy()
            out["h1"] = m.item_factors.copy()
            out["cache1"] = cache.scores.copy()
            out["loss1"] = ref.compute_loss(m, data, cfg)
        reports.append(ref.compute_loss(m, data, cfg))
    out["w10"] = m.user_factors.copy()
    out["h10"] = m.item_factors.copy()
    out["cache10"] = cache.scores.copy()
    out["loss10"] = reports[-1]
    out["losses"] = np.array(reports)
    # cross-check with the reference's own train() driver
    m2 = model.copy()
    ref.train(m2, data, cfg)
    assert np.array_equal(m2.user_factors, out["w10"])
    # large float arrays are stored in float32: parity is judged at fp32 level
    for k, v in list(out.items()):
        if isinstance(v, np.ndarray) and v.dtype == np.float64 and v.size > 1000:
            out[k] = v.astype(np.float32)
    np.savez_compressed(os.path.join(HERE, "tiny.npz"), **out)
    print("tiny: loss0 %.6f loss1 %.6f loss10 %.6f" % (out["loss0"], out["loss1"], out["loss10"]))


SMALL_CASES = [
    # (seed, U, I, nnz, d, b, alpha0, reg, nu, labels, partition)
    (1, 40, 30, 300, 8, 2, 0.1, 0.01, 1.0, "unit", None),
    (2, 37, 23, 400, 10, 4, 0.5, 0.003, 0.0, "real", None),   # remainder block
    (3, 50, 50, 500, 8, 1, 0.1, 0.05, 1.0, "real", None),     # b=1 (iCD)
    (4, 25, 45, 350, 8, 8, 0.5, 0.02, 1.0, "unit", None),     # b=d (iALS)
    (5, 60, 20, 600, 12, 5, 0.1, 0.001, 1.0, "real", None),   # remainder, skew
    (6, 30, 30, 200, 5, 2, 0.1, 0.01, 1.0, "real", [[1, 3], [0, 2, 4]]),  # permuted partition
    (7, 45, 35, 450, 16, 16, 0.1, 0.001, 1.0, "unit", None),
    (8, 33, 29, 250, 32, 8, 0.1, 0.001, 1.0, "real", None),
    (9, 80, 64, 900, 64, 32, 0.1, 0.001, 1.0, "unit", None),
    (10, 40, 40, 400, 48, 48, 0.1, 0.002, 1.0, "unit", None),
]


def make_small():
    out = {}
    for (seed, U, I, nnz, d, b, a0, reg, nu, lab, part) in SMALL_CASES:
        rng = np.random.default_rng(1000 + seed)
        users = rng.integers(0, U, nnz)
        items = rng.integers(0, I, nnz)
        # force empty rows on both sides
        users[users == U - 1] = 0
        items[items == I - 1] = 1
        labels = np.ones(nnz) if lab == "unit" else rng.uniform(0.0, 2.0, nnz)
        weights = np.ones(nnz) if lab == "unit" else rng.uniform(0.5, 2.0, nnz)
        data = ref.InteractionDataset(U, I, users, items, labels, weights)
        cfg = ref.SolverConfig(dim=d, block_size=b, unobserved_weight=a0, reg=reg,
                               reg_exponent=nu, epochs=3, seed=seed, threads=1)
        model = fp32_init(cfg, U, I)
        p = f"c{seed}_"
        out[p + "meta"] = np.array([U, I, nnz, d, b, a0, reg, nu], dtype=np.float64)
        out[p + "users"] = users
        out[p + "items"] = items
        out[p + "labels"] = labels
        out[p + "weights"] = weights
        out[p + "w0"] = model.user_factors.copy()
        out[p + "h0"] = model.item_factors.copy()
        out[p + "user_ptr"] = data.user_ptr
        out[p + "item_ptr"] = data.item_ptr
        out[p + "item_order"] = data.item_view().cache_pos
        out[p + "csr_items"] = data.items
        partition = None
        if part is not None:
            partition = ref.BlockPartition(tuple(np.array(x) for x in part), d)
            out[p + "partition"] = np.array([i for blk in part for i in blk] + [-1] +
                                            [len(blk) for blk in part])
        m = model.copy()
        cache = ref.PredictionCache.zeros(data.n_interactions)
        for e in range(3):
            ref.ialspp_epoch(m, data, cache, cfg, partition, e)
            if e == 0:
                out[p + "w1"] = m.user_factors.copy()
                out[p + "h1"] = m.item_factors.copy()
                out[p + "cache1"] = cache.scores.copy()
                out[p + "loss1"] = np.array(ref.compute_loss(m, data, cfg))
        out[p + "w3"] = m.user_factors.copy()
        out[p + "h3"] = m.item_factors.copy()
        out[p + "cache3"] = cache.scores.copy()
        out[p + "loss3"] = np.array(ref.compute_loss(m, data, cfg))
        # single block_update on the (non-first) block of the init, item side
        m = model.copy()
        cache = ref.compute_predictions(m, data)
        blocks = partition.blocks if partition is not None else ref.partition_dims(d, b).blocks
        blk = blocks[-1]
        ref.block_update(m, data, cache, cfg, blk, side="item")
        out[p + "bu_block"] = np.asarray(blk)
        out[p + "bu_h"] = m.item_factors.copy()
        out[p + "bu_cache"] = cache.scores.copy()
        out[p + "slab_w_last"] = ref.partial_gramian(model.user_factors, blk)
        out[p + "pred0"] = ref.compute_predictions(model, data).scores.copy()
        out[p + "loss0"] = np.array(ref.compute_loss(model, data, cfg))
    out["cases"] = np.array([c[0] for c in SMALL_CASES])
    np.savez_compressed(os.path.join(HERE, "small.npz"), **out)
    print("small: %d cases" % len(SMALL_CASES))


def _ragged(arrays, dtype):
    ptr = np.zeros(len(arrays) + 1, dtype=np.int64)
    ptr[1:] = np.cumsum([len(a) for a in arrays])
    flat = np.concatenate([np.asarray(a, dtype=dtype) for a in arrays]) if arrays else np.empty(0, dtype)
    return ptr, flat


def make_eval():
    from blockals import metrics as refm
    from blockals.pipeline import split_holdout
    U, I, users, items = synthetic.generate("tiny", 0)
    data = ref.InteractionDataset(U, I, users, items)
    split = split_holdout(data, 0.1, seed=0)
    cfg = ref.SolverConfig(dim=32, block_size=8, unobserved_weight=0.1, reg=1e-3,
                           reg_exponent=1.0, init_stddev=0.1, epochs=3, seed=0, threads=1)
    model = fp32_init(cfg, split.train.num_users, I)
    ref.train(model, split.train, cfg)
    hf = model.item_factors.astype(np.float32).astype(np.float64)   # what the GPU side holds
    evaluated = [f for f in split.folds if f.target_items.size > 0]
    emb = ref.fold_in_users(hf, [(f.input_items, f.input_labels, f.input_weights) for f in evaluated], cfg)
    topk = [refm.rank_items(emb[r], hf, exclude=f.input_items, k=100) for r, f in enumerate(evaluated)]
    rep = refm.evaluate_holdout(hf, split, cfg, recall_ks=(20, 50), ndcg_ks=(10, 100))
    out = {"item_factors": hf, "num_items": I, "embeddings": emb}
    out["in_ptr"], out["in_items"] = _ragged([f.input_items for f in split.folds], np.int64)
    out["tg_ptr"], out["tg_items"] = _ragged([f.target_items for f in split.folds], np.int64)
    out["topk_ptr"], out["topk"] = _ragged(topk, np.int64)
    out["recall_20"], out["recall_50"] = rep.recall_at[20], rep.recall_at[50]
    out["ndcg_10"], out["ndcg_100"] = rep.ndcg_at[10], rep.ndcg_at[100]
    out["n_evaluated"] = rep.num_users_evaluated
    # top_k_from_scores on tie-heavy integer scores, with exclusions
    rng = np.random.default_rng(5)
    sc, ex, tk, ks = [], [], [], []
    for case in range(12):
        n = int(rng.integers(1, 3000))
        s = rng.integers(-20, 20, n).astype(np.float64)
        e = rng.choice(n, int(rng.integers(0, n // 2 + 1)), replace=False) if case % 3 else np.empty(0, np.int64)
        k = int(rng.integers(1, 400)) if case != 5 else n + 10   # k beyond the pool
        sc.append(s); ex.append(e); ks.append(k)
        tk.append(refm.top_k_from_scores(s, k, exclude=e))
    out["tk_sptr"], out["tk_scores"] = _ragged(sc, np.float64)
    out["tk_eptr"], out["tk_exclude"] = _ragged(ex, np.int64)
    out["tk_optr"], out["tk_out"] = _ragged(tk, np.int64)
    out["tk_k"] = np.array(ks, dtype=np.int64)
    np.savez_compressed(os.path.join(HERE, "eval.npz"), **out)
    print("eval: %d folds, %d evaluated, recall@20 %.4f ndcg@100 %.4f" %
          (len(split.folds), rep.num_users_evaluated, rep.recall_at[20], rep.ndcg_at[100]))


if __name__ == "__main__":
    which = sys.argv[1:] or ["tiny", "small", "eval"]
    if "tiny" in which:
        make_tiny()
    if "small" in which:
        make_small()
    if "eval" in which:
        make_eval()
