"""CPU oracle for the iALS++ hot path -- TEST INFRASTRUCTURE ONLY.

This module is a float64 NumPy restatement of the reference's iALS++ epoch
(``/root/reference/pkg/src/blockals``, package ``blockals`` 0.1.0).  It exists
so that ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` have a checker and a CPU timing arm
on the GPU box, where ``/root/reference`` does not exist.  The product path
(``paper_2110_14044_b200``) never imports it.

Pinning: ``tests/test_oracle_golden.py`` checks every function here against
golden vectors produced by the *unmodified reference* (``tests/golden/
make_golden.py`` imports ``blockals`` from ``/root/reference/pkg/src`` in the
CPU container and writes ``tests/golden/*.npz``).  Parity is therefore pinned
to the reference itself, not only to this restatement.

Each function cites the reference lines it restates.  The structure is my
own: rows are batched on a x1.25 geometric degree grid (finer than the
reference's power-of-two buckets, ``data.py:54-85``) with zero-weight padding
entries; like the reference, the batched solve is LAPACK gesv
(``solvers.py:101-114``) and a failing batch is diagnosed row by row with a
Cholesky to name the row and pivot.
"""

from __future__ import annotations

import math

import numpy as np

__all__ = [
    "SingularRow", "build_csr", "effective_reg", "init_factors", "partition",
    "predictions", "gramian", "partial_gramian", "side_pass", "ialspp_epoch",
    "train", "loss", "cache_drift", "systematic_rows",
    "fold_in", "top_k", "recall_at_k", "ndcg_at_k", "evaluate",
]

_ROW_BATCH_ELEMS = 1 << 21     # gathered (rows x degree x block) elements per batch
_GRID = 1.25                   # degree classes: widths on a geometric grid


class SingularRow(np.linalg.LinAlgError):
    """Non-positive pivot in a row's block Hessian (``linalg.py:18-28``,
    ``solvers.py:101-114``): carries the offending ``row`` and ``pivot``."""

    def __init__(self, row, pivot):
        super().__init__(f"normal equations singular for row {row} (pivot {pivot})")
        self.row, self.pivot = int(row), int(pivot)


# --------------------------------------------------------------------------- data
def _stable_bucket_order(keys: np.ndarray, nbuckets: int):
    """Stable bucket order of ``keys`` and the bucket offsets: (order, ptr).

    ``order`` lists element indices bucket by bucket, keeping input order
    inside a bucket (a stable counting sort, written with NumPy's stable
    merge sort), ``ptr`` is the exclusive prefix sum of the histogram.
    """
    counts = np.bincount(keys, minlength=nbuckets).astype(np.int64)
    ptr = np.zeros(nbuckets + 1, dtype=np.int64)
    np.cumsum(counts, out=ptr[1:])
    order = np.argsort(keys, kind="mergesort").astype(np.int64)
    return order, ptr


def build_csr(num_users, num_items, users, items, labels=None, weights=None):
    """Canonical user-major interaction order and both side views.

    Restates ``InteractionDataset.__init__`` (data.py:98-134) and
    ``user_view``/``item_view`` (data.py:148-162): a stable sort by user gives
    the canonical order (duplicates kept, data.py:95-96), ``user_ptr`` is the
    cumulative user histogram, ``item_order`` is the stable item-major
    permutation of canonical positions and ``item_ptr`` its histogram.
    """
    users = np.ascontiguousarray(users, dtype=np.int64)
    items = np.ascontiguousarray(items, dtype=np.int64)
    n = users.size
    labels = np.ones(n) if labels is None else np.asarray(labels, dtype=np.float64)
    weights = np.ones(n) if weights is None else np.asarray(weights, dtype=np.float64)
    order, user_ptr = _stable_bucket_order(users, int(num_users))
    out = {
        "num_users": int(num_users), "num_items": int(num_items),
        "users": users[order], "items": items[order],
        "labels": labels[order], "weights": weights[order],
        "user_ptr": user_ptr,
    }
    item_order, item_ptr = _stable_bucket_order(out["items"], int(num_items))
    out["item_order"] = item_order
    out["item_ptr"] = item_ptr
    return out


def side_view(csr, side):
    """(ptr, cols, labels, weights, cache_pos) of one side (data.py:148-162)."""
    if side == "user":
        return (csr["user_ptr"], csr["items"], csr["labels"], csr["weights"],
                np.arange(csr["users"].size, dtype=np.int64))
    perm = csr["item_order"]
    return (csr["item_ptr"], csr["users"][perm], csr["labels"][perm],
            csr["weights"][perm], perm)


# -------------------------------------------------------------------------- model
def effective_reg(counts, opposite_size, reg, alpha0, exponent):
    """``reg * (count + alpha0 * opposite_size) ** exponent`` (model.py:144-150)."""
    base = np.asarray(counts, dtype=np.float64) + alpha0 * opposite_size
    return reg * base ** exponent


def init_factors(num_users, num_items, dim, init_stddev=0.1, seed=0):
    """W then H, i.i.d. N(0, (init_stddev/sqrt(dim))^2) from one PCG64 stream
    (model.py:123-134)."""
    rng = np.random.default_rng(seed)
    scale = init_stddev / math.sqrt(dim)
    w = rng.normal(0.0, scale, size=(int(num_users), int(dim)))
    h = rng.normal(0.0, scale, size=(int(num_items), int(dim)))
    return w, h


def partition(dim, block_size):
    """Contiguous blocks with the remainder last (solvers.py:83-92)."""
    if not 1 <= block_size <= dim:
        raise ValueError("block_size must be in [1, dim]")
    return [np.arange(s, min(s + block_size, dim)) for s in range(0, dim, block_size)]


def predictions(w, h, users, items, chunk=None):
    """yhat_k = <w[users_k], h[items_k]> in canonical order (model.py:153-165)."""
    if chunk is None:     # bound the gathered temporaries to ~256 MB
        chunk = max(1024, (1 << 25) // max(1, w.shape[1]))
    out = np.empty(users.size)
    for s in range(0, users.size, chunk):
        e = min(s + chunk, users.size)
        out[s:e] = np.einsum("kd,kd->k", w[users[s:e]], h[items[s:e]])
    return out


# ------------------------------------------------------------------------- linalg
def gramian(m):
    """M^T M (linalg.py:31-36)."""
    m = np.asarray(m, dtype=np.float64)
    return m.T @ m


def partial_gramian(m, block):
    """The d x |block| slab M^T M[:, block] (linalg.py:39-45)."""
    m = np.asarray(m, dtype=np.float64)
    return m.T @ m[:, np.asarray(block)]


def _first_bad_pivot(mat):
    """Index of the first non-positive pivot of an (assumed failing) Cholesky."""
    a = np.array(mat, dtype=np.float64)
    n = a.shape[0]
    for j in range(n):
        d = a[j, j] - a[j, :j] @ a[j, :j]
        if not d > 0:
            return j
        a[j, j] = math.sqrt(d)
        a[j + 1:, j] = (a[j + 1:, j] - a[j + 1:, :j] @ a[j, :j]) / a[j, j]
    return n - 1


# ------------------------------------------------------------------------- solver
def side_pass(ptr, cols, labels, weights, cache_pos, fixed, update, cache, block,
              slab, alpha0, lam_rows, rows=None):
    """One exact Newton step on ``block`` of every row of one side.

    Restates ``_newton_side_pass`` (solvers.py:152-186), stages 1-7:
      h_k = F[col_k, pi]; rho_k = a_k (yhat_k - y_k); g = sum rho_k h_k
      g += alpha0 * U[r,:] @ slab + lam_r U[r,pi]
      Hs = sum a_k h_k h_k^T + alpha0 slab[pi,:] + lam_r I
      delta = Hs^-1 g; U[r,pi] -= delta; yhat_k -= h_k . delta
    ``update`` and ``cache`` are modified in place.  ``rows`` optionally
    restricts the pass to a subset of rows (used for bounded CPU timing).
    """
    block = np.asarray(block)
    p = block.size
    slab_pp = slab[block, :]
    # block columns of the fixed side plus one all-zero sentinel row that padded
    # entries point at (weight 0, label 0, cache slot -> scratch)
    fixed_blk = np.zeros((fixed.shape[0] + 1, p))
    fixed_blk[:-1] = fixed[:, block]
    sentinel = fixed.shape[0]
    counts = np.diff(ptr)
    if rows is None:
        rows = np.arange(counts.size)
    rows = np.asarray(rows, dtype=np.int64)
    deg = counts[rows]
    # batch rows whose degree rounds up to the same width on a x1.25 geometric grid
    width = np.where(deg > 0, np.ceil(_GRID ** np.ceil(np.log(np.maximum(deg, 1)) / np.log(_GRID))),
                     0).astype(np.int64)
    width = np.maximum(width, deg)
    eye = np.eye(p)
    cache_ext = np.append(cache, 0.0)
    scratch = cache.size
    for n in np.unique(width):
        grp = rows[width == n]
        step = max(1, _ROW_BATCH_ELEMS // max(1, int(n) * p))
        for s in range(0, grp.size, step):
            r = grp[s:s + step]
            off = np.arange(n)[None, :]
            valid = off < counts[r][:, None]                         # (m, n)
            idx = np.where(valid, ptr[r][:, None] + off, 0)
            x = fixed_blk[np.where(valid, cols[idx], sentinel)]      # (m, n, p)
            a = np.where(valid, weights[idx], 0.0)
            pos = np.where(valid, cache_pos[idx], scratch)
            rho = a * (cache_ext[pos] - np.where(valid, labels[idx], 0.0))
            w_full = update[r]
            w_blk = w_full[:, block]
            lam = lam_rows[r]
            g = np.matmul(rho[:, None, :], x)[:, 0, :]
            g += alpha0 * (w_full @ slab) + lam[:, None] * w_blk
            hs = np.matmul(np.swapaxes(x * a[:, :, None], 1, 2), x)
            hs += alpha0 * slab_pp + lam[:, None, None] * eye
            try:
                delta = np.linalg.solve(hs, g[:, :, None])[:, :, 0]
            except np.linalg.LinAlgError:
                for i in range(r.size):
                    try:
                        np.linalg.cholesky(hs[i])
                    except np.linalg.LinAlgError:
                        raise SingularRow(r[i], _first_bad_pivot(hs[i])) from None
                raise
            update[np.ix_(r, block)] = w_blk - delta
            cache_ext[pos] -= np.matmul(x, delta[:, :, None])[:, :, 0]
            cache_ext[scratch] = 0.0
    cache[:] = cache_ext[:-1]


def side_regs(csr, alpha0, reg, exponent):
    """(lam_users, lam_items) (solvers.py:210-213)."""
    lu = effective_reg(np.diff(csr["user_ptr"]), csr["num_items"], reg, alpha0, exponent)
    li = effective_reg(np.diff(csr["item_ptr"]), csr["num_users"], reg, alpha0, exponent)
    return lu, li


def ialspp_epoch(w, h, csr, cache, alpha0, reg, exponent, blocks):
    """One iALS++ epoch in place (solvers.py:340-375): recompute the cache,
    then for each block a user pass against H's slab and an item pass against
    the (already updated) W's slab.  Returns the per-phase seconds dict."""
    import time
    lam_u, lam_i = side_regs(csr, alpha0, reg, exponent)
    t = {"cache": 0.0, "gramian": 0.0, "user": 0.0, "item": 0.0}
    t0 = time.perf_counter()
    cache[:] = predictions(w, h, csr["users"], csr["items"])
    t["cache"] += time.perf_counter() - t0
    uview, iview = side_view(csr, "user"), side_view(csr, "item")
    for block in blocks:
        t0 = time.perf_counter()
        slab = partial_gramian(h, block)
        t["gramian"] += time.perf_counter() - t0
        t0 = time.perf_counter()
        side_pass(*uview, h, w, cache, block, slab, alpha0, lam_u)
        t["user"] += time.perf_counter() - t0
        t0 = time.perf_counter()
        slab = partial_gramian(w, block)
        t["gramian"] += time.perf_counter() - t0
        t0 = time.perf_counter()
        side_pass(*iview, w, h, cache, block, slab, alpha0, lam_i)
        t["item"] += time.perf_counter() - t0
    return t


def train(w, h, csr, alpha0, reg, exponent, block_size, epochs):
    """``epochs`` iALS++ epochs (solvers.py:378-413); returns the cache."""
    cache = np.zeros(csr["users"].size)
    blocks = partition(w.shape[1], block_size)
    for _ in range(epochs):
        ialspp_epoch(w, h, csr, cache, alpha0, reg, exponent, blocks)
    return cache


def loss(w, h, csr, alpha0, reg, exponent):
    """Weighted squared error + alpha0 <W^T W, H^T H> + frequency-scaled L2
    (model.py:168-188)."""
    s = predictions(w, h, csr["users"], csr["items"])
    err = s - csr["labels"]
    obs = float(np.dot(csr["weights"] * err, err))
    unobs = alpha0 * float(np.sum(gramian(w) * gramian(h)))
    lu, li = side_regs(csr, alpha0, reg, exponent)
    l2 = float(np.dot(lu, np.einsum("ud,ud->u", w, w)))
    l2 += float(np.dot(li, np.einsum("id,id->i", h, h)))
    return obs + unobs + l2


def cache_drift(cache, w, h, csr):
    """max |cached - fresh| / (1 + |fresh|) (model.py:191-198)."""
    fresh = predictions(w, h, csr["users"], csr["items"])
    return float(np.max(np.abs(cache - fresh) / (1.0 + np.abs(fresh)), initial=0.0))


def systematic_rows(counts, stride, run=64):
    """A low-variance row sample for bounded CPU timing of a side pass.

    Returns ``(head, tail)``: ``head`` = the ``run`` highest-degree rows (timed
    in full, weight 1 -- they dominate heavy-tailed item sides), ``tail`` =
    every ``stride``-th run of ``run`` consecutive rows of the remaining
    degree-sorted list (weight ``stride``; rows of equal degree still batch as
    in a full pass)."""
    order = np.argsort(-np.asarray(counts), kind="stable")
    if stride <= 1:
        return np.sort(order), np.empty(0, dtype=np.int64)
    head, rest = order[:run], order[run:]
    starts = np.arange(0, rest.size, stride * run)
    tail = np.concatenate([rest[s:s + run] for s in starts]) if starts.size else rest[:0]
    return np.sort(head), np.sort(tail)


# ----------------------------------------------------------- fold-in / ranking
# (pinned by tests/golden/eval.npz from the reference)

def fold_in(item_factors, histories, alpha0, reg, exponent):
    """Exact least-squares embedding per history (project_user / fold_in_users,
    solvers.py:416-466): (sum a h h' + alpha0 G + lam I)^-1 sum a y h with
    lam = reg (n + alpha0 I)^exponent; an empty history gives zeros."""
    hf = np.asarray(item_factors, dtype=np.float64)
    n_items, d = hf.shape
    g = hf.T @ hf
    out = np.zeros((len(histories), d))
    for r, (its, lbl, wts) in enumerate(histories):
        its = np.asarray(its, dtype=np.int64)
        n = its.size
        lbl = np.ones(n) if lbl is None else np.asarray(lbl, dtype=np.float64)
        wts = np.ones(n) if wts is None else np.asarray(wts, dtype=np.float64)
        rows = hf[its]
        hess = rows.T @ (rows * wts[:, None]) + alpha0 * g
        hess[np.arange(d), np.arange(d)] += reg * (n + alpha0 * n_items) ** exponent
        out[r] = np.linalg.solve(hess, rows.T @ (wts * lbl))
    return out


def top_k(scores, k, exclude=None):
    """Indices of the k largest scores, ties by ascending index, excluded and
    non-finite scores never returned (top_k_from_scores, metrics.py:31-57)."""
    s = np.asarray(scores, dtype=np.float64).copy()
    if exclude is not None and len(exclude):
        s[np.asarray(exclude, dtype=np.intp)] = -np.inf
    cand = np.flatnonzero(np.isfinite(s))
    order = np.lexsort((cand, -s[cand]))
    return cand[order][:min(int(k), cand.size)]


def recall_at_k(topk, targets, k):
    """Hits among the first k over min(k, |targets|) (metrics.py:66-72)."""
    t = set(np.asarray(targets).tolist())
    hits = sum(1 for i in list(topk)[:k] if i in t)
    return hits / min(k, len(t))


def ndcg_at_k(topk, targets, k):
    """Binary-relevance NDCG truncated at k (metrics.py:75-92)."""
    t = set(np.asarray(targets).tolist())
    dcg = sum(1.0 / math.log2(p + 1) for p, i in enumerate(list(topk)[:k], start=1) if i in t)
    ideal = sum(1.0 / math.log2(p + 1) for p in range(1, min(k, len(t)) + 1))
    return dcg / ideal


def evaluate(item_factors, folds, alpha0, reg, exponent, recall_ks, ndcg_ks):
    """evaluate_holdout (metrics.py:95-119) over (input_items, labels, weights,
    target_items) tuples; returns ({k: recall}, {k: ndcg}, n_evaluated)."""
    ev = [f for f in folds if len(f[3]) > 0]
    emb = fold_in(item_factors, [(f[0], f[1], f[2]) for f in ev], alpha0, reg, exponent)
    hf = np.asarray(item_factors, dtype=np.float64)
    kmax = max(list(recall_ks) + list(ndcg_ks))
    rs = {k: 0.0 for k in recall_ks}
    ns = {k: 0.0 for k in ndcg_ks}
    for r, f in enumerate(ev):
        tk = top_k(hf @ emb[r], kmax, exclude=f[0])
        for k in recall_ks:
            rs[k] += recall_at_k(tk, f[3], k)
        for k in ndcg_ks:
            ns[k] += ndcg_at_k(tk, f[3], k)
    n = len(ev)
    return {k: v / n for k, v in rs.items()}, {k: v / n for k, v in ns.items()}, n
