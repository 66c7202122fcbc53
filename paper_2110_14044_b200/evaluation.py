"""Fold-in and ranking evaluation on the device.

Host mirror of the reference's ``project_user`` / ``fold_in_users``
(/root/reference/pkg/src/blockals/solvers.py:416-466) and ``metrics.py``
(``top_k_from_scores``, ``rank_items``, ``recall_at_k``, ``ndcg_at_k``,
``evaluate_holdout``, metrics.py:31-119), same names, arguments and errors.

* Fold-in solves, per history, the same regularized least squares as a user
  pass.  On the device that is one user pass of the block sweep with a single
  block of width d from a zero embedding and a zero cache: the Newton step
  from w = 0 is the closed-form solve (any d: widths above 256 take the
  batched wide solver, csrc/ials_sweep_wide.cuh).
* Scores are the repo's own 3xTF32 tensor-core GEMM (``ials_scores``: the TMA
  GEMM of the epoch with 128-item output tiles, FP32-accurate); the exclusion
  of each user's input items and the top-k with the reference's tie order run
  in ``ials_topk`` (csrc/ials_topk.cuh).  ``top_k_from_scores`` on the
  caller's float64 scores ranks the f64 values themselves (``ials_topk64``).
* recall / NDCG are the reference's set arithmetic on the top-k lists.
* k above 1024 (the kernel's selection buffer) uses a stable device sort of
  the row instead (torch.sort), with the same order.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from ._runtime import default_engine_session
from .data import InteractionDataset
from .engine import _ptr, current_stream_handle
from .model import FactorModel, PredictionCache, SolverConfig
from .solvers import block_update

__all__ = ["MetricReport", "project_user", "fold_in_users", "top_k_from_scores", "rank_items",
           "recall_at_k", "ndcg_at_k", "evaluate_holdout"]

_MAX_K = 1024


@dataclass
class MetricReport:
    """Per-k metric means over the evaluated user set."""

    recall_at: dict
    ndcg_at: dict
    num_users_evaluated: int


def fold_in_users(item_factors, histories, config: SolverConfig, device=None) -> np.ndarray:
    """Embeddings for a batch of histories, one per (items, labels, weights)
    (labels / weights may be None); shape (len(histories), dim)."""
    if config is None:
        raise ValueError("config is required")
    hf = np.ascontiguousarray(item_factors, dtype=np.float64)
    n_items, d = hf.shape
    users, items, labels, weights = [], [], [], []
    for row, (its, lbl, wts) in enumerate(histories):
        its = np.asarray(its, dtype=np.int64)
        users.append(np.full(its.size, row, dtype=np.int64))
        items.append(its)
        labels.append(np.ones(its.size) if lbl is None else np.asarray(lbl, dtype=np.float64))
        weights.append(np.ones(its.size) if wts is None else np.asarray(wts, dtype=np.float64))
    out = np.zeros((len(histories), d))
    if not histories or not sum(a.size for a in items):
        return out   # empty histories: the right-hand side is zero
    data = InteractionDataset(len(histories), n_items, np.concatenate(users), np.concatenate(items),
                              np.concatenate(labels), np.concatenate(weights))
    model = FactorModel(out, hf)
    cache = PredictionCache.zeros(data.n_interactions)   # exact for the zero embedding
    block_update(model, data, cache, config.with_(dim=d, block_size=d), np.arange(d), "user", device)
    return model.user_factors


def project_user(item_factors, items, labels=None, weights=None,
                 config: SolverConfig | None = None, item_gram=None, device=None) -> np.ndarray:
    """Embedding for a single interaction history against fixed item factors
    (``item_gram`` is accepted for signature parity; the device forms its own)."""
    if config is None:
        raise ValueError("config is required")
    return fold_in_users(item_factors, [(items, labels, weights)], config, device)[0]


def _padded_f32(a, device) -> torch.Tensor:
    """A 2-d float32 device copy whose row stride is a multiple of 4 floats
    (the TMA maps of ials_scores), padding columns zero."""
    a = np.asarray(a, dtype=np.float32)
    n, d = a.shape
    ld = (d + 3) & ~3
    t = torch.zeros((max(n, 1), ld), dtype=torch.float32, device=device)[:n]
    t[:, :d] = torch.from_numpy(np.ascontiguousarray(a)).to(device)
    return t


def device_scores(E: torch.Tensor, H: torch.Tensor, d: int) -> torch.Tensor:
    """E @ H^T (rows of E x rows of H) with ials_scores; E / H from _padded_f32."""
    rt = default_engine_session(E.device)
    n_u, n_i = E.shape[0], H.shape[0]
    out = torch.empty((max(n_u, 1), max(n_i, 1)), dtype=torch.float32, device=E.device)[:n_u, :n_i]
    rc = rt.lib.ials_scores(rt.session.handle, _ptr(E), E.stride(0), n_u, _ptr(H), H.stride(0), n_i,
                            d, _ptr(out), out.stride(0), current_stream_handle(E.device))
    rt.session.check(rc, "scores")
    return out


def _topk_device(scores: torch.Tensor, k: int, ex_ptr=None, ex_cols=None, as_tensor=False):
    """Rows of a device score matrix (fp32: ials_topk, f64: ials_topk64) ->
    top-k index lists, or the (index, count) device tensors."""
    rt = default_engine_session(scores.device)
    n_rows, n_cols = scores.shape
    out = torch.empty((max(n_rows, 1), k), dtype=torch.int32, device=scores.device)
    counts = torch.empty(max(n_rows, 1), dtype=torch.int32, device=scores.device)
    fn = rt.lib.ials_topk64 if scores.dtype == torch.float64 else rt.lib.ials_topk
    rc = fn(rt.session.handle, n_rows, n_cols, _ptr(scores), scores.stride(0), _ptr(ex_ptr),
            _ptr(ex_cols), k, _ptr(out), _ptr(counts), current_stream_handle(scores.device))
    rt.session.check(rc, "topk")
    if as_tensor:
        return out[:n_rows], counts[:n_rows]
    o, c = out.cpu().numpy(), counts.cpu().numpy()
    return [o[r, :c[r]].astype(np.int64) for r in range(n_rows)]


def _exclusion_csr(exclude, device):
    if exclude is None:
        return None, None
    ex = np.asarray(list(exclude) if not isinstance(exclude, np.ndarray) else exclude, dtype=np.int64)
    if not ex.size:
        return None, None
    return (torch.tensor([0, ex.size], dtype=torch.int32, device=device),
            torch.from_numpy(ex.astype(np.int32)).to(device))


def _top_k_row(scores: torch.Tensor, k, exclude) -> np.ndarray:
    if k < 1:
        raise ValueError("k must be positive")
    kk = int(min(k, max(scores.numel(), 1)))
    if kk > _MAX_K:
        # beyond the in-kernel selection buffer: a full stable sort of the row
        # on the device (descending; equal scores keep ascending index order)
        s = scores.reshape(-1).clone()
        ex = _exclusion_csr(exclude, scores.device)[1]
        if ex is not None:
            s[ex.long()] = -float("inf")
        s = torch.where(torch.isfinite(s), s + 0.0, torch.full_like(s, -float("inf")))
        pool = int(torch.isfinite(s).sum())
        order = torch.sort(s, descending=True, stable=True).indices
        return order[:min(kk, pool)].cpu().numpy().astype(np.int64)
    ptr, cols = _exclusion_csr(exclude, scores.device)
    return _topk_device(scores.reshape(1, -1).contiguous(), kk, ptr, cols)[0]


def top_k_from_scores(scores, k, exclude=None, device=None) -> np.ndarray:
    """Indices of the k largest scores, ties broken by ascending index;
    excluded indices and non-finite scores never appear."""
    if k < 1:
        raise ValueError("k must be positive")
    rt = default_engine_session(device)
    # the caller's float64 scores are ranked as float64 (ials_topk64): no
    # rounding can merge or reorder near-ties before the selection
    s = torch.from_numpy(np.ascontiguousarray(scores, dtype=np.float64)).to(rt.device)
    return _top_k_row(s, k, exclude)


def rank_items(user_embedding, item_factors, exclude=None, k=10, device=None) -> np.ndarray:
    """Top-k item indices for a user embedding, excluding ``exclude``."""
    rt = default_engine_session(device)
    hf = np.asarray(item_factors)
    H = _padded_f32(hf, rt.device)
    E = _padded_f32(np.asarray(user_embedding, dtype=np.float64).reshape(1, -1), rt.device)
    return _top_k_row(device_scores(E, H, hf.shape[1])[0], k, exclude)


def recall_at_k(topk, targets, k) -> float:
    """Hits among the first k over ``min(k, |targets|)``."""
    targets = set(np.asarray(targets).tolist())
    if not targets:
        raise ValueError("targets must be nonempty")
    hits = sum(1 for item in list(topk)[:k] if item in targets)
    return hits / min(k, len(targets))


def ndcg_at_k(topk, targets, k) -> float:
    """Truncated NDCG with binary relevance (ideal DCG puts all targets first)."""
    targets = set(np.asarray(targets).tolist())
    if not targets:
        raise ValueError("targets must be nonempty")
    dcg = sum(1.0 / math.log2(p + 1) for p, item in enumerate(list(topk)[:k], start=1)
              if item in targets)
    ideal = sum(1.0 / math.log2(p + 1) for p in range(1, min(k, len(targets)) + 1))
    return dcg / ideal


def evaluate_holdout(item_factors, split, config, recall_ks=(20, 50), ndcg_ks=(100,),
                     device=None, users_per_batch=None) -> MetricReport:
    """Fold in every held-out user, rank unseen items, average the metrics.
    Users with an empty target fold are skipped; input-fold items are
    excluded from each user's candidates.  ``split`` is a HoldoutSplit-like
    object with ``folds`` or a list of folds (``input_items``,
    ``input_labels``, ``input_weights``, ``target_items``)."""
    if not recall_ks and not ndcg_ks:
        raise ValueError("at least one k is required")
    folds = split.folds if hasattr(split, "folds") else list(split)
    evaluated = [f for f in folds if np.asarray(f.target_items).size > 0]
    if not evaluated:
        raise ValueError("no holdout users with target interactions")
    k_max = max(list(recall_ks) + list(ndcg_ks))
    if k_max > _MAX_K:
        raise ValueError(f"device top-k supports k <= {_MAX_K}")
    emb = fold_in_users(item_factors, [(f.input_items, f.input_labels, f.input_weights)
                                       for f in evaluated], config, device)
    rt = default_engine_session(device)
    dev = rt.device
    d = np.asarray(item_factors).shape[1]
    H = _padded_f32(item_factors, dev)
    n_items = H.shape[0]
    E = _padded_f32(emb, dev)
    ex = [np.asarray(f.input_items, dtype=np.int64) for f in evaluated]
    ex_ptr = np.zeros(len(ex) + 1, dtype=np.int64)
    ex_ptr[1:] = np.cumsum([a.size for a in ex])
    ex_cols = torch.from_numpy(np.concatenate(ex).astype(np.int32) if ex_ptr[-1] else
                               np.zeros(1, np.int32)).to(dev)
    if users_per_batch is None:   # score matrices of at most ~1 GB
        users_per_batch = max(1, (1 << 28) // max(n_items, 1))
    recall_sums = {k: 0.0 for k in recall_ks}
    ndcg_sums = {k: 0.0 for k in ndcg_ks}
    k_run = min(k_max, n_items)
    for r0 in range(0, len(evaluated), users_per_batch):
        r1 = min(len(evaluated), r0 + users_per_batch)
        scores = device_scores(E[r0:r1], H, d)
        ptr = torch.from_numpy((ex_ptr[r0:r1 + 1] - ex_ptr[r0]).astype(np.int32)).to(dev)
        cols = ex_cols[int(ex_ptr[r0]):] if ex_ptr[r1] > ex_ptr[r0] else ex_cols
        tops = _topk_device(scores, k_run, ptr, cols)
        for r in range(r0, r1):
            topk, targets = tops[r - r0], evaluated[r].target_items
            for k in recall_ks:
                recall_sums[k] += recall_at_k(topk, targets, k)
            for k in ndcg_ks:
                ndcg_sums[k] += ndcg_at_k(topk, targets, k)
    n = len(evaluated)
    return MetricReport({k: v / n for k, v in recall_sums.items()},
                        {k: v / n for k, v in ndcg_sums.items()}, n)
