"""Seeded synthetic interaction sets with the BASELINE.json shapes.

The reference's own generator (``data.py:165-208``) draws a fixed number of
items per user from a low-rank score, which cannot produce the Zipf item
popularity and lognormal per-user counts of the named ML20M / MSD shapes
(SURVEY.md §8d).  This module is the stand-in for those datasets; none of
their records are reproduced -- only their sizes and distribution shapes.

Recipe:
  * NumPy PCG64 seeded with ``seed``;
  * per-user counts ~ lognormal(mu, sigma) rounded and clipped to [1, I],
    with ``mu`` calibrated so that the expected total hits the target nnz;
  * each user's items are drawn *without replacement* with
    P(rank r) ∝ r^-s (successive sampling: with-replacement draws, first
    occurrences kept), ranks mapped to item ids by a random permutation;
  * labels y = 1 and weights a = 1 (implicit feedback);
  * the COO list is returned in a shuffled order so that the stable
    user-major sort of the CSR build is exercised.
"""

from __future__ import annotations

import hashlib
import math
from dataclasses import dataclass

import numpy as np

__all__ = ["SHAPES", "Shape", "generate", "digest"]


@dataclass(frozen=True)
class Shape:
    name: str
    num_users: int
    num_items: int
    target_nnz: int
    zipf_s: float
    sigma: float = 0.67


#: Config keys of SURVEY.md §8 (T, M/SW/L1/L2 share the ML20M-like shape, X is MSD-like).
SHAPES = {
    "tiny": Shape("tiny", 2_000, 1_000, 50_000, 1.0),
    "mid": Shape("mid", 136_677, 20_108, 10_000_000, 1.0),
    "msd": Shape("msd", 571_355, 41_140, 33_600_000, 1.1),
}


def _expected_total(mu, sigma, n_users, n_items, z):
    c = np.clip(np.rint(np.exp(mu + sigma * z)), 1, n_items)
    return float(c.sum())


def _user_counts(rng, shape: Shape):
    z = rng.standard_normal(shape.num_users)
    lo, hi = -5.0, 12.0
    for _ in range(60):   # bisection on mu: total count of this draw == target
        mid = 0.5 * (lo + hi)
        if _expected_total(mid, shape.sigma, shape.num_users, shape.num_items, z) < shape.target_nnz:
            lo = mid
        else:
            hi = mid
    mu = 0.5 * (lo + hi)
    return np.clip(np.rint(np.exp(mu + shape.sigma * z)), 1, shape.num_items).astype(np.int64)


def _first_occurrences(key, n_old):
    """Indices (>= n_old, in input order) of entries of ``key`` whose value
    does not occur earlier in ``key`` (stable sort-based dedupe)."""
    order = np.argsort(key, kind="stable")
    ks = key[order]
    first = np.ones(ks.size, dtype=bool)
    first[1:] = ks[1:] != ks[:-1]
    idx = order[first]
    idx = idx[idx >= n_old]
    idx.sort()
    return idx


def _draw_without_replacement(rng, counts, n_items, s):
    """Per-user distinct item ranks, successive sampling from P(r) ∝ (r+1)^-s."""
    weights = (np.arange(1, n_items + 1, dtype=np.float64)) ** (-s)
    cdf = np.cumsum(weights)
    cdf /= cdf[-1]
    n_users = counts.size
    have = np.zeros(n_users, dtype=np.int64)
    seen = np.empty(0, dtype=np.int64)
    got_users, got_ranks = [], []
    over = 1.5
    pending = np.flatnonzero(counts > 0)
    while pending.size:
        m = np.maximum(np.ceil((counts[pending] - have[pending]) * over).astype(np.int64) + 4, 8)
        uu = np.repeat(pending, m)
        rr = np.searchsorted(cdf, rng.random(uu.size), side="right")
        rr = np.minimum(rr, n_items - 1)
        key = uu * n_items + rr
        keep = _first_occurrences(np.concatenate([seen, key]), seen.size) - seen.size
        uu, rr, key = uu[keep], rr[keep], key[keep]
        # at most (counts - have) new items per user, in draw order
        order = np.argsort(uu, kind="stable")
        uu, rr, key = uu[order], rr[order], key[order]
        per = np.bincount(uu, minlength=n_users)
        start = np.concatenate([[0], np.cumsum(per)[:-1]])
        within = np.arange(uu.size) - start[uu]
        ok = within < (counts - have)[uu]
        uu, rr, key = uu[ok], rr[ok], key[ok]
        got_users.append(uu)
        got_ranks.append(rr)
        have += np.bincount(uu, minlength=n_users)
        seen = np.concatenate([seen, key])
        pending = np.flatnonzero(have < counts)
        over *= 2.0
    return np.concatenate(got_users), np.concatenate(got_ranks)


def generate(shape: str | Shape, seed: int = 0):
    """Return ``(num_users, num_items, users, items)`` (int64 COO, shuffled)."""
    if isinstance(shape, str):
        shape = SHAPES[shape]
    rng = np.random.default_rng(seed)
    counts = _user_counts(rng, shape)
    id_of_rank = rng.permutation(shape.num_items)
    users, ranks = _draw_without_replacement(rng, counts, shape.num_items, shape.zipf_s)
    items = id_of_rank[ranks]
    shuffle = rng.permutation(users.size)
    return (shape.num_users, shape.num_items,
            np.ascontiguousarray(users[shuffle], dtype=np.int64),
            np.ascontiguousarray(items[shuffle], dtype=np.int64))


def digest(users, items) -> str:
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(users, dtype=np.int64).tobytes())
    h.update(np.ascontiguousarray(items, dtype=np.int64).tobytes())
    return h.hexdigest()


def subsample_users(num_users, num_items, users, items, keep_users, seed=0):
    """Instance restricted to ``keep_users`` users (renumbered 0..k-1)."""
    rng = np.random.default_rng(seed)
    sel = np.sort(rng.choice(num_users, size=keep_users, replace=False))
    remap = -np.ones(num_users, dtype=np.int64)
    remap[sel] = np.arange(keep_users)
    mask = remap[users] >= 0
    return keep_users, num_items, remap[users[mask]], items[mask]
