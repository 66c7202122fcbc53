"""Interaction storage: canonical user-major CSR plus the item-major mirror.

Host mirror of the reference ``InteractionDataset`` / ``SideView``
(``data.py:26-52, 88-162``): the same constructor, validation errors,
attributes and view semantics, so callers of the reference can pass either
class.  The CSR arrays are bit-identical to the reference's (stable sort by
user for the canonical order, stable item-major permutation; checked by
``tests/test_host.py`` against the golden fixtures).  The reference's padded
degree buckets (``data.py:54-85``) are a NumPy batching device and are not
rebuilt: the GPU schedules rows by degree instead (engine.DeviceSide.schedule).
"""

from __future__ import annotations

import numpy as np

__all__ = ["InteractionDataset", "SideView"]


class SideView:
    """One side's adjacency: entries of row ``r`` are ``ptr[r]:ptr[r+1]``;
    ``cache_pos`` maps each entry to its canonical (user-major) cache slot."""

    def __init__(self, n_rows, n_cols, ptr, cols, labels, weights, cache_pos):
        self.n_rows, self.n_cols = int(n_rows), int(n_cols)
        self.ptr, self.cols = ptr, cols
        self.labels, self.weights = labels, weights
        self.cache_pos = cache_pos
        self.n_entries = int(cols.size)

    @property
    def counts(self) -> np.ndarray:
        return np.diff(self.ptr)

    def row_slice(self, row: int) -> slice:
        return slice(int(self.ptr[row]), int(self.ptr[row + 1]))


def _histogram_offsets(keys, n):
    ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(keys, minlength=n), out=ptr[1:])
    return ptr


class InteractionDataset:
    """Weighted, labelled (user, item) observations; duplicates are kept."""

    def __init__(self, num_users, num_items, users, items, labels=None, weights=None):
        users = np.ascontiguousarray(users, dtype=np.int64)
        items = np.ascontiguousarray(items, dtype=np.int64)
        if users.ndim != 1 or items.ndim != 1 or users.shape != items.shape:
            raise ValueError("users and items must be 1-d arrays of equal length")
        num_users, num_items = int(num_users), int(num_items)
        if min(num_users, num_items) < 1:
            raise ValueError("dataset needs at least one user and one item")
        n = users.size
        labels = np.ones(n) if labels is None else np.ascontiguousarray(labels, dtype=np.float64)
        weights = np.ones(n) if weights is None else np.ascontiguousarray(weights, dtype=np.float64)
        if labels.shape != (n,) or weights.shape != (n,):
            raise ValueError("labels and weights must match the interaction count")
        if n:
            if users.min() < 0 or users.max() >= num_users:
                raise ValueError("user index out of range")
            if items.min() < 0 or items.max() >= num_items:
                raise ValueError("item index out of range")
            if not np.all(np.isfinite(labels)):
                raise ValueError("labels must be finite")
            if not np.all(np.isfinite(weights)) or np.any(weights <= 0):
                raise ValueError("weights must be finite and strictly positive")
        canon = np.argsort(users, kind="stable")        # canonical user-major order
        self.num_users, self.num_items = num_users, num_items
        self.users, self.items = users[canon], items[canon]
        self.labels, self.weights = labels[canon], weights[canon]
        self.user_ptr = _histogram_offsets(self.users, num_users)
        self._item_order = np.argsort(self.items, kind="stable")
        self.item_ptr = _histogram_offsets(self.items, num_items)
        self._views = {}
        self._device = {}

    @property
    def n_interactions(self) -> int:
        return int(self.users.size)

    @property
    def user_counts(self) -> np.ndarray:
        return np.diff(self.user_ptr)

    @property
    def item_counts(self) -> np.ndarray:
        return np.diff(self.item_ptr)

    @property
    def item_order(self) -> np.ndarray:
        return self._item_order

    def user_view(self) -> SideView:
        if "user" not in self._views:
            self._views["user"] = SideView(self.num_users, self.num_items, self.user_ptr,
                                           self.items, self.labels, self.weights,
                                           np.arange(self.n_interactions, dtype=np.int64))
        return self._views["user"]

    def item_view(self) -> SideView:
        if "item" not in self._views:
            p = self._item_order
            self._views["item"] = SideView(self.num_items, self.num_users, self.item_ptr,
                                           self.users[p], self.labels[p], self.weights[p], p)
        return self._views["item"]
