"""Float64 CPU implementation of the ShardedTrainer compute ops -- TEST ONLY.
Wraps the oracle so the multi-rank orchestration (sharding, all-reduce of
slabs, all-gather of column blocks, dual-cache delta corrections) can be
checked with the gloo backend on CPU."""

import numpy as np
import torch

from oracle import ialspp_oracle as orc


class CpuOps:
    dtype = torch.float64

    @staticmethod
    def _rows(side):
        return np.repeat(np.arange(side.n_rows), np.diff(side.ptr))

    def predictions(self, side, A_rows, B, out):
        r = torch.from_numpy(self._rows(side))
        c = torch.from_numpy(np.asarray(side.cols, dtype=np.int64))
        out[:] = (A_rows[r] * B[c]).sum(1)

    def correct(self, side, A_rows, b0, D, out):
        b = D.shape[1]
        r = torch.from_numpy(self._rows(side))
        c = torch.from_numpy(np.asarray(side.cols, dtype=np.int64))
        out += (A_rows[r, b0:b0 + b] * D[c]).sum(1)

    def gram(self, M_rows, b0, b):
        return M_rows.T @ M_rows[:, b0:b0 + b]

    def sweep(self, side, fixed, own_rows, b0, b, slab, alpha0, cache, side_id):
        n = side.nnz
        ones = np.ones(n)
        orc.side_pass(side.ptr, np.asarray(side.cols, dtype=np.int64),
                      ones if side.labels is None else side.labels,
                      ones if side.weights is None else side.weights,
                      np.arange(n), fixed.numpy(), own_rows.numpy(), cache.numpy(),
                      np.arange(b0, b0 + b), slab.numpy(), alpha0, side.lam)

    def check(self):
        pass

    def apply_block(self, recv, nmax, bounds, rank, old_local, X, b0, b):
        delta = torch.empty((X.shape[0], b), dtype=X.dtype)
        for r, (lo, hi) in enumerate(bounds):
            new = recv[r * nmax: r * nmax + (hi - lo)]
            old = old_local if r == rank else X[lo:hi, b0:b0 + b].clone()
            if r != rank:
                X[lo:hi, b0:b0 + b] = new
            delta[lo:hi] = new - old
        return delta

