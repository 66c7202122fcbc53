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
        if side_id == 0 and getattr(self, "_gd", None) is not None:
            np.testing.assert_allclose(self._gd[b0:b0 + b].numpy(), slab[b0:b0 + b].numpy(),
                                       rtol=1e-10, atol=1e-12)
            self.rot_checks += 1
        n = side.nnz
        ones = np.ones(n)
        orc.side_pass(side.ptr, np.asarray(side.cols, dtype=np.int64),
                      ones if side.labels is None else side.labels,
                      ones if side.weights is None else side.weights,
                      np.arange(n), fixed.numpy(), own_rows.numpy(), cache.numpy(),
                      np.arange(b0, b0 + b), slab.numpy(), alpha0, side.lam)

    # ---- the rotated-pass protocol of GpuOps (distributed.py): one extra
    # all-reduce of the stacked diagonal Gram blocks at epoch start.  Here the
    # "decomposition" just keeps the all-reduced blocks, and every user sweep
    # checks them against its all-reduced slab -- which proves the collective
    # ran on every rank with the blocks of the epoch's initial H.
    rot_checks = 0

    def rot_supported(self, d, b, max_user_degree, unit_weights):
        return bool(getattr(self, "enable_rot", False) and unit_weights and d % b == 0)

    def diag_gram(self, M_rows, b):
        d = M_rows.shape[1]
        return torch.cat([M_rows[:, z:z + b].T @ M_rows[:, z:z + b] for z in range(0, d, b)], 0)

    def rot_prepare(self, gd, own_rows, n_fixed, b):
        self._gd = gd.clone()

    def rot_end(self):
        self._gd = None

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

