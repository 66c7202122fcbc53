"""Multi-GPU iALS++ epoch: row shards, replicated tables, NCCL collectives.

SURVEY.md §8e.  One process per GPU (``torch.distributed``).  Users and items
are split into contiguous, nnz-balanced shards; W and H are replicated on every
rank.  Per block pi:

  1. slab(H)[:, pi]: partial over the local item rows -> all-reduce (d x b)
  2. user sweep on the local user rows
  3. all-gather of the updated column block W[:, pi] (U_r x b per rank)
  4. slab(W)[:, pi]: partial over the local user rows -> all-reduce
  5. item sweep on the local item rows
  6. all-gather of H[:, pi]

Score caches are never moved (dual-cache delta scheme): each rank keeps C_u
(its users' entries, user-major) and C_i (its items' entries, item-major),
both recomputed at epoch start.  The reference's single cache is updated by
every pass for every entry; here, before a pass, the local cache is corrected
for the other side's last half-epoch:

  user pass of block pi : C_u[k] += <W[u, pi-1], dH[i, pi-1]>
  item pass of block pi : C_i[k] += <H[i, pi],   dW[u, pi]>

with dX = X_new - X_old of the column block that was just all-gathered.  In
exact arithmetic this equals the reference's cache maintenance
(``solvers.py:186``), so the iterates are the reference's (up to rounding).

The compute steps go through an ``ops`` object: ``GpuOps`` (the product: the
libials_b200 kernels, fp32) or, in tests only, a float64 CPU implementation
wrapping the oracle, which lets the sharding / collective / correction logic
be verified with the ``gloo`` backend on CPU (tests/test_distributed.py).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

__all__ = ["shard_bounds", "LocalSide", "ShardedTrainer", "GpuOps"]


def shard_bounds(ptr, world, row_weight=0.0):
    """Contiguous row ranges [lo_r, hi_r) balancing nnz (+ row_weight per row)."""
    ptr = np.asarray(ptr, dtype=np.int64)
    n = ptr.size - 1
    cost = ptr.astype(np.float64) + row_weight * np.arange(n + 1)
    targets = cost[-1] * np.arange(world + 1) / world
    cuts = np.searchsorted(cost, targets, side="left")
    cuts[0], cuts[-1] = 0, n
    cuts = np.maximum.accumulate(np.clip(cuts, 0, n))
    return [(int(cuts[r]), int(cuts[r + 1])) for r in range(world)]


@dataclass
class LocalSide:
    """Rows [lo, hi) of one side: a rebased CSR whose entries index the local
    cache (identity positions), cols = global ids of the other side."""

    lo: int
    hi: int
    ptr: np.ndarray       # (hi - lo + 1,) int64, ptr[0] == 0
    cols: np.ndarray      # global ids of the fixed side
    labels: np.ndarray | None
    weights: np.ndarray | None
    lam: np.ndarray       # effective regularizer of the local rows
    base: int             # offset of the first local entry in the full side view
    n_fixed: int

    @property
    def n_rows(self):
        return self.hi - self.lo

    @property
    def nnz(self):
        return int(self.ptr[-1])


def make_local_side(ptr, cols, labels, weights, lam, lo, hi, n_fixed):
    ptr = np.asarray(ptr, dtype=np.int64)
    s, e = int(ptr[lo]), int(ptr[hi])
    return LocalSide(lo, hi, ptr[lo:hi + 1] - s, np.asarray(cols[s:e]),
                     None if labels is None else np.asarray(labels[s:e]),
                     None if weights is None else np.asarray(weights[s:e]),
                     np.asarray(lam[lo:hi]), s, n_fixed)


class GpuOps:
    """The product compute path: libials_b200 kernels on this rank's GPU."""

    def __init__(self, device):
        from .engine import Session
        self.device = torch.device(device)
        self.sess = Session(self.device.index or 0)
        self.dtype = torch.float32
        self._sides = {}
        self._ws = None

    SEG = 256   # entries per row segment of the gather-dot kernels

    def _dev(self, side: LocalSide):
        key = id(side)
        if key not in self._sides:
            from .engine import DeviceSide
            ds = DeviceSide(self.device, side.ptr, side.cols, side.labels, side.weights, None,
                            side.lam, side.n_fixed)
            counts = np.diff(side.ptr)
            nseg = (counts + self.SEG - 1) // self.SEG
            row = np.repeat(np.arange(side.n_rows), nseg)
            first = np.concatenate([[0], np.cumsum(nseg)[:-1]])
            beg = side.ptr[:-1][row] + (np.arange(row.size) - first[row]) * self.SEG
            end = np.minimum(beg + self.SEG, side.ptr[1:][row])
            to = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.int32)).to(self.device)
            ds.segs = (int(row.size), to(row), to(beg), to(end))
            self._sides[key] = ds
        return self._sides[key]

    def _workspace(self, nbytes):
        if self._ws is None or self._ws.numel() < nbytes:
            self._ws = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, device=self.device)
        return self._ws

    def _stream(self):
        from .engine import current_stream_handle
        return current_stream_handle(self.device)

    def predictions(self, side, A_rows, B, out):
        from .engine import _ptr
        ds = self._dev(side)
        n, r, bg, en = ds.segs
        rc = self.sess.lib.ials_predictions_segments(
            self.sess.handle, n, _ptr(r), _ptr(bg), _ptr(en), _ptr(ds.cols), _ptr(A_rows),
            A_rows.stride(0), _ptr(B), B.stride(0), A_rows.shape[1], _ptr(out), self._stream())
        self.sess.check(rc, "predictions")

    def correct(self, side, A_rows, b0, D, out):
        from .engine import _ptr
        ds = self._dev(side)
        n, r, bg, en = ds.segs
        rc = self.sess.lib.ials_cache_correct(self.sess.handle, n, _ptr(r), _ptr(bg), _ptr(en),
                                              _ptr(ds.cols), _ptr(A_rows), A_rows.stride(0), b0,
                                              _ptr(D), D.stride(0), D.shape[1], _ptr(out),
                                              self._stream())
        self.sess.check(rc, "cache_correct")

    # ---- tensor-core GEMMs on this rank's row shards (b in 33..128, like
    # ials_epoch): K-major copies of a shard live in a per-shard workspace
    def tc_enable(self, M_rows, b):
        """Keep K-major copies of the shard ``M_rows`` (a row slice of W or H)
        for block width ``b``; returns False if the tensor-core path does not
        apply (then gram / sweep use the FP32 SIMT kernels)."""
        d = M_rows.shape[1]
        if not (32 < b <= 128 and d % 4 == 0 and M_rows.stride(0) % 4 == 0
                and M_rows.data_ptr() % 16 == 0):
            return False
        n = M_rows.shape[0]
        nb = int(self.sess.lib.ials_shard_gemm_bytes(n, d, b))
        if not hasattr(self, "_shards"):
            self._shards = {}
        self._shards[M_rows.data_ptr()] = (torch.empty(nb, dtype=torch.uint8, device=self.device), n, b)
        self.tc_sync(M_rows, 0, d)
        return True

    def _shard(self, M_rows):
        return getattr(self, "_shards", {}).get(M_rows.data_ptr())

    def tc_sync(self, M_rows, c0, cw):
        from .engine import _ptr
        sh = self._shard(M_rows)
        if sh is None:
            return
        ws, n, b = sh
        rc = self.sess.lib.ials_shard_sync(self.sess.handle, _ptr(M_rows), M_rows.stride(0), n,
                                           M_rows.shape[1], b, c0, cw, _ptr(ws), ws.numel(),
                                           self._stream())
        self.sess.check(rc, "shard_sync")

    def gram(self, M_rows, b0, b):
        from .engine import _ptr
        d = M_rows.shape[1]
        out = torch.empty((d, b), dtype=self.dtype, device=self.device)
        sh = self._shard(M_rows)
        if sh is not None and b <= sh[2]:
            ws, n, bw = sh
            rc = self.sess.lib.ials_shard_gramian(self.sess.handle, n, d, bw, b0, b, _ptr(out),
                                                  _ptr(ws), ws.numel(), self._stream())
            self.sess.check(rc, "shard_gramian")
            return out
        if M_rows.shape[0] == 0:
            return out.zero_()
        ws = self._workspace(int(self.sess.lib.ials_workspace_bytes(1, M_rows.shape[0], d, b, 0, 0)))
        rc = self.sess.lib.ials_partial_gramian(self.sess.handle, _ptr(M_rows), M_rows.shape[0],
                                                M_rows.stride(0), d, b0, b, _ptr(out), _ptr(ws),
                                                ws.numel(), self._stream())
        self.sess.check(rc, "partial_gramian")
        return out

    # ---- rotated user passes (b = 128): the sharded form of ials_epoch's
    # (eigenbasis of G_pp, Woodbury tiles for the short rows)
    def rot_supported(self, d, b, max_user_degree, unit_weights):
        """Whether the user passes of this run can be rotated.  Decided from
        GLOBAL quantities only, so every rank takes the same branch (the
        branch adds an all-reduce)."""
        return bool(unit_weights and self.sess.lib.ials_rotation_available(d, b)
                    and max_user_degree <= int(self.sess.lib.ials_heavy_threshold(b)))

    def diag_gram(self, M_rows, b):
        """Partial diagonal Gram blocks of the (item) shard: (d x b), rows
        [z b, (z+1) b) = M[:, z]^T M[:, z]; None off the tensor-core path."""
        from .engine import _ptr
        sh = self._shard(M_rows)
        if sh is None or sh[2] != b:
            return None
        ws, n, _ = sh
        d = M_rows.shape[1]
        out = torch.empty((d, b), dtype=self.dtype, device=self.device)
        rc = self.sess.lib.ials_shard_diag_gramian(self.sess.handle, n, d, b, _ptr(out), _ptr(ws),
                                                   ws.numel(), self._stream())
        self.sess.check(rc, "shard_diag_gramian")
        return out

    def rot_prepare(self, gd, own_rows, n_fixed, b):
        """Decompose every (all-reduced) diagonal block; the user sweeps of
        this epoch then run rotated."""
        from .engine import _ptr
        d = own_rows.shape[1]
        n = own_rows.shape[0]
        nb = int(self.sess.lib.ials_shard_rot_bytes(n, n_fixed, d, b))
        if getattr(self, "_rot_ws", None) is None or self._rot_ws.numel() < nb:
            self._rot_ws = torch.empty(nb, dtype=torch.uint8, device=self.device)
        rc = self.sess.lib.ials_shard_rot_prepare(self.sess.handle, d, b, _ptr(gd), n, n_fixed,
                                                  _ptr(self._rot_ws), self._rot_ws.numel(),
                                                  self._stream())
        self.sess.check(rc, "shard_rot_prepare")
        self._rot = (own_rows.data_ptr(), b)

    def rot_end(self):
        self._rot = None

    def sweep(self, side, fixed, own_rows, b0, b, slab, alpha0, cache, side_id):
        from .engine import _ptr
        import ctypes
        ds = self._dev(side)
        sch = ds.schedule(b)
        d = own_rows.shape[1]
        ws = self._workspace(int(self.sess.lib.ials_workspace_bytes(
            max(ds.n_rows, 1), max(fixed.shape[0], 1), d, b, sch.n_slices, sch.n_heavy)))
        sh = self._shard(own_rows)
        if (side_id == 0 and getattr(self, "_rot", None) == (own_rows.data_ptr(), b)
                and sh is not None and sch.n_heavy == 0):
            if own_rows.shape[0] > 0:
                sws = sh[0]
                rc = self.sess.lib.ials_shard_user_pass_rot(
                    self.sess.handle, ctypes.byref(ds.struct), ctypes.byref(sch.struct), _ptr(fixed),
                    fixed.stride(0), _ptr(own_rows), own_rows.stride(0), d, b0, b, _ptr(slab),
                    float(alpha0), _ptr(cache), _ptr(sws), sws.numel(), _ptr(self._rot_ws),
                    self._rot_ws.numel(), _ptr(ws), ws.numel(), self._stream())
                self.sess.check(rc, "shard_user_pass_rot")
                self.tc_sync(own_rows, b0, b)
            return
        if sh is not None and b <= sh[2] and own_rows.shape[0] > 0:
            # projection alpha0 * own @ slab on the tensor core, then the sweep
            sws, n, bw = sh
            proj = torch.empty((n, b), dtype=self.dtype, device=self.device)
            rc = self.sess.lib.ials_shard_projection(self.sess.handle, _ptr(own_rows),
                                                     own_rows.stride(0), n, d, bw, b, _ptr(slab),
                                                     float(alpha0), _ptr(proj), _ptr(sws),
                                                     sws.numel(), self._stream())
            self.sess.check(rc, "shard_projection")
            rc = self.sess.lib.ials_side_pass_projected(
                self.sess.handle, ctypes.byref(ds.struct), ctypes.byref(sch.struct), _ptr(fixed),
                fixed.stride(0), _ptr(own_rows), own_rows.stride(0), d, b0, b, _ptr(slab),
                _ptr(proj), float(alpha0), _ptr(cache), side_id, _ptr(ws), ws.numel(),
                self._stream())
            self.sess.check(rc, "side_pass_projected")
            self.tc_sync(own_rows, b0, b)   # the shard's block changed
            return
        rc = self.sess.lib.ials_side_pass(self.sess.handle, ctypes.byref(ds.struct),
                                          ctypes.byref(sch.struct), _ptr(fixed), fixed.stride(0),
                                          _ptr(own_rows), own_rows.stride(0), d, b0, b,
                                          _ptr(slab), float(alpha0), _ptr(cache), side_id,
                                          _ptr(ws), ws.numel(), self._stream())
        self.sess.check(rc, "side_pass")

    def apply_block(self, recv, nmax, bounds, rank, old_local, X, b0, b):
        """Remote rows of the gathered block into X, and the block's change
        (n x b, new - old) for the other side's cache correction."""
        from .engine import _ptr
        if not hasattr(self, "_bounds") or self._bounds[0] != tuple(bounds):
            flat = [lo for lo, _ in bounds] + [bounds[-1][1]]
            self._bounds = (tuple(bounds),
                            torch.tensor(flat, dtype=torch.int32, device=self.device))
        n = X.shape[0]
        delta = torch.empty((n, b), dtype=self.dtype, device=self.device)
        rc = self.sess.lib.ials_shard_apply_block(
            self.sess.handle, _ptr(recv), nmax, _ptr(self._bounds[1]), len(bounds), rank,
            _ptr(old_local), _ptr(X), X.stride(0), b0, b, _ptr(delta), n, self._stream())
        self.sess.check(rc, "shard_apply_block")
        return delta

    # ---- the whole epoch behind the C ABI (ials_epoch_sharded): the same steps
    # as ShardedTrainer.epoch over these ops, with NCCL collectives issued by
    # the library on its own communicator (no Python between the kernels)
    def make_comm(self, rank, world, group=None):
        """The library's communicator over the ranks of ``group`` (collective:
        rank 0's NCCL unique id travels by torch.distributed)."""
        import ctypes
        lib = self.sess.lib
        idp = None
        if world > 1:
            ident = ctypes.create_string_buffer(128)
            if rank == 0:
                self.sess.check(lib.ials_comm_unique_id(ident), "comm_unique_id")
            box = [ident.raw if rank == 0 else None]
            src = dist.get_global_rank(group, 0) if group is not None else 0
            dist.broadcast_object_list(box, src=src, group=group)
            ident = ctypes.create_string_buffer(box[0], 128)
            idp = ctypes.cast(ident, ctypes.c_void_p)
        h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            self.sess.check(lib.ials_comm_create(self.sess.handle, idp, rank, world, ctypes.byref(h)),
                            "comm_create")
        self._comm = h
        self._comm_shape = (rank, world)
        return h

    def close_comm(self):
        if getattr(self, "_comm", None):
            self.sess.lib.ials_comm_destroy(self._comm)
            self._comm = None

    def __del__(self):
        try:
            self.close_comm()
        except Exception:
            pass

    def epoch_native(self, us, is_, user_bounds, item_bounds, W, H, b, alpha0, rotate, Cu, Ci):
        from . import _lib
        from .engine import _ptr
        import ctypes
        lib = self.sess.lib
        rank, world = self._comm_shape
        du, di = self._dev(us), self._dev(is_)
        su, si = du.schedule(b), di.schedule(b)
        segs = []
        for ds in (du, di):
            n, r, bg, en = ds.segs
            segs.append(_lib.IalsSegs(n, _ptr(r).value, _ptr(bg).value, _ptr(en).value))
        I32 = ctypes.c_int32 * (world + 1)
        ub = I32(*([lo for lo, _ in user_bounds] + [user_bounds[-1][1]]))
        ib = I32(*([lo for lo, _ in item_bounds] + [item_bounds[-1][1]]))
        d = W.shape[1]
        nb = int(lib.ials_epoch_sharded_bytes(ub, ib, world, rank, d, b, max(su.n_slices, si.n_slices),
                                              max(su.n_heavy, si.n_heavy)))
        if nb == 0:
            raise ValueError("epoch_sharded: bad bounds")
        if getattr(self, "_ews", None) is None or self._ews.numel() < nb:
            self._ews = torch.empty(nb, dtype=torch.uint8, device=self.device)
        rc = lib.ials_epoch_sharded(
            self.sess.handle, self._comm, ctypes.byref(du.struct), ctypes.byref(su.struct),
            ctypes.byref(segs[0]), ctypes.byref(di.struct), ctypes.byref(si.struct),
            ctypes.byref(segs[1]), ub, ib, _ptr(W), W.stride(0), _ptr(H), H.stride(0), d, b,
            float(alpha0), int(bool(rotate)), _ptr(Cu), _ptr(Ci), _ptr(self._ews),
            self._ews.numel(), self._stream())
        self.sess.check(rc, "epoch_sharded")

    def check(self):
        self.sess.raise_if_singular()


class ShardedTrainer:
    """One rank's share of a sharded iALS++ run (call collectively on all ranks)."""

    def __init__(self, data, W, H, alpha0, reg, exponent, ops, group=None, native=None):
        self.ops = ops
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.alpha0 = float(alpha0)
        U, I = int(data["num_users"]), int(data["num_items"])
        self.U, self.I = U, I
        up, ip = np.asarray(data["user_ptr"]), np.asarray(data["item_ptr"])
        lam_u = reg * (np.diff(up) + alpha0 * I) ** exponent
        lam_i = reg * (np.diff(ip) + alpha0 * U) ** exponent
        self.user_bounds = shard_bounds(up, self.world)
        self.item_bounds = shard_bounds(ip, self.world, row_weight=1.0)
        ulo, uhi = self.user_bounds[self.rank]
        ilo, ihi = self.item_bounds[self.rank]
        self.us = make_local_side(up, data["user_cols"], data.get("labels"), data.get("weights"),
                                  lam_u, ulo, uhi, I)
        order = np.asarray(data["item_order"])
        lab_i = None if data.get("labels") is None else np.asarray(data["labels"])[order]
        wt_i = None if data.get("weights") is None else np.asarray(data["weights"])[order]
        self.is_ = make_local_side(ip, data["item_cols"], lab_i, wt_i, lam_i, ilo, ihi, U)
        self.W, self.H = W, H          # replicated full tables (this rank's device)
        dev, dt = W.device, W.dtype
        self.Cu = torch.zeros(self.us.nnz, dtype=dt, device=dev)
        self.Ci = torch.zeros(self.is_.nnz, dtype=dt, device=dev)
        self._umax = max(h - l for l, h in self.user_bounds)
        self._imax = max(h - l for l, h in self.item_bounds)
        # global facts the rotated-pass decision rests on (identical on every rank)
        self._max_user_degree = int(np.diff(up).max()) if U > 0 else 0
        self._unit = data.get("labels") is None and data.get("weights") is None
        # the epoch behind the C ABI (ials_epoch_sharded, its own NCCL
        # communicator) when the ops provide it; ``native=False`` / IALS_SHARD_NATIVE=0
        # keeps the orchestration below in Python (the form the gloo tests cover)
        import os
        self.native = bool(native if native is not None else os.environ.get("IALS_SHARD_NATIVE", "1") != "0")
        self.native = self.native and hasattr(ops, "epoch_native") and W.dtype == torch.float32
        if self.native:
            ops.make_comm(self.rank, self.world, group)

    # ---------------------------------------------------------------- comms
    def _allreduce(self, t):
        if self.world > 1:
            dist.all_reduce(t, group=self.group)
        return t

    def _start_exchange(self, X, bounds, nmax, b0, b):
        """Start the all-gather of this rank's rows of X[:, b0:b0+b] (padded to
        nmax rows per rank, one contiguous receive buffer); returns (work, recv)."""
        lo, hi = bounds[self.rank]
        key = (id(bounds), b)
        bufs = self.__dict__.setdefault("_xbufs", {})
        if key not in bufs:
            send = torch.zeros((nmax, b), dtype=X.dtype, device=X.device)
            recv = send if self.world == 1 else torch.empty((self.world * nmax, b), dtype=X.dtype,
                                                            device=X.device)
            bufs[key] = (send, recv)
        send, recv = bufs[key]
        send[: hi - lo] = X[lo:hi, b0:b0 + b]
        work = None
        if self.world > 1:
            work = dist.all_gather_into_tensor(recv, send, group=self.group, async_op=True)
        return work, recv

    def _finish_exchange(self, work, recv, X, bounds, nmax, b0, b, old_local):
        """Wait for the all-gather, write the other ranks' rows into X; the
        block's change new - old for every row (n x b)."""
        if work is not None:
            work.wait()
        return self.ops.apply_block(recv, nmax, bounds, self.rank, old_local, X, b0, b)

    # ---------------------------------------------------------------- epoch
    def epoch(self, block_size):
        """Per block: the user pass on the local users, the all-gather of their
        new W[:, pi] rows overlapped with the partial item-side slab, the item
        pass, the all-gather of H[:, pi] overlapped with the next block's
        partial user-side slab.  Only the local rows are copied before a sweep
        (the change of a remote row is formed while its new values land), so
        no full-table pass remains per block."""
        W, H, ops = self.W, self.H, self.ops
        d = W.shape[1]
        if self.native and block_size <= 256:
            rot = (self.I > 0 and self.U > 0
                   and ops.rot_supported(d, block_size, self._max_user_degree, self._unit)
                   and 32 < block_size <= 128 and d % 4 == 0 and W.stride(0) % 4 == 0
                   and H.stride(0) % 4 == 0)
            ops.epoch_native(self.us, self.is_, self.user_bounds, self.item_bounds, W, H, block_size,
                             self.alpha0, rot, self.Cu, self.Ci)
            return
        ulo, uhi = self.user_bounds[self.rank]
        ilo, ihi = self.item_bounds[self.rank]
        Wl, Hl = W[ulo:uhi], H[ilo:ihi]
        if hasattr(ops, "tc_enable"):   # K-major copies of both shards (no-op when b is off the TC path)
            for M in (Wl, Hl):
                ops.tc_enable(M, block_size)
        # rotated user passes: every block's G_pp = H[:, pi]^T H[:, pi] is final
        # here (H[:, pi] changes only in block pi's item pass, after its user
        # pass), so the ranks' partial diagonal blocks go through ONE all-reduce
        # (d x b floats) and every rank decomposes the same matrices
        rot = (hasattr(ops, "rot_supported") and self.I > 0 and self.U > 0
               and ops.rot_supported(d, block_size, self._max_user_degree, self._unit))
        if rot:
            gd = ops.diag_gram(Hl, block_size)
            rot = gd is not None
        if rot:
            ops.rot_prepare(self._allreduce(gd), Wl, self.I, block_size)
        ops.predictions(self.us, Wl, H, self.Cu)
        ops.predictions(self.is_, Hl, W, self.Ci)
        prev = None        # (b0, b, dH) of the last item pass
        g_h = ops.gram(Hl, 0, min(block_size, d))
        for b0 in range(0, d, block_size):
            b = min(block_size, d - b0)
            # ---- user pass
            if prev is not None:
                ops.correct(self.us, Wl, prev[0], prev[2], self.Cu)
            slab = self._allreduce(g_h)
            w_old = Wl[:, b0:b0 + b].clone()          # local rows only
            ops.sweep(self.us, H, Wl, b0, b, slab, self.alpha0, self.Cu, 0)
            work, recv = self._start_exchange(W, self.user_bounds, self._umax, b0, b)
            g_w = ops.gram(Wl, b0, b)                  # overlaps the all-gather
            dW = self._finish_exchange(work, recv, W, self.user_bounds, self._umax, b0, b, w_old)
            # ---- item pass
            ops.correct(self.is_, Hl, b0, dW, self.Ci)
            slab = self._allreduce(g_w)
            h_old = Hl[:, b0:b0 + b].clone()
            ops.sweep(self.is_, W, Hl, b0, b, slab, self.alpha0, self.Ci, 1)
            work, recv = self._start_exchange(H, self.item_bounds, self._imax, b0, b)
            if b0 + b < d:                             # the next block's slab partial, overlapped
                g_h = ops.gram(Hl, b0 + b, min(block_size, d - b0 - b))
            dH = self._finish_exchange(work, recv, H, self.item_bounds, self._imax, b0, b, h_old)
            prev = (b0, b, dH)
        # bring C_u up to date with the last item pass
        if prev is not None:
            ops.correct(self.us, Wl, prev[0], prev[2], self.Cu)
        if rot:
            ops.rot_end()

    def gather_cache(self):
        """The canonical (user-major) cache, assembled on every rank."""
        if self.world == 1:
            return self.Cu.clone()
        nmax = max(int(self.us.nnz), 1)
        sizes = torch.tensor([self.us.nnz], device=self.Cu.device)
        all_sizes = [torch.zeros_like(sizes) for _ in range(self.world)]
        dist.all_gather(all_sizes, sizes, group=self.group)
        nmax = int(max(s.item() for s in all_sizes))
        send = torch.zeros(max(nmax, 1), dtype=self.Cu.dtype, device=self.Cu.device)
        send[: self.us.nnz] = self.Cu
        recv = [torch.empty_like(send) for _ in range(self.world)]
        dist.all_gather(recv, send, group=self.group)
        return torch.cat([recv[r][: int(all_sizes[r].item())] for r in range(self.world)])
