"""Device-resident iALS++ engine: torch-owned buffers + calls into libials_b200.

``torch`` is used for device memory, streams and CUDA graphs only; all
arithmetic of the hot path runs in the hand-written sm_100a kernels behind
the C ABI (``include/ials_b200.h``).

Layout in HBM (fp32 factors, int32 indices):
  * W (U x d), H (I x d)      row-major factor tables, mutated in place
  * cache (S)                 scores in canonical user-major order
  * user side: ptr (U+1), cols = item ids (S), optional labels / weights (S)
  * item side: ptr (I+1), cols = user ids (S), pos = canonical slot (S), ...
  * per side and block-tile width: the light/heavy row schedule
  * one workspace buffer (slab, split-K partials, alpha0*U@slab, heavy partials)
"""

from __future__ import annotations

import ctypes
from ctypes import c_void_p
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib


class SingularBlock(np.linalg.LinAlgError):
    """Raised from the device error word; mapped to SingularMatrixError."""

    def __init__(self, row, pivot, side):
        super().__init__(f"normal equations singular for {side} row {row} (pivot {pivot})")
        self.row, self.pivot, self.side = int(row), int(pivot), side


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def block_tile(b: int) -> int:
    for bt in (8, 16, 32, 64, 128):
        if b <= bt:
            return bt
    return 256


def current_stream_handle(device) -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


class Session:
    """One ``ials_session`` on one device (error word + last message)."""

    def __init__(self, device: int = 0):
        self.lib = _lib.load()
        if not torch.cuda.is_available():
            raise RuntimeError("no CUDA device: the iALS++ B200 solver has no CPU path")
        self.device = torch.device("cuda", device)
        h = ctypes.c_void_p()
        rc = self.lib.ials_session_create(device, ctypes.byref(h))
        if rc != 0:
            raise RuntimeError(_lib.last_error(None))
        self.handle = h

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                self.lib.ials_session_destroy(self.handle)
        except Exception:
            pass

    def check(self, rc: int, what: str = ""):
        if rc == _lib.IALS_OK:
            return
        msg = _lib.last_error(self.handle)
        if rc in (_lib.IALS_E_INVALID, _lib.IALS_E_NOMEM):
            raise ValueError(f"{what}: {msg}")
        raise RuntimeError(f"{what}: {msg}")

    def tc_redo_rows(self, reset: bool = False) -> int:
        """Rows the fused tensor-core sweep handed back to the SIMT sweep."""
        n = ctypes.c_int64()
        self.check(self.lib.ials_tc_redo_rows(self.handle, current_stream_handle(self.device),
                                              ctypes.byref(n), int(reset)), "tc_redo_rows")
        return int(n.value)

    def reset_singular(self):
        self.check(self.lib.ials_reset_singular(self.handle, current_stream_handle(self.device)),
                   "reset_singular")

    def raise_if_singular(self):
        row, piv, side = ctypes.c_int64(), ctypes.c_int32(), ctypes.c_int32()
        rc = self.lib.ials_check_singular(self.handle, current_stream_handle(self.device),
                                          ctypes.byref(row), ctypes.byref(piv), ctypes.byref(side))
        if rc == _lib.IALS_E_SINGULAR:
            raise SingularBlock(row.value, piv.value, "user" if side.value == 0 else "item")
        self.check(rc, "check_singular")


@dataclass
class Schedule:
    tensors: dict
    struct: _lib.IalsSched
    n_light: int
    n_heavy: int
    n_slices: int


class DeviceSide:
    """One side of the interaction matrix on the device (SideView, data.py:26-52)."""

    def __init__(self, device, ptr, cols, labels, weights, pos, lam, n_fixed):
        # host arrays, or device tensors straight from build_csr_device
        ptr = ptr.cpu().numpy().astype(np.int64) if isinstance(ptr, torch.Tensor) else np.asarray(ptr, dtype=np.int64)
        self.n_rows = int(ptr.size - 1)
        self.n_fixed = int(n_fixed)
        self.nnz = int(ptr[-1])
        if self.nnz >= 2 ** 31 - 1:
            raise ValueError("more than 2^31-1 interactions are not supported")
        self.counts = np.diff(ptr)
        tdt = {np.int32: torch.int32, np.float32: torch.float32}
        to = lambda a, dt: (a.to(device=device, dtype=tdt[dt]).contiguous() if isinstance(a, torch.Tensor)
                            else torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).to(device))
        self.ptr = to(ptr, np.int32)
        self.cols = to(cols, np.int32)
        self.labels = None if labels is None else to(labels, np.float32)
        self.weights = None if weights is None else to(weights, np.float32)
        self.pos = None if pos is None else to(pos, np.int32)
        self.lam = to(lam, np.float32)
        # row of every entry (the entry-parallel cache pass)
        self.rows = to(np.repeat(np.arange(self.n_rows, dtype=np.int32), self.counts), np.int32)
        self.device = device
        self.struct = _lib.IalsSide(self.n_rows, self.n_fixed, self.nnz, _ptr(self.ptr).value,
                                    _ptr(self.cols).value, _ptr(self.labels).value,
                                    _ptr(self.weights).value, _ptr(self.pos).value,
                                    _ptr(self.lam).value, _ptr(self.rows).value)
        self._sched = {}

    def set_lam(self, lam):
        self.lam.copy_(torch.from_numpy(np.ascontiguousarray(lam, dtype=np.float32)))

    def schedule(self, b: int) -> Schedule:
        """Light rows in descending degree; heavy rows split into fixed slices."""
        lib = _lib.load()
        # keyed by what the plan depends on: the library's heavy-row threshold
        # and slice length for this width
        bt = (int(lib.ials_heavy_threshold(b)), int(lib.ials_slice_len(b)))
        if bt in self._sched:
            return self._sched[bt]
        plan = plan_schedule(self.ptr.cpu().numpy(), bt[0], bt[1])
        to = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.int32)).to(self.device)
        t = {k: to(v) for k, v in plan.items()}
        deg_light = self.counts[plan["light"]]   # descending: the counts are prefix lengths
        st = _lib.IalsSched(int(plan["light"].size), _ptr(t["light"]).value,
                            int(plan["heavy"].size), _ptr(t["heavy"]).value,
                            _ptr(t["slice0"]).value, int(plan["beg"].size),
                            _ptr(t["slice_heavy"]).value, _ptr(t["beg"]).value,
                            _ptr(t["end"]).value,
                            int(np.count_nonzero(deg_light > 64)),
                            int(np.count_nonzero(deg_light > 32)))
        sch = Schedule(t, st, int(plan["light"].size), int(plan["heavy"].size),
                       int(plan["beg"].size))
        self._sched[bt] = sch
        return sch


def plan_schedule(ptr, heavy_threshold: int, slice_len: int) -> dict:
    """Row schedule of one side (host logic, NumPy).

    * light rows (degree <= threshold), sorted by descending degree so the
      longest rows start first (LPT order);
    * heavy rows, also by descending degree, each cut into ceil(n/slice_len)
      slices of consecutive entries [beg, end); ``slice0[h]`` is the first
      slice of heavy row h and ``slice_heavy[s]`` the heavy row of slice s.
    """
    ptr = np.asarray(ptr, dtype=np.int64)
    counts = np.diff(ptr)
    order = np.argsort(-counts, kind="stable")
    heavy_mask = counts[order] > heavy_threshold
    light, heavy = order[~heavy_mask], order[heavy_mask]
    nsl = (counts[heavy] + slice_len - 1) // slice_len
    slice0 = np.zeros(heavy.size + 1, dtype=np.int64)
    np.cumsum(nsl, out=slice0[1:])
    n_slices = int(slice0[-1])
    slice_heavy = np.repeat(np.arange(heavy.size), nsl)
    within = np.arange(n_slices) - slice0[slice_heavy]
    beg = ptr[heavy][slice_heavy] + within * slice_len
    end = np.minimum(beg + slice_len, ptr[heavy + 1][slice_heavy])
    return {"light": light, "heavy": heavy, "slice0": slice0, "slice_heavy": slice_heavy,
            "beg": beg, "end": end}


def effective_reg(counts, opposite_size, reg, alpha0, exponent):
    """reg * (count + alpha0 * opposite)^exponent in fp64 (model.py:144-150)."""
    base = np.asarray(counts, dtype=np.float64) + alpha0 * opposite_size
    return reg * base ** exponent


class DeviceProblem:
    """Both side views of an interaction set, resident on one device."""

    def __init__(self, device, num_users, num_items, user_ptr, user_cols, item_ptr, item_cols,
                 item_pos, labels=None, weights=None):
        self.device = torch.device(device)
        self.num_users, self.num_items = int(num_users), int(num_items)
        lab_u = wt_u = lab_i = wt_i = None
        if labels is not None and not np.all(labels == 1.0):
            lab_u, lab_i = labels, np.asarray(labels)[item_pos]
        if weights is not None and not np.all(weights == 1.0):
            wt_u, wt_i = weights, np.asarray(weights)[item_pos]
        self.users = DeviceSide(self.device, user_ptr, user_cols, lab_u, wt_u, None,
                                np.zeros(self.num_users), self.num_items)
        self.items = DeviceSide(self.device, item_ptr, item_cols, lab_i, wt_i, item_pos,
                                np.zeros(self.num_items), self.num_users)
        self.nnz = self.users.nnz
        self._reg_key = None

    @classmethod
    def from_dataset(cls, data, device):
        """From a reference-compatible ``InteractionDataset`` (duck-typed)."""
        iv = data.item_view()
        return cls(device, data.num_users, data.num_items, data.user_ptr, data.items,
                   data.item_ptr, iv.cols, iv.cache_pos, data.labels, data.weights)

    @classmethod
    def from_device_csr(cls, csr, device=None):
        """From ``csr.build_csr_device`` (both views already on the device;
        labels and weights all ones, the BASELINE configuration)."""
        dev = device if device is not None else csr.user_cols.device
        return cls(dev, csr.num_users, csr.num_items, csr.user_ptr, csr.user_cols, csr.item_ptr,
                   csr.item_cols, csr.item_pos)

    def set_regularizer(self, alpha0, reg, exponent):
        key = (float(alpha0), float(reg), float(exponent))
        if key == self._reg_key:
            return
        self.users.set_lam(effective_reg(self.users.counts, self.num_items, reg, alpha0, exponent))
        self.items.set_lam(effective_reg(self.items.counts, self.num_users, reg, alpha0, exponent))
        self._reg_key = key


class Engine:
    """Stream-ordered launcher for one problem on one device."""

    def __init__(self, problem: DeviceProblem, session: Session | None = None):
        self.p = problem
        self.device = problem.device
        self.sess = session or Session(self.device.index or 0)
        self.lib = self.sess.lib
        self._ws = None

    # ------------------------------------------------------------ workspace
    def workspace(self, d, b):
        sch_u = self.p.users.schedule(b)
        sch_i = self.p.items.schedule(b)
        need = int(self.lib.ials_workspace_bytes(
            max(self.p.num_users, 1), max(self.p.num_items, 1), d, b,
            max(sch_u.n_slices, sch_i.n_slices), max(sch_u.n_heavy, sch_i.n_heavy)))
        # room for the epoch's tensor-core GEMM path (K-major factor copies)
        need += int(self.lib.ials_epoch_tc_bytes(max(self.p.num_users, 1),
                                                 max(self.p.num_items, 1), d, b))
        need = max(need, int(self.lib.ials_loss_workspace_bytes(d)))
        if self._ws is None or self._ws.numel() < need:
            self._ws = torch.empty(need, dtype=torch.uint8, device=self.device)
        return self._ws

    def stream(self):
        return current_stream_handle(self.device)

    # ------------------------------------------------------------ primitives
    def predictions(self, W, H, out):
        d = W.shape[1]
        rc = self.lib.ials_predictions(self.sess.handle, self.p.users.n_rows, _ptr(self.p.users.ptr),
                                       _ptr(self.p.users.cols), _ptr(W), W.stride(0), _ptr(H),
                                       H.stride(0), d, _ptr(out), self.stream())
        self.sess.check(rc, "predictions")

    def partial_gramian(self, M, b0, b, out):
        d = M.shape[1]
        ws = self.workspace(d, b)
        rc = self.lib.ials_partial_gramian(self.sess.handle, _ptr(M), M.shape[0], M.stride(0), d,
                                           b0, b, _ptr(out), _ptr(ws), ws.numel(), self.stream())
        self.sess.check(rc, "partial_gramian")

    def side_pass(self, side: str, fixed, own, b0, b, slab, alpha0, cache):
        s = self.p.users if side == "user" else self.p.items
        sch = s.schedule(b)
        d = own.shape[1]
        ws = self.workspace(d, b)
        rc = self.lib.ials_side_pass(self.sess.handle, ctypes.byref(s.struct), ctypes.byref(sch.struct),
                                     _ptr(fixed), fixed.stride(0), _ptr(own), own.stride(0), d, b0,
                                     b, _ptr(slab), float(alpha0), _ptr(cache),
                                     0 if side == "user" else 1, _ptr(ws), ws.numel(),
                                     self.stream())
        self.sess.check(rc, f"{side} side pass")

    def epoch(self, W, H, cache, b, alpha0, events=None):
        """One uniform-block iALS++ epoch entirely on the device.  `events`
        (torch.cuda.Event list, 2 + 4 * blocks) are recorded at the phase
        boundaries (see ials_epoch_events)."""
        d = W.shape[1]
        ws = self.workspace(d, b)
        su, si = self.p.users.schedule(b), self.p.items.schedule(b)
        if events:
            for e in events:
                if not e.cuda_event:   # created lazily by torch on first record
                    e.record(torch.cuda.current_stream(self.device))
            arr = (c_void_p * len(events))(*[c_void_p(e.cuda_event) for e in events])
            self.sess.check(self.lib.ials_epoch_events(arr, len(events)), "epoch events")
        try:
            rc = self.lib.ials_epoch(self.sess.handle, ctypes.byref(self.p.users.struct),
                                     ctypes.byref(su.struct), ctypes.byref(self.p.items.struct),
                                     ctypes.byref(si.struct), _ptr(W), W.stride(0), _ptr(H),
                                     H.stride(0), d, b, float(alpha0), _ptr(cache), _ptr(ws),
                                     ws.numel(), self.stream())
        finally:
            if events:
                self.lib.ials_epoch_events(None, 0)
        self.sess.check(rc, "epoch")

    def epoch_passes(self, W, H, cache, b, alpha0, pass0, npass, recompute_cache=False):
        """Passes [pass0, pass0 + npass) of ``epoch`` (pass 2k = user pass of
        block k, 2k + 1 = its item pass), through the same C code path."""
        d = W.shape[1]
        ws = self.workspace(d, b)
        su, si = self.p.users.schedule(b), self.p.items.schedule(b)
        rc = self.lib.ials_epoch_range(self.sess.handle, ctypes.byref(self.p.users.struct),
                                       ctypes.byref(su.struct), ctypes.byref(self.p.items.struct),
                                       ctypes.byref(si.struct), _ptr(W), W.stride(0), _ptr(H),
                                       H.stride(0), d, b, float(alpha0), _ptr(cache), _ptr(ws),
                                       ws.numel(), self.stream(), int(pass0), int(npass),
                                       int(bool(recompute_cache)))
        self.sess.check(rc, "epoch_range")

    def epoch_host(self, W_host, H_host, W, H, cache, b, alpha0, W_out=None, H_out=None,
                   cache_out=None):
        """One epoch for a model in (pinned) host tensors: ials_epoch_host
        stages W / H in, runs the epoch, and writes W / H (and the cache if
        ``cache_out`` is given) back, overlapping the copies with the epoch."""
        d = W.shape[1]
        ws = self.workspace(d, b)
        su, si = self.p.users.schedule(b), self.p.items.schedule(b)
        W_out = W_host if W_out is None else W_out
        H_out = H_host if H_out is None else H_out
        rc = self.lib.ials_epoch_host(self.sess.handle, ctypes.byref(self.p.users.struct),
                                      ctypes.byref(su.struct), ctypes.byref(self.p.items.struct),
                                      ctypes.byref(si.struct), _ptr(W_host), _ptr(W_out),
                                      W_host.stride(0), _ptr(H_host), _ptr(H_out), H_host.stride(0),
                                      _ptr(W), W.stride(0), _ptr(H), H.stride(0), d, b,
                                      float(alpha0), _ptr(cache), _ptr(cache_out), _ptr(ws),
                                      ws.numel(), self.stream())
        self.sess.check(rc, "epoch_host")

    def epoch_host64(self, W_host, H_host, W, H, cache, b, alpha0, staging, cache_out=None,
                     events=None):
        """One epoch for the reference's float64 model in host memory (NumPy
        arrays, C-contiguous): ials_epoch_host64 copies W / H in through device
        f64 staging, runs the epoch, and writes W / H (and the maintained
        cache, if ``cache_out`` is given) back in place, the copies and casts
        overlapped with the epoch on a second stream.  Stream-ordered: the
        host arrays are final once the current stream has synchronised."""
        d = W.shape[1]
        ws = self.workspace(d, b)
        su, si = self.p.users.schedule(b), self.p.items.schedule(b)
        hp = lambda a: ctypes.c_void_p(a.ctypes.data) if a is not None else ctypes.c_void_p(0)
        if events:
            for e in events:
                if not e.cuda_event:
                    e.record(torch.cuda.current_stream(self.device))
            arr = (c_void_p * len(events))(*[c_void_p(e.cuda_event) for e in events])
            self.sess.check(self.lib.ials_epoch_events(arr, len(events)), "epoch events")
        try:
            rc = self.lib.ials_epoch_host64(
                self.sess.handle, ctypes.byref(self.p.users.struct), ctypes.byref(su.struct),
                ctypes.byref(self.p.items.struct), ctypes.byref(si.struct), hp(W_host), hp(W_host),
                W_host.strides[0] // 8, hp(H_host), hp(H_host), H_host.strides[0] // 8, _ptr(W),
                W.stride(0), _ptr(H), H.stride(0), d, b, float(alpha0), _ptr(cache), hp(cache_out),
                _ptr(staging), staging.numel(), _ptr(ws), ws.numel(), self.stream())
        finally:
            if events:
                self.lib.ials_epoch_events(None, 0)
        self.sess.check(rc, "epoch_host64")

    def epoch_graph(self, W, H, cache, b, alpha0):
        """The same epoch captured once as a CUDA graph and replayed (one
        launch per epoch instead of ~10 per block; matters for small configs).
        The graph is keyed on the buffers, so W / H / cache must stay the same
        tensors between calls."""
        key = (W.data_ptr(), H.data_ptr(), cache.data_ptr(), int(b), float(alpha0))
        entry = getattr(self, "_graphs", {}).get(key)
        if entry is None or entry[1] is not self._ws:
            # (re)captured when the workspace the graph baked in was replaced;
            # each graph keeps its own workspace tensor alive
            self.epoch(W, H, cache, b, alpha0)          # attributes / workspace set up
            torch.cuda.synchronize(self.device)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self.epoch(W, H, cache, b, alpha0)
            entry = (g, self._ws)
            self.__dict__.setdefault("_graphs", {})[key] = entry
        entry[0].replay()

    def loss_terms(self, W, H):
        """Device fp64 loss pieces; returns a (4,) float64 CUDA tensor."""
        d = W.shape[1]
        ws = self.workspace(d, 1)
        need = int(self.lib.ials_loss_workspace_bytes(d))
        if ws.numel() < need:
            self._ws = ws = torch.empty(need, dtype=torch.uint8, device=self.device)
        out = torch.empty(4, dtype=torch.float64, device=self.device)
        rc = self.lib.ials_loss_terms(self.sess.handle, ctypes.byref(self.p.users.struct),
                                      ctypes.byref(self.p.items.struct), _ptr(W), W.stride(0),
                                      _ptr(H), H.stride(0), d, _ptr(out), _ptr(ws), ws.numel(),
                                      self.stream())
        self.sess.check(rc, "loss_terms")
        return out

    def loss(self, W, H, alpha0):
        t = self.loss_terms(W, H).cpu().numpy()
        return float(t[0] + alpha0 * t[1] + t[2] + t[3])
