"""Per-device runtime: the ials session, a scratch workspace, and the cache of
device-resident problems attached to datasets."""

from __future__ import annotations

import ctypes
import weakref

import numpy as np
import torch

from . import _lib
from .engine import DeviceProblem, Engine, Session, _ptr, current_stream_handle

_RUNTIMES = {}


def _device_index(device):
    if device is None:
        if not torch.cuda.is_available():
            raise RuntimeError("no CUDA device: the iALS++ B200 solver has no CPU path")
        return torch.cuda.current_device()
    return torch.device(device).index or 0


class Runtime:
    def __init__(self, index: int):
        self.session = Session(index)
        self.device = self.session.device
        self.lib = self.session.lib
        self._ws = None
        self._problems = weakref.WeakKeyDictionary()

    def workspace(self, nbytes):
        if self._ws is None or self._ws.numel() < nbytes:
            self._ws = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, device=self.device)
        return self._ws

    def gramian(self, M, b0, b, out):
        d = M.shape[1]
        ws = self.workspace(int(self.lib.ials_workspace_bytes(1, M.shape[0], d, b, 0, 0)))
        rc = self.lib.ials_partial_gramian(self.session.handle, _ptr(M), M.shape[0], M.stride(0),
                                           d, b0, b, _ptr(out), _ptr(ws), ws.numel(),
                                           current_stream_handle(self.device))
        self.session.check(rc, "partial_gramian")

    def engine_for(self, data) -> Engine:
        """Device CSR of ``data`` (built once per dataset object and device)."""
        try:
            eng = self._problems.get(data)
        except TypeError:
            eng = None
        if eng is None:
            eng = Engine(DeviceProblem.from_dataset(data, self.device), self.session)
            try:
                self._problems[data] = eng
            except TypeError:
                pass
        return eng


def default_engine_session(device=None) -> Runtime:
    idx = _device_index(device)
    rt = _RUNTIMES.get(idx)
    if rt is None:
        rt = _RUNTIMES[idx] = Runtime(idx)
    return rt


def to_device_f32(arr, device) -> torch.Tensor:
    a = np.ascontiguousarray(arr, dtype=np.float32)
    return torch.from_numpy(a).to(device, non_blocking=False)


# ------------------------------------------------------------ page-locked host arrays
_PINNED = {}


def pin_host_array(arr: np.ndarray) -> bool:
    """Page-lock ``arr``'s memory in place (ials_host_register) once, so the
    epoch's host copies run asynchronously beside the kernels.  The range is
    released when ``arr`` itself is garbage-collected (it keeps its buffer
    alive until then).  Returns False if the driver refused (the copies then
    still work, from pageable memory)."""
    if arr.nbytes == 0:
        return False
    key = (arr.ctypes.data, arr.nbytes)
    if key in _PINNED:
        return True
    lib = _lib.load()
    if lib.ials_host_register(ctypes.c_void_p(key[0]), ctypes.c_size_t(key[1])) != 0:
        return False

    def _release(k=key):
        if _PINNED.pop(k, None) is not None:
            try:
                _lib.load().ials_host_unregister(ctypes.c_void_p(k[0]))
            except Exception:
                pass
    try:
        _PINNED[key] = weakref.finalize(arr, _release)
    except TypeError:      # not weak-referenceable: release right away (pageable copies)
        _PINNED[key] = True
        _release()
        return False
    return True
