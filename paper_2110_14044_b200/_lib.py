"""ctypes binding of ``libials_b200.so`` (the C ABI in ``include/ials_b200.h``).

The library is built in-tree by ``__graft_entry__.build()`` (or
``python -m paper_2110_14044_b200.build``).  There is no fallback: if the
shared object is missing or a CUDA device is absent, using the solver raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libials_b200.so")
if os.environ.get("IALS_LIB") == "checked":   # the bounds-checked build (build.py --checked)
    LIB_PATH = os.path.join(HERE, "libials_b200_checked.so")

IALS_OK = 0
IALS_E_INVALID = -1
IALS_E_SINGULAR = -2
IALS_E_CUDA = -3
IALS_E_NOMEM = -4

c_i32, c_i64, c_p, c_sz, c_f = ctypes.c_int32, ctypes.c_int64, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_float


class IalsSide(ctypes.Structure):
    """``ials_side`` (one SideView on the device, data.py:26-52)."""
    _fields_ = [("n_rows", c_i32), ("n_fixed", c_i32), ("nnz", c_i64), ("ptr", c_p),
                ("cols", c_p), ("labels", c_p), ("weights", c_p), ("pos", c_p), ("lam", c_p),
                ("rows", c_p)]


class IalsSched(ctypes.Structure):
    """``ials_sched`` (light / heavy row schedule of one side)."""
    _fields_ = [("n_light", c_i32), ("light_rows", c_p), ("n_heavy", c_i32),
                ("heavy_rows", c_p), ("heavy_slice0", c_p), ("n_slices", c_i32),
                ("slice_heavy", c_p), ("slice_begin", c_p), ("slice_end", c_p),
                ("n_deg_gt64", c_i32), ("n_deg_gt32", c_i32)]


class IalsSegs(ctypes.Structure):
    """``ials_segs`` (row segments the multi-GPU gather-dot kernels walk)."""
    _fields_ = [("n", c_i32), ("row", c_p), ("beg", c_p), ("end", c_p)]


#: every symbol include/ials_b200.h declares, with its ctypes signature
SIGNATURES = {
    "ials_version": (c_i32, []),
    "ials_session_create": (c_i32, [c_i32, ctypes.POINTER(c_p)]),
    "ials_session_destroy": (c_i32, [c_p]),
    "ials_last_error": (c_i32, [c_p, ctypes.c_char_p, c_sz]),
    "ials_reset_singular": (c_i32, [c_p, c_p]),
    "ials_check_singular": (c_i32, [c_p, c_p, ctypes.POINTER(c_i64), ctypes.POINTER(c_i32),
                                    ctypes.POINTER(c_i32)]),
    "ials_set_tensor_cores": (c_i32, [c_i32]),
    "ials_tc_redo_rows": (c_i32, [c_p, c_p, ctypes.POINTER(c_i64), c_i32]),
    "ials_set_tc_cond_max": (c_f, [c_f]),
    "ials_debug_timestamps": (c_i32, [c_p]),
    "ials_heavy_threshold": (c_i64, [c_i32]),
    "ials_slice_len": (c_i64, [c_i32]),
    "ials_workspace_bytes": (c_sz, [c_i32, c_i32, c_i32, c_i32, c_i32, c_i32]),
    "ials_epoch_tc_bytes": (c_sz, [c_i32, c_i32, c_i32, c_i32]),
    "ials_epoch_events": (c_i32, [ctypes.POINTER(c_p), c_i32]),
    "ials_predictions": (c_i32, [c_p, c_i32, c_p, c_p, c_p, c_i32, c_p, c_i32, c_i32, c_p, c_p]),
    "ials_predictions_segments": (c_i32, [c_p, c_i32, c_p, c_p, c_p, c_p, c_p, c_i32, c_p, c_i32,
                                          c_i32, c_p, c_p]),
    "ials_cache_correct": (c_i32, [c_p, c_i32, c_p, c_p, c_p, c_p, c_p, c_i32, c_i32, c_p, c_i32,
                                   c_i32, c_p, c_p]),
    "ials_partial_gramian": (c_i32, [c_p, c_p, c_i32, c_i32, c_i32, c_i32, c_i32, c_p, c_p,
                                     c_sz, c_p]),
    "ials_side_pass": (c_i32, [c_p, ctypes.POINTER(IalsSide), ctypes.POINTER(IalsSched), c_p,
                               c_i32, c_p, c_i32, c_i32, c_i32, c_i32, c_p, c_f, c_p, c_i32,
                               c_p, c_sz, c_p]),
    "ials_epoch": (c_i32, [c_p, ctypes.POINTER(IalsSide), ctypes.POINTER(IalsSched),
                           ctypes.POINTER(IalsSide), ctypes.POINTER(IalsSched), c_p, c_i32, c_p,
                           c_i32, c_i32, c_i32, c_f, c_p, c_p, c_sz, c_p]),
    "ials_topk64": (c_i32, [c_p, c_i32, c_i32, c_p, c_i64, c_p, c_p, c_i32, c_p, c_p, c_p]),
    "ials_scores": (c_i32, [c_p, c_p, c_i32, c_i32, c_p, c_i32, c_i32, c_i32, c_p, c_i32, c_p]),
    "ials_shard_apply_block": (c_i32, [c_p, c_p, c_i32, c_p, c_i32, c_i32, c_p, c_p, c_i32, c_i32,
                                       c_i32, c_p, c_i32, c_p]),
    "ials_set_rotation": (c_i32, [c_i32]),
    "ials_sym_eig": (c_i32, [c_p, c_i32, c_i32, c_p, c_i32, c_i64, c_p, c_p, c_p, c_p]),
    "ials_host_register": (c_i32, [c_p, c_sz]),
    "ials_host_unregister": (c_i32, [c_p]),
    "ials_host64_staging_bytes": (c_sz, [c_i32, c_i32, c_i32, c_i64]),
    "ials_epoch_host64": (c_i32, [c_p, ctypes.POINTER(IalsSide), ctypes.POINTER(IalsSched),
                                  ctypes.POINTER(IalsSide), ctypes.POINTER(IalsSched), c_p, c_p,
                                  c_i64, c_p, c_p, c_i64, c_p, c_i32, c_p, c_i32, c_i32, c_i32, c_f,
                                  c_p, c_p, c_p, c_sz, c_p, c_sz, c_p]),
    "ials_epoch_range": (c_i32, [c_p, ctypes.POINTER(IalsSide), ctypes.POINTER(IalsSched),
                                 ctypes.POINTER(IalsSide), ctypes.POINTER(IalsSched), c_p, c_i32,
                                 c_p, c_i32, c_i32, c_i32, c_f, c_p, c_p, c_sz, c_p, c_i32, c_i32,
                                 c_i32]),
    "ials_epoch_host": (c_i32, [c_p, ctypes.POINTER(IalsSide), ctypes.POINTER(IalsSched),
                                ctypes.POINTER(IalsSide), ctypes.POINTER(IalsSched), c_p, c_p, c_i64,
                                c_p, c_p, c_i64, c_p, c_i32, c_p, c_i32, c_i32, c_i32, c_f, c_p, c_p,
                                c_p, c_sz, c_p]),
    "ials_loss_workspace_bytes": (c_sz, [c_i32]),
    "ials_build_csr_workspace_bytes": (c_sz, [c_i64]),
    "ials_launch_count": (c_i64, []),
    "ials_shard_gemm_bytes": (c_sz, [c_i32, c_i32, c_i32]),
    "ials_shard_sync": (c_i32, [c_p, c_p, c_i32, c_i32, c_i32, c_i32, c_i32, c_i32, c_p, c_sz, c_p]),
    "ials_shard_gramian": (c_i32, [c_p, c_i32, c_i32, c_i32, c_i32, c_i32, c_p, c_p, c_sz, c_p]),
    "ials_shard_projection": (c_i32, [c_p, c_p, c_i32, c_i32, c_i32, c_i32, c_i32, c_p, c_f, c_p,
                                      c_p, c_sz, c_p]),
    "ials_side_pass_projected": (c_i32, [c_p, ctypes.POINTER(IalsSide), ctypes.POINTER(IalsSched),
                                         c_p, c_i32, c_p, c_i32, c_i32, c_i32, c_i32, c_p, c_p, c_f,
                                         c_p, c_i32, c_p, c_sz, c_p]),
    "ials_shard_rot_bytes": (c_sz, [c_i32, c_i32, c_i32, c_i32]),
    "ials_rotation_available": (c_i32, [c_i32, c_i32]),
    "ials_shard_diag_gramian": (c_i32, [c_p, c_i32, c_i32, c_i32, c_p, c_p, c_sz, c_p]),
    "ials_shard_rot_prepare": (c_i32, [c_p, c_i32, c_i32, c_p, c_i32, c_i32, c_p, c_sz, c_p]),
    "ials_shard_user_pass_rot": (c_i32, [c_p, ctypes.POINTER(IalsSide), ctypes.POINTER(IalsSched),
                                         c_p, c_i32, c_p, c_i32, c_i32, c_i32, c_i32, c_p, c_f, c_p,
                                         c_p, c_sz, c_p, c_sz, c_p, c_sz, c_p]),
    "ials_comm_unique_id": (c_i32, [c_p]),
    "ials_comm_create": (c_i32, [c_p, c_p, c_i32, c_i32, ctypes.POINTER(c_p)]),
    "ials_comm_wrap": (c_i32, [c_p, c_p, c_i32, c_i32, ctypes.POINTER(c_p)]),
    "ials_comm_destroy": (c_i32, [c_p]),
    "ials_epoch_sharded_bytes": (c_sz, [c_p, c_p, c_i32, c_i32, c_i32, c_i32, c_i32, c_i32]),
    "ials_epoch_sharded": (c_i32, [c_p, c_p, ctypes.POINTER(IalsSide), ctypes.POINTER(IalsSched),
                                   ctypes.POINTER(IalsSegs), ctypes.POINTER(IalsSide),
                                   ctypes.POINTER(IalsSched), ctypes.POINTER(IalsSegs), c_p, c_p,
                                   c_p, c_i32, c_p, c_i32, c_i32, c_i32, c_f, c_i32, c_p, c_p, c_p,
                                   c_sz, c_p]),
    "ials_topk": (c_i32, [c_p, c_i32, c_i32, c_p, c_i64, c_p, c_p, c_i32, c_p, c_p, c_p]),
    "ials_build_csr": (c_i32, [c_p, c_i32, c_i32, c_i64, c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_p,
                               c_p, c_sz, c_p]),
    "ials_loss_terms": (c_i32, [c_p, ctypes.POINTER(IalsSide), ctypes.POINTER(IalsSide), c_p,
                                c_i32, c_p, c_i32, c_i32, c_p, c_p, c_sz, c_p]),
}

_lib = None
_lock = threading.Lock()


class ExtensionMissing(RuntimeError):
    pass


def load(path: str = LIB_PATH):
    """Load (once) and type the shared library; raises if it is absent."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise ExtensionMissing(
                f"{path} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`"
                " (there is no CPU fallback for the iALS++ solver)")
        lib = ctypes.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def last_error(session) -> str:
    buf = ctypes.create_string_buffer(512)
    load().ials_last_error(session, buf, 512)
    return buf.value.decode(errors="replace")
