"""Dense kernels of the reference API surface (reference ``linalg.py``).

``partial_gramian`` / ``gramian`` run on the B200 (K-slab, split-K FP32 with a
fixed-order reduction).  ``check_block`` and ``SingularMatrixError`` keep the
reference's validation rules and error type (``linalg.py:18-28, 48-57``).
"""

from __future__ import annotations

import numpy as np

__all__ = ["SingularMatrixError", "check_block", "gramian", "partial_gramian"]


class SingularMatrixError(np.linalg.LinAlgError):
    """A block Hessian hit a non-positive pivot; ``pivot`` is the zero-based
    pivot index and ``row`` the row whose normal equations failed."""

    def __init__(self, message, pivot=None, row=None):
        super().__init__(message)
        self.pivot = pivot
        self.row = row


def check_block(block, dim) -> np.ndarray:
    """Nonempty, strictly increasing, in-range column index set (linalg.py:48-57)."""
    block = np.asarray(block, dtype=np.intp)
    if block.ndim != 1 or block.size == 0:
        raise ValueError("block must be a nonempty 1-d index set")
    if block.min() < 0 or block.max() >= dim:
        raise ValueError(f"block indices out of range for dimension {dim}")
    if block.size > 1 and np.any(np.diff(block) <= 0):
        raise ValueError("block indices must be strictly increasing")
    return block


def _as_matrix(mat):
    mat = np.asarray(mat, dtype=np.float64)
    if mat.ndim != 2:
        raise ValueError("expected a 2-d array")
    return mat


def partial_gramian(mat, block, device=None) -> np.ndarray:
    """The d x |block| slab M^T M[:, block] (linalg.py:39-45), computed on the GPU."""
    import torch

    from ._runtime import default_engine_session, to_device_f32

    mat = _as_matrix(mat)
    block = check_block(block, mat.shape[1])
    sess = default_engine_session(device)
    d = mat.shape[1]
    b = int(block.size)
    contiguous = bool(np.all(np.diff(block) == 1))
    if contiguous:
        m = to_device_f32(mat, sess.device)
        b0 = int(block[0])
        width = d
    else:
        # append the selected columns and take the slab of the appended range
        m = to_device_f32(np.concatenate([mat, mat[:, block]], axis=1), sess.device)
        b0, width = d, d + b
    out = torch.empty((width, b), dtype=torch.float32, device=sess.device)
    sess.gramian(m, b0, b, out)
    return out[:d].double().cpu().numpy()


def gramian(mat, device=None) -> np.ndarray:
    """M^T M (linalg.py:31-36), on the GPU."""
    mat = _as_matrix(mat)
    return partial_gramian(mat, np.arange(mat.shape[1]), device)
