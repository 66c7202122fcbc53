"""Device CSR construction.

``build_csr_device`` produces, on the GPU, exactly the integer arrays the
reference builds on the host in ``InteractionDataset.__init__`` and its
``user_view`` / ``item_view`` (/root/reference/pkg/src/blockals/data.py:98-134,
148-162): the stable user-major order, both row-pointer arrays, both column
arrays and the item view's ``cache_pos`` permutation.  The sorts are the
stable LSD radix sorts of ``ials_build_csr`` (include/ials_b200.h); the
validation and its ``ValueError`` messages follow data.py:101-120.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from ._runtime import default_engine_session
from .engine import _ptr, current_stream_handle


@dataclass
class DeviceCSR:
    """int32 device tensors; names follow the reference's attributes."""
    num_users: int
    num_items: int
    order: torch.Tensor      # argsort(users, stable): canonical position -> input index
    user_ptr: torch.Tensor   # (U+1,)
    user_cols: torch.Tensor  # items in canonical order (user view cols)
    item_ptr: torch.Tensor   # (I+1,)
    item_cols: torch.Tensor  # users in item-major order (item view cols)
    item_pos: torch.Tensor   # item view cache_pos (canonical position of each item-major entry)

    @property
    def n_interactions(self) -> int:
        return int(self.user_cols.numel())


def _as_ids(a, device, name):
    if isinstance(a, torch.Tensor):
        t = a.to(device=device)
    else:
        t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.int64)).to(device)
    if t.dim() != 1:
        raise ValueError("users and items must be 1-d arrays of equal length")
    return t


def build_csr_device(num_users, num_items, users, items, device=None) -> DeviceCSR:
    """Build both CSR views on the device.  ``users`` / ``items`` are 1-d id
    arrays (NumPy or torch, any integer dtype); ids are range-checked like the
    reference before anything is sorted."""
    rt = default_engine_session(device)
    dev = rt.device
    num_users, num_items = int(num_users), int(num_items)
    if num_users < 1 or num_items < 1:
        raise ValueError("dataset needs at least one user and one item")
    u = _as_ids(users, dev, "users")
    i = _as_ids(items, dev, "items")
    if u.numel() != i.numel():
        raise ValueError("users and items must be 1-d arrays of equal length")
    n = int(u.numel())
    if n >= 2 ** 31 - 1:
        raise ValueError("more than 2^31-1 interactions are not supported")
    if n:
        lo_u, hi_u = (int(x) for x in torch.aminmax(u))
        lo_i, hi_i = (int(x) for x in torch.aminmax(i))
        if lo_u < 0 or hi_u >= num_users:
            raise ValueError("user index out of range")
        if lo_i < 0 or hi_i >= num_items:
            raise ValueError("item index out of range")
    u32 = u.to(torch.int32).contiguous()
    i32 = i.to(torch.int32).contiguous()
    e = lambda m: torch.empty(max(m, 1), dtype=torch.int32, device=dev)[:m]
    out = DeviceCSR(num_users, num_items, e(n), e(num_users + 1), e(n), e(num_items + 1), e(n), e(n))
    lib = rt.lib
    ws = rt.workspace(int(lib.ials_build_csr_workspace_bytes(n)))
    rc = lib.ials_build_csr(rt.session.handle, num_users, num_items, n, _ptr(u32), _ptr(i32),
                            _ptr(out.user_ptr), _ptr(out.user_cols), _ptr(out.order),
                            _ptr(out.item_ptr), _ptr(out.item_cols), _ptr(out.item_pos),
                            _ptr(ws), ws.numel(), current_stream_handle(dev))
    rt.session.check(rc, "build_csr")
    return out
