"""torch.library operator over the K5 embedding-bag (``torch.ops.agile.embedding_bag``).

The op is the framework-facing form of ``agile_embbag_sharded`` (include/agile_b200.h): sum
pooling of fp32 rows held in an AGILE context's page store, read through its HBM page cache,
fixed pooling factor (``idx`` of shape [B, T, L]) or variable-length bags (flat ``idx`` with
``offsets`` of length B*T + 1, torch ``embedding_bag``'s include_last_offset convention, bag
(b, t) = offsets[b*T + t] .. offsets[b*T + t + 1]).  Tables are whole tables here: the page key of
each table's first page (``table_key0``, dev << 36 | page) and its row count.  Accumulation is fp64,
rounded once to fp32.  The context is passed as its integer handle (``AgileSystem.handle``), so
the op carries no Python object and can sit inside captured CUDA graphs / torch.compile regions
as an opaque call.  CUDA tensors only; there is no CPU kernel (no CPU fallback).
"""

from __future__ import annotations

from typing import Optional

import numpy as np
import torch

from . import _lib

_TAB = np.dtype([("key0", "<u8"), ("row0", "<i8"), ("rows", "<i8"), ("table_rows", "<i8"),
                 ("out_offset", "<u4"), ("flags", "<u4")])


def _tables(table_key0: torch.Tensor, table_rows: torch.Tensor, D: int) -> torch.Tensor:
    T = table_key0.numel()
    d = np.zeros(T, dtype=_TAB)
    d["key0"] = table_key0.detach().cpu().numpy().view(np.uint64)
    d["rows"] = d["table_rows"] = table_rows.detach().cpu().numpy()
    d["out_offset"] = np.arange(T, dtype=np.uint32) * (4 * D)
    return torch.from_numpy(d.view(np.uint8).copy()).to(table_key0.device)


@torch.library.custom_op("agile::embedding_bag", mutates_args=())
def embedding_bag(handle: int, idx: torch.Tensor, offsets: Optional[torch.Tensor], table_key0: torch.Tensor,
                  table_rows: torch.Tensor, D: int, prefetch_distance: int = 0) -> torch.Tensor:
    if not idx.is_cuda:
        raise ValueError("agile::embedding_bag runs on CUDA tensors only")
    T = table_key0.numel()
    if offsets is None:
        B, T2, L = idx.shape
        if T2 != T:
            raise ValueError("idx must be [B, T, L] with T = len(table_key0)")
    else:
        nb = offsets.numel() - 1
        if nb % T:
            raise ValueError("offsets must hold B * T + 1 entries")
        B, L = nb // T, 0
    idx = idx.contiguous().to(torch.int64)
    off = offsets.contiguous().to(torch.int64) if offsets is not None else None
    out = torch.empty((B, T, D), dtype=torch.float32, device=idx.device)
    cnt = torch.zeros(2, dtype=torch.int64, device=idx.device)
    tabs = _tables(table_key0, table_rows, D)
    st = torch.cuda.current_stream(idx.device).cuda_stream
    lib = _lib.load()
    rc = lib.agile_embbag_sharded(C_ptr(handle), idx.data_ptr(), off.data_ptr() if off is not None else None,
                                  tabs.data_ptr(), out.data_ptr(), T * D * 4, cnt.data_ptr(), B, T, L, D,
                                  prefetch_distance, 0, 0, st)
    _lib.check(C_ptr(handle), rc, "agile::embedding_bag")
    return out


@embedding_bag.register_fake
def _(handle, idx, offsets, table_key0, table_rows, D, prefetch_distance=0):
    T = table_key0.shape[0]
    B = idx.shape[0] if offsets is None else (offsets.shape[0] - 1) // T
    return idx.new_empty((B, T, D), dtype=torch.float32)


def C_ptr(handle: int):
    import ctypes
    return ctypes.c_void_p(handle)
