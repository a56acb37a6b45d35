"""Embedding-bag oracle over paged tables (test infrastructure only).

No reference ancestor beyond the gather stand-in (bench/sweeps.py:1-9): the new
op is pooled[b, t, :] = sum_l table_t[idx[b, t, l], :] in fp32, where table t occupies pages
[key0_t, key0_t + ceil(rows_t / rows_per_page)) of the store and row r lives in page
key0_t + r // rows_per_page at slot r % rows_per_page (rows_per_page = 4096 / (4 * D)).
Page contents come from oracle.pages.page_floats (the synthetic store fill).
Summation order is l = 0..L-1 left to right in fp32, the order the GPU warp uses per lane.
"""

from __future__ import annotations

import numpy as np

from .pages import page_floats

DEV_SHIFT = 36


def embbag_reference(seed: int, dev: int, table_key0, idx: np.ndarray, D: int) -> np.ndarray:
    B, T, L = idx.shape
    rpp = 4096 // (4 * D)
    key0 = np.asarray(table_key0, dtype=np.uint64) & np.uint64((1 << DEV_SHIFT) - 1)
    page = key0[None, :, None] + (idx.astype(np.uint64) // np.uint64(rpp))
    slot = (idx % rpp).astype(np.int64)
    uniq, inv = np.unique(page.reshape(-1), return_inverse=True)
    fl = page_floats(seed, dev, uniq).reshape(len(uniq), rpp, D)
    rows = fl[inv, slot.reshape(-1)].reshape(B, T, L, D)
    out = np.zeros((B, T, D), dtype=np.float32)
    for l in range(L):
        out += rows[:, :, l, :]
    return out
