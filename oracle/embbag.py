"""Embedding-bag oracle over paged tables (test infrastructure only).

No reference ancestor beyond the gather stand-in (bench/sweeps.py:1-9): the new
op is pooled[b, t, :] = fp32(sum_l table_t[idx[b, t, l], :]) with the sum taken in fp64, where table t occupies pages
[key0_t, key0_t + ceil(rows_t / rows_per_page)) of the store and row r lives in page
key0_t + r // rows_per_page at slot r % rows_per_page (rows_per_page = 4096 / (4 * D)).
Page contents come from oracle.pages.page_floats (the synthetic store fill).
The fp64 sum is exact for the synthetic tables (values on a 2^-23 grid in [-1, 1), fewer than 2^29
terms), so the result is the correctly rounded exact sum whatever the summation order: the GPU
warp's, a bag split into chunks, or a table split by rows over ranks whose fp64 partial sums are
added after the exchange (sharded_embbag_reference).
"""

from __future__ import annotations

import numpy as np

from .pages import page_floats, row_floats

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
    return rows.astype(np.float64).sum(axis=2).astype(np.float32)


def embbag_rows_reference(seed: int, idx: np.ndarray, D: int, tables=None) -> np.ndarray:
    """Global DLRM pooling over row-keyed tables (pages.row_floats): pooled[b, t, :] =
    fp32(sum_l row(t, idx[b, t, l])) with the sum in fp64.  `tables` names the global table id
    of every column of idx (default 0..T-1).  This is the single-device answer every sharding
    of the tables over ranks must reproduce bit for bit."""
    B, T, L = idx.shape
    tables = list(range(T)) if tables is None else list(tables)
    out = np.empty((B, T, D), dtype=np.float32)
    for j, t in enumerate(tables):
        col = idx[:, j, :].reshape(-1)
        uniq, inv = np.unique(col, return_inverse=True)
        vals = row_floats(seed, t, uniq, D).astype(np.float64)
        out[:, j, :] = vals[inv].reshape(B, L, D).sum(axis=1).astype(np.float32)
    return out


def embbag_offsets_reference(seed: int, idx_flat: np.ndarray, offsets: np.ndarray, T: int, D: int,
                             tables=None) -> np.ndarray:
    """Variable-length bags (torch embedding_bag's include_last_offset layout): bag i = b*T + t
    pools idx_flat[offsets[i]:offsets[i+1]] of table t (row-keyed values, fp64 sum, fp32 out);
    an empty bag pools to zeros."""
    nb = len(offsets) - 1
    tables = list(range(T)) if tables is None else list(tables)
    out = np.zeros((nb // T, T, D), dtype=np.float32)
    for i in range(nb):
        s, e = int(offsets[i]), int(offsets[i + 1])
        if e > s:
            v = row_floats(seed, tables[i % T], idx_flat[s:e], D).astype(np.float64)
            out[i // T, i % T] = v.sum(axis=0).astype(np.float32)
    return out
