"""ctypes wrapper of oracle/agile_oracle.c — the timed CPU baseline (kind "port") and a fast
checker for large embedding-bag parity cases.  Test infrastructure only (oracle/__init__.py)."""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

_SO = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_build", "libagile_oracle.so")
_lib = None


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            raise FileNotFoundError(f"{_SO} missing: run __graft_entry__.build()")
        lib = C.CDLL(_SO)
        lib.oracle_cache_create.restype = C.c_void_p
        lib.oracle_cache_create.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64]
        lib.oracle_cache_destroy.argtypes = [C.c_void_p]
        lib.oracle_cache_stats.argtypes = [C.c_void_p, C.c_void_p]
        lib.oracle_embbag.restype = C.c_int
        lib.oracle_embbag.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                      C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32, C.c_int]
        lib.oracle_cache_rowkeyed.argtypes = [C.c_void_p, C.c_uint32]
        _lib = lib
    return _lib


class CpuEmbeddingCache:
    """Set-associative clock cache over the synthetic page store, on host threads."""

    def __init__(self, lines: int, ways: int, seed: int, row_dim: int = 0):
        """row_dim = D: tables are row-keyed (pages.row_floats, the bench's store fill); 0: page-keyed
        (pages.page_floats)."""
        self._lib = _load()
        self._h = self._lib.oracle_cache_create(lines, ways, seed)
        if not self._h:
            raise ValueError("lines must be a multiple of ways")
        if row_dim:
            self._lib.oracle_cache_rowkeyed(self._h, row_dim)

    def embbag(self, idx: np.ndarray, key0: np.ndarray, rows: np.ndarray, D: int, threads: int = 1, tables=None):
        """pooled [B, T, D]; tables = global table id of every column (row-keyed mode)."""
        idx = np.ascontiguousarray(idx, dtype=np.int64)
        B, T, L = idx.shape
        out = np.empty((B, T, D), dtype=np.float32)
        k0 = np.ascontiguousarray(key0, dtype=np.uint64)
        r = np.ascontiguousarray(rows, dtype=np.int64)
        tid = np.ascontiguousarray(np.arange(T) if tables is None else tables, dtype=np.int64)
        rc = self._lib.oracle_embbag(self._h, idx.ctypes.data, k0.ctypes.data, r.ctypes.data, tid.ctypes.data,
                                     out.ctypes.data, B, T, L, D, threads)
        if rc == -2:
            from paper_2504_19365_b200.errors import OutOfRange
            raise OutOfRange("embedding index outside its table")
        if rc:
            raise ValueError("oracle_embbag failed")
        return out

    def stats(self):
        s = (C.c_uint64 * 3)()
        self._lib.oracle_cache_stats(self._h, s)
        return {"hits": int(s[0]), "misses": int(s[1]), "evictions": int(s[2])}

    def close(self):
        if self._h:
            self._lib.oracle_cache_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()
