"""ctypes front of oracle/graph_oracle.c (test infrastructure only): BFS levels, SpMV and PageRank
restated sequentially in C for the BASELINE-scale checks (tools/graph_bench.py --check,
tests/test_oracle_graph.py)."""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

_SO = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_build", "libgraph_oracle.so")
_lib = None


def _load():
    global _lib
    if _lib is None:
        _lib = C.CDLL(_SO)
        vp, i64 = C.c_void_p, C.c_int64
        _lib.oracle_bfs.restype = i64
        _lib.oracle_bfs.argtypes = [vp, vp, i64, i64, vp]
        _lib.oracle_spmv.restype = None
        _lib.oracle_spmv.argtypes = [vp, vp, vp, vp, i64, C.c_float, C.c_float, vp]
        _lib.oracle_pagerank.restype = None
        _lib.oracle_pagerank.argtypes = [vp, vp, vp, i64, C.c_int, C.c_double, vp]
    return _lib


def bfs_levels(row_ptr: np.ndarray, col: np.ndarray, source: int) -> np.ndarray:
    row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int64)
    col = np.ascontiguousarray(col, dtype=np.int32)
    V = len(row_ptr) - 1
    level = np.empty(V, dtype=np.int32)
    _load().oracle_bfs(row_ptr.ctypes.data, col.ctypes.data, V, int(source), level.ctypes.data)
    return level


def spmv_f32(row_ptr, col, val, x, alpha=1.0, beta=0.0) -> np.ndarray:
    row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int64)
    col = np.ascontiguousarray(col, dtype=np.int32)
    x = np.ascontiguousarray(x, dtype=np.float32)
    V = len(row_ptr) - 1
    y = np.empty(V, dtype=np.float32)
    vp = None if val is None else np.ascontiguousarray(val, dtype=np.float32).ctypes.data
    _load().oracle_spmv(row_ptr.ctypes.data, col.ctypes.data, vp, x.ctypes.data, V, alpha, beta, y.ctypes.data)
    return y


def pagerank_f32(rowT, colT, outdeg, iters=10, d=0.85) -> np.ndarray:
    rowT = np.ascontiguousarray(rowT, dtype=np.int64)
    colT = np.ascontiguousarray(colT, dtype=np.int32)
    outdeg = np.ascontiguousarray(outdeg, dtype=np.int64)
    V = len(rowT) - 1
    r = np.empty(V, dtype=np.float32)
    _load().oracle_pagerank(rowT.ctypes.data, colT.ctypes.data, outdeg.ctypes.data, V, iters, d, r.ctypes.data)
    return r
