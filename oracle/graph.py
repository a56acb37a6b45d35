"""Graph oracle (test infrastructure only): BFS levels and SpMV / PageRank on a CSR, restated on
the CPU (numpy / scipy).  No reference ancestor (SPEC.md:9 drops the graph apps); parity is
levels bit-exact and fp32 sums within 1e-5 relative."""

from __future__ import annotations

import numpy as np


def bfs_levels(row_ptr: np.ndarray, col: np.ndarray, source: int) -> np.ndarray:
    V = len(row_ptr) - 1
    level = np.full(V, -1, dtype=np.int32)
    level[source] = 0
    frontier = np.array([source], dtype=np.int64)
    cur = 0
    while len(frontier):
        starts, ends = row_ptr[frontier], row_ptr[frontier + 1]
        lens = ends - starts
        if lens.sum() == 0:
            break
        idx = np.repeat(starts - np.concatenate([[0], np.cumsum(lens)[:-1]]), lens) + np.arange(lens.sum())
        nb = col[idx].astype(np.int64)
        nb = np.unique(nb[level[nb] == -1])
        level[nb] = cur + 1
        frontier = nb
        cur += 1
    return level


def spmv(row_ptr, col, vals, x):
    import scipy.sparse as sp
    V = len(row_ptr) - 1
    A = sp.csr_matrix((vals.astype(np.float64), col.astype(np.int64), row_ptr.astype(np.int64)), shape=(V, len(x)))
    return A @ x.astype(np.float64)


def pagerank(rowT, colT, outdeg, iters=10, d=0.85):
    V = len(rowT) - 1
    r = np.full(V, 1.0 / V)
    ones = np.ones(len(colT))
    inv = np.where(outdeg > 0, 1.0 / np.maximum(outdeg, 1), 0.0)
    for _ in range(iters):
        r = (1 - d) / V + d * spmv(rowT, colT, ones, r * inv)
    return r
