"""CPU: the C graph oracle (oracle/graph_oracle.c, used for the BASELINE-scale checks) agrees with
the numpy restatement (oracle/graph.py) on random CSR graphs."""

import numpy as np
import pytest

from oracle import cgraph
from oracle.graph import bfs_levels, pagerank, spmv


def _csr(V, E, seed):
    rng = np.random.default_rng(seed)
    src = np.sort(rng.integers(0, V, size=E))
    col = rng.integers(0, V, size=E).astype(np.int32)
    row_ptr = np.zeros(V + 1, dtype=np.int64)
    np.add.at(row_ptr, src + 1, 1)
    return np.cumsum(row_ptr), col


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_c_bfs_matches_numpy(seed):
    row_ptr, col = _csr(3000, 12000, seed)
    for src in (0, 17, 2999):
        assert np.array_equal(cgraph.bfs_levels(row_ptr, col, src), bfs_levels(row_ptr, col, src))


def test_c_spmv_matches_scipy():
    row_ptr, col = _csr(2000, 30000, 5)
    rng = np.random.default_rng(6)
    val = (rng.random(30000) * 2 - 1).astype(np.float32)
    x = (rng.random(2000) * 2 - 1).astype(np.float32)
    y = cgraph.spmv_f32(row_ptr, col, val, x, 1.0, 0.0)
    exp = spmv(row_ptr, col, val, x)
    assert np.all(np.abs(y - exp) <= 1e-6 * np.abs(exp) + 1e-30)


def test_c_pagerank_matches_numpy():
    row_ptr, col = _csr(1500, 20000, 8)
    outdeg = np.bincount(col, minlength=1500).astype(np.int64)   # in-edge CSR: col = source vertex
    r = cgraph.pagerank_f32(row_ptr, col, outdeg, 10)
    exp = pagerank(row_ptr, col, outdeg, 10)
    assert np.max(np.abs(r - exp) / exp) < 1e-5
