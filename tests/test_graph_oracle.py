"""CPU: the graph oracle on hand-checkable graphs."""

import numpy as np

from oracle.graph import bfs_levels, pagerank, spmv


def test_bfs_small():
    # 0->1, 0->2, 1->3, 3->4, 5 isolated
    row_ptr = np.array([0, 2, 3, 3, 4, 4, 4])
    col = np.array([1, 2, 3, 4])
    assert bfs_levels(row_ptr, col, 0).tolist() == [0, 1, 1, 2, 3, -1]


def test_spmv_and_pagerank_small():
    row_ptr = np.array([0, 2, 3])
    col = np.array([0, 1, 0])
    vals = np.array([2.0, 1.0, 3.0])
    assert np.allclose(spmv(row_ptr, col, vals, np.array([1.0, 10.0])), [12.0, 3.0])
    r = pagerank(np.array([0, 1, 2]), np.array([1, 0]), np.array([1, 1]), iters=20)
    assert np.allclose(r, [0.5, 0.5])
