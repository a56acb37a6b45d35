"""GPU parity of BFS (levels bit-exact) and SpMV / PageRank (1e-5 relative) over a paged CSR."""

import numpy as np
import pytest
import torch

from oracle.graph import bfs_levels, pagerank, spmv
from paper_2504_19365_b200.bench.graph import (build_csr, edge_values, pages_for, rmat_edges, run_bfs,
                                               run_pagerank, run_spmv, write_paged)

pytestmark = pytest.mark.gpu


def _graph(scale, seed=1, transpose=False):
    dev = torch.device("cuda", 0)
    src, dst, V = rmat_edges(scale, 16, seed, dev)
    row_ptr, col = build_csr(dst, src, V) if transpose else build_csr(src, dst, V)
    return dev, src, dst, V, row_ptr, col


@pytest.mark.parametrize("prefetch", [False, True])
@pytest.mark.parametrize("frac", [0.25, 1.5])
def test_bfs_levels_match_oracle(gpu_system, prefetch, frac):
    dev, src, dst, V, row_ptr, col = _graph(13)
    E = col.numel()
    lines = max(64, int(frac * pages_for(E)) // 32 * 32)
    s = gpu_system(cache_lines=lines, ways=32, blocks=pages_for(E) + 8, pairs=16, engine_warps=16, warps=8)
    write_paged(s, 0, 0, col)
    rp = row_ptr.cpu().numpy()
    deg = np.diff(rp)
    source = int(np.nonzero(deg)[0][7])
    level, st = run_bfs(s, row_ptr, V, source, 0, prefetch)
    exp = bfs_levels(rp, col.cpu().numpy(), source)
    assert np.array_equal(level.cpu().numpy(), exp)
    assert st["edges"] == int(deg[exp >= 0].sum())      # every reached vertex is expanded once


@pytest.mark.parametrize("prefetch", [False, True])
def test_spmv_matches_oracle(gpu_system, prefetch):
    dev, src, dst, V, row_ptr, col = _graph(12, seed=3)
    E = col.numel()
    vals = edge_values(E, 3, dev)
    npg = pages_for(E)
    s = gpu_system(cache_lines=max(64, (2 * npg // 4) // 32 * 32), ways=32, blocks=2 * npg + 8, pairs=16,
                   engine_warps=16, warps=8)
    nxt = write_paged(s, 0, 0, col)
    write_paged(s, 0, nxt, vals)
    x = torch.rand(V, device=dev)
    y, st = run_spmv(s, row_ptr, V, 0, nxt, x, 1, prefetch)
    exp = spmv(row_ptr.cpu().numpy(), col.cpu().numpy(), vals.cpu().numpy(), x.cpu().numpy())
    got = y.cpu().numpy().astype(np.float64)
    assert np.max(np.abs(got - exp) / np.maximum(np.abs(exp), 1.0)) < 1e-5
    assert st["edges"] == E


def test_pagerank_matches_oracle(gpu_system):
    dev, src, dst, V, rowT, colT = _graph(12, seed=5, transpose=True)
    outdeg = torch.bincount(src, minlength=V)
    E = colT.numel()
    s = gpu_system(cache_lines=max(64, (pages_for(E) // 4) // 32 * 32), ways=32, blocks=pages_for(E) + 8,
                   pairs=16, engine_warps=16, warps=8)
    write_paged(s, 0, 0, colT)
    r, st = run_pagerank(s, rowT, V, 0, outdeg, 10)
    exp = pagerank(rowT.cpu().numpy(), colT.cpu().numpy(), outdeg.cpu().numpy(), 10)
    got = r.cpu().numpy().astype(np.float64)
    assert np.max(np.abs(got - exp) / np.maximum(np.abs(exp), 1e-12)) < 1e-4
