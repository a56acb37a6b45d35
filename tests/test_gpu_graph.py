"""GPU parity of BFS (levels bit-exact) and SpMV / PageRank (1e-5 relative, north_star) over a paged CSR,
against the CPU restatement in oracle/graph.py, for sync (prefetch distance 0) and async modes and
for caches smaller and larger than the paged arrays."""

import numpy as np
import pytest
import torch

from oracle.graph import bfs_levels, pagerank, pagerank_f32, spmv
from paper_2504_19365_b200.bench.graph import (edge_values, pages_for, pick_source, rmat_csr, run_bfs,
                                               run_pagerank, run_spmv, write_paged)

pytestmark = pytest.mark.gpu


def _graph(scale, seed=1, transpose=False):
    dev = torch.device("cuda", 0)
    row_ptr, col, outdeg = rmat_csr(scale, 16, seed, dev, transpose=transpose, chunk=1 << 16)
    return dev, row_ptr, col, outdeg


def test_rmat_csr_is_sorted_and_deterministic():
    dev, rp, col, od = _graph(12, seed=9)
    _, rp2, col2, _ = _graph(12, seed=9)
    assert torch.equal(rp, rp2) and torch.equal(col, col2)
    r, c = rp.cpu().numpy(), col.cpu().numpy()
    assert r[0] == 0 and r[-1] == len(c) == (1 << 12) * 16
    for v in range(0, 1 << 12, 97):   # ascending within rows
        seg = c[r[v]:r[v + 1]]
        assert np.all(seg[1:] >= seg[:-1])
    assert int(od.sum()) == len(c)


@pytest.mark.parametrize("pd", [0, 2])
@pytest.mark.parametrize("frac", [0.25, 1.5])
def test_bfs_levels_match_oracle(gpu_system, pd, frac):
    dev, row_ptr, col, _ = _graph(14)
    V = row_ptr.numel() - 1
    E = col.numel()
    lines = max(64, int(frac * pages_for(E)) // 32 * 32)
    s = gpu_system(cache_lines=lines, ways=32, blocks=pages_for(E) + 8, pairs=16, engine_warps=16, warps=8)
    write_paged(s, 0, 0, col)
    rp = row_ptr.cpu().numpy()
    for seed in (0, 1):
        s.reset()
        source = pick_source(row_ptr, seed)
        level, st = run_bfs(s, row_ptr, V, source, 0, pd)
        exp = bfs_levels(rp, col.cpu().numpy(), source)
        assert np.array_equal(level.cpu().numpy(), exp)
        deg = np.diff(rp)
        assert st["edges"] == int(deg[exp >= 0].sum())      # every reached vertex is expanded once
        assert st["levels"] == int(exp.max()) + 1          # one launch per non-empty frontier


def test_bfs_isolated_source(gpu_system):
    # a source without out-edges: one level, only the source reached
    rp = torch.tensor([0, 0, 2, 3], dtype=torch.int64, device="cuda")
    col = torch.tensor([0, 2, 1], dtype=torch.int32, device="cuda")
    s = gpu_system(cache_lines=64, ways=32, blocks=8, pairs=4, engine_warps=4, warps=2)
    write_paged(s, 0, 0, col)
    level, st = run_bfs(s, rp, 3, 0, 0, 0)
    assert level.cpu().tolist() == [0, -1, -1]
    level, st = run_bfs(s, rp, 3, 1, 0, 1)
    assert level.cpu().tolist() == [1, 0, 1]


@pytest.mark.parametrize("pd", [0, 2])
def test_spmv_matches_oracle(gpu_system, pd):
    dev, row_ptr, col, _ = _graph(13, seed=3)
    V = row_ptr.numel() - 1
    E = col.numel()
    vals = edge_values(E, 3, dev)
    npg = pages_for(E)
    s = gpu_system(cache_lines=max(64, (2 * npg // 4) // 32 * 32), ways=32, blocks=2 * npg + 8, pairs=16,
                   engine_warps=16, warps=8)
    nxt = write_paged(s, 0, 0, col)
    write_paged(s, 0, nxt, vals)
    x = torch.rand(V, device=dev, generator=torch.Generator(device=dev).manual_seed(5 + pd))
    y, st = run_spmv(s, row_ptr, V, E, 0, nxt, x, 1, pd)
    rp_, col_, vals_, x_ = row_ptr.cpu().numpy(), col.cpu().numpy(), vals.cpu().numpy(), x.cpu().numpy()
    exp = spmv(rp_, col_, vals_, x_)
    got = y.cpu().numpy().astype(np.float64)
    # 1e-5 relative to |y| (north_star).  The kernel sums exact fp64 products in fp64 and rounds
    # once, so its error is half an fp32 ulp of y plus ~1e-16 of the row's term magnitudes: the
    # second term only shows when a row's +-1 weights cancel to below 1e-10 of its magnitude.
    mag = spmv(rp_, col_, np.abs(vals_), np.abs(x_))
    assert np.all(np.abs(got - exp) <= 1e-5 * np.abs(exp) + 1e-12 * mag)
    assert st["edges"] == E
    # deterministic summation order: a second run is bit-identical
    y2, _ = run_spmv(s, row_ptr, V, E, 0, nxt, x, 1, pd)
    assert torch.equal(y, y2)


def test_spmv_hub_rows_span_chunks(gpu_system):
    # rows far longer than a 1024-edge chunk, empty rows between them, a last partial chunk
    dev = torch.device("cuda", 0)
    deg = torch.tensor([0, 5000, 0, 0, 3, 2500, 1, 0, 1024, 7], dtype=torch.int64)
    rp = torch.zeros(len(deg) + 1, dtype=torch.int64)
    rp[1:] = torch.cumsum(deg, 0)
    E = int(rp[-1])
    g = torch.Generator().manual_seed(4)
    col = torch.randint(0, len(deg), (E,), generator=g, dtype=torch.int32)
    vals = torch.rand(E, generator=g) * 2 - 1
    x = torch.rand(len(deg), generator=g)
    npg = pages_for(E)
    s = gpu_system(cache_lines=64, ways=32, blocks=2 * npg + 8, pairs=4, engine_warps=4, warps=2)
    nxt = write_paged(s, 0, 0, col.to(dev))
    write_paged(s, 0, nxt, vals.to(dev))
    y, _ = run_spmv(s, rp.to(dev), len(deg), E, 0, nxt, x.to(dev), 1, 1)
    exp = spmv(rp.numpy(), col.numpy(), vals.numpy(), x.numpy())
    mag = spmv(rp.numpy(), col.numpy(), np.abs(vals.numpy()), np.abs(x.numpy()))
    assert np.all(np.abs(y.cpu().numpy() - exp) <= 1e-5 * np.abs(exp) + 1e-12 * mag)


def test_pagerank_matches_oracle(gpu_system):
    dev, rowT, colT, outdeg = _graph(12, seed=5, transpose=True)
    V = rowT.numel() - 1
    E = colT.numel()
    s = gpu_system(cache_lines=max(64, (pages_for(E) // 4) // 32 * 32), ways=32, blocks=pages_for(E) + 8,
                   pairs=16, engine_warps=16, warps=8)
    write_paged(s, 0, 0, colT)
    r, st = run_pagerank(s, rowT, V, E, 0, outdeg, 10, prefetch_distance=2)
    exp = pagerank(rowT.cpu().numpy(), colT.cpu().numpy(), outdeg.cpu().numpy(), 10)
    got = r.cpu().numpy().astype(np.float64)
    assert np.max(np.abs(got - exp) / np.abs(exp)) < 1e-5       # north_star: 1e-5 relative
    # against the restatement with the GPU path's roundings: within one fp32 ulp (the fp64 row
    # sums may differ in their last bits between summation orders)
    f32 = pagerank_f32(rowT.cpu().numpy(), colT.cpu().numpy(), outdeg.cpu().numpy(), 10)
    assert np.max(np.abs(r.cpu().numpy() - f32) / f32) < 2.5e-7


def test_rmat22_bfs_spmv_pagerank_match_c_oracle(gpu_system):
    """RMAT scale 22 (4.2 M vertices, 67 M edges), cache = 25 % of the paged arrays, async mode,
    against the C oracle (oracle/graph_oracle.c): BFS levels bit-exact, SpMV and PageRank within
    1e-5 relative."""
    from oracle import cgraph
    dev, row_ptr, col, _ = _graph(22, seed=4)
    V, E = row_ptr.numel() - 1, col.numel()
    npg = pages_for(E)
    s = gpu_system(cache_lines=max(64, (2 * npg // 4) // 32 * 32), ways=32, blocks=2 * npg + 8, pairs=64,
                   sq_depth=256, cq_depth=256, engine_warps=64, warps=16)
    nxt = write_paged(s, 0, 0, col)
    vals = edge_values(E, 4, dev)
    write_paged(s, 0, nxt, vals)
    rp = row_ptr.cpu().numpy()
    col_h = col.cpu().numpy()
    src = pick_source(row_ptr, 0)
    level, _ = run_bfs(s, row_ptr, V, src, 0, 2)
    assert np.array_equal(level.cpu().numpy(), cgraph.bfs_levels(rp, col_h, src))
    x = torch.rand(V, device=dev)
    s.reset()
    y, _ = run_spmv(s, row_ptr, V, E, 0, nxt, x, 1, 2)
    vh, xh = vals.cpu().numpy(), x.cpu().numpy()
    exp = cgraph.spmv_f32(rp, col_h, vh, xh).astype(np.float64)
    mag = cgraph.spmv_f32(rp, col_h, np.abs(vh), np.abs(xh)).astype(np.float64)
    assert np.all(np.abs(y.cpu().numpy() - exp) <= 1e-5 * np.abs(exp) + 1e-12 * mag)
    # PageRank on the transpose (in-edge CSR) of a second graph
    _, rowT, colT, outdeg = _graph(22, seed=5, transpose=True)
    ET = colT.numel()
    s2 = gpu_system(cache_lines=max(64, (pages_for(ET) // 4) // 32 * 32), ways=32, blocks=pages_for(ET) + 8, pairs=64,
                    sq_depth=256, cq_depth=256, engine_warps=64, warps=16)
    write_paged(s2, 0, 0, colT)
    r, _ = run_pagerank(s2, rowT, V, ET, 0, outdeg, 10, prefetch_distance=2)
    pexp = cgraph.pagerank_f32(rowT.cpu().numpy(), colT.cpu().numpy(), outdeg.cpu().numpy(), 10).astype(np.float64)
    assert np.max(np.abs(r.cpu().numpy() - pexp) / pexp) < 1e-5
