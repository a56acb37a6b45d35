"""GPU: the 1D-partitioned graph workloads (§8(e)) on one B200, rank by rank.  Every rank of a
G-way vertex partition gets its own context (cache, queue pairs, service, engine, page store
holding only its rows' col_idx / value pages) on cuda:0; the per-level frontier all-gather and
the per-iteration x all-gather are replayed in-process (bfs_partitioned / pagerank_partitioned
with the rank list).  Levels, SpMV sums and PageRank vectors must equal the single-GPU run bit
for bit, and BFS levels the CPU oracle."""

import numpy as np
import pytest
import torch

from conftest import small_config
from oracle.graph import bfs_levels
from paper_2504_19365_b200 import AgileSystem
from paper_2504_19365_b200.bench.graph import (BfsRank, PagerankRank, bfs_partitioned, edge_values, load_part,
                                               pages_for, pagerank_partitioned, partition_1d, pick_source,
                                               rmat_csr, run_bfs, run_pagerank, run_spmv, write_paged)

pytestmark = pytest.mark.gpu
DEV = torch.device("cuda", 0)


def _system(pages, frac=0.3):
    lines = max(64, int(frac * pages) // 32 * 32)
    return AgileSystem(small_config(cache_lines=lines, ways=32, blocks=pages + 8, pairs=16, engine_warps=16,
                                    warps=8), device=0)


@pytest.mark.parametrize("G", [2, 4])
def test_partitioned_bfs_matches_single_gpu(G):
    row_ptr, col, _ = rmat_csr(13, 16, 4, DEV, chunk=1 << 16)
    V, E = row_ptr.numel() - 1, col.numel()
    rp_h, col_h = row_ptr.cpu().numpy(), col.cpu().numpy()
    parts = partition_1d(rp_h, G)
    systems = [_system(p.pages) for p in parts]
    try:
        loaded = [load_part(s, p, row_ptr, col) for s, p in zip(systems, parts)]
        with _system(pages_for(E)) as one:
            write_paged(one, 0, 0, col)
            for seed in (0, 3):
                source = pick_source(row_ptr, seed)
                single, _ = run_bfs(one, row_ptr, V, source, 0, 0)
                ranks = [BfsRank(s, p, rp, V, source, prefetch_distance=seed % 3, col_key0=ck)
                         for s, p, (rp, ck, _) in zip(systems, parts, loaded)]
                bfs_partitioned(ranks)
                exp = bfs_levels(rp_h, col_h, source)
                assert np.array_equal(single.cpu().numpy(), exp)
                for r in ranks:
                    assert torch.equal(r.level, single), "partitioned levels differ from one GPU's"
                edges = sum(int(r.counters[0]) for r in ranks)
                assert edges == int(np.diff(rp_h)[exp >= 0].sum())     # each reached vertex expanded once
    finally:
        for s in systems:
            s.close()


@pytest.mark.parametrize("G", [2, 4])
def test_partitioned_pagerank_and_spmv_match_single_gpu(G):
    rowT, colT, outdeg = rmat_csr(13, 16, 6, DEV, transpose=True, chunk=1 << 16)
    V, E = rowT.numel() - 1, colT.numel()
    parts = partition_1d(rowT.cpu().numpy(), G)
    vals = edge_values(E, 6, DEV)
    systems = [_system(2 * p.pages) for p in parts]
    try:
        loaded = [load_part(s, p, rowT, colT, vals) for s, p in zip(systems, parts)]
        with _system(2 * pages_for(E)) as one:
            nxt = write_paged(one, 0, 0, colT)
            write_paged(one, 0, nxt, vals)
            r1, _ = run_pagerank(one, rowT, V, E, 0, outdeg, 10, prefetch_distance=1)
            ranks = [PagerankRank(s, p, rp, V, outdeg, prefetch_distance=2, col_key0=ck)
                     for s, p, (rp, ck, _) in zip(systems, parts, loaded)]
            pagerank_partitioned(ranks, 10)
            assert torch.equal(torch.cat([r.r for r in ranks]), r1), "partitioned PageRank differs"
            # weighted SpMV over the partition's rows, x global
            x = torch.rand(V, device=DEV, generator=torch.Generator(device=DEV).manual_seed(2))
            y1, _ = run_spmv(one, rowT, V, E, 0, nxt, x, 1, 0)
            ys = []
            for s, p, (rp, ck, vk) in zip(systems, parts, loaded):
                y = torch.empty(p.v1 - p.v0, dtype=torch.float32, device=DEV)
                s.spmv_rows(rp, p.v1 - p.v0, p.e_end, V, ck, vk, x, y, 1.0, 0.0, 1)
                s.sync()
                ys.append(y)
            assert torch.equal(torch.cat(ys), y1), "partitioned SpMV differs"
    finally:
        for s in systems:
            s.close()
