"""Graph workloads over a paged CSR (BASELINE configs[2] BFS, [3] SpMV/PageRank; new — the
reference has no graph driver).

* RMAT / Kronecker generator (Graph500 parameters A, B, C = 0.57, 0.19, 0.19; edge factor 16),
  vertex labels permuted, directed edges kept as generated (duplicates/self-loops included, as
  Graph500 does).  Built on the GPU with torch.
* CSR: row_ptr int64 [V+1] resident in HBM; col_idx int32 (and SpMV values fp32) laid out in the
  emulated device's page store, 1024 entries per 4 KiB page, read through the HBM cache.
* BFS: level-synchronous top-down, one fused launch per level, next-frontier pages prefetched as
  vertices are discovered.  SpMV: y = A x with next-row-block prefetch; PageRank: 10 iterations of
  r <- (1-d)/V + d * A^T (r / outdeg) on the transposed CSR with unit weights.
"""

from __future__ import annotations

import time

import numpy as np

ENTRIES_PER_PAGE = 1024


def rmat_edges(scale: int, edge_factor: int, seed: int, device, abc=(0.57, 0.19, 0.19)):
    import torch
    V = 1 << scale
    E = V * edge_factor
    g = torch.Generator(device=device).manual_seed(seed)
    a, b, c = abc
    src = torch.zeros(E, dtype=torch.int64, device=device)
    dst = torch.zeros(E, dtype=torch.int64, device=device)
    for lvl in range(scale):
        r = torch.rand(E, generator=g, device=device)
        sb = (r >= a + b).to(torch.int64)
        db = ((r >= a) & (r < a + b) | (r >= a + b + c)).to(torch.int64)
        src |= sb << lvl
        dst |= db << lvl
    perm = torch.randperm(V, generator=g, device=device)
    return perm[src], perm[dst], V


def build_csr(src, dst, V):
    """CSR by source: row_ptr int64 [V+1], col int32 [E] (stable by destination within a row)."""
    import torch
    key = src * V + dst
    key, _ = torch.sort(key)
    s = key // V
    col = (key % V).to(torch.int32)
    counts = torch.bincount(s, minlength=V)
    row_ptr = torch.zeros(V + 1, dtype=torch.int64, device=src.device)
    row_ptr[1:] = torch.cumsum(counts, 0)
    return row_ptr, col


def edge_values(E: int, seed: int, device):
    """Synthetic fp32 SpMV weights in [-1, 1) (hash of the edge index)."""
    import torch
    g = torch.Generator(device=device).manual_seed(seed + 7)
    return torch.rand(E, generator=g, device=device) * 2 - 1


def pages_for(n: int) -> int:
    return (n + ENTRIES_PER_PAGE - 1) // ENTRIES_PER_PAGE


def write_paged(system, dev: int, first_page: int, arr_gpu) -> int:
    """Copy a 4-byte-element GPU array into the pinned page store starting at first_page."""
    import torch
    view = system.store_view(dev)
    n = arr_gpu.numel()
    flat = view[first_page:first_page + pages_for(n)].reshape(-1).view(np.int32)[:n]
    torch.from_numpy(flat).copy_(arr_gpu.view(torch.int32))
    return first_page + pages_for(n)


def run_bfs(system, row_ptr, V, source: int, col_key0: int, prefetch: bool = True):
    """Levels int32 [V] (-1 unreachable), plus stats."""
    import torch
    dev = row_ptr.device
    level = torch.full((V,), -1, dtype=torch.int32, device=dev)
    level[source] = 0
    fa = torch.zeros(V, dtype=torch.int32, device=dev)
    fb = torch.zeros(V, dtype=torch.int32, device=dev)
    fa[0] = source
    n_in = 1
    cnt = torch.zeros(1, dtype=torch.int32, device=dev)
    ctr = torch.zeros(2, dtype=torch.int64, device=dev)
    st = torch.cuda.current_stream(dev)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(st)
    cur = 0
    levels = 0
    while n_in:
        cnt.zero_()
        system.bfs_level(row_ptr, level, fa, n_in, fb, cnt, col_key0, cur, prefetch, ctr, stream=st.cuda_stream)
        n_in = int(cnt.item())
        fa, fb = fb, fa
        cur += 1
        levels += 1
    e1.record(st)
    system.sync(st.cuda_stream)
    ms = e0.elapsed_time(e1)
    edges = int(ctr[0].item())
    return level, {"levels": levels, "ms": ms, "edges": edges, "teps": edges / (ms / 1e3) if ms else 0.0,
                   "wall_s": time.perf_counter() - t0}


def run_spmv(system, row_ptr, V, col_key0, val_key0, x, iters: int = 1, prefetch: bool = True):
    import torch
    dev = row_ptr.device
    y = torch.empty(V, dtype=torch.float32, device=dev)
    ctr = torch.zeros(2, dtype=torch.int64, device=dev)
    st = torch.cuda.current_stream(dev)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(iters):
        system.spmv(row_ptr, V, col_key0, val_key0, x, y, 1.0, 0.0, prefetch, ctr, stream=st.cuda_stream)
    e1.record(st)
    system.sync(st.cuda_stream)
    ms = e0.elapsed_time(e1)
    return y, {"ms": ms, "edges": int(ctr[0].item()), "gflops": 2 * int(ctr[0].item()) / (ms / 1e3) / 1e9}


def run_pagerank(system, rowT, V, colT_key0, outdeg, iters: int = 10, d: float = 0.85, prefetch: bool = True):
    """r <- (1-d)/V + d * A^T (r / outdeg) on the transposed CSR (in-edges), unit weights."""
    import torch
    dev = rowT.device
    r = torch.full((V,), 1.0 / V, dtype=torch.float32, device=dev)
    y = torch.empty_like(r)
    inv = torch.where(outdeg > 0, 1.0 / outdeg.clamp(min=1).float(), torch.zeros_like(r))
    ctr = torch.zeros(2, dtype=torch.int64, device=dev)
    st = torch.cuda.current_stream(dev)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(iters):
        x = r * inv
        system.spmv(rowT, V, colT_key0, None, x, y, d, (1 - d) / V, prefetch, ctr, stream=st.cuda_stream)
        r, y = y, r
    e1.record(st)
    system.sync(st.cuda_stream)
    return r, {"ms": e0.elapsed_time(e1), "edges": int(ctr[0].item())}


def run_graph(cfg, kind: str):
    """CLI experiments `bfs` / `spmv`: RMAT graph_scale, cache = graph_cache_fraction of edge bytes."""
    import copy

    import torch

    from . import BenchResult
    from ..system import AgileSystem
    dev = torch.device("cuda", torch.cuda.current_device())
    src, dst, V = rmat_edges(cfg.graph_scale, cfg.graph_edge_factor, cfg.system.seed, dev)
    if kind == "spmv":
        # PageRank runs on the transpose (in-edges)
        row_ptr, col = build_csr(dst, src, V)
        outdeg = torch.bincount(src, minlength=V)
    else:
        row_ptr, col = build_csr(src, dst, V)
    E = col.numel()
    vals = edge_values(E, cfg.system.seed, dev) if kind == "spmv" else None
    sc = copy.deepcopy(cfg.system)
    npages = pages_for(E) * (2 if vals is not None else 1)
    sc.device.num_blocks = max(npages, 1)
    lines = max(64, int(cfg.graph_cache_fraction * npages))
    sc.cache.bytes = 0
    sc.cache.lines = -(-lines // 32) * 32
    sc.cache.ways = 32
    res = BenchResult(header=["kind", "scale", "vertices", "edges", "prefetch", "ms", "rate"], rows=[], info={})
    with AgileSystem(sc) as system:
        nxt = write_paged(system, 0, 0, col)
        val_key0 = None
        if vals is not None:
            write_paged(system, 0, nxt, vals)
            val_key0 = nxt
        for pf in (False, True):
            system.reset()
            if kind == "bfs":
                deg = row_ptr[1:] - row_ptr[:-1]
                cand = torch.nonzero(deg > 0).flatten()
                g = torch.Generator(device="cpu").manual_seed(cfg.system.seed)
                source = int(cand[torch.randint(len(cand), (1,), generator=g).item()].item())
                _, st = run_bfs(system, row_ptr, V, source, 0, pf)
                res.rows.append(("bfs", cfg.graph_scale, V, E, int(pf), round(st["ms"], 3), round(st["teps"] / 1e9, 6)))
                res.info[f"bfs_levels_pf{int(pf)}"] = st["levels"]
            else:
                _, st = run_pagerank(system, row_ptr, V, 0, outdeg, cfg.pagerank_iters, prefetch=pf)
                res.rows.append(("pagerank", cfg.graph_scale, V, E, int(pf), round(st["ms"], 3),
                                 round(st["edges"] / (st["ms"] / 1e3) / 1e9, 6)))
                x = torch.rand(V, device=dev)
                system.reset()
                _, s2 = run_spmv(system, row_ptr, V, 0, val_key0, x, 1, pf)
                res.rows.append(("spmv", cfg.graph_scale, V, E, int(pf), round(s2["ms"], 3), round(s2["gflops"], 6)))
    return res
