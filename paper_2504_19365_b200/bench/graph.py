"""Graph workloads over a paged CSR (BASELINE configs[2] BFS, [3] SpMV/PageRank; new — the
reference has no graph driver).

* RMAT / Kronecker generator (Graph500 parameters A, B, C = 0.57, 0.19, 0.19; edge factor 16),
  vertex labels permuted, directed edges kept as generated (duplicates/self-loops included, as
  Graph500 does).  Built on the GPU with torch in bounded memory (scale 27 = 2^31 edges).
* CSR: row_ptr int64 [V+1] resident in HBM; col_idx int32 (and SpMV values fp32) laid out in the
  emulated device's page store, 1024 entries per 4 KiB page, read through the HBM cache.
* BFS (agile_bfs): level-synchronous top-down over a sorted frontier, one fused launch per level;
  warps walk the frontier's edge list in chunks, async mode prefetches the pages of the chunks a
  warp grabbed ahead.  SpMV (agile_spmv): page-aligned edge chunks, deterministic row sums;
  PageRank: 10 iterations of r <- (1-d)/V + d * A^T (r / outdeg) on the in-edge CSR.
"""

from __future__ import annotations

import numpy as np

ENTRIES_PER_PAGE = 1024


def _rmat_chunk(n: int, scale: int, g, device, abc):
    """n RMAT edges (src, dst) int64 from generator g: per bit level, one uniform picks the quadrant."""
    import torch
    a, b, c = abc
    src = torch.zeros(n, dtype=torch.int64, device=device)
    dst = torch.zeros(n, dtype=torch.int64, device=device)
    for lvl in range(scale):
        r = torch.rand(n, generator=g, device=device)
        src |= (r >= a + b).to(torch.int64) << lvl
        dst |= (((r >= a) & (r < a + b)) | (r >= a + b + c)).to(torch.int64) << lvl
    return src, dst


def rmat_csr(scale: int, edge_factor: int, seed: int, device, transpose: bool = False,
             abc=(0.57, 0.19, 0.19), chunk: int = 1 << 27):
    """RMAT / Kronecker graph as CSR, built on the GPU in bounded memory (scale 27 = 2^31 edges).

    Edges are drawn in chunks, vertex labels permuted (Graph500), duplicates and self-loops kept.
    CSR by source (by destination with transpose=True, the in-edge CSR PageRank needs): keys
    src << scale | dst are sorted in buckets of the leading source bits (each bucket stays below
    2^31 keys), so col_idx is ascending within every row and the CSR is identical run to run.
    Returns row_ptr int64 [V+1], col int32 [E], out-degree int64 [V] (of the original direction).
    """
    import torch
    V = 1 << scale
    E = V * edge_factor
    g = torch.Generator(device=device).manual_seed(seed)
    perm = torch.randperm(V, generator=g, device=device)
    keys = torch.empty(E, dtype=torch.int64, device=device)
    outdeg = torch.zeros(V, dtype=torch.int64, device=device)
    for c0 in range(0, E, chunk):
        n = min(chunk, E - c0)
        src, dst = _rmat_chunk(n, scale, g, device, abc)
        src, dst = perm[src], perm[dst]
        outdeg += torch.bincount(src, minlength=V)
        if transpose:
            src, dst = dst, src
        keys[c0:c0 + n] = (src << scale) | dst
        del src, dst
    nb = 1
    while E // nb >= (1 << 30):
        nb *= 2
    col = torch.empty(E, dtype=torch.int32, device=device)
    deg = torch.zeros(V, dtype=torch.int64, device=device)
    pos = 0
    shift = 2 * scale - (nb.bit_length() - 1)
    for bkt in range(nb):
        sel = keys[(keys >> shift) == bkt] if nb > 1 else keys
        sel, _ = torch.sort(sel)
        col[pos:pos + sel.numel()] = (sel & (V - 1)).to(torch.int32)
        deg += torch.bincount(sel >> scale, minlength=V)
        pos += sel.numel()
        del sel
    del keys
    row_ptr = torch.zeros(V + 1, dtype=torch.int64, device=device)
    row_ptr[1:] = torch.cumsum(deg, 0)
    return row_ptr, col, outdeg


def edge_values(E: int, seed: int, device):
    """Synthetic fp32 SpMV weights in [-1, 1)."""
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


def pick_source(row_ptr, seed: int) -> int:
    """A seeded random vertex with out-degree > 0 (Graph500 search keys)."""
    import torch
    deg = row_ptr[1:] - row_ptr[:-1]
    cand = torch.nonzero(deg > 0).flatten()
    g = torch.Generator(device="cpu").manual_seed(seed)
    return int(cand[torch.randint(len(cand), (1,), generator=g).item()].item())


def run_bfs(system, row_ptr, V, source: int, col_key0: int, prefetch_distance: int = 0):
    """Levels int32 [V] (-1 unreachable), plus stats (levels, edges, page misses, ms, teps)."""
    import torch
    level = torch.empty(V, dtype=torch.int32, device=row_ptr.device)
    st = system.bfs(row_ptr, V, source, col_key0, level, prefetch_distance)
    st["teps"] = st["edges"] / (st["ms"] / 1e3) if st["ms"] else 0.0
    return level, st


def _timed(fn):
    import torch
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    fn()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


def run_spmv(system, row_ptr, V, E, col_key0, val_key0, x, iters: int = 1, prefetch_distance: int = 0):
    import torch
    y = torch.empty(V, dtype=torch.float32, device=row_ptr.device)
    ctr = torch.zeros(2, dtype=torch.int64, device=row_ptr.device)
    ms = _timed(lambda: [system.spmv(row_ptr, V, E, col_key0, val_key0, x, y, 1.0, 0.0, prefetch_distance, ctr)
                         for _ in range(iters)])
    system.sync()
    c = ctr.cpu().numpy()
    return y, {"ms": ms, "edges": int(c[0]), "page_misses": int(c[1]), "gflops": 2 * int(c[0]) / (ms / 1e3) / 1e9}


def run_pagerank(system, rowT, V, E, colT_key0, outdeg, iters: int = 10, d: float = 0.85, prefetch_distance: int = 0):
    """r <- (1-d)/V + d * A^T (r / outdeg) on the in-edge CSR, unit weights."""
    import torch
    r = torch.full((V,), 1.0 / V, dtype=torch.float32, device=rowT.device)
    y = torch.empty_like(r)
    inv = torch.where(outdeg > 0, 1.0 / outdeg.clamp(min=1).float(), torch.zeros_like(r))
    ctr = torch.zeros(2, dtype=torch.int64, device=rowT.device)

    def body():
        nonlocal r, y
        for _ in range(iters):
            x = r * inv
            system.spmv(rowT, V, E, colT_key0, None, x, y, d, (1 - d) / V, prefetch_distance, ctr)
            r, y = y, r
    ms = _timed(body)
    system.sync()
    c = ctr.cpu().numpy()
    return r, {"ms": ms, "edges": int(c[0]), "page_misses": int(c[1])}


def run_graph(cfg, kind: str):
    """CLI experiments `bfs` / `spmv`: RMAT graph_scale, cache = graph_cache_fraction of the paged
    bytes; sync (prefetch distance 0) and async (graph_prefetch) runs on a cold cache each."""
    import copy

    import torch

    from . import BenchResult
    from ..system import AgileSystem
    dev = torch.device("cuda", torch.cuda.current_device())
    seed = cfg.system.seed
    if kind == "spmv":
        row_ptr, col, outdeg = rmat_csr(cfg.graph_scale, cfg.graph_edge_factor, seed, dev, transpose=True)
    else:
        row_ptr, col, outdeg = rmat_csr(cfg.graph_scale, cfg.graph_edge_factor, seed, dev)
    V = row_ptr.numel() - 1
    E = col.numel()
    vals = edge_values(E, seed, dev) if kind == "spmv" else None
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
        del col, vals
        for pd in (0, cfg.graph_prefetch):
            system.reset()
            if kind == "bfs":
                source = pick_source(row_ptr, seed)
                _, st = run_bfs(system, row_ptr, V, source, 0, pd)
                res.rows.append(("bfs", cfg.graph_scale, V, E, pd, round(st["ms"], 3), round(st["teps"] / 1e9, 6)))
                res.info[f"bfs_levels_pd{pd}"] = st["levels"]
            else:
                _, st = run_pagerank(system, row_ptr, V, E, 0, outdeg, cfg.pagerank_iters, prefetch_distance=pd)
                res.rows.append(("pagerank", cfg.graph_scale, V, E, pd, round(st["ms"], 3),
                                 round(st["edges"] / (st["ms"] / 1e3) / 1e9, 6)))
                x = torch.rand(V, device=dev)
                system.reset()
                _, s2 = run_spmv(system, row_ptr, V, E, 0, val_key0, x, 1, pd)
                res.rows.append(("spmv", cfg.graph_scale, V, E, pd, round(s2["ms"], 3), round(s2["gflops"], 6)))
    return res


# ----------------------------------------------------------------------------- multi-GPU (§8(e))
# 1D vertex partition: rank r owns vertices [v0, v1) = an equal share of V, i.e. their CSR rows and
# the col_idx (and SpMV value) pages of those rows in its own page store, read through its own
# cache and queue pairs.  The rank's store starts at the unpartitioned CSR's page holding its first
# edge (local position = global position - base, base page-aligned), so its edges fall into the
# same 1024-edge chunks a single GPU uses: every SpMV row sum is formed in the same order and the
# sharded results are bit-identical to one GPU's.  Exchanges (torch.distributed, NCCL on GPUs):
#   BFS:      per level, all-gather of every rank's next-frontier bitmap (V/8 bytes), OR-reduced;
#   PageRank: per iteration, all-gather of the owned slices of x = r / outdeg (4 V / N bytes each).

from dataclasses import dataclass as _dataclass


@_dataclass
class GraphPart:
    rank: int
    world: int
    v0: int
    v1: int
    base: int      # page-aligned global edge position of the rank's first stored entry
    e_end: int     # local end position (global row_ptr[v1] - base)

    @property
    def pages(self) -> int:
        return pages_for(self.e_end)


def partition_1d(row_ptr_host: np.ndarray, world: int):
    V = len(row_ptr_host) - 1
    assert V % (32 * world) == 0, "V must split into word-aligned equal vertex ranges"
    parts = []
    for r in range(world):
        v0, v1 = r * V // world, (r + 1) * V // world
        e0, e1 = int(row_ptr_host[v0]), int(row_ptr_host[v1])
        base = e0 - e0 % ENTRIES_PER_PAGE
        parts.append(GraphPart(r, world, v0, v1, base, e1 - base))
    return parts


def load_part(system, part: GraphPart, row_ptr, col, vals=None):
    """Write the rank's col (and value) pages into its store; returns (local row_ptr, col_key0,
    val_key0) — row_ptr local = global[v0 : v1 + 1] - base."""
    rp = (row_ptr[part.v0:part.v1 + 1] - part.base).contiguous()
    e1 = part.base + part.e_end
    nxt = write_paged(system, 0, 0, col[part.base:e1])
    vk = None
    if vals is not None:
        write_paged(system, 0, nxt, vals[part.base:e1])
        vk = nxt
    return rp, 0, vk


def bits_to_ids(words, offset: int = 0):
    """Ascending vertex ids of the set bits of an int32 bitmap (bit k of word w = vertex 32 w + k)."""
    import torch
    w = words.to(torch.int64) & 0xFFFFFFFF
    nz = torch.nonzero(w).flatten()
    if nz.numel() == 0:
        return torch.empty(0, dtype=torch.int32, device=words.device)
    ar = torch.arange(32, device=words.device)
    bits = ((w[nz].unsqueeze(1) >> ar) & 1).bool()
    ids = (nz.unsqueeze(1) * 32 + ar)[bits]
    return (ids + offset).to(torch.int32)


class BfsRank:
    """One rank of the partitioned BFS: expands the frontier vertices it owns (agile_bfs_level);
    visited / level are kept globally on every rank and merged after each level's exchange."""

    def __init__(self, system, part: GraphPart, row_ptr_local, V: int, source: int, prefetch_distance: int = 0,
                 col_key0: int = 0):
        import torch
        dev = row_ptr_local.device
        self.s, self.part, self.rp, self.V, self.pd, self.ck = system, part, row_ptr_local, V, prefetch_distance, col_key0
        self.nw = (V + 31) // 32
        self.visited = torch.zeros(self.nw, dtype=torch.int32, device=dev)
        self.visited[source // 32] = torch.tensor(1 << (source % 32), dtype=torch.int64).to(torch.int32)
        self.level = torch.full((V,), -1, dtype=torch.int32, device=dev)
        self.level[source] = 0
        own = part.v0 <= source < part.v1
        self.frontier = torch.tensor([source] if own else [], dtype=torch.int32, device=dev)
        self.cur = 0
        self.counters = torch.zeros(2, dtype=torch.int64, device=dev)

    def expand(self):
        import torch
        nb = torch.zeros(self.nw, dtype=torch.int32, device=self.rp.device)
        if self.frontier.numel():
            self.s.bfs_level(self.rp, self.part.v0, self.frontier, self.visited, nb, self.level, self.cur, self.ck,
                             self.pd, self.counters)
        return nb

    def merge(self, nb_global) -> int:
        new = nb_global & ~self.visited
        self.visited |= nb_global
        ids = bits_to_ids(new)
        if ids.numel():
            self.level[ids.long()] = self.cur + 1
        w0, w1 = self.part.v0 // 32, (self.part.v1 + 31) // 32
        self.frontier = bits_to_ids(nb_global[w0:w1], self.part.v0)
        self.cur += 1
        return int(bits_to_ids(nb_global).numel())


def _or_reduce(stack):
    import functools
    import torch
    return functools.reduce(torch.bitwise_or, list(stack))


def bfs_partitioned(ranks, allgather=None):
    """Level-synchronous BFS over partition ranks.  `ranks`: this process's rank objects — one
    (multi-process: allgather = torch.distributed all-gather of a tensor into [world, ...]) or all
    of them (single process: the all-gather is the list itself).  Returns levels run."""
    levels = 0
    while True:
        nbs = [r.expand() for r in ranks]
        gathered = allgather(nbs[0]) if allgather is not None else nbs
        nb = _or_reduce(gathered)
        levels += 1
        n = [r.merge(nb) for r in ranks][0]
        if n == 0:
            return levels


class PagerankRank:
    """One rank of the partitioned PageRank: r over its owned vertices, SpMV over its rows."""

    def __init__(self, system, part: GraphPart, row_ptr_local, V: int, outdeg, d: float = 0.85,
                 prefetch_distance: int = 0, col_key0: int = 0):
        import torch
        dev = row_ptr_local.device
        self.s, self.part, self.rp, self.V, self.d, self.pd, self.ck = system, part, row_ptr_local, V, d, prefetch_distance, col_key0
        n = part.v1 - part.v0
        self.r = torch.full((n,), 1.0 / V, dtype=torch.float32, device=dev)
        self.y = torch.empty_like(self.r)
        od = outdeg[part.v0:part.v1]
        self.inv = torch.where(od > 0, 1.0 / od.clamp(min=1).float(), torch.zeros_like(self.r))
        self.counters = torch.zeros(2, dtype=torch.int64, device=dev)

    def x_local(self):
        return self.r * self.inv

    def step(self, x_global):
        self.s.spmv_rows(self.rp, self.part.v1 - self.part.v0, self.part.e_end, self.V, self.ck, None, x_global,
                         self.y, self.d, (1 - self.d) / self.V, self.pd, self.counters)
        self.r, self.y = self.y, self.r


def pagerank_partitioned(ranks, iters: int, allgather=None):
    import torch
    for _ in range(iters):
        xs = [r.x_local() for r in ranks]
        x = torch.cat(list(allgather(xs[0]))) if allgather is not None else torch.cat(xs)
        for r in ranks:
            r.step(x)
