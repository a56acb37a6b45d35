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


# ------------------------------------------------------------------ partitioned restatements
# CPU stand-ins for one rank of the 1D-partitioned BFS / PageRank (bench/graph.py BfsRank /
# PagerankRank): the same expand / merge / step interface, so the exchange logic (all-gather of
# frontier bitmaps and x slices over torch.distributed) is tested on CPU with gloo.

def _row_sum_f32(row_ptr, col, x32, rows, d, V):
    """fp32(d * sum_e fp64(x[col[e]]) + (1 - d) / V) per row, the kernel's rounding."""
    out = np.empty(len(rows), dtype=np.float32)
    xd = x32.astype(np.float64)
    for i, r in enumerate(rows):
        s = xd[col[row_ptr[r]:row_ptr[r + 1]]].sum()
        out[i] = np.float32(np.float64(np.float32(d)) * s + np.float64(np.float32((1 - d) / V)))
    return out


class OracleBfsRank:
    """numpy expand of the owned frontier; merge() is bench.graph.BfsRank.merge (torch on CPU)."""

    def __init__(self, part, row_ptr, col, V, source):
        import torch
        from paper_2504_19365_b200.bench.graph import BfsRank
        self.part, self.row_ptr, self.col, self.V = part, row_ptr, col, V
        self.nw = (V + 31) // 32
        self.visited = torch.zeros(self.nw, dtype=torch.int32)
        self.visited[source // 32] = torch.tensor(1 << (source % 32), dtype=torch.int64).to(torch.int32)
        self.level = torch.full((V,), -1, dtype=torch.int32)
        self.level[source] = 0
        own = part.v0 <= source < part.v1
        self.frontier = torch.tensor([source] if own else [], dtype=torch.int32)
        self.cur = 0
        self.merge = BfsRank.merge.__get__(self)

    def expand(self):
        import torch
        vis = self.visited.numpy().view(np.uint32)
        bits = np.zeros(self.nw, dtype=np.uint32)
        for v in self.frontier.numpy():
            for u in self.col[self.row_ptr[v]:self.row_ptr[v + 1]]:
                if not (vis[u >> 5] >> (u & 31)) & 1:
                    bits[u >> 5] |= np.uint32(1 << (u & 31))
                    self.level[int(u)] = self.cur + 1
        self.visited |= torch.from_numpy(bits.view(np.int32))
        return torch.from_numpy(bits.view(np.int32).copy())


class OraclePagerankRank:
    def __init__(self, part, rowT, colT, V, outdeg, d=0.85):
        import torch
        self.part, self.rowT, self.colT, self.V, self.d = part, rowT, colT, V, d
        n = part.v1 - part.v0
        self.r = torch.full((n,), 1.0 / V, dtype=torch.float32)
        od = torch.from_numpy(np.asarray(outdeg[part.v0:part.v1]))
        self.inv = torch.where(od > 0, 1.0 / od.clamp(min=1).float(), torch.zeros_like(self.r))

    def x_local(self):
        return self.r * self.inv

    def step(self, x_global):
        import torch
        rows = np.arange(self.part.v0, self.part.v1)
        self.r = torch.from_numpy(_row_sum_f32(self.rowT, self.colT, x_global.numpy(), rows, self.d, self.V))


def pagerank_f32(rowT, colT, outdeg, iters=10, d=0.85):
    """PageRank with the GPU path's roundings (x = fp32(r * fp32(1/outdeg)), row sums in fp64,
    r rounded to fp32 per iteration): the partitioned runs must reproduce it bit for bit."""
    import torch
    V = len(rowT) - 1
    r = torch.full((V,), 1.0 / V, dtype=torch.float32)
    od = torch.from_numpy(np.asarray(outdeg))
    inv = torch.where(od > 0, 1.0 / od.clamp(min=1).float(), torch.zeros_like(r))
    for _ in range(iters):
        x = (r * inv).numpy()
        r = torch.from_numpy(_row_sum_f32(rowT, colT, x, np.arange(V), d, V))
    return r.numpy()
