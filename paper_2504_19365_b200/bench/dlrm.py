"""DLRM embedding-bag driver (BASELINE configs[1] and [4]; new workload — the reference's
ancestor is the synthetic gather of bench/sweeps.py:1-9, which "stands in for embedding lookups").

* 26 Criteo-shaped tables (Kaggle cardinalities scaled to a byte budget), dim 128, fp32 rows,
  8 rows per 4 KiB page, laid out contiguously in the emulated device's page store.
* Indices: bounded Zipf(alpha) ranks per table, optionally scattered over rows by a bijective
  multiplicative hash (hashed categorical ids), deterministic per (seed, batch).
* Table-wise + row-wise sharding over G ranks (plan_shards), balanced by bytes and lookups;
  K5 writes every rank's pooled rows straight into the peer-major all-to-all send buffer, one
  unpadded all_to_all_single exchanges them, combine() adds the row-wise partials.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import os

import numpy as np

# Criteo Kaggle categorical cardinalities (26 sparse features)
CRITEO_KAGGLE = (1460, 583, 10131227, 2202608, 305, 24, 12517, 633, 3, 93145, 5683, 8351593, 3194,
                 27, 14992, 5461306, 10, 5652, 2173, 4, 7046547, 18, 15, 286181, 105, 142572)


def table_rows(total_bytes: int, dim: int = 128, tables: int = 26) -> np.ndarray:
    """Row counts with the Criteo skew, scaled so the tables total ~total_bytes."""
    base = np.array([CRITEO_KAGGLE[i % len(CRITEO_KAGGLE)] for i in range(tables)], dtype=np.float64)
    scale = total_bytes / (base.sum() * dim * 4)
    return np.maximum(1, np.floor(base * scale)).astype(np.int64)


def layout(rows: np.ndarray, dim: int, dev: int = 0, first_page: int = 0):
    """Contiguous page ranges per table: returns (key0[T] uint64, total_pages)."""
    rpp = 4096 // (4 * dim)
    pages = (rows + rpp - 1) // rpp
    start = first_page + np.concatenate([[0], np.cumsum(pages)[:-1]])
    key0 = (np.uint64(dev) << np.uint64(36)) | start.astype(np.uint64)
    return key0, int(first_page + pages.sum())


def _scatter_mult(n: int) -> int:
    m = 2654435761 % n if n > 1 else 1
    while math.gcd(m, n) != 1:
        m += 1
    return m


def zipf_rows(rng: np.random.Generator, n: int, size, alpha: float, scatter: bool) -> np.ndarray:
    """Bounded Zipf over ranks 1..n (inverse-CDF of the continuous approximation), mapped to rows."""
    u = rng.random(size)
    if abs(alpha - 1.0) < 1e-9:
        r = np.exp(u * np.log(n + 1.0))
    else:
        a1 = 1.0 - alpha
        r = (1.0 + u * ((n + 1.0) ** a1 - 1.0)) ** (1.0 / a1)
    rank = np.clip(np.floor(r).astype(np.int64) - 1, 0, n - 1)
    if not scatter or n == 1:
        return rank
    return (rank * _scatter_mult(n) + 12345) % n


def make_batch(seed: int, step: int, rows: np.ndarray, B: int, L: int, alpha: float, scatter: bool,
               tables=None) -> np.ndarray:
    """int64 [B, len(tables), L]; table t's indices depend only on (seed, step, t), so every rank
    generates exactly its own tables' slice of the global batch."""
    tables = range(len(rows)) if tables is None else tables
    return np.stack([zipf_rows(np.random.default_rng([seed, step, int(t)]), int(rows[t]), (B, L), alpha, scatter)
                     for t in tables], axis=1)


def gpu_zipf_batch(gen, rows_t, B: int, L: int, alpha: float, scatter: bool, device):
    """Same bounded-Zipf construction on the GPU (torch), for untimed cache warm-up batches."""
    import torch
    cols = []
    for n in rows_t.tolist():
        u = torch.rand((B, L), generator=gen, device=device, dtype=torch.float64)
        if abs(alpha - 1.0) < 1e-9:
            r = torch.exp(u * np.log(n + 1.0))
        else:
            a1 = 1.0 - alpha
            r = (1.0 + u * ((n + 1.0) ** a1 - 1.0)) ** (1.0 / a1)
        rank = torch.clamp(torch.floor(r).to(torch.int64) - 1, 0, n - 1)
        if scatter and n > 1:
            rank = (rank * _scatter_mult(n) + 12345) % n
        cols.append(rank)
    return torch.stack(cols, dim=1).contiguous()


# ----------------------------------------------------------------------------- sharding (configs[4])

# one agile_table_shard (include/agile_b200.h) per table piece of a launch
TAB_DTYPE = np.dtype([("key0", "<u8"), ("row0", "<i8"), ("rows", "<i8"), ("table_rows", "<i8"),
                      ("out_offset", "<u4"), ("flags", "<u4")])
assert TAB_DTYPE.itemsize == 40
PARTIAL_F64 = 1


@dataclass
class Piece:
    """Rows [row0, row0 + rows) of global table `table`; `partial`: the table is split by rows over
    several ranks, so this rank sends its fp64 partial sums and the sample's owner adds them."""
    table: int
    row0: int
    rows: int
    partial: bool


@dataclass
class ShardPlan:
    """Table-wise + row-wise sharding of the DLRM tables over `world` ranks (TWRW).

    Small tables stay whole and are spread by lookup count; large tables are cut into page-aligned
    row ranges so every rank holds about 1/world of the table bytes and of the lookups.  Row-wise
    pieces pool fp64 partial sums; because the kernel accumulates in fp64 (exact for the synthetic
    rows), the receiver's fp64 sum of the partials rounds to the same fp32 as a single device."""
    world: int
    dim: int
    rows: np.ndarray
    pieces: list   # per rank: [Piece], whole tables first, then partials

    @property
    def rpp(self) -> int:
        return 4096 // (4 * self.dim)

    def rank_tables(self, rank: int) -> np.ndarray:
        return np.array([p.table for p in self.pieces[rank]], dtype=np.int64)

    def row_bytes(self, rank: int) -> int:
        """bytes of one sample's output row on `rank`: D fp32 per whole table, D fp64 per piece"""
        return sum(self.dim * (8 if p.partial else 4) for p in self.pieces[rank])

    def n_whole(self, rank: int) -> int:
        return sum(1 for p in self.pieces[rank] if not p.partial)

    def rank_layout(self, rank: int, dev: int = 0, first_page: int = 0):
        """(descs [P] TAB_DTYPE, first page of every piece [P], total pages) of the rank's store."""
        ps = self.pieces[rank]
        descs = np.zeros(len(ps), dtype=TAB_DTYPE)
        first = np.zeros(len(ps), dtype=np.int64)
        page, off = first_page, 0
        for j, p in enumerate(ps):
            first[j] = page
            descs[j] = ((dev << 36) | page, p.row0, p.rows, int(self.rows[p.table]), off,
                        PARTIAL_F64 if p.partial else 0)
            page += (p.rows + self.rpp - 1) // self.rpp
            off += self.dim * (8 if p.partial else 4)
        return descs, first, page

    def balance(self, lookups_by_table=None) -> dict:
        """max/mean over ranks of table bytes and of lookups (expected: proportional to the rows of
        a piece, or counted: lookups_by_table[t] = callable(row0, rows) -> lookups in the range)."""
        by = np.array([sum(p.rows for p in ps) for ps in self.pieces], dtype=np.float64)
        if lookups_by_table is None:
            lk = np.array([sum(p.rows / self.rows[p.table] for p in ps) for ps in self.pieces])
        else:
            lk = np.array([sum(lookups_by_table[p.table](p.row0, p.rows) for p in ps) for ps in self.pieces],
                          dtype=np.float64)
        return {"bytes": float(by.max() / by.mean()), "lookups": float(lk.max() / lk.mean()),
                "pieces": [len(ps) for ps in self.pieces]}


def plan_shards(rows: np.ndarray, world: int, dim: int = 128, eps: float = 0.03,
                small_frac: float = 0.05) -> ShardPlan:
    """Greedy TWRW plan.  Tables are taken largest first.  A table whose pages exceed small_frac of
    a rank's byte target is cut into page-aligned row ranges, each put on the rank with the lowest
    normalised load max(lookups / target, bytes / target) and sized to fill it up to (1 + eps) of
    both targets.  Smaller tables stay whole, on the rank with the fewest lookups (ties: bytes)."""
    rows = np.asarray(rows, dtype=np.int64)
    T = len(rows)
    rpp = 4096 // (4 * dim)
    pages = (rows + rpp - 1) // rpp
    tl, tb = T / world, pages.sum() / world
    ll = np.zeros(world)
    lb = np.zeros(world)
    raw = [[] for _ in range(world)]
    for t in np.argsort(-rows, kind="stable"):
        n = int(rows[t])
        if world == 1 or pages[t] <= small_frac * tb:
            g = int(np.lexsort((lb, ll))[0])
            raw[g].append((int(t), 0, n))
            ll[g] += 1
            lb[g] += pages[t]
            continue
        r0 = 0
        while r0 < n:
            g = int(np.argmin(np.maximum(ll / tl, lb / tb)))
            rem = n - r0
            fit = min(((1 + eps) * tl - ll[g]) * n, ((1 + eps) * tb - lb[g]) * rpp)
            take = rem if fit >= rem else min(rem, max(rpp, int(fit) // rpp * rpp))
            raw[g].append((int(t), r0, take))
            ll[g] += take / n
            lb[g] += (take + rpp - 1) // rpp
            r0 += take
    split = {t for ps in raw for (t, r0, k) in ps if k < rows[t]}
    pieces = []
    for ps in raw:
        whole = [Piece(t, r0, k, False) for (t, r0, k) in sorted(ps) if t not in split]
        part = [Piece(t, r0, k, True) for (t, r0, k) in sorted(ps) if t in split]
        pieces.append(whole + part)
    return ShardPlan(world=world, dim=dim, rows=rows, pieces=pieces)


def fill_rank_store(system, plan: ShardPlan, rank: int, seed: int, dev: int = 0) -> None:
    """Write the rank's pieces into its page store, row-keyed (oracle/pages.py row_floats)."""
    descs, first, _ = plan.rank_layout(rank, dev)
    for j, p in enumerate(plan.pieces[rank]):
        system.fill_rows(dev, seed, int(first[j]), p.table, p.row0, p.rows, plan.dim)


def combine(plan: ShardPlan, recv, n_local: int):
    """Received bytes (all_to_all_single output: peer q's [n_local, row_bytes(q)] blocks in rank
    order) -> pooled [n_local, T, D] fp32 in global table order: whole tables copied, row-wise
    pieces summed in fp64 (exact) and rounded once."""
    import torch
    D, T = plan.dim, len(plan.rows)
    out = torch.empty((n_local, T, D), dtype=torch.float32, device=recv.device)
    split = sorted({p.table for ps in plan.pieces for p in ps if p.partial})
    slot = {t: i for i, t in enumerate(split)}
    acc = torch.zeros((n_local, len(split), D), dtype=torch.float64, device=recv.device) if split else None
    off = 0
    for q, ps in enumerate(plan.pieces):
        rb = plan.row_bytes(q)
        blk = recv[off:off + n_local * rb].view(n_local, rb)
        off += n_local * rb
        nw = plan.n_whole(q)
        if nw:
            tw = torch.as_tensor([p.table for p in ps[:nw]], dtype=torch.long, device=recv.device)
            out[:, tw] = blk[:, :nw * D * 4].contiguous().view(torch.float32).view(n_local, nw, D)
        if len(ps) > nw:
            sl = torch.as_tensor([slot[p.table] for p in ps[nw:]], dtype=torch.long, device=recv.device)
            acc.index_add_(1, sl, blk[:, nw * D * 4:].contiguous().view(torch.float64).view(n_local, len(ps) - nw, D))
    if split:
        out[:, torch.as_tensor(split, dtype=torch.long, device=recv.device)] = acc.to(torch.float32)
    return out


def exchange(plan: ShardPlan, send, rank: int, batch: int):
    """One all_to_all_single of the kernel's output rows: `send` is the rank's [batch, row_bytes]
    uint8 buffer, peer-major along the batch (samples [p*batch/G, (p+1)*batch/G) go to rank p),
    unpadded: rank q's rows are row_bytes(q) wide (input/output split sizes per peer)."""
    import torch
    import torch.distributed as dist
    G = plan.world
    nl = batch // G
    rb = plan.row_bytes(rank)
    out_splits = [nl * plan.row_bytes(q) for q in range(G)]
    recv = torch.empty(sum(out_splits), dtype=torch.uint8, device=send.device)
    dist.all_to_all_single(recv, send.view(-1), out_splits, [nl * rb] * G)
    return combine(plan, recv, nl)


def pool_rank_reference(plan: ShardPlan, rank: int, idx: np.ndarray, seed: int) -> np.ndarray:
    """CPU restatement of the rank's K5 output rows ([B, row_bytes] uint8) from row-keyed tables:
    whole tables fp32(fp64 sum), row pieces the fp64 partial over the rows they hold.  Test
    infrastructure for the exchange (the gloo test) — the GPU path writes these bytes itself."""
    from oracle.pages import row_floats
    B = idx.shape[0]
    D = plan.dim
    cols = []
    for j, p in enumerate(plan.pieces[rank]):
        ix = idx[:, j, :]
        m = (ix >= p.row0) & (ix < p.row0 + p.rows)
        acc = np.zeros((B, D), dtype=np.float64)
        if m.any():
            uniq, inv = np.unique(ix[m], return_inverse=True)
            vals = row_floats(seed, p.table, uniq, D).astype(np.float64)
            bi = np.nonzero(m)[0]
            np.add.at(acc, bi, vals[inv])
        cols.append(acc.view(np.uint8) if p.partial else acc.astype(np.float32).view(np.uint8))
    return np.ascontiguousarray(np.concatenate(cols, axis=1)) if cols else np.zeros((B, 0), np.uint8)


# ----------------------------------------------------------------------------- DLRM model + pipeline

class DlrmModel:
    """DLRM forward (Criteo-style): bottom MLP 13-512-256-128 on dense features, pairwise dot
    interaction of the 26 pooled embeddings + dense vector, top MLP 479(+pad)-1024-1024-512-256-1.
    bf16 weights/activations on the tensor cores through torch (the MLPs run outside the hot path,
    BASELINE north star); `repeat` re-runs the top MLP to scale compute for CTC studies."""

    def __init__(self, device, dim=128, tables=26, dense=13, repeat=1, seed=0):
        import torch
        g = torch.Generator(device="cpu").manual_seed(seed)
        self.dim, self.tables, self.repeat = dim, tables, repeat
        def mlp(sizes):
            return [((torch.randn(b, a, generator=g) / a ** 0.5).to(device, torch.bfloat16),
                     torch.zeros(b, device=device, dtype=torch.bfloat16)) for a, b in zip(sizes[:-1], sizes[1:])]
        self.bot = mlp([dense, 512, 256, dim])
        n = tables + 1
        self.inter = n * (n - 1) // 2
        self.top = mlp([self.inter + dim, 1024, 1024, 512, 256, 1])
        self.iu = torch.triu_indices(n, n, offset=1, device=device)

    @staticmethod
    def _run(layers, x):
        import torch
        for i, (w, b) in enumerate(layers):
            x = torch.nn.functional.linear(x, w, b)
            if i + 1 < len(layers):
                x = torch.relu(x)
        return x

    def forward(self, dense, pooled):
        import torch
        z = self._run(self.bot, dense)                                  # [B, dim]
        feats = torch.cat([z.unsqueeze(1), pooled.to(torch.bfloat16)], dim=1)   # [B, 27, dim]
        inter = torch.bmm(feats, feats.transpose(1, 2))[:, self.iu[0], self.iu[1]]
        x = torch.cat([z, inter], dim=1)
        out = None
        for _ in range(self.repeat):
            out = self._run(self.top, x)
        return torch.sigmoid(out)

    def capture(self, dense, pooled, repeat: int, sm_carveout: int = 0):
        """The forward as one CUDA graph over the fixed `pooled` buffer.  Eager, the MLPs are
        host-launch-bound (~10 small GEMMs per top-MLP pass at batch 2048): the GPU would idle
        between kernels and a "compute" phase would really be CPU time.  Replaying a graph makes
        the MLP phase GPU time, so the compute/communication ratio is the device's."""
        import torch
        self.repeat = repeat
        # sm_carveout: SMs cuBLAS leaves free (CUBLASLT_MATMUL_DESC_SM_COUNT_TARGET), for a graph
        # that runs beside a gather holding those SMs; persistent GEMMs sized to all 148 SMs
        # would otherwise need a second wave
        prev = torch._C._get_sm_carveout_experimental()
        torch._C._set_sm_carveout_experimental(sm_carveout if sm_carveout else None)
        try:
            return self._capture(dense, pooled)
        finally:
            torch._C._set_sm_carveout_experimental(prev)

    def _capture(self, dense, pooled):
        import torch
        side = torch.cuda.Stream(dense.device)
        side.wait_stream(torch.cuda.current_stream(dense.device))
        with torch.cuda.stream(side):
            for _ in range(2):
                self.forward(dense, pooled)
        torch.cuda.current_stream(dense.device).wait_stream(side)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            res = self.forward(dense, pooled)
        g.result = res
        return g


def mlp_graph_ms(graph, reps: int = 10) -> float:
    """Device time of one replay (CUDA events on the current stream, after a warm replay)."""
    import torch
    graph.replay()
    st = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(reps):
        graph.replay()
    b.record(st)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def run_pipeline(system, batches, key0, rows, mlps, outs, mode: str, side_ctas: int = 16,
                 prefetch_distance: int = 0, profile: bool = False):
    """Time len(batches) DLRM steps.  `mlps[k]` is a captured forward graph reading the pooled
    buffer `outs[k]` ([B, T, D], k = 0, 1: double buffering).
      sync:     gather(i) -> MLPs(i) on one stream (bench/ctc.py:27-44: compute starts once the
                epoch's data arrived), always buffer 0.
      async:    gather(i+1) runs on a high-priority side stream, bounded to `side_ctas` user CTAs,
                into the other buffer while MLPs(i) run on the main stream (bench/ctc.py:47-70: the
                next epoch's reads are issued before this epoch's compute); a step costs
                max(gather, MLPs) instead of their sum.
      prefetch: batch-level AGILE prefetch (gpu_api.py:139-162) of batch i+1 beside MLPs(i), then
                a full-grid gather(i+1) that finds its pages resident.
    Two AGILE launches never overlap (one context: same stream, or ordered by events)."""
    import torch
    dev = batches[0].device
    B, T, L = batches[0].shape
    D = outs[0].shape[-1]
    main = torch.cuda.current_stream(dev)
    # lower = higher: the side launch's CTAs dispatch ahead of the MLPs' (AGILE_SIDE_PRIORITY=0: equal)
    side = torch.cuda.Stream(dev, priority=int(os.environ.get("AGILE_SIDE_PRIORITY", "-1")))
    cnt = torch.zeros(2, dtype=torch.int64, device=dev)
    pcnt = torch.zeros(2, dtype=torch.int64, device=dev)
    n = len(batches)
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(main)
    if mode == "sync":
        for i in range(n):
            system.embbag(batches[i], key0, rows, outs[0], cnt, prefetch_distance=prefetch_distance,
                          stream=main.cuda_stream)
            mlps[0].replay()
    elif mode == "async":
        ev_g = [torch.cuda.Event() for _ in range(n)]
        ev_m = [torch.cuda.Event() for _ in range(n)]
        side.wait_event(t0)
        system.embbag(batches[0], key0, rows, outs[0], cnt, prefetch_distance=prefetch_distance,
                      stream=side.cuda_stream, user_ctas=side_ctas)
        ev_g[0].record(side)
        for i in range(n):
            if i + 1 < n:
                # buffer (i+1)%2 was last read by MLPs(i-1)
                if i >= 1:
                    side.wait_event(ev_m[i - 1])
                system.embbag(batches[i + 1], key0, rows, outs[(i + 1) % 2], cnt, prefetch_distance=prefetch_distance,
                              stream=side.cuda_stream, user_ctas=side_ctas)
                ev_g[i + 1].record(side)
            main.wait_event(ev_g[i])
            mlps[i % 2].replay()
            ev_m[i].record(main)
    elif mode == "prefetch":
        ev_p = [torch.cuda.Event(enable_timing=profile) for _ in range(n)]
        ev_e = [torch.cuda.Event(enable_timing=profile) for _ in range(n)]
        ev_m = [torch.cuda.Event(enable_timing=profile) for _ in range(n)]
        side.wait_event(t0)
        system.embbag_prefetch(batches[0], key0, rows, D, pcnt, side_ctas, stream=side.cuda_stream)
        ev_p[0].record(side)
        for i in range(n):
            main.wait_event(ev_p[i])
            system.embbag(batches[i], key0, rows, outs[0], cnt, prefetch_distance=0, stream=main.cuda_stream)
            ev_e[i].record(main)
            if i + 1 < n:
                side.wait_event(ev_e[i])
                system.embbag_prefetch(batches[i + 1], key0, rows, D, pcnt, side_ctas, stream=side.cuda_stream)
                ev_p[i + 1].record(side)
            mlps[0].replay()
            ev_m[i].record(main)
    else:
        raise ValueError(f"unknown pipeline mode {mode!r}")
    t1.record(main)
    torch.cuda.synchronize()
    system.sync(main.cuda_stream)
    c = cnt.cpu().numpy()
    res = {"ms": t0.elapsed_time(t1), "lookups": int(c[0]), "miss_lookups": int(c[1]),
           "lookups_per_s": n * B * T * L / (t0.elapsed_time(t1) / 1e3)}
    if profile and mode == "prefetch" and n > 2:
        # per step under overlap: prefetch(i+1) = ev_e[i] -> ev_p[i+1]; MLPs(i) = ev_e[i] -> ev_m[i];
        # gather(i+1) = max(ev_p[i+1], ev_m[i]) -> ev_e[i+1]
        pf = [ev_e[i].elapsed_time(ev_p[i + 1]) for i in range(1, n - 1)]
        ml = [ev_e[i].elapsed_time(ev_m[i]) for i in range(1, n - 1)]
        ga = [ev_m[i].elapsed_time(ev_e[i + 1]) for i in range(1, n - 1)]
        res.update({"prefetch_ms": sum(pf) / len(pf), "mlp_ms": sum(ml) / len(ml), "gather_ms": sum(ga) / len(ga)})
    return res


def run_dlrm(cfg, trace: bool = False):
    """CLI experiment `dlrm`: DLRM steps on one GPU, sync vs async (BenchResult rows)."""
    import torch
    from . import BenchResult
    from ..system import AgileSystem
    dev = torch.device("cuda", torch.cuda.current_device())
    sc = cfg.system
    cache_bytes = sc.cache.bytes or sc.cache.lines * 4096
    total = cfg.dlrm_table_bytes or 4 * cache_bytes
    rows = table_rows(total, cfg.dlrm_dim, cfg.dlrm_tables)
    key0, pages = layout(rows, cfg.dlrm_dim)
    import copy
    sc = copy.deepcopy(sc)
    sc.device.num_blocks = max(sc.device.num_blocks, pages)
    result = BenchResult(header=["mode", "batches", "t_ns", "lookups_per_s", "miss_lookups"], rows=[], info={})
    with AgileSystem(sc) as system:
        system.fill_store(0, sc.seed, kind="f32")
        model = DlrmModel(dev, cfg.dlrm_dim, cfg.dlrm_tables)
        dense = torch.randn(cfg.dlrm_batch, 13, device=dev, dtype=torch.bfloat16)
        outs = [torch.zeros((cfg.dlrm_batch, cfg.dlrm_tables, cfg.dlrm_dim), dtype=torch.float32, device=dev)
                for _ in range(2)]
        mlps = [model.capture(dense, o, 1) for o in outs]
        k0 = torch.from_numpy(key0.view(np.int64)).to(dev)
        r = torch.from_numpy(rows).to(dev)
        nb = cfg.dlrm_batches
        for mode, base in (("sync", 0), ("async", nb)):
            bat = [torch.from_numpy(make_batch(sc.seed, base + i, rows, cfg.dlrm_batch, cfg.dlrm_pooling,
                                               cfg.dlrm_zipf, cfg.dlrm_scatter)).to(dev) for i in range(nb)]
            res = run_pipeline(system, bat, k0, r, mlps, outs, mode)
            result.rows.append((mode, nb, int(res["ms"] * 1e6), round(res["lookups_per_s"], 3), res["miss_lookups"]))
    return result
