"""DLRM embedding-bag driver (BASELINE configs[1] and [4]; new workload — the reference's
ancestor is the synthetic gather of bench/sweeps.py:1-9, which "stands in for embedding lookups").

* 26 Criteo-shaped tables (Kaggle cardinalities scaled to a byte budget), dim 128, fp32 rows,
  8 rows per 4 KiB page, laid out contiguously in the emulated device's page store.
* Indices: bounded Zipf(alpha) ranks per table, optionally scattered over rows by a bijective
  multiplicative hash (hashed categorical ids), deterministic per (seed, batch).
* Table-wise sharding over G ranks, balanced by bytes (largest first); pooled outputs of a
  rank's tables are [B, T_g, D], i.e. already in the peer-major layout all_to_all_single
  splits along B.
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


def shard_tables(rows: np.ndarray, G: int):
    """Table-wise assignment balanced by bytes (largest first onto the lightest rank)."""
    load = [0] * G
    owner = np.zeros(len(rows), dtype=np.int64)
    for t in np.argsort(-rows, kind="stable"):
        g = int(np.argmin(load))
        owner[t] = g
        load[g] += int(rows[t])
    return [np.nonzero(owner == g)[0] for g in range(G)], owner


@dataclass
class DlrmShard:
    """One rank's share: its tables, their rows and page keys in the rank's own store."""
    tables: np.ndarray
    rows: np.ndarray
    key0: np.ndarray
    pages: int


def build_shard(all_rows: np.ndarray, tables: np.ndarray, dim: int) -> DlrmShard:
    rows = all_rows[tables]
    key0, pages = layout(rows, dim)
    return DlrmShard(tables=tables, rows=rows, key0=key0, pages=pages)


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


def exchange_pooled(pooled_local, groups, rank: int, world: int):
    """Table-wise model parallel -> data parallel: rank r holds pooled[B, T_r, D] for its tables;
    after one all_to_all_single every rank holds pooled[B/world, T, D] for its sample slice, tables
    in global order.  pooled_local's B dimension is already peer-major (slice p goes to rank p)."""
    import torch
    import torch.distributed as dist
    B, Tr, D = pooled_local.shape
    tmax = max(len(g) for g in groups)
    send = torch.zeros((world, B // world, tmax, D), dtype=pooled_local.dtype, device=pooled_local.device)
    send[:, :, :Tr] = pooled_local.view(world, B // world, Tr, D)
    recv = torch.empty_like(send)
    dist.all_to_all_single(recv, send)
    T = sum(len(g) for g in groups)
    out = torch.empty((B // world, T, D), dtype=pooled_local.dtype, device=pooled_local.device)
    for q in range(world):
        out[:, torch.as_tensor(groups[q], dtype=torch.long, device=out.device)] = recv[q, :, :len(groups[q])]
    return out
