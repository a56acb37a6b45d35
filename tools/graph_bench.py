"""Graph workloads at the BASELINE scales on one GPU (GPU-box tool; prints one JSON line per run).

  python tools/graph_bench.py bfs  [scale=26] [cache_frac=0.25]
  python tools/graph_bench.py spmv [scale=27] [cache_frac=0.25] [iters=10]

configs[2]: BFS on RMAT scale 26, cache = 25% of the col_idx bytes.
configs[3]: SpMV + PageRank (10 iterations) on RMAT scale 27 with next-chunk prefetch.
Both run in sync (prefetch distance 0) and async (distance 2) mode on a cold cache; levels /
results of the two modes are compared (bit-exact BFS levels; identical SpMV sums).
"""
import faulthandler
import json
import os
import sys
import time

faulthandler.enable()


def note(msg):
    print(f"[graph_bench {time.strftime('%H:%M:%S')}] {msg}", file=sys.stderr, flush=True)

sys.path.insert(0, os.getcwd())
import torch

from paper_2504_19365_b200 import AgileSystem, SystemConfig
from paper_2504_19365_b200.bench.graph import (edge_values, pages_for, pick_source, rmat_csr, run_bfs,
                                               run_pagerank, run_spmv, write_paged)

LINK_PEAK = 51.4   # GB/s, profiles/link_probe_r01.json (zero-copy 4 KiB gather)


def make_system(npages, frac, ew=128, sw=48):
    cfg = SystemConfig()
    cfg.device.num_blocks = npages
    cfg.device.emulation = "link"
    lines = max(64, int(frac * npages))
    cfg.cache.lines = -(-lines // 32) * 32
    cfg.cache.ways = 32
    cfg.queues.pairs_per_device = 128
    cfg.engine.warps = ew
    cfg.service.warps = sw
    cfg.service.idle_max_ns = 1600
    cfg.debug_locks = False
    return AgileSystem(cfg, device=0)


def bfs(scale, frac):
    dev = torch.device("cuda", 0)
    t0 = time.time()
    row_ptr, col, _ = rmat_csr(scale, 16, 1, dev)
    V, E = row_ptr.numel() - 1, col.numel()
    gen_s = time.time() - t0
    s = make_system(pages_for(E), frac)
    write_paged(s, 0, 0, col)
    del col
    torch.cuda.empty_cache()
    out = {}
    ref = None
    for pd in (0, 2):
        runs = []
        for seed in range(3):
            s.reset()
            src = pick_source(row_ptr, seed)
            f0 = s.stats()["fills"]
            level, st = run_bfs(s, row_ptr, V, src, 0, pd)
            st["fills"] = s.stats()["fills"] - f0   # every page the engine moved (prefetches too)
            if pd == 0 and seed == 0:
                ref = level.clone()
            if pd == 2 and seed == 0:
                st["levels_equal_sync"] = bool(torch.equal(level, ref))
            runs.append(st)
        ms = sum(r["ms"] for r in runs) / len(runs)
        edges = sum(r["edges"] for r in runs) / len(runs)
        misses = sum(r["fills"] for r in runs) / len(runs)
        out[pd] = {"ms": ms, "gteps": edges / ms / 1e6, "edges": edges, "levels": runs[0]["levels"],
                   "page_fills": misses, "link_gbs": misses * 4096 / ms / 1e6,
                   "link_frac": misses * 4096 / ms / 1e6 / LINK_PEAK,
                   "levels_equal_sync": runs[0].get("levels_equal_sync")}
    line = {"workload": "bfs", "scale": scale, "vertices": V, "edges": E, "cache_frac": frac,
            "cache_lines": s.num_lines, "gen_s": gen_s, "sync": out[0], "async": out[2],
            "async_vs_sync": out[0]["ms"] / out[2]["ms"]}
    if os.environ.get("GRAPH_CHECK", "1") == "1":
        # the C oracle (oracle/graph_oracle.c) over the same CSR: col_idx straight from the pinned
        # page store the GPU read it from, row_ptr copied back
        from oracle import cgraph
        t1 = time.time()
        col_h = s.store_view(0).reshape(-1)[:E * 4].view("<i4")
        exp = cgraph.bfs_levels(row_ptr.cpu().numpy(), col_h, pick_source(row_ptr, 0))
        line["oracle"] = {"levels_equal_oracle": bool((ref.cpu().numpy() == exp).all()), "kind": "oracle/graph_oracle.c",
                          "seconds": time.time() - t1}
    print(json.dumps(line), flush=True)
    s.close()


def spmv(scale, frac, iters):
    dev = torch.device("cuda", 0)
    t0 = time.time()
    note(f"spmv scale {scale}: generating")
    rowT, colT, outdeg = rmat_csr(scale, 16, 2, dev, transpose=True)
    V, E = rowT.numel() - 1, colT.numel()
    vals = edge_values(E, 2, dev)
    gen_s = time.time() - t0
    npg = pages_for(E)
    s = make_system(2 * npg, frac)
    nxt = write_paged(s, 0, 0, colT)
    write_paged(s, 0, nxt, vals)
    del colT, vals
    torch.cuda.empty_cache()
    x = torch.rand(V, device=dev)
    res = {}
    ys = {}
    rs = {}
    for pd in (0, 2):
        note(f"spmv pd={pd}")
        s.reset()
        f0 = s.stats()["fills"]
        y, st = run_spmv(s, rowT, V, E, 0, nxt, x, 1, pd)
        st["page_misses"] = s.stats()["fills"] - f0   # engine fills, prefetches included
        ys[pd] = y
        s.reset()
        f0 = s.stats()["fills"]
        note(f"pagerank pd={pd}")
        rs[pd], pr = run_pagerank(s, rowT, V, E, 0, outdeg, iters, prefetch_distance=pd)
        pr["page_misses"] = s.stats()["fills"] - f0
        res[pd] = {"spmv_ms": st["ms"], "spmv_gflops": st["gflops"], "spmv_page_fills": st["page_misses"],
                   "spmv_link_gbs": st["page_misses"] * 4096 / st["ms"] / 1e6,
                   "spmv_link_frac": st["page_misses"] * 4096 / st["ms"] / 1e6 / LINK_PEAK,
                   "pagerank_ms": pr["ms"], "pagerank_gteps": pr["edges"] / pr["ms"] / 1e6,
                   "pagerank_page_fills": pr["page_misses"],
                   "pagerank_link_frac": pr["page_misses"] * 4096 / pr["ms"] / 1e6 / LINK_PEAK}
    line = {"workload": "spmv_pagerank", "scale": scale, "vertices": V, "edges": E, "cache_frac": frac,
            "cache_lines": s.num_lines, "gen_s": gen_s, "iters": iters, "sync": res[0], "async": res[2],
            "spmv_equal_sync": bool(torch.equal(ys[0], ys[2])),
            "spmv_async_vs_sync": res[0]["spmv_ms"] / res[2]["spmv_ms"],
            "pagerank_async_vs_sync": res[0]["pagerank_ms"] / res[2]["pagerank_ms"]}
    if os.environ.get("GRAPH_CHECK", "1") == "1":
        # the C oracle over the same CSR (col / val straight from the pinned page store): y within
        # 1e-5 relative (north_star; guarded by sum |a x| for cancelling rows), PageRank within 1e-5
        import numpy as np
        from oracle import cgraph
        t1 = time.time()
        note("oracle: spmv")
        view = s.store_view(0).reshape(-1)    # bytes of the pinned store
        colT_h = view[:E * 4].view("<i4")
        vals_h = view[nxt * 4096:nxt * 4096 + E * 4].view("<f4")
        rp = rowT.cpu().numpy()
        xh = x.cpu().numpy()
        exp = cgraph.spmv_f32(rp, colT_h, vals_h, xh).astype(np.float64)
        mag = cgraph.spmv_f32(rp, colT_h, np.abs(vals_h), np.abs(xh)).astype(np.float64)
        got = ys[0].cpu().numpy().astype(np.float64)
        err = np.abs(got - exp) / np.maximum(np.abs(exp), 1e-30)
        ok = np.abs(got - exp) <= 1e-5 * np.abs(exp) + 1e-12 * mag
        note("oracle: pagerank")
        pr_exp = cgraph.pagerank_f32(rp, colT_h, outdeg.cpu().numpy(), iters).astype(np.float64)
        pr_err = np.abs(rs[0].cpu().numpy().astype(np.float64) - pr_exp) / pr_exp
        line["oracle"] = {"kind": "oracle/graph_oracle.c", "spmv_within_1e-5": bool(ok.all()),
                          "spmv_median_rel_err": float(np.median(err)),
                          "pagerank_max_rel_err": float(pr_err.max()), "pagerank_within_1e-5": bool(pr_err.max() < 1e-5),
                          "seconds": time.time() - t1}
    print(json.dumps(line), flush=True)
    s.close()


if __name__ == "__main__":
    kind = sys.argv[1]
    if kind == "bfs":
        bfs(int(sys.argv[2]) if len(sys.argv) > 2 else 26, float(sys.argv[3]) if len(sys.argv) > 3 else 0.25)
    else:
        spmv(int(sys.argv[2]) if len(sys.argv) > 2 else 27, float(sys.argv[3]) if len(sys.argv) > 3 else 0.25,
             int(sys.argv[4]) if len(sys.argv) > 4 else 10)
