"""DLRM path probes on one GPU (not part of the product; GPU-box tool).

  python tools/dlrm_probe.py prefetch   # prefetch-only launch time vs user CTAs on fresh batches
  python tools/dlrm_probe.py hit        # all-hit embedding-bag replay (HBM roofline of hits)
  python tools/dlrm_probe.py hitprof    # hit replays for an ncu capture (-k regex:agile_kernel -s 4 -c 1)
"""
import json
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import numpy as np
import torch

from paper_2504_19365_b200 import AgileSystem, SystemConfig
from paper_2504_19365_b200.bench.dlrm import table_rows, layout, gpu_zipf_batch

B, T, L, D = 2048, 26, 20, 128


def system(cache_gib, table_gib, ways=32, ew=128, sw=48):
    rows = table_rows(int(table_gib * (1 << 30)), D, T)
    key0, pages = layout(rows, D)
    cfg = SystemConfig()
    cfg.device.num_blocks = pages
    cfg.device.emulation = "link"
    cfg.cache.bytes = int(cache_gib * (1 << 30))
    cfg.cache.ways = ways
    cfg.queues.pairs_per_device = 128
    cfg.engine.warps = ew
    cfg.service.warps = sw
    cfg.service.idle_max_ns = 1600
    cfg.debug_locks = False
    s = AgileSystem(cfg, device=0)
    s.fill_store(0, 5, kind="f32")
    dev = torch.device("cuda", 0)
    return s, rows, torch.from_numpy(key0.view(np.int64)).to(dev), torch.from_numpy(rows).to(dev)


def timed(fn, st):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    fn()
    b.record(st)
    torch.cuda.synchronize()
    return a.elapsed_time(b)


def main():
    mode = sys.argv[1] if len(sys.argv) > 1 else "hit"
    dev = torch.device("cuda", 0)
    st = torch.cuda.current_stream(dev)
    gen = torch.Generator(device=dev).manual_seed(1)
    out = torch.empty((B, T, D), dtype=torch.float32, device=dev)
    cnt = torch.zeros(2, dtype=torch.int64, device=dev)
    if mode == "prefetch":
        s, rows_np, key0, rows = system(16, 64)
        full, infra = s.embbag_grid()
        for _ in range(60):   # warm the cache to steady state
            s.embbag(gpu_zipf_batch(gen, rows_np, B, L, 1.05, True, dev), key0, rows, out, cnt, prefetch_distance=0)
        s.sync(st.cuda_stream)
        for uc in (8, 16, 32, 64, full):
            ms_p, ms_g, fills = [], [], []
            for _ in range(4):
                bat = gpu_zipf_batch(gen, rows_np, B, L, 1.05, True, dev)
                f0 = s.stats()["fills"]
                ms_p.append(timed(lambda: s.embbag_prefetch(bat, key0, rows, D, cnt, uc, stream=st.cuda_stream), st))
                f1 = s.stats()["fills"]
                fills.append(f1 - f0)
                ms_g.append(timed(lambda: s.embbag(bat, key0, rows, out, cnt, prefetch_distance=0, stream=st.cuda_stream), st))
            fl = float(np.mean(fills))
            print(json.dumps({"user_ctas": uc, "infra_ctas": infra, "prefetch_ms": float(np.median(ms_p)),
                              "fills": fl, "link_gbs": fl * 4096 / (np.median(ms_p) / 1e3) / 1e9,
                              "gather_after_ms": float(np.median(ms_g))}), flush=True)
        # full gather of fresh batches for reference
        ms = [timed(lambda: s.embbag(gpu_zipf_batch(gen, rows_np, B, L, 1.05, True, dev), key0, rows, out, cnt,
                                     prefetch_distance=0, stream=st.cuda_stream), st) for _ in range(4)]
        print(json.dumps({"full_gather_fresh_ms": float(np.median(ms))}))
    else:
        # every page resident: tables 1 GiB in a 4 GiB cache (hit/hitprof: L2-friendly), or 10 GiB
        # of tables in the bench's 16 GiB cache (hitbig: the rows stream from HBM)
        s, rows_np, key0, rows = system(16, 10) if mode == "hitbig" else system(4, 1)
        bat = gpu_zipf_batch(gen, rows_np, B, L, 1.05, True, dev)
        for _ in range(3):
            s.embbag(bat, key0, rows, out, cnt, prefetch_distance=0, stream=st.cuda_stream)
        s.sync(st.cuda_stream)
        reps = 2 if mode == "hitprof" else 20
        cnt.zero_()
        ms = timed(lambda: [s.embbag(bat, key0, rows, out, cnt, prefetch_distance=0, stream=st.cuda_stream)
                            for _ in range(reps)], st) / reps
        alg = B * T * L * (D * 4 + 8) + B * T * D * 4
        c = cnt.cpu().numpy()
        print(json.dumps({"mode": mode, "hit_ms": ms, "lookups_per_s": B * T * L / ms * 1e3, "alg_gbs": alg / ms / 1e6,
                          "miss_lookups": int(c[1]), "grid": s.embbag_grid()}))
    s.close()


if __name__ == "__main__":
    main()
