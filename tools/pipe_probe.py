"""DLRM async-pipeline probe on one GPU (GPU-box tool, not part of the product).

For each (engine warps, service warps) context: calibrate the MLP graph to a compute/communication
ratio near 1, pick the fastest MLP graph over cuBLAS SM carve-outs for the sync baseline, then time
the async (bounded side-stream gather) and prefetch (bounded AGILE prefetch + full gather)
pipelines for each side-CTA bound and carve-out.

  COMBOS=128/48,64/16 UCS=16,32,64 CARVE=0,16,32 python tools/pipe_probe.py [cache_gib] [table_gib]
"""
import json
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np
import torch

from paper_2504_19365_b200 import AgileSystem, SystemConfig
from paper_2504_19365_b200.bench.dlrm import (table_rows, layout, gpu_zipf_batch, DlrmModel, run_pipeline,
                                              mlp_graph_ms)

B, T, L, D = 2048, 26, 20, 128


def make(cache_gib, table_gib, ew, sw):
    rows = table_rows(int(table_gib * (1 << 30)), D, T)
    key0, pages = layout(rows, D)
    cfg = SystemConfig()
    cfg.device.num_blocks = pages
    cfg.device.emulation = "link"
    cfg.cache.bytes = int(cache_gib * (1 << 30))
    cfg.cache.ways = 32
    cfg.queues.pairs_per_device = 128
    cfg.engine.warps = ew
    cfg.service.warps = sw
    cfg.service.idle_max_ns = 1600
    side = os.environ.get("SIDE")
    if side:
        cfg.engine.side_warps, cfg.service.side_warps = (int(x) for x in side.split("/"))
    cfg.debug_locks = False
    cfg.engine.copy = os.environ.get("ENGINE_COPY", "registers")
    s = AgileSystem(cfg, device=0)
    s.fill_store(0, 5, kind="f32")
    dev = torch.device("cuda", 0)
    return s, rows, torch.from_numpy(key0.view(np.int64)).to(dev), torch.from_numpy(rows).to(dev)


def main():
    cache_gib = float(sys.argv[1]) if len(sys.argv) > 1 else 4
    table_gib = float(sys.argv[2]) if len(sys.argv) > 2 else 16
    dev = torch.device("cuda", 0)
    st = torch.cuda.current_stream(dev)
    gen = torch.Generator(device=dev).manual_seed(1)
    outs = [torch.zeros((B, T, D), dtype=torch.float32, device=dev) for _ in range(2)]
    cnt = torch.zeros(2, dtype=torch.int64, device=dev)
    model = DlrmModel(dev, D, T)
    dense = torch.randn(B, 13, device=dev, dtype=torch.bfloat16)
    combos = [tuple(int(x) for x in c.split("/")) for c in os.environ.get("COMBOS", "128/48,64/16").split(",")]
    ucs = [int(x) for x in os.environ.get("UCS", "16,32,64").split(",")]
    cos = [int(x) for x in os.environ.get("CARVE", "0,16,32").split(",")]
    modes = os.environ.get("MODES", "async,prefetch").split(",")
    n = 10
    for ew, sw in combos:
        s, rows_np, key0, rows = make(cache_gib, table_gib, ew, sw)
        full, infra = s.embbag_grid()
        for _ in range(int(1.3 * s.num_lines / 69000) + 4):
            s.embbag(gpu_zipf_batch(gen, rows_np, B, L, 1.05, True, dev), key0, rows, outs[0], cnt, prefetch_distance=0)
        s.sync(st.cuda_stream)
        f1 = mlp_graph_ms(model.capture(dense, outs[0], 1))
        f9 = mlp_graph_ms(model.capture(dense, outs[0], 9))
        per = max((f9 - f1) / 8, 1e-3)
        bat = [gpu_zipf_batch(gen, rows_np, B, L, 1.05, True, dev) for _ in range(n)]
        r = run_pipeline(s, bat, key0, rows, [model.capture(dense, o, 1) for o in outs], outs, "sync")
        g_ms = r["ms"] / n - f1
        rep = max(1, int(round((g_ms - f1) / per)) + 1)
        graphs, mlp_ms = {}, {}
        for co in cos:
            graphs[co] = [model.capture(dense, o, rep, sm_carveout=co) for o in outs]
            mlp_ms[co] = mlp_graph_ms(graphs[co][0], 3)
        best = min(cos, key=lambda k: mlp_ms[k])
        bat = [gpu_zipf_batch(gen, rows_np, B, L, 1.05, True, dev) for _ in range(n)]
        sync_ms = run_pipeline(s, bat, key0, rows, graphs[best], outs, "sync")["ms"] / n
        print(json.dumps({"engine_copy": s.engine_copy, "side": os.environ.get("SIDE"), "engine_warps": ew, "service_warps": sw, "infra_ctas": infra, "gather_ms": g_ms,
                          "mlp_ms_by_carveout": mlp_ms, "sync_carveout": best, "sync_ms": sync_ms}), flush=True)
        for mode in modes:
            for uc in ucs:
                for co in cos:
                    bat = [gpu_zipf_batch(gen, rows_np, B, L, 1.05, True, dev) for _ in range(n)]
                    rr = run_pipeline(s, bat, key0, rows, graphs[co], outs, mode, side_ctas=uc, profile=True)
                    ms = rr["ms"] / n
                    print(json.dumps({"ew": ew, "sw": sw, "mode": mode, "user_ctas": uc, "carveout": co,
                                      "ms": ms, "speedup": sync_ms / ms, "parts": {k: rr[k] for k in
                                      ("prefetch_ms", "mlp_ms", "gather_ms") if k in rr},
                                      "ideal": (g_ms + mlp_ms[best]) / max(g_ms, mlp_ms[best])}), flush=True)
        s.close()
        del graphs


if __name__ == "__main__":
    main()
