"""DLRM async-pipeline probe on one GPU (GPU-box tool, not part of the product).

For each (engine warps, service warps) context and each side-stream user-CTA bound, time the
sync and async DLRM pipelines at a compute/communication ratio near 1, plus the MLP graph alone
while an idle bounded gather context holds its SMs.

  python tools/pipe_probe.py [cache_gib] [table_gib]
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
    cfg.debug_locks = False
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
    combos = [tuple(int(x) for x in c.split("/")) for c in os.environ.get("COMBOS", "128/48,64/16,32/8").split(",")]
    pds = [int(x) for x in os.environ.get("PDS", "0").split(",")]
    ucs = [int(x) for x in os.environ.get("UCS", "8,16,32,64,0").split(",")]
    for ew, sw in combos:
        s, rows_np, key0, rows = make(cache_gib, table_gib, ew, sw)
        full, infra = s.embbag_grid()
        for _ in range(int(1.3 * s.num_lines / 69000) + 4):
            s.embbag(gpu_zipf_batch(gen, rows_np, B, L, 1.05, True, dev), key0, rows, outs[0], cnt, prefetch_distance=0)
        s.sync(st.cuda_stream)
        # gather time on fresh batches (full grid)
        bat = [gpu_zipf_batch(gen, rows_np, B, L, 1.05, True, dev) for _ in range(8)]
        f1 = mlp_graph_ms(model.capture(dense, outs[0], 1))
        f9 = mlp_graph_ms(model.capture(dense, outs[0], 9))
        per = max((f9 - f1) / 8, 1e-3)
        r = run_pipeline(s, bat, key0, rows, [model.capture(dense, o, 1) for o in outs], outs, "sync")
        g_ms = r["ms"] / len(bat) - f1
        rep = max(1, int(round((g_ms - f1) / per)) + 1)
        mlps = [model.capture(dense, o, rep) for o in outs]
        mlp_ms = mlp_graph_ms(mlps[0], 3)
        for uc, pd in [(u if u else full, p) for u in ucs for p in pds]:
            res = {}
            for mode in ("sync", "async"):
                bat = [gpu_zipf_batch(gen, rows_np, B, L, 1.05, True, dev) for _ in range(10)]
                res[mode] = run_pipeline(s, bat, key0, rows, mlps, outs, mode, side_ctas=uc,
                                         prefetch_distance=pd)["ms"] / 10
            # gather alone with this bound (fresh batches)
            bat = [gpu_zipf_batch(gen, rows_np, B, L, 1.05, True, dev) for _ in range(6)]
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            for x in bat:
                s.embbag(x, key0, rows, outs[0], cnt, prefetch_distance=pd, user_ctas=uc, stream=st.cuda_stream)
            b.record(st)
            torch.cuda.synchronize()
            gb = a.elapsed_time(b) / len(bat)
            print(json.dumps({"engine_warps": ew, "service_warps": sw, "infra_ctas": infra, "user_ctas": uc, "pd": pd,
                              "gather_ms_full": g_ms, "gather_ms_bounded": gb, "mlp_ms": mlp_ms,
                              "sync_ms": res["sync"], "async_ms": res["async"],
                              "speedup": res["sync"] / res["async"],
                              "ideal": (g_ms + mlp_ms) / max(g_ms, mlp_ms)}), flush=True)
        s.close()
        del mlps


if __name__ == "__main__":
    main()
