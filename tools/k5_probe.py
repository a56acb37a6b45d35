"""K5 (embedding-bag) hit-path probe on one GPU (GPU-box tool, not part of the product).

  python tools/k5_probe.py [uniform|zipf] [reps]
    uniform: 12 GiB of row-keyed tables resident in a 16 GiB cache, batch indices uniform over all
             rows (1.06 M distinct rows per batch, 545 MB of rows >> L2): the replayed batch is
             all hits and its rows stream from HBM — the no-reuse roofline case.
    zipf:    the bench's hashed Zipf 1.05 batch over the same tables (L2 reuse of hot rows).
Prints one JSON line: ms per launch, algorithmic GB/s and fraction of the measured HBM peak.
Profile: K5_SOLO=1 ncu -k regex:agile_user_kernel -c 1 python tools/k5_probe.py uniform 1: the
warm-up runs take the launch mode the co-residency probe picks (fused under ncu: they need the
engine for their misses), then the timed all-hit replays switch to split-solo (the infra grid
is not launched at all: launch mode "users"; all hits need no engine), so the capture is the
production user kernel with its own register budget and grid.
"""
import json
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np
import torch

from paper_2504_19365_b200 import AgileSystem, SystemConfig
from paper_2504_19365_b200.bench.dlrm import fill_rank_store, gpu_zipf_batch, plan_shards, table_rows

B, T, L, D = 2048, 26, 20, 128


def main():
    mode = sys.argv[1] if len(sys.argv) > 1 else "uniform"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    dev = torch.device("cuda", 0)
    rows = table_rows(12 << 30, D, T)
    plan = plan_shards(rows, 1, D)
    descs, _, pages = plan.rank_layout(0)
    cfg = SystemConfig()
    cfg.device.num_blocks = pages
    cfg.device.emulation = "link"
    cfg.cache.bytes = 16 << 30
    cfg.cache.ways = 32
    cfg.queues.pairs_per_device = 128
    cfg.queues.sq_depth = 256
    cfg.queues.cq_depth = 256
    cfg.engine.warps = int(os.environ.get("K5_ENGINE_WARPS", 128))
    cfg.service.warps = int(os.environ.get("K5_SERVICE_WARPS", 48))
    cfg.service.idle_max_ns = 1600
    cfg.engine.copy = os.environ.get("K5_ENGINE_COPY", "registers")
    cfg.debug_locks = False
    s = AgileSystem(cfg, device=0)
    if os.environ.get("K5_SOLO") == "1":
        # warm-up runs need the engine: one fused grid (ncu with a kernel filter lets the
        # co-residency probe's kernels overlap, yet serialises the user kernel it profiles)
        s.set_launch_mode("fused")
    fill_rank_store(s, plan, 0, 5)
    gen = torch.Generator(device=dev).manual_seed(3)
    if mode == "uniform":
        rt = torch.from_numpy(rows).to(dev)
        u = torch.rand((B, T, L), generator=gen, device=dev, dtype=torch.float64)
        idx = (u * rt.view(1, T, 1)).to(torch.int64).contiguous()
    else:
        idx = gpu_zipf_batch(gen, rows, B, L, 1.05, True, dev)
    tabs = torch.from_numpy(descs.view(np.uint8).copy()).to(dev)
    out = torch.empty((B, plan.row_bytes(0)), dtype=torch.uint8, device=dev)
    cnt = torch.zeros(2, dtype=torch.int64, device=dev)
    st = torch.cuda.current_stream(dev)
    for _ in range(2):   # fill, then make sure every page is resident
        s.embbag_sharded(idx, tabs, out, cnt, D, stream=st.cuda_stream)
    s.sync(st.cuda_stream)
    if os.environ.get("K5_SOLO") == "1":
        s.set_launch_mode("users")
    cnt.zero_()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(reps):
        s.embbag_sharded(idx, tabs, out, cnt, D, stream=st.cuda_stream)
    b.record(st)
    s.sync(st.cuda_stream)
    ms = a.elapsed_time(b) / reps
    alg = B * T * L * (D * 4 + 8) + B * T * D * 4
    try:
        peak = float(json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"])
    except Exception:
        peak = 6650.0
    c = cnt.cpu().numpy()
    print(json.dumps({"mode": mode, "ms": ms, "alg_gbs": alg / ms / 1e6, "frac": alg / ms / 1e6 / peak,
                      "lookups_per_s": B * T * L / ms * 1e3, "miss_lookups": int(c[1]),
                      "lib": os.environ.get("AGILE_LIB", "default"), "engine_copy": cfg.engine.copy, "launch": s.launch_mode,
                      "grid": s.embbag_grid()}), flush=True)
    s.close()


if __name__ == "__main__":
    main()
