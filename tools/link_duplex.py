"""Host-link sharing probe on one GPU (GPU-box tool): does a D2H (or H2D) DMA copy overlap the
link-bound device step (zero-copy page reads from host memory), or do they share one budget?
Bench config; prints one JSON line with the times of each alone and of both together.
  step   agile_embbag_sharded on device-resident indices (misses read host pages over the link)
  d2h    the pooled output (B*T*D fp32, 27.3 MB) copied device -> pinned host
  h2d    the indices (B*T*L int64, 8.5 MB) copied pinned host -> device
"""
import json
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np
import torch

import bench
from paper_2504_19365_b200 import AgileSystem, SystemConfig
from paper_2504_19365_b200.bench.dlrm import fill_rank_store, gpu_zipf_batch, plan_shards, table_rows

B, T, L, D = bench.B, bench.T, bench.L, bench.D


def main():
    steps = 10
    dev = torch.device("cuda", 0)
    rows_all = table_rows(64 << 30, D, T)
    plan = plan_shards(rows_all, 1, D)
    descs, _, pages = plan.rank_layout(0)
    cfg = SystemConfig()
    cfg.device.num_blocks = pages
    cfg.device.emulation = "link"
    cfg.cache.bytes = 16 << 30
    cfg.cache.ways = 32
    cfg.queues.pairs_per_device = 128
    cfg.engine.warps = 128
    cfg.service.warps = 48
    cfg.service.idle_max_ns = 1600
    cfg.debug_locks = False
    s = AgileSystem(cfg, device=0)
    fill_rank_store(s, plan, 0, bench.SEED)
    st = torch.cuda.current_stream(dev)
    cp = torch.cuda.Stream(dev)
    gen = torch.Generator(device=dev).manual_seed(1)
    tabs = torch.from_numpy(descs.view(np.uint8).copy()).to(dev)
    out = torch.empty((B, plan.row_bytes(0)), dtype=torch.uint8, device=dev)
    cnt = torch.zeros(2, dtype=torch.int64, device=dev)
    for _ in range(90):
        s.embbag_sharded(gpu_zipf_batch(gen, rows_all, B, L, bench.ALPHA, True, dev), tabs, out, cnt, D,
                         stream=st.cuda_stream)
    s.sync(st.cuda_stream)
    batches = [gpu_zipf_batch(gen, rows_all, B, L, bench.ALPHA, True, dev) for _ in range(3 * steps)]
    hout = torch.empty(out.numel(), dtype=torch.uint8).pin_memory()
    hidx = torch.empty(batches[0].shape, dtype=batches[0].dtype).pin_memory()
    didx = torch.empty_like(batches[0])
    res = {}

    def timed(fn):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        cp_done = torch.cuda.Event()
        cp_done.record(cp)
        st.wait_event(cp_done)
        b.record(st)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / steps

    def steps_on(k0):
        for k in range(steps):
            s.embbag_sharded(batches[k0 + k], tabs, out, cnt, D, stream=st.cuda_stream)

    def copies(kind):
        start = torch.cuda.Event()
        start.record(st)
        cp.wait_event(start)
        with torch.cuda.stream(cp):
            for _ in range(steps):
                if kind == "d2h":
                    hout.copy_(out.view(-1), non_blocking=True)
                else:
                    didx.copy_(hidx, non_blocking=True)

    res["step"] = timed(lambda: steps_on(0))
    res["d2h"] = timed(lambda: copies("d2h"))
    res["h2d"] = timed(lambda: copies("h2d"))
    res["step+d2h"] = timed(lambda: (copies("d2h"), steps_on(steps)))
    res["step+h2d"] = timed(lambda: (copies("h2d"), steps_on(2 * steps)))
    res["d2h_gbps"] = out.numel() / res["d2h"] / 1e6
    res["h2d_gbps"] = hidx.numel() * 8 / res["h2d"] / 1e6
    print(json.dumps(res), flush=True)
    s.close()


if __name__ == "__main__":
    main()
