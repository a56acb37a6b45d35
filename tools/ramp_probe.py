"""Per-launch fixed cost of the bench step (GPU-box tool): one launch over k bench batches
(batch 2048*k x 26 x 20, fresh hashed-Zipf indices) for k = 1, 2, 4 at the bench config (16 GiB cache
over 64 GiB of tables, link mode); ms per batch-equivalent and page fills per batch.  A per-launch
ramp (first misses submitted, last fills drained, infra start/stop) shows as ms(k=1) > ms(k=4)."""
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
    gen = torch.Generator(device=dev).manual_seed(1)
    tabs = torch.from_numpy(descs.view(np.uint8).copy()).to(dev)
    cnt = torch.zeros(2, dtype=torch.int64, device=dev)
    out4 = torch.empty((4 * B, plan.row_bytes(0)), dtype=torch.uint8, device=dev)
    for _ in range(90):
        s.embbag_sharded(gpu_zipf_batch(gen, rows_all, B, L, bench.ALPHA, True, dev), tabs, out4[:B], cnt, D,
                         stream=st.cuda_stream)
    s.sync(st.cuda_stream)
    res = {}
    for rep in range(2):
        for k in (1, 2, 4):
            n = 8 // k
            bats = [torch.cat([gpu_zipf_batch(gen, rows_all, B, L, bench.ALPHA, True, dev) for _ in range(k)])
                    for _ in range(n)]
            cnt.zero_()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            for x in bats:
                s.embbag_sharded(x, tabs, out4[:k * B], cnt, D, stream=st.cuda_stream)
            b.record(st)
            s.sync(st.cuda_stream)
            c = cnt.cpu().numpy()
            res[f"k{k}_r{rep}"] = {"ms_per_batch": a.elapsed_time(b) / 8, "miss_lookups_per_batch": int(c[1]) / 8}
    print(json.dumps(res), flush=True)
    s.close()


if __name__ == "__main__":
    main()
