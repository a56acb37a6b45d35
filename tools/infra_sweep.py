"""Engine / service size sweep at the bench config (GPU-box tool): ms per bench batch (one launch per
batch, fresh hashed-Zipf indices) and the per-batch CQE stalls / fills / completions, for each
(engine warps, service warps[, engine pages]) given as EW/SW pairs in $COMBOS."""
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
    gen = torch.Generator(device=dev).manual_seed(1)
    tabs = torch.from_numpy(descs.view(np.uint8).copy()).to(dev)
    cnt = torch.zeros(2, dtype=torch.int64, device=dev)
    st = torch.cuda.current_stream(dev)
    for combo in os.environ.get("COMBOS", "128/48,128/96,192/48,96/48").split(","):
        ew, sw = (int(x) for x in combo.split("/"))
        cfg = SystemConfig()
        cfg.device.num_blocks = pages
        cfg.device.emulation = "link"
        cfg.cache.bytes = 16 << 30
        cfg.cache.ways = 32
        cfg.queues.pairs_per_device = int(os.environ.get("QPS", 128))
        cfg.engine.warps = ew
        cfg.service.warps = sw
        cfg.service.idle_max_ns = 1600
        cfg.debug_locks = False
        s = AgileSystem(cfg, device=0)
        fill_rank_store(s, plan, 0, bench.SEED)
        out = torch.empty((B, plan.row_bytes(0)), dtype=torch.uint8, device=dev)
        for _ in range(90):
            s.embbag_sharded(gpu_zipf_batch(gen, rows_all, B, L, bench.ALPHA, True, dev), tabs, out, cnt, D,
                             stream=st.cuda_stream)
        s.sync(st.cuda_stream)
        bats = [gpu_zipf_batch(gen, rows_all, B, L, bench.ALPHA, True, dev) for _ in range(10)]
        s0 = s.stats()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        uc = int(os.environ.get("UCTAS", 0))
        for x in bats:
            s.embbag_sharded(x, tabs, out, cnt, D, user_ctas=uc, stream=st.cuda_stream)
        b.record(st)
        s.sync(st.cuda_stream)
        s1 = s.stats()
        d = {k: (s1[k] - s0[k]) / len(bats) for k in s1 if s1[k] != s0[k]}
        print(json.dumps({"ew": ew, "sw": sw, "qps": cfg.queues.pairs_per_device, "user_ctas": int(os.environ.get("UCTAS", 0)), "ms_per_batch": a.elapsed_time(b) / len(bats),
                          "per_batch": d}), flush=True)
        s.close()
        del out


if __name__ == "__main__":
    main()
