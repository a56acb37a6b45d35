"""End-to-end (host buffers) DLRM step probe on one GPU (GPU-box tool): where does the e2e step
lose time against the device-timed step?  Bench config (16 GiB cache over 64 GiB of tables),
fresh Zipf batches; prints one JSON line per variant:
  device      agile_embbag_sharded on device-resident indices (the bench's `value` path)
  h2d_only    pinned H2D of the indices + the device run, output left on the device
  pipelined   agile_embbag_host_submit / _wait over two staging slots (the bench's `e2e`)
  serial      agile_embbag_host (copy in, run, copy out, synchronise) per step
"""
import json
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import numpy as np
import torch

import bench
from paper_2504_19365_b200 import AgileSystem, SystemConfig
from paper_2504_19365_b200.bench.dlrm import fill_rank_store, gpu_zipf_batch, make_batch, plan_shards, table_rows

B, T, L, D = bench.B, bench.T, bench.L, bench.D


def main():
    steps = 10
    print("numa:", bench.bind_local_numa(0), file=sys.stderr)
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
    out = torch.empty((B, plan.row_bytes(0)), dtype=torch.uint8, device=dev)
    cnt = torch.zeros(2, dtype=torch.int64, device=dev)
    for _ in range(90):
        s.embbag_sharded(gpu_zipf_batch(gen, rows_all, B, L, bench.ALPHA, True, dev), tabs, out, cnt, D,
                         stream=st.cuda_stream)
    s.sync(st.cuda_stream)
    hb = [make_batch(bench.SEED, 1000 + k, rows_all, B, L, bench.ALPHA, True) for k in range(4 * steps)]
    pinned = [torch.from_numpy(x).pin_memory() for x in hb]
    res = {}
    # device
    db = [p.to(dev) for p in pinned[:steps]]
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for k in range(steps):
        s.embbag_sharded(db[k], tabs, out, cnt, D, stream=st.cuda_stream)
    b.record(st)
    s.sync(st.cuda_stream)
    res["device"] = a.elapsed_time(b) / steps
    # h2d only
    dbuf = torch.empty_like(db[0])
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k in range(steps):
        dbuf.copy_(pinned[steps + k], non_blocking=True)
        s.embbag_sharded(dbuf, tabs, out, cnt, D, stream=st.cuda_stream)
    s.sync(st.cuda_stream)
    res["h2d_only"] = (time.perf_counter() - t0) * 1e3 / steps
    # pipelined host entry (the bench's e2e)
    keyh = torch.from_numpy(descs["key0"].view(np.int64).copy()).pin_memory().numpy().view(np.uint64)
    rowsh = torch.from_numpy(rows_all.copy()).pin_memory().numpy()
    outs = [torch.empty((B, T, D), dtype=torch.float32).pin_memory().numpy() for _ in range(2)]
    cnts = [np.zeros(2, dtype=np.uint64) for _ in range(2)]
    hnp = [p.numpy() for p in pinned]
    t0 = time.perf_counter()
    for k in range(steps):
        slot = k % 2
        if k >= 2:
            s.embbag_host_wait(slot)
        s.embbag_host_submit(hnp[2 * steps + k], keyh, rowsh, D, outs[slot], cnts[slot], slot, prefetch_distance=0)
    for slot in (0, 1):
        s.embbag_host_wait(slot)
    res["pipelined"] = (time.perf_counter() - t0) * 1e3 / steps
    # serial host entry
    t0 = time.perf_counter()
    for k in range(steps):
        s.embbag_host(hnp[3 * steps + k], keyh, rowsh, D, prefetch_distance=0, out=outs[0])
    res["serial"] = (time.perf_counter() - t0) * 1e3 / steps
    print(json.dumps({k: {"ms_per_step": v, "lookups_per_s": B * T * L / v * 1e3} for k, v in res.items()}), flush=True)
    s.close()


if __name__ == "__main__":
    main()
