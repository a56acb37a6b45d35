"""Timeline of one bench step (GPU-box tool): trace one DLRM embedding-bag launch at the bench config
(after the cache is warm) and histogram the engine's page-copy starts (`fetch`) and completions
(`complete`) in 50 us bins from the first event: shows how fast the link fills at the start of the
launch and how it drains at the end."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np
import torch

import bench
from paper_2504_19365_b200 import AgileSystem, SystemConfig, TraceRecorder
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
    s = AgileSystem(cfg, device=0, recorder=TraceRecorder(), trace_capacity=0)
    fill_rank_store(s, plan, 0, bench.SEED)
    st = torch.cuda.current_stream(dev)
    gen = torch.Generator(device=dev).manual_seed(1)
    tabs = torch.from_numpy(descs.view(np.uint8).copy()).to(dev)
    cnt = torch.zeros(2, dtype=torch.int64, device=dev)
    out = torch.empty((B, plan.row_bytes(0)), dtype=torch.uint8, device=dev)
    for _ in range(90):
        s.embbag_sharded(gpu_zipf_batch(gen, rows_all, B, L, bench.ALPHA, True, dev), tabs, out, cnt, D,
                         stream=st.cuda_stream)
    s.sync(st.cuda_stream)
    bat = gpu_zipf_batch(gen, rows_all, B, L, bench.ALPHA, True, dev)
    s._lib.agile_trace_enable(s._ctx, C.c_uint64(1 << 22))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    s.embbag_sharded(bat, tabs, out, cnt, D, stream=st.cuda_stream)
    b.record(st)
    s.sync(st.cuda_stream)
    ev = s.events().records
    t = {k: np.array([r[0] for r in ev if r[3] == k], dtype=np.int64) for k in ("fetch", "complete", "enqueue", "cqe_process")}
    t0 = min(int(x.min()) for x in t.values() if len(x))
    res = {"launch_ms_traced": a.elapsed_time(b), "n": {k: len(v) for k, v in t.items()}}
    for k, v in t.items():
        if len(v):
            res[k + "_first_us"] = (int(v.min()) - t0) / 1e3
            res[k + "_last_us"] = (int(v.max()) - t0) / 1e3
    comp = np.sort(t["complete"] - t0)
    edges = np.arange(0, comp.max() + 50_000, 50_000)
    res["complete_per_50us"] = np.histogram(comp, edges)[0].tolist()
    enq = np.sort(t["enqueue"] - t0)
    res["enqueue_per_50us"] = np.histogram(enq, edges)[0].tolist()
    fet = np.sort(t["fetch"] - t0)
    res["fetch_per_50us"] = np.histogram(fet, edges)[0].tolist()
    # per command: enqueue -> fetch -> complete latencies, by the enqueue's 50 us bin
    stages = {}
    seen = {}
    for tt, who, mod, act, det in ev:
        if act == "enqueue":
            q, slot = det[0], det[2]
            seen[(q, slot)] = seen.get((q, slot), 0) + 1
            stages[(q, slot, seen[(q, slot)])] = {"enqueue": tt}
        elif act in ("fetch", "complete", "doorbell"):
            if act == "doorbell":
                continue
            q, slot = (det[1], det[2])
            k = (q, slot, seen.get((q, slot), 0))
            if k in stages:
                stages[k][act] = tt
    lat_f, lat_c = {}, {}
    for v in stages.values():
        if "fetch" in v and "complete" in v:
            bi = int((v["enqueue"] - t0) // 50_000)
            lat_f.setdefault(bi, []).append(v["fetch"] - v["enqueue"])
            lat_c.setdefault(bi, []).append(v["complete"] - v["fetch"])
    res["enq_to_fetch_us_by_enqueue_bin"] = [round(float(np.mean(lat_f[i])) / 1e3, 1) if i in lat_f else None
                                             for i in range(len(edges) - 1)]
    res["fetch_to_complete_us_by_enqueue_bin"] = [round(float(np.mean(lat_c[i])) / 1e3, 1) if i in lat_c else None
                                                  for i in range(len(edges) - 1)]
    print(json.dumps(res), flush=True)
    s.close()


if __name__ == "__main__":
    main()
