"""Trace the default CTC config (GPU-box tool): per-command stage latencies, sync and async."""
import os
import sys
from collections import defaultdict

sys.path.insert(0, os.getcwd())
import numpy as np

from paper_2504_19365_b200 import AgileSystem, TraceRecorder
from paper_2504_19365_b200.bench.ctc import request_keys
from paper_2504_19365_b200.cli import build_config

cfg = build_config("ctc_sweep")
cfg.epochs = 4
for mode in (False, True):
    s = AgileSystem(cfg.system, recorder=TraceRecorder(), device=0)
    keys = request_keys(cfg)
    r = s.run_reads(keys, cfg.tasks, cfg.reads_per_task, cfg.epochs, mode, int(os.environ.get("COMPUTE_NS", "0")))
    ev = s.events().records
    stages = defaultdict(dict)
    seen = defaultdict(int)
    order = {"enqueue": 0, "fetch": 1, "complete": 2, "cqe_post": 3, "cqe_process": 4}
    for t, who, mod, act, det in ev:
        if act == "enqueue":
            q, slot = det[0], det[2]
            seen[(q, slot)] += 1
            stages[(q, slot, seen[(q, slot)])]["enqueue"] = t
        elif act in ("fetch", "complete", "cqe_post", "cqe_process"):
            q, slot = {"fetch": (det[1], det[2]), "complete": (det[1], det[2]),
                       "cqe_post": (det[0], det[2]), "cqe_process": (det[3], det[2])}[act]
            stages[(q, slot, seen[(q, slot)])][act] = t
    names = ["enqueue", "fetch", "complete", "cqe_post", "cqe_process"]
    print("mode", "async" if mode else "sync", "t_ns", r["t_ns"], "epochs", np.diff(r["epoch_t"]))
    for a, b in zip(names, names[1:]):
        d = [v[b] - v[a] for v in stages.values() if a in v and b in v]
        if d:
            print(f"  {a}->{b}: mean {np.mean(d):.0f} p50 {np.median(d):.0f} max {np.max(d):.0f} n {len(d)}")
    # per-epoch timeline (commands grouped by enqueue order, 128 per epoch)
    cmds = sorted((v for v in stages.values() if "enqueue" in v), key=lambda v: v["enqueue"])
    per = cfg.tasks * cfg.reads_per_task
    prev_end = None
    for e in range(len(cmds) // per):
        g = cmds[e * per:(e + 1) * per]
        col = lambda k: sorted(v[k] for v in g if k in v)
        enq, fet, com, post, proc = (col(k) for k in names)
        row = {"first_enq": enq[0], "last_enq": enq[-1] - enq[0], "first_fetch": fet[0] - enq[0],
               "16th_fetch": fet[min(15, len(fet) - 1)] - enq[0], "last_complete": com[-1] - enq[0],
               "last_post": post[-1] - enq[0], "last_process": proc[-1] - enq[0]}
        if prev_end is not None:
            row["gap_from_prev_last_process"] = enq[0] - prev_end
        prev_end = proc[-1]
        print("  epoch", e, row)
    enq = sorted(v["enqueue"] for v in stages.values() if "enqueue" in v)
    print("  enqueue times (first 5 / per-epoch spans):", enq[:3], [enq[i * 128 + 127] - enq[i * 128] for i in range(len(enq) // 128)])
    s.close()

# fine timeline of the first two issue rounds of lane u0 / u1 (sync mode, 1 epoch)
cfg.epochs = 1
s = AgileSystem(cfg.system, recorder=TraceRecorder(), device=0)
r = s.run_reads(request_keys(cfg), cfg.tasks, cfg.reads_per_task, 1, False, 0)
ev = s.events().records
for t, who, mod, act, det in ev:
    if who in ("u0", "u1", "u15") and t < 80000:
        print(t, who, mod, act, det)
s.close()
