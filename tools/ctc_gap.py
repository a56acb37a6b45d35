"""CTC default config, sync mode, 2 epochs, traced (GPU-box tool): every device event between the
last device completion of epoch 0 and the first doorbell of epoch 1 — where the epoch gap goes."""
import os
import sys

sys.path.insert(0, os.getcwd())
from paper_2504_19365_b200 import AgileSystem, TraceRecorder
from paper_2504_19365_b200.bench.ctc import request_keys
from paper_2504_19365_b200.cli import build_config

cfg = build_config("ctc_sweep")
for kv in sys.argv[1:]:
    k, v = kv.split("=")
    obj = cfg.system
    parts = k.split(".")
    for p in parts[:-1]:
        obj = getattr(obj, p)
    setattr(obj, parts[-1], type(getattr(obj, parts[-1]))(v))
for rep in range(2):
    s = AgileSystem(cfg.system, recorder=TraceRecorder(), device=0)
    r = s.run_reads(request_keys(cfg), cfg.tasks, cfg.reads_per_task, 3, False, 0)
    ev = s.events().records
    print("rep", rep, "t_ns", r["t_ns"], "epoch_t", list(r["epoch_t"]))
    comp = sorted(t for t, who, mod, act, det in ev if act == "complete")
    t_last = comp[127]
    t_next = comp[255]
    for t, who, mod, act, det in ev:
        if t_last - 3000 <= t <= t_last + 70000 and act not in ("fetch",):
            print(t - t_last, who, mod, act, det)
    s.close()
