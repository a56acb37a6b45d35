"""CTC default-config probe (GPU-box tool): per-epoch times and barrier latency, sync vs async."""
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np

from paper_2504_19365_b200 import AgileSystem
from paper_2504_19365_b200.bench.ctc import request_keys
from paper_2504_19365_b200.cli import build_config

cfg = build_config("ctc_sweep", sys.argv[1] if len(sys.argv) > 1 and sys.argv[1] != "-" else None)
for kv in sys.argv[2:]:
    k, v = kv.split("=")
    obj = cfg.system
    parts = k.split(".")
    for p in parts[:-1]:
        obj = getattr(obj, p)
    setattr(obj, parts[-1], type(getattr(obj, parts[-1]))(v))
s = AgileSystem(cfg.system, device=0)
keys = request_keys(cfg)
T, R, E = cfg.tasks, cfg.reads_per_task, cfg.epochs
s.reset()
r0 = s.run_reads(keys, T, R, E, False, 0)
comm = r0["t_ns"] / E
st = s.stats()
print("calib t_ns", r0["t_ns"], "per epoch", comm, "epochs", np.diff(r0["epoch_t"])[:6],
      "mean barrier ns", st["barrier_latency_sum"] / max(1, st["barrier_count"]))
for mode in (False, True):
    s.reset()
    r = s.run_reads(keys, T, R, E, mode, int(comm))
    st = s.stats()
    print("async" if mode else "sync ", r["t_ns"], np.diff(r["epoch_t"])[:6], "mean barrier ns",
          st["barrier_latency_sum"] / max(1, st["barrier_count"]))
s.close()
