"""Trace the queue_sweep gather (8 QPs) sync vs async (GPU-box tool): per-epoch action counts/time."""
import copy
import os
import sys
from collections import Counter

sys.path.insert(0, os.getcwd())
import numpy as np

from paper_2504_19365_b200 import AgileSystem, TraceRecorder
from paper_2504_19365_b200.bench.sweeps import gather_sets
from paper_2504_19365_b200.cli import build_config
from paper_2504_19365_b200.system import make_key

cfg = build_config("queue_sweep")
blocks = gather_sets(cfg)
sc = copy.deepcopy(cfg.system)
sc.queues.pairs_per_device = 8
sc.queues.sq_depth = 64
sc.queues.cq_depth = 64
sc.cache.lines = max(sc.cache.lines, 4 * cfg.tasks * cfg.gathers_per_epoch)
sc.device.num_blocks = max(sc.device.num_blocks, cfg.block_pool)
print("tasks", cfg.tasks, "epochs", cfg.epochs, "gathers", cfg.gathers_per_epoch, "compute", cfg.compute_ns_per_gather,
      "lines", sc.cache.lines, "ways", sc.cache.ways, "emu", sc.device.emulation)
for mode in ("sync", "async"):
    s = AgileSystem(copy.deepcopy(sc), recorder=TraceRecorder())
    keys = make_key(np.zeros_like(blocks), blocks)
    r = s.run_gather(keys, cfg.tasks, cfg.epochs, cfg.gathers_per_epoch, mode == "async",
                     cfg.gathers_per_epoch * cfg.compute_ns_per_gather)
    ev = s.events().records
    st = s.stats()
    print(mode, "t_ns", r["t_ns"], {k: st[k] for k in ("hits", "misses", "fills", "resets", "sq_full", "retries", "attaches")})
    print("  ", Counter((e[2], e[3]) for e in ev).most_common(12))
    enq = sorted(e[0] for e in ev if e[3] == "enqueue")
    print("   enqueue deciles (us):", [round(enq[int(len(enq) * q / 10)] / 1e3) for q in range(10)] if enq else None)
    # pass boundaries: every 32 enqueues is one warp pass (32 tasks x one gather)
    print("   pass starts (us):", [round(enq[i] / 1e3, 1) for i in range(0, min(len(enq), 32 * 40), 32)])
    hits = sorted(e[0] for e in ev if e[3] == "hit")
    print("   hit starts (us):", [round(hits[i] / 1e3, 1) for i in range(0, min(len(hits), 32 * 40), 32)])
    s.close()
