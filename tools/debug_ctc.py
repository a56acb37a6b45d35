import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, "tests")
import numpy as np
from conftest import small_config
from paper_2504_19365_b200 import AgileSystem
from paper_2504_19365_b200.system import make_key
T, R, E = [int(x) for x in sys.argv[1:4]]
s = AgileSystem(small_config(cache_lines=8192, ways=32, blocks=1 << 16, pairs=16, sq_depth=256, cq_depth=256,
                             emulation="model", engine_warps=8, warps=4), device=0)
keys = make_key(np.zeros(E * T * R), np.arange(E * T * R)).reshape(E, T, R)
r0 = s.run_reads(keys, T, R, E, False, 0); comm = r0["t_ns"] / E
print("calib", r0["t_ns"], np.diff(r0["epoch_t"]))
for mode in (False, True):
    s.reset()
    r = s.run_reads(keys, T, R, E, mode, int(comm))
    print("async" if mode else "sync ", r["t_ns"], np.diff(r["epoch_t"]), {k: v for k, v in s.stats().items() if k in ("sq_full", "cqe_stalls", "misses", "barrier_count")}, "mean barrier ns", s.stats()["barrier_latency_sum"] / max(1, s.stats()["barrier_count"]))
