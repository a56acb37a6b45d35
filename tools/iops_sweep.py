"""Closed-loop 4 KiB IOPS sweep in link mode (GPU-box tool): engine / service warp counts x
concurrency, completions per second through async_read with service-side waiter delivery
(profiles/iops_p.txt)."""
import sys, os, json
sys.path.insert(0, os.getcwd()); sys.path.insert(0, "tests")
from conftest import small_config
from paper_2504_19365_b200 import AgileSystem
res = []
for ew, sw in [(64, 16), (64, 32), (64, 64), (96, 64)]:
    for conc in (4096, 16384):
        s = AgileSystem(small_config(pairs=128, sq_depth=256, cq_depth=256, cache_lines=1 << 17, ways=32,
                                     blocks=1 << 20, emulation="link", engine_warps=ew, warps=sw), device=0)
        r = s.run_loop(conc, warmup_ns=2_000_000, measure_ns=20_000_000)
        st = s.stats()
        gbps = r["completions"] * 4096 / r["window_ns"]
        res.append(dict(ew=ew, sw=sw, conc=conc, gbps=round(gbps, 2), miops=round(r["completions"] / r["window_ns"] * 1e3, 3),
                        mean_lat_us=round(st["barrier_latency_sum"] / max(1, st["barrier_count"]) / 1e3, 1), sq_full=st["sq_full"]))
        print(res[-1], flush=True)
        s.close()
