import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, "tests")
import numpy as np
from conftest import small_config
from paper_2504_19365_b200 import AgileSystem, TraceRecorder
conc = int(sys.argv[1]) if len(sys.argv) > 1 else 512
s = AgileSystem(small_config(pairs=8, sq_depth=256, cq_depth=256, cache_lines=8192, ways=32, blocks=1 << 18,
                             emulation="model", engine_warps=16, warps=4), recorder=TraceRecorder(), device=0)
r = s.run_loop(conc, warmup_ns=0, measure_ns=10**10, max_per_task=8)
st = s.stats(); print(r, {k: st[k] for k in ("completions", "cqe_stalls", "sq_full", "fetched")})
recs = s.events().records
fetch = {}; comp = []; post = []; enq = []; iss = {}
for t, who, mod, act, d in recs:
    if act == "enqueue": enq.append(t)
    if act == "fetch": fetch[(d[1], d[2])] = t
    if act == "complete": comp.append((t, t - fetch.get((d[1], d[2]), t)))
comp.sort()
ct = np.array([c[0] for c in comp]); lat = np.array([c[1] for c in comp])
print("n", len(ct), "span us", (ct[-1] - ct[0]) / 1e3, "rate M/s", len(ct) / (ct[-1] - ct[0]) * 1e3)
print("fetch->complete us p10/50/90", np.percentile(lat, [10, 50, 90]) / 1e3)
gaps = np.diff(ct); print("completion gaps us p50/p90/p99/max", np.percentile(gaps, [50, 90, 99]) / 1e3, gaps.max() / 1e3)
# completions per 17.7us window
w = ((ct - ct[0]) // 17712).astype(int); cnt = np.bincount(w); print("per-17.7us window completions (first 40)", cnt[:40].tolist())
en = np.array(sorted(enq)); f = np.array(sorted(fetch.values()))
print("enqueued by t", [(int((x - ct[0]) / 1e3), int((en <= x).sum()), int((f <= x).sum()), int((ct <= x).sum())) for x in np.linspace(ct[0], ct[-1], 12)])
