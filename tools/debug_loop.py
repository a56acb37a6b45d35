import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, "tests")
import numpy as np
from collections import defaultdict
from conftest import small_config
from paper_2504_19365_b200 import AgileSystem, TraceRecorder
s = AgileSystem(small_config(pairs=8, sq_depth=256, cq_depth=256, cache_lines=4096, ways=32, blocks=1 << 16,
                             emulation="model", engine_warps=8, warps=4), recorder=TraceRecorder(), device=0)
r = s.run_loop(64, warmup_ns=0, measure_ns=10**10, max_per_task=20)
print(r, s.stats())
recs = s.events().records
ev = defaultdict(dict)
for t, who, mod, act, d in recs:
    if act == "enqueue": key = (d[0], d[1]); ev[key].setdefault("list", []).append({"enq": t})
    elif act in ("sqe_issued",): ev[(d[0], d[1])]["list"][-1]["iss"] = t
    elif act == "fetch": ev[(d[1], d[2])]["list"][-1]["fetch"] = t
    elif act == "complete": ev[(d[1], d[2])]["list"][-1]["done"] = t
    elif act == "cqe_post": ev[(d[0], d[2])]["list"][-1]["post"] = t
    elif act == "cqe_process": ev[(d[3], d[2])]["list"][-1]["proc"] = t
rows = [x for v in ev.values() for x in v["list"] if len(x) == 6]
a = {k: np.array([x[k] for x in rows]) for k in ("enq", "iss", "fetch", "done", "post", "proc")}
for k1, k2 in (("enq", "iss"), ("iss", "fetch"), ("fetch", "done"), ("done", "post"), ("post", "proc"), ("enq", "proc")):
    dd = a[k2] - a[k1]
    print(f"{k1}->{k2}: p50 {np.percentile(dd,50):.0f} p90 {np.percentile(dd,90):.0f} max {dd.max():.0f} ns")
print("span", a["proc"].max() - a["enq"].min(), "n", len(rows))
# gaps between one warp's consecutive enqueue batches
en = np.sort(a["enq"]); print("enqueue time quantiles", np.percentile(np.diff(en), [50, 90, 99]))
