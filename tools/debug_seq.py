import json, sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
sys.path.insert(0, "tests"); from conftest import small_config
from paper_2504_19365_b200 import AgileSystem, TraceRecorder
g = json.load(open("tests/golden/golden.json"))["a1_full_stack"]
s = AgileSystem(small_config(cache_lines=16, ways=0, blocks=256), recorder=TraceRecorder(), device=0)
n = 45
out, vic, _ = s.run_seq(np.zeros(n), g["stream"][:n])
print("out", list(out))
print("vic", [int(v) if v != np.uint64(2**64-1) else -1 for v in vic])
print("stream", g["stream"][:n])
recs = s.events().records
for r in recs:
    if r[2] == "cache" or r[3] in ("sqe_release",):
        print(r)
