"""Per-source-line STL/LDL counts of one kernel in a cubin (nvdisasm -gi line info, innermost frame).

  python tools/spill_lines.py file.cubin kernel_substring [line_lo line_hi]
"""
import collections
import re
import subprocess
import sys

dis = subprocess.run(["nvdisasm", "-gi", sys.argv[1]], capture_output=True, text=True).stdout
fn_sub = sys.argv[2]
lo, hi = (int(sys.argv[3]), int(sys.argv[4])) if len(sys.argv) > 4 else (0, 1 << 30)
fn, inner, newgrp, chain = None, None, True, []
cnt = collections.Counter()
tot = collections.Counter()
for ln in dis.splitlines():
    m = re.match(r"\s*\.text\.(\S+):", ln)
    if m:
        fn = m.group(1)
        continue
    if not fn or fn_sub not in fn:
        continue
    m = re.search(r'## File "([^"]+)", line (\d+)', ln)
    if m:
        if newgrp:
            inner = (m.group(1).split("/")[-1], int(m.group(2)))
            chain = []
            newgrp = False
        chain.append(int(m.group(2)))
        continue
    m = re.search(r"/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", ln)
    if m:
        newgrp = True
        op = m.group(1).split(".")[0]
        tot[op] += 1
        if op in ("STL", "LDL") and inner and any(lo <= x <= hi for x in chain):
            cnt[(inner, op)] += 1
for k, v in sorted(cnt.items(), key=lambda x: -x[1])[:40]:
    print(v, k)
print("total", {k: tot[k] for k in ("STL", "LDL", "LDG", "STG", "CALL")})
