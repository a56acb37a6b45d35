"""Aggregate an ncu SASS source page (instructions executed, stall samples) per CUDA source line.

  ncu -i rep.ncu-rep --page source --csv --print-source sass > sass.csv
  python tools/sass_lines.py sass.csv lib.so EmbBagWork [top]

Rows are matched to `nvdisasm -gi` line info of the same cubin by their offset within the kernel
(ncu reports absolute addresses; the kernel's first instruction is its base).  The innermost
source line and the outermost call site inside the workload file are both reported.
"""
import collections
import csv
import os
import re
import subprocess
import sys
import tempfile


def line_map(so, fn_sub):
    d = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=d, check=True, capture_output=True)
    cub = [os.path.join(d, f) for f in os.listdir(d) if f.endswith(".cubin")][0]
    dis = subprocess.run(["nvdisasm", "-gi", cub], capture_output=True, text=True).stdout
    cur, inner, outer, out, block = None, None, None, {}, []
    for ln in dis.splitlines():
        m = re.match(r"\.text\.(\S+):", ln)
        if m:
            cur = m.group(1) if fn_sub in m.group(1) and ("agile_kernel" in m.group(1) or "agile_user_kernel" in m.group(1)) else None
            continue
        if cur is None:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            block.append(f"{os.path.basename(m.group(1))}:{m.group(2)}")
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(\S.*?);", ln)
        if m:
            if block:   # a chain is printed innermost first, then each enclosing call site
                inner = block[0]
                work = [b for b in block if "agile_work" in b]
                outer = work[-1] if work else block[-1]
                block = []
            out[int(m.group(1), 16)] = (inner, outer, m.group(2).strip())
    return out


def main():
    csv_path, so, fn_sub = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    rows = list(csv.reader(open(csv_path)))
    hdr = rows[1]
    ia, ix, iss = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    data = [(int(r[ia], 16), float(r[ix] or 0), float(r[iss] or 0)) for r in rows[2:]
            if len(r) > ix and r[ia].startswith("0x")]
    base = data[0][0]
    lm = line_map(so, fn_sub)
    tot_i = sum(x for _, x, _ in data) or 1
    tot_s = sum(s for _, _, s in data) or 1
    by_in, by_out = collections.Counter(), collections.Counter()
    st_in, st_out = collections.Counter(), collections.Counter()
    ops = collections.Counter()
    for a, x, s in data:
        inner, outer, sass = lm.get(a - base, ("?", "?", "?"))
        by_in[inner] += x
        st_in[inner] += s
        by_out[outer] += x
        st_out[outer] += s
        ops[sass.split()[0].split(".")[0] if sass != "?" else "?"] += x
    print(f"total warp instructions {tot_i:.0f}, stall samples {tot_s:.0f}")
    print("--- by innermost line: inst% stall% line")
    for k, v in sorted(by_in.items(), key=lambda kv: -(kv[1] / tot_i + st_in[kv[0]] / tot_s))[:top]:
        print(f"{100 * v / tot_i:6.2f} {100 * st_in[k] / tot_s:6.2f}  {k}")
    print("--- by call site: inst% stall% line")
    for k, v in sorted(by_out.items(), key=lambda kv: -(kv[1] / tot_i + st_out[kv[0]] / tot_s))[:top // 2]:
        print(f"{100 * v / tot_i:6.2f} {100 * st_out[k] / tot_s:6.2f}  {k}")
    print("--- opcodes: inst%")
    for k, v in ops.most_common(25):
        print(f"{100 * v / tot_i:6.2f}  {k}")


if __name__ == "__main__":
    main()
