#!/bin/bash
# round-2 batch n: grouped set-lock claims — full GPU suite, CTC / queue / cache sweeps, CTC probe,
# IOPS at link speed, bench step.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest -q -m gpu tests > gpurun_out/tests_n.log 2>&1
echo "suite rc=$?"; grep -E "^FAILED|passed|failed" gpurun_out/tests_n.log | tail -8
timeout 300 python tools/ctc_probe.py - 2>&1 | tail -3
for e in ctc_sweep queue_sweep cache_sweep; do
  timeout 600 python -m paper_2504_19365_b200.cli $e > gpurun_out/${e}_r02n.csv 2> gpurun_out/${e}.err; echo "$e rc=$?"; cat gpurun_out/${e}_r02n.csv
done
timeout 600 python bench.py --quick --steps 10 --warmup 3 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench', d['value'], d['ms_per_step'], d['roofline']['frac'])"
