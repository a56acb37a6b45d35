#!/bin/bash
# round-2 batch c: bulk-copy (TMA) engine — full GPU parity suite, infra sizing sweep on the all-hit
# replay and on the link-bound bench step, IOPS at link speed.  Outputs under gpurun_out/.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest -q -m gpu tests > gpurun_out/tests_c.log 2>&1
echo "tests rc=$?"; grep -E "^FAILED|passed|failed" gpurun_out/tests_c.log | tail -8
for ew in 128 64 32; do
  for sw in 48 16; do
    K5_ENGINE_WARPS=$ew K5_SERVICE_WARPS=$sw timeout 300 python tools/k5_probe.py uniform 20 2>>gpurun_out/k5_c.err \
      | sed "s/^{/{\"ew\": $ew, \"sw\": $sw, /" | tee -a gpurun_out/k5_c.jsonl
  done
done
for ew in 128 64 32; do
  for sw in 48 16; do
    timeout 400 python bench.py --quick --steps 10 --warmup 3 --engine-warps $ew --service-warps $sw 2>>gpurun_out/bench_c.err \
      | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(json.dumps({'ew': $ew, 'sw': $sw, 'value': d['value'], 'ms': d['ms_per_step'], 'link_frac': d['roofline']['frac'], 'iops': d['roofline']['iops']}))" \
      | tee -a gpurun_out/bench_c.jsonl
  done
done
timeout 300 python tools/iops_sweep.py > gpurun_out/iops_c.txt 2>&1; echo "iops rc=$?"; tail -12 gpurun_out/iops_c.txt
