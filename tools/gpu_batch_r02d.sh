#!/bin/bash
# round-2 batch d: engine A/B (register-staged vs bulk-copy variants) on the bench step and the
# all-hit replay; new parity tests (device API, torch op).  Outputs under gpurun_out/.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest -q -m gpu tests/test_gpu_device_api.py tests/test_gpu_torch_op.py tests/test_gpu_array_get.py > gpurun_out/tests_d.log 2>&1
echo "tests rc=$?"; grep -E "^FAILED|passed|failed" gpurun_out/tests_d.log | tail -8
for lib in paper_2504_19365_b200/libagile_b200.so tools/bin/libeng_reg.so tools/bin/libeng_b6.so tools/bin/libeng_b4m3.so; do
  for rep in 1 2; do
    AGILE_LIB=$lib timeout 400 python bench.py --quick --steps 10 --warmup 3 2>>gpurun_out/bench_d.err \
      | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(json.dumps({'lib': '$lib'.split('/')[-1], 'value': d['value'], 'ms': d['ms_per_step'], 'link_frac': d['roofline']['frac'], 'iops': d['roofline']['iops']}))" \
      | tee -a gpurun_out/bench_d.jsonl
  done
  AGILE_LIB=$lib timeout 300 python tools/k5_probe.py uniform 20 2>>gpurun_out/k5_d.err | tee -a gpurun_out/k5_d.jsonl
done
