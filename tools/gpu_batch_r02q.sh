#!/bin/bash
# round-2 batch q: K5 adaptive grabs (no block held ahead in sync mode) vs fixed 4-bag lookahead.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest -q -m gpu tests/test_gpu_embbag.py tests/test_gpu_dlrm_shard.py tests/test_gpu_torch_op.py > gpurun_out/tests_q.log 2>&1
echo "tests rc=$?"; grep -E "^FAILED|passed|failed" gpurun_out/tests_q.log | tail -4
for rep in 1 2; do
for lib in paper_2504_19365_b200/libagile_b200.so tools/bin/libk5_grab4.so; do
  for cp in registers bulk; do
    for m in uniform zipf; do
      AGILE_LIB=$lib K5_ENGINE_COPY=$cp timeout 300 python tools/k5_probe.py $m 20 2>>gpurun_out/k5_q.err | tee -a gpurun_out/k5_q.jsonl
    done
  done
  AGILE_LIB=$lib timeout 600 python bench.py --quick --steps 10 --warmup 3 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench', '$lib', d['value'], d['ms_per_step'], d['roofline']['frac'])"
done
done
