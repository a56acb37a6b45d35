#!/bin/bash
# round-2 batch r: K5 adaptive grabs with a tail of 2 bags per warp vs the fixed 4-bag lookahead; edge tests.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest -q -m gpu tests/test_gpu_embbag.py tests/test_gpu_dlrm_shard.py tests/test_gpu_edges.py > gpurun_out/tests_r.log 2>&1
echo "tests rc=$?"; grep -E "^FAILED|passed|failed" gpurun_out/tests_r.log | tail -6
for rep in 1 2 3; do
for lib in paper_2504_19365_b200/libagile_b200.so tools/bin/libk5_grab4.so; do
  for m in uniform zipf; do
    AGILE_LIB=$lib timeout 300 python tools/k5_probe.py $m 20 2>>gpurun_out/k5_r.err | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$lib', d['mode'], round(d['ms'],4), round(d['frac'],3))"
  done
  AGILE_LIB=$lib timeout 600 python bench.py --quick --steps 10 --warmup 3 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench', '$lib', d['value'], d['ms_per_step'], d['roofline']['frac'])"
done
done
