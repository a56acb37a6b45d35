#!/bin/bash
# A/B of K5 builds (tools/bin/libk5_*.so, built here with -D switches) on the all-hit replays,
# plus the embedding-bag parity tests on the default build.  GPU-box tool; outputs in gpurun_out/.
TAG=${TAG:-v}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_embbag.py tests/test_gpu_dlrm_shard.py tests/test_gpu_cache.py > gpurun_out/k5_tests_${TAG}.log 2>&1
echo "k5 tests rc=$?"; tail -2 gpurun_out/k5_tests_${TAG}.log
for lib in ${LIBS:-tools/bin/libk5_*.so}; do
  for m in uniform zipf; do
    AGILE_LIB=$lib timeout 300 python tools/k5_probe.py $m 20 2>>gpurun_out/k5_var.err | tee -a gpurun_out/k5_var_${TAG}.jsonl
  done
done
