#!/bin/bash
# round-2 batch: new-code parity tests, K5 variant timings + ncu captures of the production user
# kernel (solo mode), TMA bulk-copy probe, CTC stage trace.  Outputs under gpurun_out/.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest -q -m gpu tests/test_gpu_embbag.py tests/test_gpu_dlrm_shard.py tests/test_gpu_cache.py \
  tests/test_gpu_array_get.py tests/test_gpu_queue.py > gpurun_out/tests_b.log 2>&1
echo "tests rc=$?"; tail -4 gpurun_out/tests_b.log
for lib in tools/bin/libk5_bag.so tools/bin/libk5_48.so tools/bin/libk5_44.so tools/bin/libk5_36.so; do
  for m in uniform zipf; do
    AGILE_LIB=$lib timeout 300 python tools/k5_probe.py $m 20 2>>gpurun_out/k5_var.err | tee -a gpurun_out/k5_var_b.jsonl
  done
done
for v in bag 48 36; do
  AGILE_LIB=tools/bin/libk5_$v.so K5_SOLO=1 timeout 600 ncu --set full --import-source on --clock-control none \
    -k regex:agile_user_kernel -c 1 -o gpurun_out/k5u_$v -f python tools/k5_probe.py uniform 1 > gpurun_out/k5u_$v.log 2>&1
  echo "ncu $v rc=$?"; tail -1 gpurun_out/k5u_$v.log
done
timeout 300 ./tools/bin/probe_bulk 8 > gpurun_out/probe_bulk.jsonl 2>&1; echo "bulk rc=$?"; cat gpurun_out/probe_bulk.jsonl
timeout 300 python tools/ctc_trace.py > gpurun_out/ctc_trace.txt 2>&1; echo "ctc trace rc=$?"; head -30 gpurun_out/ctc_trace.txt
