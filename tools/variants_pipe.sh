#!/bin/bash
mkdir -p gpurun_out
for v in ${VARIANTS:-p2 p4}; do
  export AGILE_LIB=tools/bin/v_$v.so
  echo "== $v"
  timeout 300 python -m pytest tests/test_gpu_embbag.py tests/test_gpu_queue.py -q -m gpu -x --timeout 120 2>&1 | tail -1
  COMBOS=${COMBOS:-128/48,64/16,32/16} PDS=0 UCS=${UCS:-32,64} CARVE=${CARVE:-0,32} timeout 900 python tools/pipe_probe.py 4 16 2>&1 | grep '^{'
done
