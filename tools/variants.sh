#!/bin/bash
# A/B of prebuilt library variants (tools/bin/v_*.so) on the hit path and the bounded gather
mkdir -p gpurun_out
for v in ${VARIANTS:-s2 d2 d3 d4}; do
  export AGILE_LIB=tools/bin/v_$v.so
  echo "== $v"
  timeout 300 python -m pytest tests/test_gpu_embbag.py -q -m gpu -x --timeout 120 2>&1 | tail -1
  timeout 300 python tools/dlrm_probe.py hit 2>&1 | tail -1
  timeout 300 python tools/dlrm_probe.py hitbig 2>&1 | tail -1
  COMBOS=128/48 PDS=0 UCS=${UCS:-16,32} timeout 600 python tools/pipe_probe.py 4 16 2>&1 | tail -2
done
