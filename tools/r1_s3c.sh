#!/bin/bash
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_embbag.py -q -m gpu -x --timeout 240 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python tools/dlrm_probe.py hit > gpurun_out/hit.txt 2>&1; echo "hit rc=$?"; cat gpurun_out/hit.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:agile_kernel -s 4 -c 1 \
  -o gpurun_out/prof_hit2 python tools/dlrm_probe.py hitprof > gpurun_out/prof_hit.log 2>&1; echo "ncu rc=$?"
