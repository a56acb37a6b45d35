#!/bin/bash
# DLRM probes + hit-path ncu capture (1 GPU)
mkdir -p gpurun_out
python __graft_entry__.py > /dev/null
timeout 600 python tools/dlrm_probe.py prefetch > gpurun_out/prefetch_sweep.txt 2>&1; echo "prefetch rc=$?"
timeout 300 python tools/dlrm_probe.py hit > gpurun_out/hit.txt 2>&1; echo "hit rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:agile_kernel -s 3 -c 1 \
  -o gpurun_out/prof_hit python tools/dlrm_probe.py hitprof > gpurun_out/prof_hit.log 2>&1; echo "ncu rc=$?"
cat gpurun_out/prefetch_sweep.txt gpurun_out/hit.txt
