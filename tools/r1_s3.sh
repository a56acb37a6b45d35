#!/bin/bash
# session-3 probe: pipeline modes in the bench + ncu of the all-hit embbag launch
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -3 gpurun_out/bench.err
timeout 900 ncu --set full --import-source on --clock-control none -k regex:agile_kernel -s 4 -c 1 \
  -o gpurun_out/prof_hit python tools/dlrm_probe.py hitprof > gpurun_out/prof_hit.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/prof_hit.log
