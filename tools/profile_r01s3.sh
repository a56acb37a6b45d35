#!/bin/bash
# round-1 session-3 ncu evidence (fused launch mode: the serialising profiler cannot run the split
# launch's two co-running grids)
mkdir -p gpurun_out
export AGILE_LAUNCH=fused
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:agile --csv \
  --log-file gpurun_out/launches_bench.csv python bench.py --quick --steps 4 --warmup 3 > gpurun_out/launches_bench.json 2>&1; echo "launch list rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:agile_fused_kernel -s 4 -c 1 \
  -o gpurun_out/prof_hit_fused python tools/dlrm_probe.py hitprof > gpurun_out/prof_hit_fused.log 2>&1; echo "hit rc=$?"
unset AGILE_LAUNCH
timeout 300 python tools/dlrm_probe.py hitbig > gpurun_out/hitbig_split.txt 2>&1; cat gpurun_out/hitbig_split.txt | tail -1
