#!/bin/bash
# ncu evidence for the embedding-bag step.  The production launch runs two grids concurrently
# (infra + PDL user grid); ncu serialises kernels, so the captures use the fused single-grid mode
# (AGILE_LAUNCH=fused: same device code, roles by arrival ticket, one register budget).
mkdir -p gpurun_out
export AGILE_LAUNCH=fused
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --quick --steps 6 --warmup 3 ${BENCH_ARGS} > gpurun_out/prof_bench_launches.json 2>&1; echo "launches rc=$?"
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:agile_fused_kernel -s ${SKIP:-12} -c 1 \
  -o gpurun_out/prof_embbag python bench.py --quick --steps 3 --warmup 3 ${BENCH_ARGS} > gpurun_out/prof_full.log 2>&1; echo "full rc=$?"
tail -2 gpurun_out/prof_full.log
