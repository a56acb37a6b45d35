#!/bin/bash
# ncu evidence for the embedding-bag fused kernel (1 GPU): launch list of a bench run + one full
# capture of a steady-state timed launch (2 GiB cache config so replays stay cheap)
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --quick --steps 6 --warmup 3 --cache-gib 2 --warm-batches 8 > gpurun_out/prof_bench_launches.json 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:agile_kernel -s 11 -c 1 \
  -o gpurun_out/prof_embbag python bench.py --quick --steps 2 --warmup 3 --cache-gib 2 --warm-batches 8 \
  > gpurun_out/prof_full.log 2>&1
ls -la gpurun_out/*.ncu-rep
