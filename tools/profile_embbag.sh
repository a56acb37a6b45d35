#!/bin/bash
# ncu evidence for the embedding-bag fused kernel (1 GPU): launch list + one full capture per mode
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --quick --steps 4 --warmup 3 --cache-gib 2 > gpurun_out/prof_bench_launches.json 2>&1
for pd in 1 0; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:agile_kernel -s 4 -c 1 \
    -o gpurun_out/prof_embbag_pd$pd python bench.py --quick --steps 2 --warmup 3 --cache-gib 2 --prefetch $pd \
    > gpurun_out/prof_pd$pd.log 2>&1
done
ls -la gpurun_out/*.ncu-rep
