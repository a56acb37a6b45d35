#!/bin/bash
# ncu evidence for one DLRM step = memset + infra grid + PDL user grid running concurrently.
# Kernel replay serialises launches, which the two co-running grids cannot survive (the infra
# grid waits for a user grid that may not start before it ends), so the step is captured as one
# range (--replay-mode range): per-step duration, DRAM bytes and the SOL sections.
mkdir -p gpurun_out
export AGILE_PROFILE_STEP=1
timeout 900 ncu --replay-mode range --clock-control none \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed \
  --csv --log-file gpurun_out/range_step.csv python bench.py --quick --steps 3 --warmup 3 ${BENCH_ARGS} > gpurun_out/range_step.log 2>&1; echo "range rc=$?"
tail -5 gpurun_out/range_step.csv
timeout 1200 ncu --replay-mode range --clock-control none --set full \
  -o gpurun_out/prof_range python bench.py --quick --steps 3 --warmup 3 ${BENCH_ARGS} > gpurun_out/range_full.log 2>&1; echo "range full rc=$?"
tail -3 gpurun_out/range_full.log
