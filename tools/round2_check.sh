#!/bin/bash
# round-2 baseline check on the GPU box: parity suite, smoke (plain and under ncu), one bench line
bash tools/gpu_check.sh
timeout 600 python bench.py > gpurun_out/bench_r02a.json 2> gpurun_out/bench_r02a.err; echo "bench rc=$?"
tail -c 3000 gpurun_out/bench_r02a.json
