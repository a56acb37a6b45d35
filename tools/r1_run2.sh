#!/bin/bash
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -q -m gpu -x --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log
timeout 300 python tools/dlrm_probe.py hit > gpurun_out/hit.txt 2>&1; echo "hit rc=$?"; cat gpurun_out/hit.txt
timeout 600 python tools/dlrm_probe.py prefetch > gpurun_out/prefetch_sweep.txt 2>&1; echo "prefetch rc=$?"; cat gpurun_out/prefetch_sweep.txt
timeout 600 python tools/graph_bench.py bfs 22 > gpurun_out/bfs22.txt 2>&1; echo "bfs22 rc=$?"; tail -3 gpurun_out/bfs22.txt
timeout 600 python tools/graph_bench.py spmv 22 0.25 3 > gpurun_out/spmv22.txt 2>&1; echo "spmv22 rc=$?"; tail -3 gpurun_out/spmv22.txt
