#!/bin/bash
# full bench line + CLI smoke of the reference experiments
mkdir -p gpurun_out
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -2 gpurun_out/bench.err
timeout 300 python -m paper_2504_19365_b200.cli ctc_sweep > gpurun_out/cli_ctc_default.csv 2>&1; echo "ctc rc=$?"
timeout 600 python -m paper_2504_19365_b200.cli ctc_sweep --config configs/ctc_paper.cfg > gpurun_out/cli_ctc_paper.csv 2>&1; echo "ctc paper rc=$?"
timeout 300 python -m paper_2504_19365_b200.cli rand_read > gpurun_out/cli_rand_read.csv 2>&1; echo "rand_read rc=$?"
timeout 300 python -m paper_2504_19365_b200.cli rand_write > gpurun_out/cli_rand_write.csv 2>&1; echo "rand_write rc=$?"
timeout 300 python -m paper_2504_19365_b200.cli queue_sweep > gpurun_out/cli_queue_sweep.csv 2>&1; echo "queue rc=$?"
timeout 300 python -m paper_2504_19365_b200.cli cache_sweep > gpurun_out/cli_cache_sweep.csv 2>&1; echo "cache rc=$?"
timeout 300 python -m paper_2504_19365_b200.cli deadlock_demo > gpurun_out/cli_deadlock.csv 2>&1; echo "deadlock rc=$?"
timeout 600 python -m paper_2504_19365_b200.cli bfs --config configs/graph_bench.cfg > gpurun_out/cli_bfs.csv 2>&1; echo "bfs rc=$?"
timeout 600 python -m paper_2504_19365_b200.cli spmv --config configs/graph_bench.cfg > gpurun_out/cli_spmv.csv 2>&1; echo "spmv rc=$?"
