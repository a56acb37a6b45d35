#!/bin/bash
# round-2 batch i: lock-chain detector tests + full suite, reference arm, SpMV/PageRank at scale 27
# with the C-oracle check.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest -q -m gpu tests > gpurun_out/tests_i.log 2>&1
echo "suite rc=$?"; grep -E "^FAILED|passed|failed" gpurun_out/tests_i.log | tail -8
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref_r02i.json 2> gpurun_out/bench_ref_r02i.err; echo "ref rc=$?"
tail -c 1500 gpurun_out/bench_ref_r02i.json
timeout 1800 python tools/graph_bench.py spmv 27 0.25 10 > gpurun_out/graph_spmv27_r02.json 2> gpurun_out/graph_spmv27.err; echo "spmv27 rc=$?"
tail -3 gpurun_out/graph_spmv27.err; tail -c 2000 gpurun_out/graph_spmv27_r02.json
