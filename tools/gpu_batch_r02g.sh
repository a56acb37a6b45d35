#!/bin/bash
# round-2 batch g: K5 deferred validation A/B, ncu of the production user kernel (users-only replay),
# RMAT-22 oracle test, graph benchmarks at the BASELINE scales with C-oracle checks.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest -q -m gpu tests/test_gpu_embbag.py tests/test_gpu_dlrm_shard.py tests/test_gpu_graph.py > gpurun_out/tests_g.log 2>&1
echo "tests rc=$?"; grep -E "^FAILED|passed|failed" gpurun_out/tests_g.log | tail -6
for lib in paper_2504_19365_b200/libagile_b200.so tools/bin/libk5_nodefer.so; do
  for cp in registers bulk; do
    for m in uniform zipf; do
      AGILE_LIB=$lib K5_ENGINE_COPY=$cp timeout 300 python tools/k5_probe.py $m 20 2>>gpurun_out/k5_g.err | tee -a gpurun_out/k5_g.jsonl
    done
  done
done
K5_SOLO=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:agile_user_kernel -c 1 \
  -o gpurun_out/k5u_users -f python tools/k5_probe.py uniform 1 > gpurun_out/k5u_users.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/k5u_users.log
timeout 1200 python tools/graph_bench.py bfs 26 0.25 > gpurun_out/graph_bfs26_r02.json 2> gpurun_out/graph_bfs26.err; echo "bfs26 rc=$?"
tail -c 1500 gpurun_out/graph_bfs26_r02.json
timeout 1800 python tools/graph_bench.py spmv 27 0.25 10 > gpurun_out/graph_spmv27_r02.json 2> gpurun_out/graph_spmv27.err; echo "spmv27 rc=$?"
tail -c 1500 gpurun_out/graph_spmv27_r02.json
