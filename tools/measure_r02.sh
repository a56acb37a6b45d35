#!/bin/bash
# Reproduces the round-2 measurements under profiles/ on one B200 (run through gpurun from the repo
# root; outputs land in gpurun_out/).  Sections can be picked with ONLY="tests bench k5 graph sweeps
# ncu sanitizer".
set -u
mkdir -p gpurun_out
want() { [ -z "${ONLY:-}" ] || [[ " $ONLY " == *" $1 "* ]]; }
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
if want tests; then
  timeout 1500 python -m pytest -q -m gpu tests > gpurun_out/tests.log 2>&1; echo "gpu tests rc=$?"; tail -1 gpurun_out/tests.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
fi
if want bench; then   # profiles/bench_r02*.json, bench_ref_r02*.json
  timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
  timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
fi
if want k5; then      # profiles/k5_variants_r02.jsonl (engine copy modes x all-hit replays)
  for cp in registers bulk; do for m in uniform zipf; do
    K5_ENGINE_COPY=$cp timeout 300 python tools/k5_probe.py $m 20 2>>gpurun_out/k5.err | tee -a gpurun_out/k5.jsonl
  done; done
fi
if want ncu; then     # profiles/ncu_k5_users_uniform_r02.csv, ncu_launches_bench_r02.csv, ncu_bench_step_fused_r02.csv
  K5_SOLO=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:agile_user_kernel -c 1 \
    -o gpurun_out/k5u_users -f python tools/k5_probe.py uniform 1 > gpurun_out/k5u_users.log 2>&1; echo "ncu k5 rc=$?"
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu_launches_bench.csv \
    python bench.py --quick --steps 4 --warmup 3 > /dev/null 2>&1; echo "launch list rc=$?"
  AGILE_LAUNCH=fused timeout 900 ncu --clock-control none \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,pcie__read_bytes.sum,pcie__write_bytes.sum,launch__registers_per_thread,launch__grid_size \
    -k regex:agile_fused_kernel -s 87 -c 2 --csv --log-file gpurun_out/ncu_bench_step_fused.csv \
    python bench.py --quick --steps 4 --warmup 3 > /dev/null 2>&1; echo "fused capture rc=$?"
fi
if want graph; then   # profiles/graph_bfs26_r02.json, graph_spmv27_r02.json (C-oracle checks included)
  timeout 1200 python tools/graph_bench.py bfs 26 0.25 > gpurun_out/graph_bfs26.json 2> gpurun_out/graph_bfs26.err; echo "bfs26 rc=$?"
  timeout 1800 python tools/graph_bench.py spmv 27 0.25 10 > gpurun_out/graph_spmv27.json 2> gpurun_out/graph_spmv27.err; echo "spmv27 rc=$?"
fi
if want sweeps; then  # profiles/ctc_sweep_r02*.csv, queue_sweep_r02*.csv, cache_sweep_r02*.csv, iops, pipeline probe
  for e in ctc_sweep queue_sweep cache_sweep; do
    timeout 600 python -m paper_2504_19365_b200.cli $e > gpurun_out/${e}.csv 2> gpurun_out/${e}.err; echo "$e rc=$?"
  done
  timeout 300 python tools/iops_sweep.py > gpurun_out/iops.txt 2>&1
  SIDE=64/16 COMBOS=128/48 UCS=24,48,96 CARVE=48,64 MODES=prefetch timeout 900 python tools/pipe_probe.py 16 64 > gpurun_out/pipe.jsonl 2>/dev/null
  timeout 300 ./tools/bin/probe_bulk 8 > gpurun_out/probe_bulk.jsonl 2>&1 || true   # nvcc -o tools/bin/probe_bulk tools/probe_bulk.cu
fi
if want sanitizer; then   # profiles/sanitizer_r02.txt
  timeout 1500 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 \
    python -m pytest -q -m gpu -x tests/test_gpu_cache.py tests/test_gpu_array_get.py \
    "tests/test_gpu_queue.py::test_two_level_coalescing" tests/test_gpu_embbag.py tests/test_gpu_dlrm_shard.py \
    tests/test_gpu_coherence.py::test_enabled_table_masks_the_hazard_on_every_seed > gpurun_out/sanitizer.txt 2>&1
  echo "memcheck rc=$?"
fi
