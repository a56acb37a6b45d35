#!/bin/bash
# round-2 batch j: CTC latency probes under config variations, the reference's sweeps via the CLI,
# ncu launch list of the bench command and a fused-mode traffic capture of one bench step.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
for v in "" "service.idle_max_ns=400" "service.warps=16" "service.idle_max_ns=400 service.warps=16 engine.warps=32"; do
  echo "== $v"; timeout 300 python tools/ctc_probe.py - $v 2>&1 | tail -3
done > gpurun_out/ctc_probe_r02.txt
cat gpurun_out/ctc_probe_r02.txt
for e in ctc_sweep queue_sweep cache_sweep; do
  timeout 600 python -m paper_2504_19365_b200.cli $e > gpurun_out/${e}_r02.csv 2> gpurun_out/${e}.err; echo "$e rc=$?"; cat gpurun_out/${e}_r02.csv
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu_launches_bench_r02.csv \
  python bench.py --quick --steps 4 --warmup 3 > gpurun_out/bench_launches.json 2> gpurun_out/bench_launches.err; echo "launch list rc=$?"
grep -c agile gpurun_out/ncu_launches_bench_r02.csv
timeout 900 ncu --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,pcie__read_bytes.sum,pcie__write_bytes.sum,launch__registers_per_thread,launch__grid_size \
  -k regex:agile_fused_kernel -s 88 -c 1 --csv --log-file gpurun_out/ncu_bench_step_fused_r02.csv \
  python bench.py --quick --steps 4 --warmup 3 > gpurun_out/bench_fused.json 2> gpurun_out/bench_fused.err; echo "fused capture rc=$?"
tail -3 gpurun_out/ncu_bench_step_fused_r02.csv
