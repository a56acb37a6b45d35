#!/bin/bash
# round-2 batch k: fused-mode traffic capture of one bench step (the launch the ncu launch list
# shows), then the final bench line and the reference arm.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
AGILE_LAUNCH=fused timeout 900 ncu --clock-control none \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,pcie__read_bytes.sum,pcie__write_bytes.sum,launch__registers_per_thread,launch__grid_size \
  -k regex:agile_fused_kernel -s 87 -c 2 --csv --log-file gpurun_out/ncu_bench_step_fused_r02.csv \
  python bench.py --quick --steps 4 --warmup 3 > gpurun_out/bench_fused.json 2> gpurun_out/bench_fused.err; echo "fused capture rc=$?"
grep agile gpurun_out/ncu_bench_step_fused_r02.csv | cut -c1-300 | head -20
timeout 900 python bench.py > gpurun_out/bench_r02k.json 2> gpurun_out/bench_r02k.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/bench_r02k.json').read().strip().splitlines()[-1])
print('value', d['value'], 'ms', d['ms_per_step'], 'link', d['roofline']['frac'], 'e2e', d['e2e']['value'], 'hit', d['roofline_hit']['frac'], 'avs', d['async_vs_sync'], d['async_vs_sync_engine'], 'clocks', d['clocks'])"
