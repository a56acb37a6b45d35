#!/bin/bash
# round-2 batch h: full bench line (pipeline with both engine copy modes), SpMV / PageRank at the
# BASELINE scale with the C-oracle check (progress on stderr), host memory report.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
free -g > gpurun_out/box_mem.txt; nproc >> gpurun_out/box_mem.txt; cat gpurun_out/box_mem.txt
timeout 900 python bench.py > gpurun_out/bench_r02h.json 2> gpurun_out/bench_r02h.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/bench_r02h.json').read().strip().splitlines()[-1])
print('value', d['value'], 'ms', d['ms_per_step'], 'link', d['roofline']['frac'], 'e2e', d['e2e']['value'], 'hit', d['roofline_hit']['frac'], 'avs', d['async_vs_sync'], d['async_vs_sync_engine'])
for p in d['dlrm_pipeline']['points']: print(p['target_ctc'], round(p['ctc'],2), round(p['speedup'],3), round(p['speedup_bulk_engine'],3), round(p['ideal'],3))"
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_r02h.json 2> gpurun_out/bench_ref_r02h.err; echo "ref rc=$?"
tail -c 1200 gpurun_out/bench_ref_r02h.json
timeout 1800 python tools/graph_bench.py spmv 27 0.25 10 > gpurun_out/graph_spmv27_r02.json 2> gpurun_out/graph_spmv27.err; echo "spmv27 rc=$?"
tail -5 gpurun_out/graph_spmv27.err; tail -c 1500 gpurun_out/graph_spmv27_r02.json
