#!/bin/bash
# K5 (embedding-bag) evidence on the GPU box: timing of the all-hit replays (no profiler), one
# full ncu capture of the production user kernel on the uniform (no-reuse) replay, and one
# range-replay capture of a bench step (both grids of the split launch running together).
# Outputs under gpurun_out/ (TAG names them).
TAG=${TAG:-r02}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
for m in uniform zipf; do
  timeout 600 python tools/k5_probe.py $m 20 2>gpurun_out/k5_$m.err | tee gpurun_out/k5_${m}_${TAG}.json
done
if [ -z "$NO_NCU" ]; then
  # production user kernel alone (solo mode: the infra grid leaves after 100 ms; all hits need no engine)
  AGILE_LAUNCH=split AGILE_SOLO_USERS=1 timeout 900 ncu --set full --import-source on --clock-control none \
    -k regex:agile_user_kernel -s 3 -c 1 -o gpurun_out/k5_uniform_${TAG} -f \
    python tools/k5_probe.py uniform 2 > gpurun_out/k5_ncu_${TAG}.log 2>&1; echo "ncu uniform rc=$?"
  tail -2 gpurun_out/k5_ncu_${TAG}.log
fi
if [ -n "$RANGE" ]; then
  export AGILE_PROFILE_STEP=1
  timeout 900 ncu --replay-mode range --clock-control none \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,pcie__read_bytes.sum,pcie__write_bytes.sum \
    --csv --log-file gpurun_out/range_step_${TAG}.csv python bench.py --quick --steps 3 --warmup 3 > gpurun_out/range_step.log 2>&1; echo "range rc=$?"
  tail -8 gpurun_out/range_step_${TAG}.csv
fi
