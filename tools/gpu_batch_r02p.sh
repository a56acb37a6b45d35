#!/bin/bash
# round-2 batch p: service waiter copies in one step (slice 8) with the register engine — suite,
# CTC / queue sweeps x3, IOPS link sweep.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest -q -m gpu tests > gpurun_out/tests_p.log 2>&1
echo "suite rc=$?"; grep -E "^FAILED|passed|failed" gpurun_out/tests_p.log | tail -8
for rep in 1 2 3; do
  for e in queue_sweep ctc_sweep; do
    timeout 600 python -m paper_2504_19365_b200.cli $e > gpurun_out/${e}_p.csv 2>/dev/null
    col=5; [ $e = ctc_sweep ] && col=4
    echo "slice8 $rep $e: $(tail -n +2 gpurun_out/${e}_p.csv | awk -F, -v c=$col '{printf "%s ", $c}' )" | tee -a gpurun_out/slice_ab_r02.txt
  done
done
timeout 300 python tools/iops_sweep.py > gpurun_out/iops_p.txt 2>&1; tail -8 gpurun_out/iops_p.txt
