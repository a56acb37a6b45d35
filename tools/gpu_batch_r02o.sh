#!/bin/bash
# round-2 batch o: grouped vs per-lane set-lock claims on the queue / cache sweeps and the CTC
# default (3 repetitions each, to separate the effect from run-to-run noise).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
for lib in paper_2504_19365_b200/libagile_b200.so tools/bin/libclaim_old.so; do
  for rep in 1 2 3; do
    for e in queue_sweep ctc_sweep; do
      AGILE_LIB=$lib timeout 600 python -m paper_2504_19365_b200.cli $e > gpurun_out/${e}_o.csv 2>/dev/null
      col=5; [ $e = ctc_sweep ] && col=4
      echo "$lib $rep $e: $(tail -n +2 gpurun_out/${e}_o.csv | awk -F, -v c=$col '{printf "%s ", $c}' )" | tee -a gpurun_out/claim_ab_r02.txt
    done
  done
done
