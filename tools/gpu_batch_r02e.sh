#!/bin/bash
# round-2 batch e: full GPU suite; K5 hit-path variants x engine copy mode; bench with each engine.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest -q -m gpu tests > gpurun_out/tests_e.log 2>&1
echo "tests rc=$?"; grep -E "^FAILED|passed|failed" gpurun_out/tests_e.log | tail -8
for lib in paper_2504_19365_b200/libagile_b200.so tools/bin/libk5_ef.so tools/bin/libk5_m3.so; do
  for cp in registers bulk; do
    for m in uniform zipf; do
      AGILE_LIB=$lib K5_ENGINE_COPY=$cp timeout 300 python tools/k5_probe.py $m 20 2>>gpurun_out/k5_e.err | tee -a gpurun_out/k5_e.jsonl
    done
  done
done
