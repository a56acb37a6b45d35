#!/bin/bash
# round-2 batch m: DLRM pipeline probe (prefetch mode parts: side prefetch / MLPs / hit gather) over
# side-CTA bounds, carve-outs, side infra sizes and engine copy modes, at the bench config.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
for eng in registers bulk; do
  for side in 64/16 32/8 128/48; do
    ENGINE_COPY=$eng SIDE=$side COMBOS=128/48 UCS=24,48,96 CARVE=48,64 MODES=prefetch \
      timeout 900 python tools/pipe_probe.py 16 64 2>>gpurun_out/pipe_m.err | tee -a gpurun_out/pipe_m.jsonl
  done
done
