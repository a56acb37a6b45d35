#!/bin/bash
# round-2 batch f: share table + MODIFIED coherence tests, device API / torch op tests, the full
# suite, and ncu captures of the production K5 user kernel (solo mode, uniform replay) with each
# engine copy mode.  Outputs under gpurun_out/.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest -q -m gpu tests/test_gpu_coherence.py tests/test_gpu_device_api.py tests/test_gpu_torch_op.py > gpurun_out/tests_f1.log 2>&1
echo "new tests rc=$?"; grep -E "^FAILED|passed|failed" gpurun_out/tests_f1.log | tail -12
timeout 1200 python -m pytest -q -m gpu tests > gpurun_out/tests_f.log 2>&1
echo "suite rc=$?"; grep -E "^FAILED|passed|failed" gpurun_out/tests_f.log | tail -8
for cp in registers bulk; do
  K5_ENGINE_COPY=$cp K5_SOLO=1 timeout 600 ncu --set full --import-source on --clock-control none \
    -k regex:agile_user_kernel -c 1 -o gpurun_out/k5u_$cp -f python tools/k5_probe.py uniform 1 > gpurun_out/k5u_$cp.log 2>&1
  echo "ncu $cp rc=$?"; tail -2 gpurun_out/k5u_$cp.log
done
