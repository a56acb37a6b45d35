#!/bin/bash
# round-2 batch l: full GPU suite (BufferBusy + nodes zeroed per run), compute-sanitizer memcheck
# over a parity subset (fused launch under the sanitizer), smoke.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest -q -m gpu tests > gpurun_out/tests_l.log 2>&1
echo "suite rc=$?"; grep -E "^FAILED|passed|failed" gpurun_out/tests_l.log | tail -8
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_l.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_l.log
timeout 1500 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 \
  python -m pytest -q -m gpu -x tests/test_gpu_cache.py tests/test_gpu_array_get.py \
  "tests/test_gpu_queue.py::test_two_level_coalescing" "tests/test_gpu_embbag.py::test_embbag_shapes" \
  tests/test_gpu_coherence.py::test_enabled_table_masks_the_hazard_on_every_seed > gpurun_out/sanitizer_r02.txt 2>&1
echo "memcheck rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/sanitizer_r02.txt | tail -5
