#!/bin/bash
# staged embbag: parity, hit roofline, pipeline probe
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests -q -m gpu -x --timeout 240 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log
timeout 300 python tools/dlrm_probe.py hit > gpurun_out/hit.txt 2>&1; echo "hit rc=$?"; cat gpurun_out/hit.txt
COMBOS=128/48 PDS=0 UCS=16,32,64,0 timeout 900 python tools/pipe_probe.py 4 16 > gpurun_out/pipe_probe3.txt 2>&1; echo "pipe rc=$?"; cat gpurun_out/pipe_probe3.txt
