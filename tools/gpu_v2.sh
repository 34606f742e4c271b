#!/bin/bash
# v2 bring-up: parity tests, per-config throughput for v2 and v1.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 600 python -m pytest tests -q -m gpu -x 2>&1 | tail -30 > gpurun_out/pytest_gpu.txt
timeout 300 python tools/perf_quick.py 2 > gpurun_out/perf_v2.txt 2>&1
timeout 300 python tools/perf_quick.py 1 > gpurun_out/perf_v1.txt 2>&1
cat gpurun_out/pytest_gpu.txt gpurun_out/perf_v2.txt gpurun_out/perf_v1.txt
