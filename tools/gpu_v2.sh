#!/bin/bash
# Kernel bring-up: parity tests (default kernel), per-config throughput for variants 3, 2, 1.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu -x 2>&1 | tail -30 > gpurun_out/pytest_gpu.txt
for v in 3 2; do timeout 300 python tools/perf_quick.py $v > gpurun_out/perf_v$v.txt 2>&1; done
cat gpurun_out/pytest_gpu.txt gpurun_out/perf_v3.txt gpurun_out/perf_v2.txt
