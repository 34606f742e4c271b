#!/bin/bash
# v3 check: parity tests, throughput, phase breakdown
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu -x --timeout=120 2>&1 | tail -15 > gpurun_out/pytest.txt
timeout 300 python tools/perf_quick.py 3 > gpurun_out/perf_v3.txt 2>&1
timeout 300 python tools/phase_timing.py run 2 4 5 > gpurun_out/phase.txt 2>&1
cat gpurun_out/pytest.txt gpurun_out/perf_v3.txt gpurun_out/phase.txt
