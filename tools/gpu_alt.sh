#!/bin/bash
# v3 instantiation experiment: default vs LHAF_V3_ALT=1 (more lanes per row) / 2 (R=200)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu -x 2>&1 | tail -3 > gpurun_out/pytest.txt
timeout 300 python tools/perf_quick.py 3 > gpurun_out/perf_v3.txt 2>&1
LHAF_V3_ALT=1 timeout 300 python tools/perf_quick.py 3 > gpurun_out/perf_v3alt.txt 2>&1
LHAF_V3_ALT=2 timeout 300 python tools/perf_quick.py 3 > gpurun_out/perf_v3alt2.txt 2>&1
cat gpurun_out/pytest.txt gpurun_out/perf_v3.txt gpurun_out/perf_v3alt.txt gpurun_out/perf_v3alt2.txt
