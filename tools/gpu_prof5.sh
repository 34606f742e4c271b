#!/bin/bash
# Full ncu capture of one v5 sieve launch on a cfg4 slice (64-term units, 592 units = 2 waves)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-v5a}
export LHAF_CTAS_PER_SM=${CPS:-2}
export LHAF_MAX_UNITS=8388608
timeout 300 python tools/prof_run.py 4 -592 > gpurun_out/plain_${TAG}.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sieve -c 1 -o gpurun_out/prof_${TAG}_cfg4 -f \
    python tools/prof_run.py 4 -592 > gpurun_out/ncu_${TAG}.log 2>&1
tail -3 gpurun_out/plain_${TAG}.log gpurun_out/ncu_${TAG}.log
