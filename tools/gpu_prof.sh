#!/bin/bash
# Full ncu captures of the sieve kernel on a cfg4 slice (64-term units, 1776 units = 4 waves
# of 444 CTAs) and a cfg2 slice.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-v2}
export LHAF_MAX_UNITS=8388608
export LHAF_V3_ALT=${LHAF_V3_ALT:-0}
timeout 300 python tools/prof_run.py 4 -1776 > gpurun_out/plain_cfg4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sieve -c 1 -o gpurun_out/prof_${TAG}_cfg4 -f \
    python tools/prof_run.py 4 -1776 > gpurun_out/ncu_cfg4.log 2>&1
unset LHAF_MAX_UNITS
timeout 300 python tools/prof_run.py 2 64 > gpurun_out/plain_cfg2.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sieve -c 1 -o gpurun_out/prof_${TAG}_cfg2 -f \
    python tools/prof_run.py 2 64 > gpurun_out/ncu_cfg2.log 2>&1
tail -3 gpurun_out/plain_cfg4.log gpurun_out/plain_cfg2.log gpurun_out/ncu_cfg4.log gpurun_out/ncu_cfg2.log
