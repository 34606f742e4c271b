#!/bin/bash
# compute-sanitizer passes (one tool per process) over tiny launches of every kernel family;
# logs under gpurun_out/sanitizer/, one summary line per (tool, case) in summary.txt
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/sanitizer
S=/usr/local/cuda/bin/compute-sanitizer
: > gpurun_out/sanitizer/summary.txt
for tool in memcheck racecheck synccheck initcheck; do
  for c in cfg1 cfg2 cfg4_tree d48_tree d48_v3 d48_v5 cfg4_v3 cfg4_v5 precise mg cutoff et; do
    log=gpurun_out/sanitizer/${tool}_${c}.log
    timeout 900 $S --tool $tool --error-exitcode 9 python tools/sanitize_case.py $c > $log 2>&1
    rc=$?
    echo "$tool $c rc=$rc $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|hazard' $log | tail -1)" >> gpurun_out/sanitizer/summary.txt
  done
done
cat gpurun_out/sanitizer/summary.txt
