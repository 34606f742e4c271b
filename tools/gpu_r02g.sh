#!/bin/bash
# round 2 final evidence (part 2): compute-sanitizer (racecheck, synccheck, memcheck) over tiny
# launches of every kernel family, the paper's Fig. 5 on the GPU to N = 60 (ET on the tree),
# full-size values (cfg4 tree x 3 matchings, cfg5 mixed mode 3 x 3)
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02g
mkdir -p $O/sanitizer
S=/usr/local/cuda/bin/compute-sanitizer
: > $O/sanitizer/summary.txt
for tool in racecheck synccheck memcheck; do
  for c in cfg1 cfg2 cfg4_tree d48_tree et d48_v3 d48_v5 precise mg cutoff; do
    log=$O/sanitizer/${tool}_${c}.log
    timeout 600 $S --tool $tool --error-exitcode 9 python tools/sanitize_case.py $c > $log 2>&1
    rc=$?
    echo "$tool $c rc=$rc $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $log | tail -1)" >> $O/sanitizer/summary.txt
  done
done
cat $O/sanitizer/summary.txt
rm -f gpurun_out/full_values.jsonl
for p in -1 7 11; do timeout 900 python tools/full_value.py 4 0 $p > /dev/null 2>> $O/full_values.err; done
for p in -1 7 11 3; do timeout 900 python tools/full_value.py 5 0 $p 3 > /dev/null 2>> $O/full_values.err; done
cp gpurun_out/full_values.jsonl $O/full_values_final.jsonl
cat $O/full_values_final.jsonl
timeout 2400 python tests/diag/et_vs_fds.py 16 24 32 40 48 52 56 60 --inst=10 > $O/et_vs_fds_fig5.jsonl 2> $O/et_vs_fds.err
cut -c1-200 $O/et_vs_fds_fig5.jsonl
