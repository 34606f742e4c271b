#!/bin/bash
# round 2: the GPU test suite, smoke, bench lines of every workload + the reference arm, the launch
# list of the default bench command, one full ncu capture of the sieve on a cfg4 slice, cutoff cost
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02b
mkdir -p $O
timeout 2400 python -m pytest tests -q -m gpu -s --timeout=1200 -p no:cacheprovider > $O/pytest_gpu.txt 2>&1
tail -3 $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
timeout 1200 python bench.py > $O/bench_cfg4.json 2> $O/bench_cfg4.err
for w in cfg2 cfg5 cfg3 n40; do
  timeout 900 python bench.py --workload $w --no-cpu > $O/bench_$w.json 2> $O/bench_$w.err
done
timeout 600 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-n40 > $O/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg4.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-n40 > $O/ncu_launch.log 2>&1
export LHAF_MAX_UNITS=8388608
timeout 300 python tools/prof_run.py 4 -1776 > $O/plain_prof.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:sieve -c 1 -o $O/prof_r02_cfg4 -f \
    python tools/prof_run.py 4 -1776 > $O/ncu_full.log 2>&1
unset LHAF_MAX_UNITS
ncu -i $O/prof_r02_cfg4.ncu-rep --page raw --csv > $O/prof_r02_cfg4_raw.csv 2>/dev/null
python tools/ncu_summary.py $O/prof_r02_cfg4_raw.csv v3_cfg4_slice > $O/ncu_summary_cfg4.json 2>&1
for a in "24 20" "30 16" "36 12"; do timeout 600 python tools/cutoff_bench.py $a >> $O/cutoff_bench.jsonl 2>>$O/cutoff_bench.err; done
cat $O/smoke.txt $O/bench_cfg4.json | cut -c1-600
