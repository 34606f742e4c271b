#!/bin/bash
# round 2, tree default: GPU suite, smoke, bench lines, the launch list of the bench command,
# DRAM traffic of a cfg4 slice (cache-control none), one full capture of the T+update kernel
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02d
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
timeout 1200 python bench.py > $O/bench_cfg4.json 2> $O/bench_cfg4.err
for w in cfg2 cfg5 cfg3 n40; do
  timeout 900 python bench.py --workload $w --no-cpu > $O/bench_$w.json 2> $O/bench_$w.err
done
timeout 600 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-n40 > $O/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg4.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-n40 > $O/ncu_launch.log 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --cache-control none \
    --clock-control none --csv --log-file $O/traffic_cfg4.csv python tools/tree_time.py 4 6 64 1 > $O/traffic.log 2>&1
python tools/traffic_sum.py $O/traffic_cfg4.csv 8388608 cfg4_slice_1024_units > $O/traffic_cfg4.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tree_bc_k --launch-skip 45 -c 1 -o $O/prof_bc -f \
    python tools/tree_time.py 4 6 512 1 > $O/ncu_bc.log 2>&1
ncu -i $O/prof_bc.ncu-rep --page raw --csv > $O/prof_bc_raw.csv 2>/dev/null
python tools/ncu_summary.py $O/prof_bc_raw.csv tree_bc_k > $O/ncu_summary_bc.json 2>&1
rm -f $O/prof_bc.ncu-rep
timeout 2400 python -m pytest tests -q -m gpu -s --timeout=1200 -p no:cacheprovider > $O/pytest_gpu.txt 2>&1
tail -3 $O/pytest_gpu.txt
cat $O/smoke.txt; cut -c1-400 $O/bench_cfg4.json
