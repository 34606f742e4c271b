#!/bin/bash
# round 2 final evidence (part 1): smoke, pytest -m gpu, bench lines of every workload and the
# reference arm, the ncu launch list of the default bench command, DRAM traffic of a cfg4 slice,
# full ncu captures of bottom-level launches of the three main tree kernels
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02f
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
cat $O/smoke.txt
timeout 2400 python -m pytest tests -q -m gpu -s --timeout=1200 -p no:cacheprovider > $O/pytest_gpu.txt 2>&1
tail -n 3 $O/pytest_gpu.txt
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
for spec in "tree_bc_k:280:1" "tree_pivot_s:280:1" "tree_leaf_r:12:1"; do
  IFS=: read name skip cnt <<< "$spec"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$name --launch-skip $skip -c $cnt \
      -o $O/p_$name -f python tools/tree_time.py 4 6 64 1 > $O/ncu_$name.log 2>&1
  ncu -i $O/p_$name.ncu-rep --page raw --csv > $O/raw_$name.csv 2>/dev/null
  python tools/ncu_summary.py $O/raw_$name.csv $name > $O/ncu_summary_$name.json 2>&1
  rm -f $O/p_$name.ncu-rep
done
for f in $O/bench_*.json; do echo $f; cut -c1-300 $f; done
