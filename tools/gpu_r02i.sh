#!/bin/bash
# round 2, session 5: HEAD evidence — smoke, pytest -m gpu, bench lines of every workload + the
# reference arm, the launch list of the default bench command, DRAM traffic of one step
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02i
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
cat $O/smoke.txt
timeout 2400 python -m pytest tests -q -m gpu -s --timeout=1200 -p no:cacheprovider > $O/pytest_gpu.txt 2>&1
tail -n 3 $O/pytest_gpu.txt
timeout 1200 python bench.py > $O/bench_cfg4.json 2> $O/bench_cfg4.err
cut -c1-300 $O/bench_cfg4.json
for w in cfg5 cfg2 n40; do
  timeout 900 python bench.py --workload $w > $O/bench_$w.json 2> $O/bench_$w.err
  cut -c1-200 $O/bench_$w.json
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-n40 > $O/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg4.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-n40 > $O/ncu_launch.log 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none --csv \
    --log-file $O/traffic_cfg4.csv python tools/tree_time.py 4 6 64 1 > $O/ncu_traffic.log 2>&1
echo done
