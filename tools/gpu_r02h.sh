#!/bin/bash
# round 2, session 4: HEAD evidence — smoke, pytest -m gpu, default bench line + launch list
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02h
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
cat $O/smoke.txt
timeout 2400 python -m pytest tests -q -m gpu -s --timeout=1200 -p no:cacheprovider > $O/pytest_gpu.txt 2>&1
tail -n 3 $O/pytest_gpu.txt
timeout 1200 python bench.py > $O/bench_cfg4.json 2> $O/bench_cfg4.err
cut -c1-600 $O/bench_cfg4.json
timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-n40 > $O/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg4.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-n40 > $O/ncu_launch.log 2>&1
echo done
