#!/bin/bash
# One GPU session: tests, smoke, bench lines, launch list and one full ncu capture.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m pytest tests -q -m gpu -x 2>&1 | tail -3 > gpurun_out/pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
python bench.py --workload cfg2 --steps 5 --warmup 3 > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
python bench.py --workload cfg4 --steps 1 --warmup 1 --no-e2e > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err
python bench.py --workload cfg2 --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2.csv \
    python bench.py --workload cfg2 --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1
python tools/prof_run.py 2 16 > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sieve -c 1 -o gpurun_out/prof_v1_cfg2 -f \
    python tools/prof_run.py 2 16 > gpurun_out/ncu_full.log 2>&1
cat gpurun_out/pytest_gpu.txt gpurun_out/smoke.txt gpurun_out/bench_cfg2.json gpurun_out/bench_cfg4.json
