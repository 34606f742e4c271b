#!/bin/bash
# One GPU session: tests, smoke, bench lines (cfg4 default, cfg2, cfg5, cfg3), reference arm,
# launch list of the default bench and full ncu captures of the sieve kernel.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-r01}
timeout 600 python -m pytest tests -q -m gpu -x --timeout=120 2>&1 | tail -3 > gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err
timeout 600 python bench.py --workload cfg2 > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err
timeout 600 python bench.py --workload cfg5 --no-cpu > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err
timeout 300 python bench.py --workload cfg3 --no-cpu > gpurun_out/bench_cfg3.json 2> gpurun_out/bench_cfg3.err
timeout 300 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 300 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg4.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1
export LHAF_MAX_UNITS=8388608
timeout 300 python tools/prof_run.py 4 -1776 > gpurun_out/plain_cfg4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sieve -c 1 -o gpurun_out/prof_${TAG}_cfg4 -f \
    python tools/prof_run.py 4 -1776 > gpurun_out/ncu_cfg4.log 2>&1
unset LHAF_MAX_UNITS
cat gpurun_out/pytest_gpu.txt gpurun_out/smoke.txt gpurun_out/bench_cfg4.json gpurun_out/bench_cfg2.json gpurun_out/bench_cfg5.json gpurun_out/bench_cfg3.json gpurun_out/bench_ref.json
tail -3 gpurun_out/bench_cfg4.err
