#!/bin/bash
# round 2, first GPU pass: the whole GPU suite (incl. the new N = 60 pins) and a short bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r02a
timeout 1500 python -m pytest tests -q -m gpu -x -s --timeout=900 > gpurun_out/r02a/pytest_gpu.txt 2>&1
tail -5 gpurun_out/r02a/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02a/smoke.txt 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/r02a/bench_cfg4.json 2> gpurun_out/r02a/bench_cfg4.err
cat gpurun_out/r02a/smoke.txt gpurun_out/r02a/bench_cfg4.json; tail -3 gpurun_out/r02a/bench_cfg4.err
