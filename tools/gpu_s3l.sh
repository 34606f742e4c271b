#!/bin/bash
# small jobs on the per-term kernel (LHAF_TREE_MIN_TERMS): the GPU suite, smoke, cfg3 / n40 bench
cd $GRAFT_REPO_ROOT
O=gpurun_out/s3l
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; cat $O/smoke.txt
timeout 2400 python -m pytest tests -q -m gpu -s --timeout=1200 -p no:cacheprovider > $O/pytest_gpu.txt 2>&1
tail -n 3 $O/pytest_gpu.txt
timeout 900 python bench.py --workload cfg3 --no-cpu > $O/bench_cfg3.json 2> $O/bench_cfg3.err
timeout 1200 python bench.py > $O/bench_cfg4.json 2> $O/bench_cfg4.err
cut -c1-400 $O/bench_cfg3.json; python -c "import json; d=json.load(open('$O/bench_cfg4.json')); print(d['value'], d['n40'], d['roofline']['frac'])"
