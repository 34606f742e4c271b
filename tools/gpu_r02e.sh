#!/bin/bash
# round 2 (session 3): confirm HEAD on the GPU (smoke, pytest -m gpu, default bench line), the
# full-size values on the tree (cfg4 / cfg5, permuted modes = independent evaluations), and the
# paper's Fig. 5 on the GPU to N = 60 (10 instances per N)
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02e
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
timeout 2400 python -m pytest tests -q -m gpu -s --timeout=1200 -p no:cacheprovider > $O/pytest_gpu.txt 2>&1
tail -3 $O/pytest_gpu.txt
timeout 1200 python bench.py > $O/bench_cfg4.json 2> $O/bench_cfg4.err
rm -f gpurun_out/full_values.jsonl
for p in -1 7 11; do timeout 900 python tools/full_value.py 4 0 $p > /dev/null 2>> $O/full_values.err; done
for m in 1 2; do for p in -1 7; do timeout 900 python tools/full_value.py 5 0 $p $m > /dev/null 2>> $O/full_values.err; done; done
cp gpurun_out/full_values.jsonl $O/full_values_tree.jsonl
timeout 3600 python tests/diag/et_vs_fds.py 16 24 32 40 48 52 56 60 --inst=10 > $O/et_vs_fds_fig5.jsonl 2> $O/et_vs_fds.err
cat $O/smoke.txt; cut -c1-700 $O/bench_cfg4.json; cat $O/full_values_tree.jsonl; cut -c1-400 $O/et_vs_fds_fig5.jsonl
