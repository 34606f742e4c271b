#!/bin/bash
# session-3 iteration b: tree/variant tests on the working-tree build, A/B, ET debug, kappa
# search (cfg5 matchings), launch list of a cfg4 slice, profiles
cd $GRAFT_REPO_ROOT
O=gpurun_out/s3b
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_tree.py tests/test_gpu_fullsize.py tests/test_gpu_variants.py tests/test_gpu_parity.py -q -x -p no:cacheprovider > $O/pytest.txt 2>&1
tail -3 $O/pytest.txt
bash tools/gpu_ab.sh s3b base v3
timeout 300 python tools/et_debug.py 48 > $O/et_debug.txt 2>&1
cat $O/et_debug.txt
timeout 600 python tools/kappa_search.py 5 12 4096 2 > $O/kappa_cfg5.jsonl 2>&1
cut -c1-300 $O/kappa_cfg5.jsonl
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_v3_cfg4.csv \
    python tools/tree_time.py 4 6 64 2 > $O/ncu_launch.log 2>&1
timeout 1500 bash tools/gpu_prof_tree.sh s3b/prof
