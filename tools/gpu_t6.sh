#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/t6
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_tree.py -x -q -p no:cacheprovider > $O/pytest_tree.txt 2>&1
tail -2 $O/pytest_tree.txt
for c in 40 2 5; do timeout 300 python tools/tree_time.py $c 6 1 2; done 2>&1 | tee $O/time.txt
timeout 300 python tools/tree_time.py 4 6 64 2 2>&1 | tee -a $O/time.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
    python tools/tree_time.py 4 6 512 1 > $O/ncu_launch.log 2>&1
