#!/bin/bash
# tree variant: full GPU suite, per-kernel launch list of a cfg4 slice, one full ncu capture of
# the update and leaf kernels
cd $GRAFT_REPO_ROOT
O=gpurun_out/t2
mkdir -p $O
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_cfg4_slice.csv \
    python tools/tree_time.py 4 6 512 1 > $O/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tree_update_k|tree_leaf_k|tree_tmat_k|tree_pivot_k" -c 4 -o $O/prof_tree_cfg4 -f \
    python tools/tree_time.py 4 6 512 1 > $O/ncu_full.log 2>&1
ncu -i $O/prof_tree_cfg4.ncu-rep --page raw --csv > $O/prof_tree_cfg4_raw.csv 2>/dev/null
timeout 2400 python -m pytest tests -q -m gpu -s --timeout=1200 -p no:cacheprovider > $O/pytest_gpu.txt 2>&1
tail -5 $O/pytest_gpu.txt
