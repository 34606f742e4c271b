#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/s3f
mkdir -p $O
bash tools/gpu_ab2.sh s3f v8:v8 v9tb16:v9tb16
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_v8_cfg4.csv \
    python tools/tree_time.py 4 6 64 2 > $O/ncu_launch.log 2>&1
PROF_SPECS="tree_bc_k:60:6 tree_pivot_s:30:2 tree_leaf_r:3:2" timeout 1500 bash tools/gpu_prof_tree.sh s3f/prof
