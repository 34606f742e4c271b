#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/s3c
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_tree.py tests/test_gpu_fullsize.py -q -x -p no:cacheprovider > $O/pytest_default.txt 2>&1
tail -2 $O/pytest_default.txt
LHAF_TREE_AMODE=3 timeout 900 python -m pytest tests/test_gpu_tree.py -q -x -p no:cacheprovider > $O/pytest_amode3.txt 2>&1
tail -2 $O/pytest_amode3.txt
bash tools/gpu_ab2.sh s3c base:base v6:v6 v6m0:v6:LHAF_BC_MODEL=0 v6a0:v6:LHAF_TREE_AMODE=0 v6a3:v6:LHAF_TREE_AMODE=3 v6a0m0:v6:LHAF_TREE_AMODE=0,LHAF_BC_MODEL=0 v5:v5 v4:v4
