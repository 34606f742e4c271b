#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/s3d
mkdir -p $O
bash tools/gpu_ab2.sh s3d base:base v2:v2 v7:v7 v7b:v7b v7a1:v7:LHAF_TREE_AMODE=1 v6a0:v6:LHAF_TREE_AMODE=0 v7b_a1:v7b:LHAF_TREE_AMODE=1
timeout 900 python -m pytest tests/test_gpu_tree.py tests/test_gpu_fullsize.py -q -x -p no:cacheprovider > $O/pytest_default.txt 2>&1
tail -n 2 $O/pytest_default.txt
LHAF_TREE_AMODE=3 timeout 900 python -m pytest tests/test_gpu_tree.py -q -x -p no:cacheprovider > $O/pytest_amode3.txt 2>&1
tail -n 2 $O/pytest_amode3.txt
rm -f gpurun_out/full_values.jsonl
for p in -1 7 11; do timeout 900 python tools/full_value.py 5 0 $p 3 > /dev/null 2>> $O/full_values.err; done
cp gpurun_out/full_values.jsonl $O/full_values_cfg5_mode3.jsonl
cat $O/full_values_cfg5_mode3.jsonl
