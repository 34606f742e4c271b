#!/bin/bash
# session-3 iteration: tree tests on the working-tree build, A/B of variants, ET debug, profiles
cd $GRAFT_REPO_ROOT
O=gpurun_out/s3a
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_tree.py tests/test_gpu_fullsize.py -q -x -p no:cacheprovider > $O/pytest_tree.txt 2>&1
tail -3 $O/pytest_tree.txt
bash tools/gpu_ab.sh s3a base v2
for n in 40 44 48; do timeout 300 python tools/et_debug.py $n >> $O/et_debug.txt 2>&1; done
LHAF_TREE_REGL=24 timeout 300 python tools/et_debug.py 48 >> $O/et_debug.txt 2>&1
cat $O/et_debug.txt
timeout 1500 bash tools/gpu_prof_tree.sh s3a/prof
