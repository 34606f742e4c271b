#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/s3e
mkdir -p $O
bash tools/gpu_ab2.sh s3e v7:v7 v8:v8 v8s100:v8s100 v8s50:v8s50 v8m0:v8:LHAF_BC_MODEL=0
timeout 1500 python -m pytest tests/test_gpu_tree.py tests/test_gpu_fullsize.py tests/test_gpu_parity.py tests/test_gpu_variants.py -q -x -p no:cacheprovider > $O/pytest.txt 2>&1
tail -n 2 $O/pytest.txt
