cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/t4
timeout 900 python -m pytest tests/test_gpu_tree.py tests/test_gpu_variants.py -x -q -p no:cacheprovider > gpurun_out/t4/pytest_tree.txt 2>&1
tail -3 gpurun_out/t4/pytest_tree.txt
for rl in 40 0; do for c in 40 2 5; do LHAF_TREE_REGL=$rl timeout 300 python tools/tree_time.py $c 6 1 2; done; LHAF_TREE_REGL=$rl timeout 300 python tools/tree_time.py 4 6 64 2; done 2>&1 | tee gpurun_out/t4/time.txt
