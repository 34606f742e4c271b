#!/bin/bash
# bounds-checked build (-DLHAF_CHECK: device asserts on shared-memory extents, level-buffer
# slots; compute-sanitizer is closed on this pool) over the tree / parity / variant tests, then
# the default build's tree tests
cd $GRAFT_REPO_ROOT
O=gpurun_out/checked
mkdir -p $O
LHAF_LIB_PATH=build/variants/check.so timeout 1800 python -m pytest tests/test_gpu_tree.py tests/test_gpu_parity.py tests/test_gpu_variants.py tests/test_gpu_fullsize.py -q -p no:cacheprovider > $O/pytest_checked.txt 2>&1
tail -n 3 $O/pytest_checked.txt; grep -c "LHAF_CHECK failed" $O/pytest_checked.txt
LHAF_LIB_PATH=build/variants/check.so timeout 600 python tools/tree_time.py 4 6 64 1 > $O/checked_cfg4_slice.txt 2>&1
LHAF_LIB_PATH=build/variants/check.so timeout 600 python tools/tree_time.py 5 6 64 1 >> $O/checked_cfg4_slice.txt 2>&1
cat $O/checked_cfg4_slice.txt
timeout 900 python -m pytest tests/test_gpu_tree.py -q -p no:cacheprovider > $O/pytest_default_tree.txt 2>&1
tail -n 2 $O/pytest_default_tree.txt
