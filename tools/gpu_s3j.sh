#!/bin/bash
# precision mode 2 (tree with double-double pivots): tests, full-size values (cfg5 mixed mode 3,
# three matchings; cfg4), and the FP64 mixed-mode-3 values with the final search (8 samples)
cd $GRAFT_REPO_ROOT
O=gpurun_out/s3j
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_tree.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -s -p no:cacheprovider > $O/pytest.txt 2>&1
tail -n 3 $O/pytest.txt; grep "N=40 blocks" $O/pytest.txt
rm -f gpurun_out/full_values.jsonl
for p in -1 7 11; do timeout 900 python tools/full_value.py 5 2 $p 3 > /dev/null 2>> $O/full_values.err; done
for p in -1 7 11; do timeout 900 python tools/full_value.py 5 0 $p 3 > /dev/null 2>> $O/full_values.err; done
for p in -1 7; do timeout 900 python tools/full_value.py 4 2 $p > /dev/null 2>> $O/full_values.err; done
cp gpurun_out/full_values.jsonl $O/full_values_dd.jsonl
cat $O/full_values_dd.jsonl; tail -3 $O/full_values.err
