#!/bin/bash
# A/B of the warp-staged leaf kernel (LHAF_TREE_LEAF=1, default) against tree_leaf_r, tree tests, ncu of the leaf
cd $GRAFT_REPO_ROOT
O=gpurun_out/leafw
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_tree.py tests/test_gpu_fullsize.py -q -m gpu -x --timeout=600 -p no:cacheprovider > $O/pytest_tree.txt 2>&1
tail -n 3 $O/pytest_tree.txt
for r in 1 2; do
for v in 0 1; do
  echo "LEAF=$v cfg4: $(LHAF_TREE_LEAF=$v timeout 300 python tools/tree_time.py 4 6 64 3 2>&1 | tail -1)" >> $O/ab.txt
  echo "LEAF=$v cfg5: $(LHAF_TREE_LEAF=$v timeout 300 python tools/tree_time.py 5 6 64 3 2>&1 | tail -1)" >> $O/ab.txt
done
done
cat $O/ab.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_leafw.csv python tools/tree_time.py 4 6 64 1 > /dev/null 2>&1
LHAF_TREE_LEAF=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_leafr.csv python tools/tree_time.py 4 6 64 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tree_leaf_w --launch-skip 4 -c 1 \
      -o $O/p_leafw -f python tools/tree_time.py 4 6 64 1 > $O/ncu_leafw.log 2>&1
ncu -i $O/p_leafw.ncu-rep --page raw --csv > $O/raw_leafw.csv 2>/dev/null
python tools/ncu_summary.py $O/raw_leafw.csv tree_leaf_w > $O/ncu_summary_leafw.json 2>&1
rm -f $O/p_leafw.ncu-rep
cat $O/ncu_summary_leafw.json | head -c 1500
