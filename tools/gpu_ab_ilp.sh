#!/bin/bash
# A/B of the recursion-ILP variants + per-kernel launch times of each (ncu launch list)
cd $GRAFT_REPO_ROOT
bash tools/gpu_ab2.sh ab_ilp r1:r1 r2:r2 r4:r4 r1b:r1 r2b:r2 r4b:r4
for v in r1 r2 r4; do
  LHAF_LIB_PATH=build/variants/$v.so timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
     --log-file gpurun_out/ab_ilp/launches_$v.csv python tools/tree_time.py 4 6 64 1 > /dev/null 2>&1
done
