#!/bin/bash
# A/B timing of library variants (build/variants/*.so via LHAF_LIB_PATH) on tree workloads, then
# the tree GPU tests on the working-tree build.  usage: tools/gpu_ab.sh OUTDIR VARIANT...
cd $GRAFT_REPO_ROOT
O=gpurun_out/$1; shift
mkdir -p $O
for v in "$@"; do
  for w in "4 6 64 3" "5 6 64 3" "40 6 1 3" "2 6 1 3"; do
    LHAF_LIB_PATH=build/variants/$v.so timeout 600 python tools/tree_time.py $w 2>&1 | sed "s/^/$v /" >> $O/ab.txt
  done
done
cat $O/ab.txt
