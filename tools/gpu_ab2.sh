#!/bin/bash
# A/B timing of (library variant, environment) pairs on the tree workloads.
# usage: tools/gpu_ab2.sh OUTDIR SPEC...   SPEC = label:variant[:VAR=V,VAR=V]
cd $GRAFT_REPO_ROOT
O=gpurun_out/$1; shift
mkdir -p $O
for spec in "$@"; do
  IFS=: read label var envs <<< "$spec"
  for w in "4 6 64 3" "5 6 64 3" "40 6 1 3" "2 6 1 3"; do
    env $(echo $envs | tr ',' ' ') LHAF_LIB_PATH=build/variants/$var.so timeout 600 python tools/tree_time.py $w 2>&1 \
      | grep -v "^value" | tail -1 | sed "s/^/$label /" >> $O/ab.txt
  done
done
cat $O/ab.txt
