#!/bin/bash
# A/B timing of alternative builds (LHAF_LIB_PATH) on the cfg4 slice and cfg5
cd $GRAFT_REPO_ROOT
for v in "$@"; do
  echo "== $v"
  LHAF_LIB_PATH=$PWD/$v timeout 300 python tools/tree_time.py 4 6 64 2 2>&1 | tail -1
  LHAF_LIB_PATH=$PWD/$v timeout 300 python tools/tree_time.py 5 6 4 2 2>&1 | tail -1
  LHAF_LIB_PATH=$PWD/$v timeout 300 python tools/tree_time.py 2 6 1 2 2>&1 | tail -2 | head -1
done
