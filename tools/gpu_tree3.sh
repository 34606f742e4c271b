#!/bin/bash
# tree variant: the per-term / full-size unit tests in the job's order, and one full ncu
# capture of a bottom-level launch of each tree kernel (cfg4 slice)
cd $GRAFT_REPO_ROOT
O=gpurun_out/t3
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -s -p no:cacheprovider -k "per_term or full_size_sieve_unit" > $O/pytest_fix.txt 2>&1
tail -3 $O/pytest_fix.txt
for k in tree_update_k:60 tree_tmat_k:60 tree_pivot_k:60 tree_leaf_k:4; do
  name=${k%%:*}; skip=${k##*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$name --launch-skip $skip -c 1 -o $O/prof_$name -f \
      python tools/tree_time.py 4 6 512 1 > $O/ncu_$name.log 2>&1
  ncu -i $O/prof_$name.ncu-rep --page raw --csv > $O/prof_${name}_raw.csv 2>/dev/null
  python tools/ncu_summary.py $O/prof_${name}_raw.csv $name > $O/sum_$name.json 2>&1
done
