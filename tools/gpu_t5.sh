#!/bin/bash
# per-kernel launch list of a cfg4 slice and full ncu captures of bottom-level tree kernels
cd $GRAFT_REPO_ROOT
O=gpurun_out/t5
mkdir -p $O
: timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
    python tools/tree_time.py 4 6 512 1 > $O/ncu_launch.log 2>&1
for k in tree_bc_k:45 tree_pivot_r:45 tree_leaf_r:6; do
  name=${k%%:*}; skip=${k##*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$name --launch-skip $skip -c 1 -o $O/prof_$name -f \
      python tools/tree_time.py 4 6 512 1 > $O/ncu_$name.log 2>&1
  ncu -i $O/prof_$name.ncu-rep --page raw --csv > $O/prof_${name}_raw.csv 2>/dev/null
  python tools/ncu_summary.py $O/prof_${name}_raw.csv $name > $O/sum_$name.json 2>&1
  ncu -i $O/prof_$name.ncu-rep --page source --csv > $O/src_$name.csv 2>/dev/null; gzip -f $O/src_$name.csv; rm -f $O/prof_$name.ncu-rep
done
