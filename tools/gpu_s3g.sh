#!/bin/bash
cd $GRAFT_REPO_ROOT
O=gpurun_out/s3g
mkdir -p $O
timeout 300 python tools/tree_time.py 4 6 64 1 > $O/plain.log 2>&1
for spec in "tree_bc_k:280:3" "tree_pivot_s:280:2"; do
  IFS=: read name skip cnt <<< "$spec"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$name --launch-skip $skip -c $cnt \
      -o $O/p_$name -f python tools/tree_time.py 4 6 64 1 > $O/ncu_$name.log 2>&1
  ncu -i $O/p_$name.ncu-rep --page raw --csv > $O/raw_$name.csv 2>/dev/null
  ncu -i $O/p_$name.ncu-rep --page source --csv --print-source sass > $O/src_$name.csv 2>/dev/null
  python tools/ncu_summary.py $O/raw_$name.csv $name > $O/sum_$name.json 2>&1
  rm -f $O/p_$name.ncu-rep
done
cat $O/sum_*.json | head -80
