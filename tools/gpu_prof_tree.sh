#!/bin/bash
# ncu --set full captures of each tree kernel on a cfg4 slice (several launches each, so that
# bottom and middle levels are both covered); raw CSV + source page exported, .ncu-rep removed
cd $GRAFT_REPO_ROOT
O=gpurun_out/${1:-prof_tree}
mkdir -p $O
timeout 300 python tools/tree_time.py 4 6 512 1 > $O/plain.log 2>&1 || exit 1
for spec in ${PROF_SPECS:-"tree_pivot_s:30:3" "tree_leaf2_r:3:2" "tree_bc_k:30:6"}; do
  IFS=: read name skip cnt <<< "$spec"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$name --launch-skip $skip -c $cnt \
      -o $O/p_$name -f python tools/tree_time.py 4 6 512 1 > $O/ncu_$name.log 2>&1
  ncu -i $O/p_$name.ncu-rep --page raw --csv > $O/raw_$name.csv 2>/dev/null
  ncu -i $O/p_$name.ncu-rep --page source --csv --print-source sass > $O/src_$name.csv 2>/dev/null
  python tools/ncu_summary.py $O/raw_$name.csv $name > $O/sum_$name.json 2>&1
  rm -f $O/p_$name.ncu-rep
done
cat $O/plain.log; for f in $O/sum_*.json; do python - "$f" <<'PY'
import json,sys
d=json.load(open(sys.argv[1])); d=d if isinstance(d,list) else [d]
for r in d: print(r["kernel"][:40], r["grid"], r["registers_per_thread"], "ms", round(r["duration_ms"],3), "warps%", round(r["warps_active_pct"],1), "issue%", round(r["issue_active_pct"],1), "fp64pipe%", round(r["fp64_pipe_active_pct"],1), r["top_stalls_per_issue"][:3])
PY
done
