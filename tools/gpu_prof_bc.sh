#!/bin/bash
# ncu --set full capture of tree_bc_k launches spread over the levels of a cfg4 slice
# (every 3rd launch from the unit depth down); raw CSV + SASS source page of the last one.
cd $GRAFT_REPO_ROOT
O=gpurun_out/${1:-prof_bc}
mkdir -p $O
timeout 300 python tools/tree_time.py 4 6 512 1 > $O/plain.log 2>&1 || exit 1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:tree_bc_k --launch-skip ${SKIP:-16} -c ${CNT:-16} \
    -o $O/p_bc -f python tools/tree_time.py 4 6 512 1 > $O/ncu_bc.log 2>&1
ncu -i $O/p_bc.ncu-rep --page raw --csv > $O/raw_bc.csv 2>/dev/null
ncu -i $O/p_bc.ncu-rep --page source --csv --print-source sass > $O/src_bc.csv 2>/dev/null
python tools/ncu_summary.py $O/raw_bc.csv tree_bc_k > $O/sum_bc.json 2>&1
rm -f $O/p_bc.ncu-rep
cat $O/plain.log
python - $O/sum_bc.json <<'PY'
import json,sys
d=json.load(open(sys.argv[1])); d=d if isinstance(d,list) else [d]
for r in d: print(r["grid"], r["block"], r["registers_per_thread"], "smem", r["smem_dynamic_bytes"], "ms", round(r["duration_ms"],3), "warps%", round(r["warps_active_pct"],1), "issue%", round(r["issue_active_pct"],1), "fp64pipe%", round(r["fp64_pipe_active_pct"],1), "fp64exec", round(r["fp64_pct_ncu"],3), r["top_stalls_per_issue"][:4], r["threads_per_inst"])
PY
