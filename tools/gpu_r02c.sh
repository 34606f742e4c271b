#!/bin/bash
# round 2: the paper's Fig. 5 on the GPU (10 instances per N to 56, 4 at N = 60), then the
# compute-sanitizer passes
cd $GRAFT_REPO_ROOT
O=gpurun_out/r02c
mkdir -p $O
timeout 3000 python tests/diag/et_vs_fds.py 16 24 32 40 48 52 56 --inst=10 > $O/et_vs_fds_fig5.jsonl 2> $O/et_vs_fds.err
timeout 2400 python tests/diag/et_vs_fds.py 60 --inst=4 >> $O/et_vs_fds_fig5.jsonl 2>> $O/et_vs_fds.err
bash tools/gpu_sanitize.sh > $O/sanitize.txt 2>&1
cp -r gpurun_out/sanitizer $O/ 2>/dev/null
cat $O/et_vs_fds_fig5.jsonl | cut -c1-300; cat $O/sanitize.txt | tail -45
