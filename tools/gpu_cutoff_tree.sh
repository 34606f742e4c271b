#!/bin/bash
# cutoff groups on the tree: tests, the cutoff benchmark against the largest single call
cd $GRAFT_REPO_ROOT
O=gpurun_out/cutoff_tree
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_tree.py tests/test_gpu_parity.py -q -x -k "cutoff" -p no:cacheprovider > $O/pytest_cutoff.txt 2>&1
tail -n 15 $O/pytest_cutoff.txt
for a in "24 20" "30 16" "36 12" "40 20"; do timeout 900 python tools/cutoff_bench.py $a >> $O/cutoff_bench.jsonl 2>>$O/cutoff_bench.err; done
python - <<'PY'
import json
for l in open('gpurun_out/cutoff_tree/cutoff_bench.jsonl'):
    d=json.loads(l); print(d['fixed_photons'], d['n_cut'], 'shared %.3f per-term %.3f separate %.3f largest %.3f ratio %.2f'%(d['shared_s'], d['shared_per_term_s'], d['separate_s'], d['largest_single_s'], d['shared_over_largest']), 'maxdiff', max(d['rel_diff_shared_per_term'][:8]))
PY
tail -3 $O/cutoff_bench.err
