"""Cutoff-batched chain-rule evaluation (App. B.5): the shared path (one series per (fixed
prefix, w_b) serving every count of the batched mode; on the tree: the batched self-pair is the
leaf level) against the per-term shared kernel (LHAF_CUTOFF_PER_TERM) and per-count sieves, device-synchronous
wall time per call (each call includes its own host planning and H2D of A, gamma).  The two
paths are the same sums in a different order: they agree to ~kappa * eps per count (kappa =
sum|term| / |lhaf|, large for heavy collisions in strongly squeezed modes).
    python tools/cutoff_bench.py [n_fixed_modes] [n_cut] [tanh r]"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import gbs_inputs as G  # noqa: E402
import paper_2108_01622_b200 as L  # noqa: E402

nfix = int(sys.argv[1]) if len(sys.argv) > 1 else 24
n_cut = int(sys.argv[2]) if len(sys.argv) > 2 else 20
rng = G.rng_for(517)
k = 60
t = float(sys.argv[3]) if len(sys.argv) > 3 else 0.6
A = G.pure_B(G.haar_unitary(k, rng), t)
g = G.complex_gaussian(k, 0.1, rng)
fixed = np.zeros(k, np.int32)
fixed[rng.choice(np.arange(1, k), nfix, replace=False)] = 1
out = {"k": k, "tanh_r": t, "fixed_photons": int(fixed.sum()), "batched_mode": 0, "n_cut": n_cut}
for name, env in (("shared", None), ("shared_per_term", "LHAF_CUTOFF_PER_TERM"), ("separate", "LHAF_CUTOFF_SEPARATE")):
    if env:
        os.environ[env] = "1"
    L.lhaf_rpt_cutoff(A, g, fixed, 0, min(n_cut, 2))   # warm-up (context, module load)
    t0 = time.perf_counter()
    v = L.lhaf_rpt_cutoff(A, g, fixed, 0, n_cut)
    out[name + "_s"] = time.perf_counter() - t0
    out[name + "_values"] = [[x.real, x.imag] for x in v[:4]]
    if env:
        os.environ.pop(env, None)
    if name == "shared":
        vs = v
    else:
        out["rel_diff_" + name] = [float(abs(a - b) / max(abs(b), 1e-300)) for a, b in zip(vs, v)]
        out["abs_vals"] = [float(abs(b)) for b in v]
out["speedup"] = out["separate_s"] / out["shared_s"]
out["speedup_vs_per_term_shared"] = out["shared_per_term_s"] / out["shared_s"]
# the paper's claim: all counts in about the time of the largest single call
reps = fixed.copy()
reps[0] = n_cut
L.lhaf_rpt(A, g, reps)
t0 = time.perf_counter()
L.lhaf_rpt(A, g, reps)
out["largest_single_s"] = time.perf_counter() - t0
out["shared_over_largest"] = out["shared_s"] / out["largest_single_s"]
_, err = L.lhaf_rpt_cutoff_ex(A, g, fixed, 0, n_cut)
out["err_est"] = [float(e) for e in err]
print(json.dumps(out))
