"""Tiny launches of every kernel family for compute-sanitizer (racecheck / synccheck / memcheck /
initcheck): a few 64-term work units of each instance, so that a sanitizer pass stays short.
    python tools/sanitize_case.py CASE   (cfg1 | cfg2 | d48_v3 | d48_v5 | cfg4_v3 | cfg4_v5 |
                                          precise | mg | cutoff | et | cfg4_tree | d48_tree)
(cfg1, cfg2 and et run the default path: the tree, variant 6)"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("LHAF_MAX_UNITS", "1073741824")  # 64-term units: few terms per launch
import numpy as np
import gbs_inputs as G
import paper_2108_01622_b200 as L

case = sys.argv[1]


def small_job(cfg, units=2, kernel=0, mixed=None):
    L.lhaf_set_kernel(kernel)
    reps = cfg.get("reps_batch", cfg.get("reps"))
    job = L.Job(cfg["A"], cfg["gamma"], reps[:8] if reps.ndim == 2 else reps,
                mixed=cfg["mixed"] if mixed is None else mixed)
    job.reset(); job.run(0, min(units, job.units)); v = job.finalize()
    print(case, "kernel", job.info.kernel, "units", min(units, job.units), "value", v[0])
    job.close()
    L.lhaf_set_kernel(0)


if case == "cfg1":
    c = G.config(1)
    print(case, L.lhaf_rpt(c["A"], c["gamma"], c["reps"]))
elif case == "cfg2":
    small_job(G.config(2), units=8)
elif case in ("d48_v3", "d48_v5"):
    small_job(G.config(5), kernel=3 if case.endswith("v3") else 5)
elif case == "cfg4_tree":
    small_job(G.config(4), units=2, kernel=6)
elif case == "d48_tree":
    small_job(G.config(5), units=2, kernel=6)
elif case in ("cfg4_v3", "cfg4_v5"):
    small_job(G.config(4), kernel=3 if case.endswith("v3") else 5)
elif case == "precise":
    L.lhaf_set_precision(1)
    small_job(G.config(4))
    L.lhaf_set_precision(0)
elif case == "mg":
    rng = G.rng_for(11)
    A = G.random_symmetric(8, rng, 0.5)
    gs = np.stack([G.complex_gaussian(8, 0.4, rng) for _ in range(4)])
    print(case, L.lhaf_rpt_multigamma(A, gs, [2, 1, 1, 0, 1, 1, 2, 0]))
elif case == "cutoff":
    rng = G.rng_for(12)
    A = G.pure_B(G.haar_unitary(6, rng), 0.7)
    print(case, L.lhaf_rpt_cutoff(A, G.complex_gaussian(6, 0.3, rng), np.array([1, 1, 0, 1, 0, 1], np.int32), 2, 6))
elif case == "et":
    rng = G.rng_for(13)
    A = G.random_symmetric(7, rng, 0.5)
    print(case, L.lhaf_rpt_et(A, G.complex_gaussian(7, 0.4, rng), [2, 1, 0, 3, 1, 0, 1]))
