"""Fig. 5 of the paper on the device path: relative error of the loop hafnian of
C = A (+) B (block diagonal, random N/2 x N/2 blocks) against lhaf(A) lhaf(B), for the
finite-difference sieve (lhaf_rpt, FP64; and in precise mode up to --precise-max N) and
inclusion/exclusion (lhaf_rpt_et: on the tree an excluded pair's children copy the parent's
leading block -- the pair is deleted), with the reference product from the CPU oracle in x87 long
double (ET tier at N/2).  Device-synchronous wall time per call.  One JSON line per N.
    python tests/diag/et_vs_fds.py [N ...] [--inst=K] [--precise-max=N]"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import gbs_inputs as G  # noqa: E402
import oracle  # noqa: E402  (reference values only)
import paper_2108_01622_b200 as L  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
inst = 10
pmax = 48
for a in sys.argv[1:]:
    if a.startswith("--inst="):
        inst = int(a.split("=")[1])
    if a.startswith("--precise-max="):
        pmax = int(a.split("=")[1])
Ns = [int(a) for a in args] or [16, 24, 32, 40, 48, 52, 56, 60]
oracle.build()
L.lhaf_rpt(np.eye(2), np.ones(2), [1, 1])  # context warm-up
for N in Ns:
    m = N // 2
    rec = {"N": N, "instances": inst, "err_fds": [], "err_et": [], "err_fds_precise": [],
           "t_fds_s": 0.0, "t_et_s": 0.0, "t_fds_precise_s": 0.0}
    for i in range(inst):
        rng = G.rng_for(5000 + 100 * N + i)
        A = G.random_symmetric(m, rng, 0.5)
        B = G.random_symmetric(m, rng, 0.5)
        ga = G.complex_gaussian(m, 0.5, rng)
        gb = G.complex_gaussian(m, 0.5, rng)
        C = np.block([[A, np.zeros((m, m))], [np.zeros((m, m)), B]])
        gc = np.concatenate([ga, gb])
        one = np.ones(m, np.int32)
        ref = oracle.lhaf(A, ga, one, method="et") * oracle.lhaf(B, gb, one, method="et")
        t0 = time.perf_counter()
        f = L.lhaf_rpt(C, gc, np.ones(N, np.int32))
        t1 = time.perf_counter()
        e = L.lhaf_rpt_et(C, gc, np.ones(N, np.int32))
        t2 = time.perf_counter()
        rec["err_fds"].append(abs(f - ref) / abs(ref))
        rec["err_et"].append(abs(e - ref) / abs(ref))
        rec["t_fds_s"] += (t1 - t0) / inst
        rec["t_et_s"] += (t2 - t1) / inst
        if N <= pmax:
            L.lhaf_set_precision(1)
            t3 = time.perf_counter()
            fp = L.lhaf_rpt(C, gc, np.ones(N, np.int32))
            rec["t_fds_precise_s"] += (time.perf_counter() - t3) / inst
            L.lhaf_set_precision(0)
            rec["err_fds_precise"].append(abs(fp - ref) / abs(ref))
    rec["median_err_fds"] = float(np.median(rec["err_fds"]))
    rec["median_err_et"] = float(np.median(rec["err_et"]))
    rec["max_err_fds"] = float(np.max(rec["err_fds"]))
    if rec["err_fds_precise"]:
        rec["median_err_fds_precise"] = float(np.median(rec["err_fds_precise"]))
    print(json.dumps(rec), flush=True)
