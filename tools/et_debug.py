"""ET (inclusion/exclusion) on the tree vs the per-term v5 kernel and the oracle on Fig. 5
block-diagonal instances: python tools/et_debug.py N [inst]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import gbs_inputs as G
import oracle
import paper_2108_01622_b200 as L

N = int(sys.argv[1]); inst = int(sys.argv[2]) if len(sys.argv) > 2 else 0
oracle.build()
m = N // 2
rng = G.rng_for(5000 + 100 * N + inst)
A = G.random_symmetric(m, rng, 0.5); B = G.random_symmetric(m, rng, 0.5)
ga = G.complex_gaussian(m, 0.5, rng); gb = G.complex_gaussian(m, 0.5, rng)
C = np.block([[A, np.zeros((m, m))], [np.zeros((m, m)), B]]); gc = np.concatenate([ga, gb])
one = np.ones(m, np.int32)
ref = oracle.lhaf(A, ga, one, method="et") * oracle.lhaf(B, gb, one, method="et")
L.lhaf_rpt_et(C, gc, np.ones(N, np.int32)); L.lhaf_rpt(C, gc, np.ones(N, np.int32))  # pool + context warm-up
for kern in (0, 6, 5):
    L.lhaf_set_kernel(kern)
    t = time.perf_counter(); e = L.lhaf_rpt_et(C, gc, np.ones(N, np.int32)); dt = time.perf_counter() - t
    print(f"N={N} ET kernel {kern}: {e} rel err {abs(e - ref) / abs(ref):.3e}  {dt:.3f} s", flush=True)
    t = time.perf_counter(); f = L.lhaf_rpt(C, gc, np.ones(N, np.int32)); dt = time.perf_counter() - t
    print(f"N={N} FDS kernel {kern}: {f} rel err {abs(f - ref) / abs(ref):.3e}  {dt:.3f} s", flush=True)
L.lhaf_set_kernel(0)
