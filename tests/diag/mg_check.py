"""GPU check of the gamma-batched evaluation (FLAG_MG) and of zero-weight deletion (ET):
values vs the oracle and the separate evaluation, and the cost of G loop vectors against one."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import gbs_inputs as G
import oracle as O
import paper_2108_01622_b200 as L

rel = lambda a, b: abs(a - b) / max(abs(b), 1e-300)
rng = G.rng_for(8801)
for trial in range(4):
    k = 6
    A = G.pure_B(G.haar_unitary(k, rng), 0.8) if trial % 2 else G.random_symmetric(k, rng, 0.6)
    reps = G.random_pattern(k, int(rng.integers(3, 12)), rng)
    gs = np.stack([G.complex_gaussian(k, 0.5, rng) for _ in range(5)] + [np.zeros(k, complex)])
    shared = L.lhaf_rpt_multigamma(A, gs, reps)
    os.environ["LHAF_MULTIGAMMA_SEPARATE"] = "1"
    sep = L.lhaf_rpt_multigamma(A, gs, reps)
    del os.environ["LHAF_MULTIGAMMA_SEPARATE"]
    errs = [rel(shared[g], O.lhaf(A, gs[g], reps)) for g in range(len(gs))]
    print(f"small reps={list(reps)}: max rel err vs oracle {max(errs):.2e}, vs separate {max(rel(a, b) for a, b in zip(shared, sep)):.2e}", flush=True)
c2 = G.config(2)
A, reps = c2["A"], c2["reps_batch"][0]
gs = np.stack([G.complex_gaussian(50, 0.2, rng) for _ in range(16)])
shared = L.lhaf_rpt_multigamma(A, gs, reps)
errs = [rel(shared[g], O.lhaf(A, gs[g], reps, method="et")) for g in range(0, 16, 5)]
print(f"d=24 G=16: max rel err vs oracle (4 sampled) {max(errs):.2e}", flush=True)
# cost at d = 48 (24 distinct modes of the cfg4 interferometer, 2^23 terms)
c4 = G.config(4)
modes = np.flatnonzero(c4["reps"])[:48]
reps48 = np.zeros(100, np.int32); reps48[modes] = 1
gs = np.stack([G.complex_gaussian(100, 0.1, rng) for _ in range(16)])
for Gn in (1, 4, 16):
    t0 = time.time(); v = L.lhaf_rpt_multigamma(c4["A"], gs[:Gn], reps48); t_sh = time.time() - t0
    print(f"d=48 G={Gn}: shared {t_sh:.3f} s", flush=True)
t0 = time.time(); v1 = L.lhaf_rpt(c4["A"], gs[0], reps48); t_single = time.time() - t0
os.environ["LHAF_MULTIGAMMA_SEPARATE"] = "1"
t0 = time.time(); vs = L.lhaf_rpt_multigamma(c4["A"], gs, reps48); t_sep = time.time() - t0
del os.environ["LHAF_MULTIGAMMA_SEPARATE"]
print(f"d=48: single call {t_single:.3f} s; 16 separate {t_sep:.3f} s; shared vs separate max rel {max(rel(a, b) for a, b in zip(v, vs[:len(v)])):.2e}", flush=True)
# ET with deletion vs sieve
m = 20
A1 = G.random_symmetric(2 * m, rng, 0.5); g1 = G.complex_gaussian(2 * m, 0.5, rng)
one = np.ones(2 * m, np.int32)
t0 = time.time(); f = L.lhaf_rpt(A1, g1, one); t_f = time.time() - t0
t0 = time.time(); e = L.lhaf_rpt_et(A1, g1, one); t_e = time.time() - t0
print(f"N=40: sieve {t_f:.3f} s, ET (deletion) {t_e:.3f} s, rel diff {rel(e, f):.2e}", flush=True)
