import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, gbs_inputs as G, oracle as orc, paper_2108_01622_b200 as L
orc.build()
cfg = G.config(5)
info = L.lhaf_plan(cfg["reps"], mixed=True)
C, v, eta, n = orc.reduced_system(cfg["A"], cfg["gamma"], cfg["reps"], mixed=True)
job = L.Job(cfg["A"], cfg["gamma"], cfg["reps"], mixed=True)
U = job.units; chunk = max(64, -(-info.T_eval // 131072)); t0 = (U - 1) * chunk; t1 = info.T_eval
print("T_eval", info.T_eval, "chunk", chunk, "last unit", t0, t1, "n", n, info.n)
# sample terms of the last unit
ts = np.unique(np.concatenate([np.arange(t0, t0 + 40), np.arange(t1 - 40, t1), np.linspace(t0, t1 - 1, 40).astype(np.int64)])).astype(np.uint64)
gg = job.terms_g(ts)
worst = []
for t, g in zip(ts, gg):
    k, w, sign, wt = orc.decode(int(t), eta)
    ref = orc.fds_term(C, v, w, n)
    worst.append((abs(g - ref) / max(abs(ref), 1e-300), int(t), abs(ref), sign, wt))
worst.sort(reverse=True)
for x in worst[:8]: print("rel %.2e t %d |g| %.3e sign %d weight %d" % x)
# unit sum: GPU terms path vs oracle range, and vs the sieve
allt = np.arange(t0, t1, dtype=np.uint64)
ga = job.terms_g(allt)
s_terms = 0
for t, g in zip(allt, ga):
    k, w, sign, wt = orc.decode(int(t), eta)
    s_terms += sign * wt * g
s_or, c = orc.fds_range(cfg["A"], cfg["gamma"], cfg["reps"], t0, t1, mixed=True)
job.reset(); job.run(U - 1, U); s_sieve = job.finalize()[0] / 2.0 ** (1 - n)
print("sum terms_g", s_terms, "oracle", s_or, "sieve", s_sieve)
