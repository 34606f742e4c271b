import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, gbs_inputs as G, oracle as orc, paper_2108_01622_b200 as L
orc.build()
cfg = G.config(5)
info = L.lhaf_plan(cfg["reps"], mixed=True)
C, v, eta, n = orc.reduced_system(cfg["A"], cfg["gamma"], cfg["reps"], mixed=True)
T1 = info.T_eval
ts = np.arange(T1 - 40, T1, dtype=np.uint64)
refs = []
for t in ts:
    k, w, sign, wt = orc.decode(int(t), eta)
    refs.append(orc.fds_term(C, v, w, n))
refs = np.array(refs)
for var in (1, 2, 3):
    L.lhaf_set_kernel(var)
    job = L.Job(cfg["A"], cfg["gamma"], cfg["reps"], mixed=True)
    gg = job.terms_g(ts)
    job.close()
    rel = np.abs(gg - refs) / np.abs(refs)
    print("variant", var, "max rel", rel.max(), "median", np.median(rel))
L.lhaf_set_kernel(0)
print("w of the worst:", orc.decode(int(T1 - 25), eta)[1])
