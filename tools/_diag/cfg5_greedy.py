"""cfg5 through the plain path: greedy matching on the doubled pattern (reps, reps) over the
2k x 2k matrix, instead of the natural pairing (i, i+k): value, kappa, time."""
import sys, os, time, json
sys.path.insert(0, os.getcwd())
import numpy as np, gbs_inputs as G, paper_2108_01622_b200 as L
cfg = G.config(5)
r = np.asarray(cfg["reps"], np.int32)
job = L.Job(cfg["A"], cfg["gamma"], np.concatenate([r, r]), mixed=False)
t0 = time.perf_counter(); job.reset(); job.run(); v = job.finalize()[0]; dt = time.perf_counter() - t0
s = job.abs_sum()[0]
print(json.dumps({"alt": os.environ.get("LHAF_V3_ALT", "0"), "value": [v.real, v.imag], "abs_sum": s, "kappa": s / abs(v), "s": dt}))
