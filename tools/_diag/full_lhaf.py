"""Full cfg5 loop hafnian (all work units) with the selected kernel instantiation: value,
sum |term| (kappa), wall time."""
import sys, os, time, json
sys.path.insert(0, os.getcwd())
import numpy as np, gbs_inputs as G, paper_2108_01622_b200 as L
cfg = G.config(int(sys.argv[1]) if len(sys.argv) > 1 else 5)
if len(sys.argv) > 2:
    L.lhaf_set_kernel(int(sys.argv[2]))  # 1 = v1 Householder baseline
job = L.Job(cfg["A"], cfg["gamma"], cfg["reps"], mixed=cfg["mixed"])
t0 = time.perf_counter(); job.reset(); job.run(); v = job.finalize()[0]; dt = time.perf_counter() - t0
s = job.abs_sum()[0]
print(json.dumps({"alt": os.environ.get("LHAF_V3_ALT", "0"), "kernel": job.info.kernel, "value": [v.real, v.imag], "abs_sum": s, "kappa": s / abs(v), "s": dt}))
