import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np, gbs_inputs as G, paper_2108_01622_b200 as L
cfg = G.config(2)
A, g, reps = cfg["A"], cfg["gamma"], cfg["reps_batch"]
L.lhaf_rpt_batch(A, g, reps[:2])
for it in range(3):
    t0 = time.perf_counter(); job = L.Job(A, g, reps); t1 = time.perf_counter()
    job.reset(); job.run(); t2 = time.perf_counter()
    v = job.finalize(); t3 = time.perf_counter(); job.close(); t4 = time.perf_counter()
    t5 = time.perf_counter(); L.lhaf_rpt_batch(A, g, reps); t6 = time.perf_counter()
    print(f"create {1e3*(t1-t0):.1f} ms run {1e3*(t2-t1):.1f} finalize {1e3*(t3-t2):.1f} close {1e3*(t4-t3):.1f} | rpt_batch {1e3*(t6-t5):.1f} ms")
