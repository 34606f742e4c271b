import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, gbs_inputs as G, paper_2108_01622_b200 as L
rng = G.rng_for(517)
k = 60
A = G.pure_B(G.haar_unitary(k, rng), float(sys.argv[1]) if len(sys.argv) > 1 else 0.9)
g = G.complex_gaussian(k, 0.1, rng)
fixed = np.zeros(k, np.int32)
fixed[rng.choice(np.arange(1, k), 30, replace=False)] = 1
for c in (2, 4, 8, 12, 16):
    reps = fixed.copy(); reps[0] = c
    job = L.Job(A, g, reps); job.reset(); job.run()
    v = job.finalize()[0]; s = job.abs_sum()[0]
    print(c, abs(v), s / abs(v), s / abs(v) * 2**-53)
    job.close()
