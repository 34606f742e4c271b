import sys, numpy as np
sys.path.insert(0, '.')
import paper_2108_01622_b200 as L, gbs_inputs as G
def telephone(N):
    t = [1, 1]
    for m in range(2, N + 1):
        t.append(t[-1] + (m - 1) * t[-2])
    return t[N]
for reps in [[6, 5, 5, 4, 4, 4, 4, 4, 4, 4, 4, 4, 4, 4], [3] * 20, [10]*6]:
    rng = G.rng_for(sum(reps) + len(reps)); k = len(reps)
    a = (rng.standard_normal(k) + 1j * rng.standard_normal(k)) * 0.6
    job = L.Job(np.outer(a, a), a, reps); job.reset(); job.run(); v = job.finalize()[0]; s = job.abs_sum()[0]
    want = telephone(sum(reps)) * np.prod(a.astype(complex) ** np.array(reps))
    print(reps[:3], 'rel err', abs(v-want)/abs(want), 'kappa', s/abs(want), 'kappa*eps', s/abs(want)*1.1e-16)
