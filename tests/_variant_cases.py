"""Seeded cases for tests/test_gpu_variants.py (shared by the test and its worker subprocess;
input generation only, no method arithmetic)."""
import numpy as np
import gbs_inputs as G


def cases():
    out = []
    # block-diagonal, pairs straddling the blocks (Fig. 5 protocol): N = 48 (E = 49,
    # the d = 60 instance / v4), N = 40 (E = 41), N = 24 (E = 25)
    for m, seed in ((24, 4801), (20, 4001), (12, 2401)):
        rng = G.rng_for(seed)
        A1 = G.random_symmetric(m, rng, 0.5)
        A2 = G.random_symmetric(m, rng, 0.5)
        g1 = G.complex_gaussian(m, 0.5, rng)
        g2 = G.complex_gaussian(m, 0.5, rng)
        Z = np.zeros((m, m), complex)
        A = np.block([[A1, Z], [Z, A2]])
        g = np.concatenate([g1, g2])
        perm = rng.permutation(2 * m)
        out.append(dict(A=A[np.ix_(perm, perm)], gamma=g[perm], reps=np.ones(2 * m, np.int32),
                        blocks=(A1, g1, A2, g2)))
    return out
