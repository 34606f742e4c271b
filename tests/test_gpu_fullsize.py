"""Full-size N = 60 parity against the oracle: the paper's own accuracy protocol.

P:139-140 (Sec. 1) claims "relative error < 10^-8 when tested up to N = 60"; the protocol is
Fig. 5's block-diagonal test (App. B.4 caption): for C = A1 (+) A2,
lhaf(C) = lhaf(A1) lhaf(A2).  Here (SURVEY 8(c) pin P10) the blocks are 30 + 30 = 60 photons,
the rows/columns of C are randomly permuted so that the sieve's pairs straddle the blocks, the
product path evaluates lhaf(C) as one d = 60 sieve (2^29 evaluated terms at E = 61 -- the
bench's cfg4 kernel instance and work-unit layout), and each factor comes from the oracle's
eigenvalue-trace tier (2^15 subsets, explicit powers in x87 long double), cross-
checked against the oracle's long-double +-1 sieve of the same block (agreement <= 1e-10, i.e.
>= 100x inside the tolerance).

Two matrix classes: iid-Gaussian blocks (Fig. 5's "random matrices", reading C18) and
Haar-GBS blocks (sub-blocks of B = U diag(tanh r) U^T, tanh r = 0.9, m = 100, loops
gamma ~ sigma 0.1 -- the cfg4 class).  Both assert the north_star's 1e-8 and print the
achieved error and the sieve's cancellation factor kappa = sum|term| / |lhaf|.
"""
import numpy as np
import pytest

import gbs_inputs as G

pytestmark = pytest.mark.gpu


def _blocks(kind, seed):
    rng = G.rng_for(seed)
    m = 30
    if kind == "gaussian":
        A1 = G.random_symmetric(m, rng, 0.5)
        A2 = G.random_symmetric(m, rng, 0.5)
        g1 = G.complex_gaussian(m, 0.5, rng)
        g2 = G.complex_gaussian(m, 0.5, rng)
    else:
        blocks = []
        for _ in range(2):
            U = G.haar_unitary(100, rng)
            B = G.pure_B(U, 0.9)
            modes = rng.choice(100, m, replace=False)
            blocks.append((B[np.ix_(modes, modes)], G.complex_gaussian(m, 0.1, rng)))
        (A1, g1), (A2, g2) = blocks
    Z = np.zeros((m, m), complex)
    A = np.block([[A1, Z], [Z, A2]])
    g = np.concatenate([g1, g2])
    perm = rng.permutation(2 * m)
    return (A1, g1, A2, g2), A[np.ix_(perm, perm)], g[perm]


@pytest.mark.parametrize("kind,seed", [("gaussian", 6001), ("haar_gbs", 6002)])
def test_block_diagonal_N60(lib, orc, kind, seed):
    (A1, g1, A2, g2), A, g = _blocks(kind, seed)
    one = np.ones(30, np.int32)
    # each factor by two independent long-double tiers -- eigenvalue-trace inclusion/exclusion
    # and the +-1 finite-difference sieve, 2^15 terms each -- whose
    # agreement (<= 1e-10 of the value: >= 100x inside the 1e-8 tolerance) is the oracle's
    # own error evidence; their a-priori bounds kappa * 2^-64 are printed alongside
    f1, s1 = orc.lhaf_et_kappa(orc.expand(A1, g1, one))
    f2, s2 = orc.lhaf_et_kappa(orc.expand(A2, g2, one))
    h1, _, a1 = orc.lhaf_fds(A1, g1, one)
    h2, _, a2 = orc.lhaf_fds(A2, g2, one)
    for f, h in ((f1, h1), (f2, h2)):
        assert abs(f - h) <= 1e-10 * abs(h), (f, h)
    want = f1 * f2
    oracle_bound = (min(s1 / abs(f1), a1 / abs(h1)) + min(s2 / abs(f2), a2 / abs(h2))) * orc.EPS_LD
    agree = max(abs(f1 - h1) / abs(h1), abs(f2 - h2) / abs(h2))
    reps = np.ones(60, np.int32)
    info = lib.lhaf_plan(reps)
    assert info.d == 60 and info.T_eval == 2 ** 29
    job = lib.Job(A, g, reps)
    job.reset()
    job.run()
    got = job.finalize()[0]
    kappa = job.abs_sum()[0] / abs(got)
    job.close()
    err = abs(got - want) / abs(want)
    print(f"P10 N=60 {kind}: lhaf = {got:.12e}, oracle = {want:.12e}, rel err {err:.2e}, "
          f"sieve kappa {kappa:.2e}, oracle ET/FDS agreement {agree:.1e}, kappa*eps_ld {oracle_bound:.1e}")
    assert err <= 1e-8, (kind, got, want, err, kappa)
