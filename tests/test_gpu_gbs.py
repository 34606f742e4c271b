"""GPU parity of the probability layer (lhaf_gbs_prob) against the oracle (oracle.gbs_prob:
explicit A_n and brute-force / ET loop hafnian), on random lossy displaced squeezed states
(mixed path) and lossless ones (pure path = mixed path), plus the textbook photon statistics
and the sum rule through the product."""
import math

import numpy as np
import pytest

import gbs_inputs as G

pytestmark = pytest.mark.gpu


def rel(a, b):
    return abs(a - b) / max(abs(b), 1e-300)


def test_gbs_prob_vs_oracle_mixed(lib, orc):
    rng = G.rng_for(1317)
    U = G.haar_unitary(4, rng)
    sig, al = G.gaussian_state(U, [0.6, 0.4, 0.5, 0.3], [0.7, 0.9, 0.8, 0.6],
                               G.complex_gaussian(4, 0.3, rng))
    for n in ([0, 0, 0, 0], [1, 0, 0, 0], [2, 1, 0, 1], [1, 1, 1, 1], [3, 0, 2, 0], [0, 4, 0, 1]):
        want = orc.gbs_prob(sig, al, n)
        got = lib.lhaf_gbs_prob(sig, al, n)
        assert rel(got.real, want.real) <= 1e-10 and abs(got.imag) <= 1e-12 * abs(want), (n, got, want)


def test_gbs_prob_pure_equals_mixed(lib, orc):
    rng = G.rng_for(1326)
    U = G.haar_unitary(5, rng)
    sig, al = G.gaussian_state(U, [0.5, 0.7, 0.3, 0.6, 0.4], 1.0, G.complex_gaussian(5, 0.25, rng))
    for n in ([1, 0, 2, 0, 1], [2, 2, 0, 1, 1], [0, 3, 0, 0, 2], [1, 1, 1, 1, 0]):
        mixed = lib.lhaf_gbs_prob(sig, al, n)
        pure = lib.lhaf_gbs_prob(sig, al, n, pure=True)
        want = orc.gbs_prob(sig, al, n)
        assert rel(pure.real, want.real) <= 1e-10 and rel(mixed.real, want.real) <= 1e-10, (n, pure, mixed, want)


def test_gbs_prob_textbook_statistics(lib):
    one = np.eye(1, dtype=complex)
    r = 0.9
    sig, al = G.gaussian_state(one, [r])
    t = math.tanh(r)
    for k in range(0, 12):   # up to 22 photons, pure path d = 22
        want = t ** (2 * k) * math.factorial(2 * k) / (4 ** k * math.factorial(k) ** 2 * math.cosh(r))
        assert rel(lib.lhaf_gbs_prob(sig, al, [2 * k], pure=True).real, want) <= 1e-12
        assert abs(lib.lhaf_gbs_prob(sig, al, [2 * k + 1]).real) <= 1e-15
    b = 1.3 + 0.4j
    sig, al = G.gaussian_state(one, [0.0], beta=[b])
    for n in range(0, 20):
        want = math.exp(-abs(b) ** 2) * abs(b) ** (2 * n) / math.factorial(n)
        assert rel(lib.lhaf_gbs_prob(sig, al, [n]).real, want) <= 1e-12


def test_gbs_sum_rule(lib, orc):
    # 3 modes, weak squeezing, loss and displacement: the probabilities over |n| <= 6 sum to
    # 1 minus the tail (P:317 normalisation; the tail beyond |n| = 6 is ~1.1e-5), and the
    # partial sum equals the oracle's (explicit A_n, brute force) over the same patterns
    rng = G.rng_for(1555)
    U = G.haar_unitary(3, rng)
    sig, al = G.gaussian_state(U, [0.2, 0.15, 0.25], [0.9, 0.8, 0.85], [0.1, 0.1j, -0.05])
    tot = 0.0
    tot_orc = 0.0
    for a in range(7):
        for b in range(7 - a):
            for c in range(7 - a - b):
                tot += lib.lhaf_gbs_prob(sig, al, [a, b, c]).real
                tot_orc += orc.gbs_prob(sig, al, [a, b, c]).real
    assert 1.0 - 2e-5 < tot < 1.0, tot
    assert abs(tot - tot_orc) <= 1e-12, (tot, tot_orc)



def test_ips_prob_vs_oracle(lib, orc):
    rng = G.rng_for(1560)
    U = G.haar_unitary(4, rng)
    B = G.pure_B(U, 0.6)
    al = G.complex_gaussian(4, 0.4, rng)
    for n in ([0, 0, 0, 0], [1, 0, 0, 0], [2, 1, 0, 1], [1, 1, 1, 1], [3, 0, 2, 0], [0, 4, 0, 1]):
        want = orc.ips_prob(B, al, n)
        assert rel(lib.lhaf_ips_prob(B, al, n), want) <= 1e-10, n
    # sum rule through the product on 2 modes
    B2 = G.random_symmetric(2, rng, 0.3)
    a2 = G.complex_gaussian(2, 0.3, rng)
    tot = sum(lib.lhaf_ips_prob(B2, a2, [i, j]) for i in range(11) for j in range(11) if i + j <= 10)
    assert 1.0 - 1e-5 < tot <= 1.0 + 1e-12, tot   # tail beyond |n| = 10: 2.8e-6


def test_gbs_prob_state_vs_oracle_and_closed_forms(lib, orc):
    # (U, r, eta, beta) -> P(n) in one product call, against the oracle's
    # gbs_prob on the independently generated state, and the squeezed-vacuum / Poisson closed forms
    rng = G.rng_for(2201)
    M = 4
    U = G.haar_unitary(M, rng)
    rs = [0.6, 0.4, 0.5, 0.3]
    eta = [0.7, 0.9, 0.8, 0.6]
    beta = G.complex_gaussian(M, 0.3, rng)
    sig, al = G.gaussian_state(U, np.array(rs), np.array(eta), beta)
    for n in ([0, 0, 0, 0], [2, 1, 0, 1], [1, 1, 1, 1], [3, 0, 2, 0]):
        want = orc.gbs_prob(sig, al, n)
        got = lib.lhaf_gbs_prob_state(U, rs, n, eta=eta, beta=beta)
        assert rel(got.real, want.real) <= 1e-10, (n, got, want)
    for n in ([1, 0, 2, 0], [2, 2, 0, 1]):  # lossless: the pure half-size path
        sig, al = G.gaussian_state(U, np.array(rs), 1.0, beta)
        assert rel(lib.lhaf_gbs_prob_state(U, rs, n, beta=beta).real, orc.gbs_prob(sig, al, n).real) <= 1e-10
    r = 0.7
    t = math.tanh(r)
    for k in range(6):
        want = t ** (2 * k) * math.factorial(2 * k) / (4 ** k * math.factorial(k) ** 2 * math.cosh(r))
        assert rel(lib.lhaf_gbs_prob_state(np.eye(1), [r], [2 * k]).real, want) <= 1e-12
    b = 0.9 - 0.4j
    for n in range(8):
        want = math.exp(-abs(b) ** 2) * abs(b) ** (2 * n) / math.factorial(n)
        assert rel(lib.lhaf_gbs_prob_state(np.eye(1), [0.0], [n], beta=[b]).real, want) <= 1e-12
