"""Pins of the Gaussian-state probability layer (App. A).

Oracle (oracle.gbs_prob) against photon statistics fixed by quantum optics textbooks:
squeezed vacuum P(2k) = tanh^{2k} r (2k)! / (4^k k!^2 cosh r), P(odd) = 0; coherent state:
Poisson e^{-|b|^2} |b|^{2n} / n!; thermal state: geometric nbar^n / (1+nbar)^{n+1}; the sum
rule sum_n P(n) = 1 on a random 2-mode lossy displaced squeezed state.  The product's host
algebra (lhaf_gbs_matrices, no device) against the closed-form A, gamma and prefactor of the
same states."""
import math

import numpy as np
import pytest

import gbs_inputs as G


def _single(r=0.0, eta=1.0, beta=None, nbar=None):
    return G.gaussian_state(np.eye(1, dtype=complex), [r], eta, None if beta is None else [beta],
                            None if nbar is None else np.array([nbar]))


def test_oracle_squeezed_vacuum(orc):
    r = 0.7
    sig, al = _single(r)
    t = math.tanh(r)
    for n in range(0, 9):
        want = 0.0 if n % 2 else t ** n * math.factorial(n) / (4 ** (n // 2) * math.factorial(n // 2) ** 2 * math.cosh(r))
        got = orc.gbs_prob(sig, al, [n])
        assert abs(got - want) <= 1e-14, (n, got, want)


def test_oracle_coherent_poisson(orc):
    b = 0.8 - 0.6j
    sig, al = _single(beta=b)
    for n in range(0, 9):
        want = math.exp(-abs(b) ** 2) * abs(b) ** (2 * n) / math.factorial(n)
        assert abs(orc.gbs_prob(sig, al, [n]) - want) <= 1e-14


def test_oracle_thermal_geometric(orc):
    nb = 0.6
    sig, al = _single(nbar=nb)
    for n in range(0, 8):
        want = nb ** n / (1 + nb) ** (n + 1)
        assert abs(orc.gbs_prob(sig, al, [n]) - want) <= 1e-14


def test_oracle_sum_rule(orc):
    # 2 modes, weak squeezing + loss + displacement: sum over n1 + n2 <= 7 within the tail
    rng = G.rng_for(317)
    U = G.haar_unitary(2, rng)
    sig, al = G.gaussian_state(U, [0.25, 0.15], [0.9, 0.8], [0.2 + 0.1j, -0.15j])
    tot = sum(orc.gbs_prob(sig, al, [a, b]).real for a in range(8) for b in range(8) if a + b <= 7)
    assert 1.0 - 1e-5 < tot <= 1.0 + 1e-12, tot


def test_host_algebra_closed_forms(lib):
    # squeezed vacuum: A = -tanh r (I2), gamma = 0, prefactor 1/cosh r
    r = 0.55
    A, g, p = lib.lhaf_gbs_matrices(*_single(r))
    assert np.allclose(A, -math.tanh(r) * np.eye(2), atol=1e-15) and np.allclose(g, 0)
    assert abs(p - 1 / math.cosh(r)) <= 1e-15
    # coherent: A = 0, gamma = (b*, b), prefactor exp(-|b|^2)
    b = 0.3 + 0.4j
    A, g, p = lib.lhaf_gbs_matrices(*_single(beta=b))
    assert np.allclose(A, 0, atol=1e-15) and np.allclose(g, [b.conjugate(), b], atol=1e-15)
    assert abs(p - math.exp(-abs(b) ** 2)) <= 1e-15
    # thermal: A = X nbar/(1+nbar), prefactor 1/(1+nbar)
    nb = 0.4
    A, g, p = lib.lhaf_gbs_matrices(*_single(nbar=nb))
    q = nb / (1 + nb)
    assert np.allclose(A, [[0, q], [q, 0]], atol=1e-15) and abs(p - 1 / (1 + nb)) <= 1e-15


def test_host_algebra_multimode(lib):
    # lossless multimode squeezing: A = B* (+) B with B = U diag(-tanh r) U^T (P:322-334 up to
    # the block order, reading C12), prefactor prod 1/cosh r_i
    rng = G.rng_for(326)
    U = G.haar_unitary(4, rng)
    r = np.array([0.3, 0.5, 0.2, 0.7])
    A, g, p = lib.lhaf_gbs_matrices(*G.gaussian_state(U, r))
    B = (U * (-np.tanh(r))[None, :]) @ U.T
    assert np.allclose(A[:4, :4], B.conj(), atol=1e-13) and np.allclose(A[4:, 4:], B, atol=1e-13)
    assert np.allclose(A[:4, 4:], 0, atol=1e-13) and np.allclose(g, 0)
    assert abs(p - np.prod(1 / np.cosh(r))) <= 1e-14


def test_host_algebra_errors(lib):
    with pytest.raises(lib.LhafError):
        lib.lhaf_gbs_matrices(np.zeros((2, 2)) - 0.5 * np.eye(2), np.zeros(2))   # sigma_Q = 0


def test_oracle_ips_single_mode(orc):
    # one mode: n photons = singles ~ Poisson(|a|^2) plus 2 x pairs ~ Poisson(|b|^2 / 2)
    a, b = 0.7 + 0.2j, 0.9 - 0.4j
    la, lb = abs(a) ** 2, abs(b) ** 2 / 2
    for n in range(0, 10):
        want = sum(math.exp(-la) * la ** (n - 2 * m) / math.factorial(n - 2 * m)
                   * math.exp(-lb) * lb ** m / math.factorial(m) for m in range(n // 2 + 1))
        got = orc.ips_prob(np.array([[b]]), np.array([a]), [n])
        assert abs(got - want) <= 1e-14 * max(1.0, want), (n, got, want)


def test_oracle_ips_sum_rule(orc):
    rng = G.rng_for(560)
    B = G.random_symmetric(2, rng, 0.3)
    al = G.complex_gaussian(2, 0.3, rng)
    tot = sum(orc.ips_prob(B, al, [i, j]) for i in range(9) for j in range(9) if i + j <= 8)
    assert 1.0 - 2e-5 < tot <= 1.0 + 1e-12, tot   # tail beyond |n| = 8: 8.5e-6


def test_product_state_constructor(lib):
    # lhaf_gbs_state (product, host arithmetic) against the closed forms of P:301-313: a single
    # squeezed mode has sigma = [[sinh^2 r + 1/2, -cosh r sinh r], [., sinh^2 r + 1/2]]; pure
    # states have det(sigma) = 4^-M; pure loss mixes with vacuum (sigma -> eta sigma + (1-eta)/2);
    # the interferometer preserves the mean photon number tr(sigma)/2 - M/2; and it agrees with
    # the test-input generator gbs_inputs.gaussian_state (written independently) to rounding
    r = 0.8
    sig, al = lib.lhaf_gbs_state(np.eye(1), [r])
    want = np.array([[np.sinh(r) ** 2 + 0.5, -np.cosh(r) * np.sinh(r)],
                     [-np.cosh(r) * np.sinh(r), np.sinh(r) ** 2 + 0.5]])
    assert np.abs(sig - want).max() <= 1e-15 and np.abs(al).max() == 0
    sig_l, _ = lib.lhaf_gbs_state(np.eye(1), [r], eta=[0.3])
    assert np.abs(sig_l - (0.3 * want + 0.35 * np.eye(2))).max() <= 1e-15
    rng = G.rng_for(2101)
    M = 5
    U = G.haar_unitary(M, rng)
    rs = rng.uniform(0.1, 0.9, M)
    sig, al = lib.lhaf_gbs_state(U, rs, beta=G.complex_gaussian(M, 0.3, rng))
    assert abs(np.linalg.det(sig) - 4.0 ** -M) <= 1e-12 * 4.0 ** -M
    assert abs(np.trace(sig).real / 2 - M / 2 - np.sum(np.sinh(rs) ** 2)) <= 1e-12
    eta = rng.uniform(0.2, 1.0, M)
    beta = G.complex_gaussian(M, 0.4, rng)
    s1, a1 = lib.lhaf_gbs_state(U, rs, eta=eta, beta=beta)
    s2, a2 = G.gaussian_state(U, rs, eta, beta)
    assert np.abs(s1 - s2).max() <= 1e-13 and np.abs(a1 - a2).max() == 0
    with pytest.raises(lib.LhafError):
        lib.lhaf_gbs_state(2 * U, rs)                  # not unitary
    with pytest.raises(lib.LhafError):
        lib.lhaf_gbs_state(U, rs, eta=np.full(M, 1.5))  # transmission > 1
