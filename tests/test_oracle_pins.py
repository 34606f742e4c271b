"""Pins of the CPU oracle (oracle/) against what the paper and the mathematics fix -- not
against itself.  CPU only (no GPU marker).  Each test names the passage / closed form.

A plausible mistake in the oracle (a dropped loop term, a wrong sign of Eq. ET_loop, a
transposed X, an off-by-one in the repeat expansion or the sieve weights) fails at least one
of: the 2x2 closed form, telephone numbers, (N-1)!!, rank-one, TMSV, coherent,
squeezed-vacuum, the GBS sum rule, the pure/mixed factorisation, block-diagonal
factorisation, and permutation invariance.
"""
import json
import math
import os

import numpy as np
import pytest

import gbs_inputs as G

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def telephone(N):  # T(N) = T(N-1) + (N-1) T(N-2): number of involutions of [N]
    t = [1, 1]
    for m in range(2, N + 1):
        t.append(t[-1] + (m - 1) * t[-2])
    return t[N]


def dfact(m):  # m!! for odd m, 1 for m <= 0
    r = 1
    while m > 1:
        r *= m
        m -= 2
    return r


def rel(a, b):
    return abs(a - b) / max(abs(b), 1e-300)


# ---------------------------------------------------------------- P1: trivial closed forms
def test_trivial_closed_forms(orc):
    a, b, d = 0.3 + 0.2j, -0.7 + 0.1j, 1.1 - 0.4j
    M2 = np.array([[a, b], [b, d]])
    for f in (orc.lhaf_brute, orc.lhaf_et):
        assert f(np.zeros((0, 0))) == 1
        assert rel(f(np.array([[a]])), a) < 1e-15
        assert rel(f(M2), b + a * d) < 1e-15          # S:184, fixes the sign reading C1
    val, T, _ = orc.lhaf_fds(np.array([[0, b], [b, 0]]), np.array([a, d]), [1, 1])
    assert T == 2 and rel(val, b + a * d) < 1e-15     # reading C4/C5 on the 2x2 case
    # f of a 2x2 block = 1/2 Tr(CX) + 1/2 v X v^T
    C = np.array([[a, b], [b, d]])
    v = np.array([a, d])
    assert rel(orc.fds_term(C, v, [1], 1), 0.5 * (2 * b) + 0.5 * (2 * a * d)) < 1e-15


def test_involution_counts(orc):
    # the brute force visits exactly the single-pair matchings: telephone numbers
    assert [orc.count_matchings(n) for n in range(13)] == [telephone(n) for n in range(13)]


# ---------------------------------------------------------------- P2/P3: all-ones matrices
@pytest.mark.parametrize("reps", [[1] * 8, [2, 1, 0, 3], [4], [3, 3], [5, 2, 2], [1] * 11, [7]])
def test_all_ones_telephone_and_double_factorial(orc, reps):
    k = len(reps)
    N = sum(reps)
    A = np.ones((k, k), complex)
    val = orc.lhaf(A, np.ones(k), reps)
    assert rel(val, telephone(N)) < 1e-14
    val0 = orc.lhaf(A, np.zeros(k), reps)
    want = dfact(N - 1) if N % 2 == 0 else 0
    assert abs(val0 - want) <= 1e-14 * max(1, want)
    f, T, _ = orc.lhaf_fds(A, np.ones(k), reps)
    assert rel(f, telephone(N)) < 1e-14


@pytest.mark.parametrize("N", [16, 24, 33])
def test_all_ones_large_N_et(orc, N):
    # eigenvalue-trace at sizes beyond brute force; exact integers T(N), (N-1)!!
    # the error must stay inside the oracle's own bound kappa * eps_ld * N^2
    A = np.ones((N, N), complex)
    np.fill_diagonal(A, 1.0)
    v, sabs = orc.lhaf_et_kappa(A)
    assert abs(v - telephone(N)) <= sabs * orc.EPS_LD * N * N
    np.fill_diagonal(A, 0.0)
    v, sabs = orc.lhaf_et_kappa(A)
    want = dfact(N - 1) if N % 2 == 0 else 0
    assert abs(v - want) <= max(sabs * orc.EPS_LD * N * N, 1e-13 * max(1, want))


# ---------------------------------------------------------------- P4: rank one
@pytest.mark.parametrize("reps", [[1, 1, 1, 1, 1, 1], [2, 1, 0, 3], [3, 2, 2, 1], [6, 1], [1] * 9])
def test_rank_one(orc, reps):
    rng = G.rng_for(42 + sum(reps))
    k = len(reps)
    a = rng.standard_normal(k) + 1j * rng.standard_normal(k)
    A = np.outer(a, a)
    N = sum(reps)
    prod = np.prod(a ** np.array(reps))
    assert rel(orc.lhaf(A, a, reps), telephone(N) * prod) < 1e-12
    want0 = dfact(N - 1) * prod if N % 2 == 0 else 0
    assert abs(orc.lhaf(A, np.zeros(k), reps) - want0) <= 1e-12 * abs(dfact(N - 1) * prod)
    f, _, _ = orc.lhaf_fds(A, a, reps)
    assert rel(f, telephone(N) * prod) < 1e-12


# ---------------------------------------------------------------- P5/P6/P7
@pytest.mark.parametrize("a_", [1, 3, 6])
def test_tmsv(orc, a_):
    t = 0.8 - 0.3j
    A = np.array([[0, t], [t, 0]])
    val = orc.lhaf(A, np.zeros(2), [a_, a_])
    assert rel(val, math.factorial(a_) * t ** a_) < 1e-13
    f, T, _ = orc.lhaf_fds(A, np.zeros(2), [a_, a_])
    assert T == a_ + 1 and rel(f, math.factorial(a_) * t ** a_) < 1e-13


def test_coherent(orc):
    rng = G.rng_for(5)
    g = rng.standard_normal(4) + 1j * rng.standard_normal(4)
    reps = [2, 0, 3, 1]
    want = np.prod(g ** np.array(reps))
    assert rel(orc.lhaf(np.zeros((4, 4)), g, reps), want) < 1e-14
    assert rel(orc.lhaf_fds(np.zeros((4, 4)), g, reps)[0], want) < 1e-14


@pytest.mark.parametrize("m", [1, 2, 5, 8])
def test_single_mode_squeezed(orc, m):
    t = 0.6 + 0.2j
    want = dfact(2 * m - 1) * t ** m
    assert rel(orc.lhaf(np.array([[t]]), np.zeros(1), [2 * m]), want) < 1e-13
    f, T, _ = orc.lhaf_fds(np.array([[t]]), np.zeros(1), [2 * m])
    assert T == m + 1 and rel(f, want) < 1e-13


def test_odd_single_mode_phantom(orc):
    # reps = (3): gamma^3 + 3 A00 gamma (reading C7)
    A00, g0 = 0.4 - 0.1j, 0.7 + 0.5j
    want = g0 ** 3 + 3 * A00 * g0
    assert rel(orc.lhaf(np.array([[A00]]), np.array([g0]), [3]), want) < 1e-14
    assert rel(orc.lhaf_fds(np.array([[A00]]), np.array([g0]), [3])[0], want) < 1e-14


# ---------------------------------------------------------------- P8: GBS sum rules
def _patterns(k, ncut):
    def rec(i, left):
        if i == k:
            yield ()
            return
        for c in range(left + 1):
            for rest in rec(i + 1, left - c):
                yield (c,) + rest
    return list(rec(0, ncut))


def test_sum_rule_mixed_lossy(orc):
    # sum_n P0 lhaf(A_n) / prod n! -> 1, lossy squeezed state of gbs_inputs
    rng = G.rng_for(9)
    k, t, eta = 3, 0.35, 0.6
    U = G.haar_unitary(k, rng)
    A2 = G.lossy_squeezed_A2(U, t, eta)
    P0 = G.lossy_vacuum_prob(t, eta, k)
    total = 0.0
    for n in _patterns(k, 8):
        val = orc.lhaf_mixed(A2, np.zeros(2 * k), list(n))
        total += P0 * val.real / np.prod([math.factorial(c) for c in n])
    assert abs(total - 1.0) < 2e-4


def test_sum_rule_pure(orc):
    # pure state (eta = 1): P(n) = P0 |lhaf(B_n)|^2 / prod n!, P0 = prod 1/cosh r
    rng = G.rng_for(10)
    k, t = 3, 0.3
    U = G.haar_unitary(k, rng)
    B = G.pure_B(U, t)
    P0 = (1.0 / np.cosh(np.arctanh(t))) ** k
    total = 0.0
    for n in _patterns(k, 10):
        val = orc.lhaf(B, np.zeros(k), list(n))
        total += P0 * abs(val) ** 2 / np.prod([math.factorial(c) for c in n])
    assert abs(total - 1.0) < 1e-4


# ---------------------------------------------------------------- P9: pure/mixed factorisation
def test_pure_mixed_factorisation(orc):
    rng = G.rng_for(11)
    k = 4
    B = G.pure_B(G.haar_unitary(k, rng), 0.7)
    g = G.complex_gaussian(k, 0.4, rng)
    A2 = np.block([[B, np.zeros((k, k))], [np.zeros((k, k)), B.conj()]])
    g2 = np.concatenate([g, g.conj()])
    for reps in ([1, 1, 1, 1], [2, 1, 0, 1], [3, 0, 1, 1]):
        mixed = orc.lhaf_mixed(A2, g2, reps)
        pure = orc.lhaf(B, g, reps)
        assert rel(mixed, abs(pure) ** 2) < 1e-12
        f, _, _ = orc.lhaf_fds(A2, g2, reps, mixed=True)
        assert rel(f, abs(pure) ** 2) < 1e-12


# ---------------------------------------------------------------- P10/P11: identities
def test_block_diagonal_and_permutation(orc):
    rng = G.rng_for(12)
    A1 = G.random_symmetric(5, rng)
    A2 = G.random_symmetric(6, rng)
    C = np.zeros((11, 11), complex)
    C[:5, :5] = A1
    C[5:, 5:] = A2
    perm = rng.permutation(11)
    Cp = C[np.ix_(perm, perm)]
    want = orc.lhaf_brute(A1) * orc.lhaf_brute(A2)
    assert rel(orc.lhaf_brute(Cp), want) < 1e-12
    assert rel(orc.lhaf_et(Cp), want) < 1e-12


def test_homogeneity_and_diagonal_irrelevance(orc):
    rng = G.rng_for(13)
    k = 7
    A = G.random_symmetric(k, rng)
    g = G.complex_gaussian(k, 1.0, rng)
    reps = [1, 0, 1, 1, 1, 1, 1]
    base = orc.lhaf(A, g, reps)
    A2 = A.copy()
    np.fill_diagonal(A2, 123.0 - 7j)                     # diagonal unused when reps <= 1
    assert rel(orc.lhaf(A2, g, reps), base) < 1e-14
    s = 2.0                                               # lhaf(s^2 A, s gamma) = s^N lhaf
    assert rel(orc.lhaf(s * s * A, s * g, reps), s ** 6 * base) < 1e-14
    reps2 = [2, 0, 1, 3, 0, 1, 1]                          # with repeats the diagonal matters
    assert rel(orc.lhaf_fds(A, g, reps2)[0], orc.lhaf(A, g, reps2)) < 1e-12
    assert rel(orc.lhaf_fds(A2, g, reps2)[0], orc.lhaf(A2, g, reps2)) < 1e-12


# ---------------------------------------------------------------- P12: matching, term counts
def test_paper_worked_example(orc):
    gold = json.load(open(os.path.join(GOLDEN, "paper_worked_example.json")))
    pairs, eta, left = orc.matched_reps(gold["reps"])
    T = int(np.prod([e + 1 for e in eta]))
    assert T == gold["terms_this_paper"] and sorted(eta, reverse=True) == gold["eta_sorted"]
    assert 2 ** (sum(gold["reps"]) // 2) == gold["terms_eigenvalue_trace"]
    assert left is None


def test_matching_examples_and_bounds(orc):
    # S:213-215 examples; bounds P:452-466; strictness rule P:485
    assert orc.matched_reps([1, 1]) == ([(0, 1)], [1], None)
    assert orc.matched_reps([4, 0]) == ([(0, 0)], [2], None)
    rng = G.rng_for(14)
    for _ in range(1000):
        k = int(rng.integers(1, 9))
        reps = [int(x) for x in rng.integers(0, 6, k)]
        pairs, eta, left = orc.matched_reps(reps)
        N = sum(reps)
        # photons accounted for exactly
        cnt = [0] * k
        for (p, q), e in zip(pairs, eta):
            cnt[p] += e
            cnt[q] += e
        if left is not None:
            cnt[left] += 1
        assert cnt == reps
        T = int(np.prod([e + 1 for e in eta])) * (2 if left is not None else 1)
        lower = np.prod([math.sqrt(c + 1) for c in reps])
        assert lower <= T * (1 + 1e-12)
        assert T <= 2 ** ((N + 1) // 2)
        if (sum(1 for c in reps if c > 1) >= 2 or any(c >= 4 for c in reps)) and N % 2 == 0:
            assert T < 2 ** (N // 2)


def test_halving_identity(orc):
    # reading C6: term(T-1-t) = term(t) (mixed-radix complement, g homogeneous of degree n)
    rng = G.rng_for(15)
    A = G.random_symmetric(4, rng)
    g = G.complex_gaussian(4, 1.0, rng)
    for reps in ([2, 1, 0, 3], [2, 2, 1, 1], [3, 3, 0, 0]):
        C, v, eta, n = orc.reduced_system(A, g, reps)
        T = int(np.prod([e + 1 for e in eta]))
        terms = []
        for t in range(T):
            _, w, sign, weight = orc.decode(t, eta)
            terms.append(sign * weight * orc.fds_term(C, v, w, n))
        for t in range(T):
            assert abs(terms[t] - terms[T - 1 - t]) <= 1e-12 * max(abs(x) for x in terms)
        full = sum(terms) / 2 ** n
        half = 2 * sum(terms[: T // 2]) / 2 ** n
        assert rel(half, full) < 1e-12 and rel(full, orc.lhaf(A, g, reps)) < 1e-12


# ---------------------------------------------------------------- P13: brute vs ET vs FDS
@pytest.mark.parametrize("seed", range(6))
def test_brute_et_fds_random(orc, seed):
    rng = G.rng_for(100 + seed)
    k = int(rng.integers(3, 7))
    A = G.random_symmetric(k, rng)
    g = G.complex_gaussian(k, 1.0, rng)
    reps = G.random_pattern(k, int(rng.integers(2, 12)), rng)
    ref = orc.lhaf(A, g, reps, method="brute")
    assert rel(orc.lhaf(A, g, reps, method="et"), ref) < 1e-11
    assert rel(orc.lhaf_fds(A, g, reps)[0], ref) < 1e-11


# ---------------------------------------------------------------- fds_range / fds_terms pins
@pytest.mark.parametrize("seed", range(5))
def test_fds_range_pinned(orc, seed):
    # fds_range (the term-range sum used as the expected value of the full-size unit tests and
    # by the CPU baseline) against brute force: the whole range times 2^{-n} is
    # lhaf; a split of [0, T) adds up; twice the first half is the whole (halving, C6); and
    # odd N / mixed pairings go through the same range routine
    rng = G.rng_for(4270 + seed)
    k = int(rng.integers(3, 7))
    A = G.random_symmetric(k, rng)
    g = G.complex_gaussian(k, 1.0, rng) if seed != 3 else np.zeros(k, complex)
    reps = G.random_pattern(k, int(rng.integers(2, 13)), rng)
    pairs, eta, left = orc.matched_reps(reps)
    eta_f = eta + ([1] if left is not None else [])
    n = sum(eta_f)
    T = int(np.prod([e + 1 for e in eta_f]))
    brute = orc.lhaf(A, g, reps, method="brute")
    s, cnt = orc.fds_range(A, g, reps, 0, T)
    assert cnt == T
    assert abs(s * 2.0 ** -n - brute) <= 1e-11 * max(abs(brute), 1e-3)
    cut = int(rng.integers(1, T)) if T > 1 else 0
    s1, c1 = orc.fds_range(A, g, reps, 0, cut)
    s2, c2 = orc.fds_range(A, g, reps, cut, T)
    assert c1 + c2 == T and abs((s1 + s2) - s) <= 1e-12 * max(abs(s), 1e-3)
    sh, _ = orc.fds_range(A, g, reps, 0, T // 2)
    assert abs(2 * sh * 2.0 ** -n - brute) <= 1e-11 * max(abs(brute), 1e-3)
    assert orc.fds_range(A, g, reps, T, T + 5)[1] == 0   # clipped at T


def test_fds_range_mixed_pinned(orc):
    # the mixed (natural pairing, reading C11) range against the brute-force lhaf of A_n
    rng = G.rng_for(4280)
    U = G.haar_unitary(3, rng)
    A2 = G.lossy_squeezed_A2(U, 0.6, 0.7)
    g2 = G.complex_gaussian(6, 0.3, rng)
    reps = np.array([2, 1, 1], np.int32)
    brute = orc.lhaf_mixed(A2, g2, reps)
    T = int(np.prod(reps + 1))
    s, cnt = orc.fds_range(A2, g2, reps, 0, T, mixed=True)
    assert cnt == T and abs(s * 2.0 ** -int(reps.sum()) - brute) <= 1e-11 * abs(brute)


def test_fds_terms_equals_fds_term(orc):
    rng = G.rng_for(4290)
    A = G.random_symmetric(6, rng)
    g = G.complex_gaussian(6, 0.7, rng)
    C, v, eta, n = orc.reduced_system(A, g, [2, 1, 0, 3, 1, 1])
    T = int(np.prod([e + 1 for e in eta]))
    W = np.array([orc.decode(t, eta)[1] for t in range(T)], np.int32)
    got = orc.fds_terms(C, v, W, n)
    for t in range(T):
        assert got[t] == orc.fds_term(C, v, W[t], n)


@pytest.mark.parametrize("seed", range(4))
def test_fds_sum_permuted_order_pinned(orc, seed):
    # fds_sum over the whole range of a PERMUTED pair order (the tree variant's order) equals
    # brute force (any order of the sieve's pairs gives the same sum), and its
    # halves add up (the term ranges the GPU's work units cover)
    rng = G.rng_for(4300 + seed)
    k = int(rng.integers(3, 7))
    A = G.random_symmetric(k, rng)
    g = G.complex_gaussian(k, 0.8, rng)
    reps = G.random_pattern(k, int(rng.integers(2, 12)), rng)
    pairs, eta, left = orc.matched_reps(reps)
    if left is not None:
        pairs, eta = pairs + [(left, -1)], eta + [1]
    perm = rng.permutation(len(pairs))
    pairs, eta = [pairs[i] for i in perm], [eta[i] for i in perm]
    C, v = orc.reduced_from_pairs(A, g, pairs)
    n = sum(eta)
    T = int(np.prod([e + 1 for e in eta]))
    s, sabs = orc.fds_sum(C, v, eta, n, 0, T)
    brute = orc.lhaf(A, g, reps, method="brute")
    assert abs(s * 2.0 ** -n - brute) <= 1e-11 * max(abs(brute), 1e-3)
    cut = T // 3
    s1, _ = orc.fds_sum(C, v, eta, n, 0, cut)
    s2, _ = orc.fds_sum(C, v, eta, n, cut, T)
    assert abs(s1 + s2 - s) <= 1e-12 * max(sabs, 1e-3)
