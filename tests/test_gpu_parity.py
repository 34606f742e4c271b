"""GPU parity: the sm_100a path (through the C-ABI of include/lhaf.h) against the CPU oracle.

Tolerances (north_star, BASELINE.json): relative error <= 1e-10 for N <= 24 photons,
<= 1e-8 for N <= 60; integer decode bit-exact (tests/test_host.py).  Where the exact value
is 0 or tiny (odd N with gamma = 0), the comparison is absolute against the oracle's own
sum |term| scale (reading C18).  Every oracle value used here is computed live by oracle/
(the paper's printed values -- the worked example of P:133-135 -- sit in tests/golden/ with
their citations and are used by the CPU pin tests).
"""
import json
import math
import os

import numpy as np
import pytest

import gbs_inputs as G

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def tol_for(N):
    return 1e-10 if N <= 24 else 1e-8


def rel(a, b):
    return abs(a - b) / max(abs(b), 1e-300)


def telephone(N):
    t = [1, 1]
    for m in range(2, N + 1):
        t.append(t[-1] + (m - 1) * t[-2])
    return t[N]


def dfact(m):
    r = 1
    while m > 1:
        r *= m
        m -= 2
    return r


def test_cfg1_vs_bruteforce(lib, orc):
    cfg = G.config(1)
    ref = orc.lhaf(cfg["A"], cfg["gamma"], cfg["reps"], method="brute")   # 12x12, 140152 matchings
    got = lib.lhaf_rpt(cfg["A"], cfg["gamma"], cfg["reps"])
    assert rel(got, ref) <= 1e-10, (got, ref)


@pytest.mark.parametrize("seed", range(24))
def test_random_small_patterns(lib, orc, seed):
    rng = G.rng_for(500 + seed)
    k = int(rng.integers(1, 9))
    N = int(rng.integers(1, 17))
    A = G.pure_B(G.haar_unitary(k, rng), 0.8) if seed % 2 else G.random_symmetric(k, rng)
    g = np.zeros(k, complex) if seed % 5 == 0 else G.complex_gaussian(k, 0.5, rng)
    reps = G.random_pattern(k, N, rng)
    ref, T, sabs = orc.lhaf_fds(A, g, reps)
    got = lib.lhaf_rpt(A, g, reps)
    if abs(ref) < 1e-6 * sabs:          # exact zero (odd N, no loops) or extreme cancellation
        assert abs(got - ref) <= 1e-12 * sabs
    else:
        assert rel(got, ref) <= 1e-10, (reps, got, ref)


@pytest.mark.parametrize("seed", range(6))
def test_mixed_small(lib, orc, seed):
    rng = G.rng_for(600 + seed)
    k = int(rng.integers(2, 6))
    U = G.haar_unitary(k, rng)
    A2 = G.lossy_squeezed_A2(U, 0.7, 0.5)
    g2 = np.zeros(2 * k, complex) if seed % 2 else G.complex_gaussian(2 * k, 0.3, rng)
    reps = G.random_pattern(k, int(rng.integers(1, 8)), rng)
    ref = orc.lhaf_mixed(A2, g2, reps)
    got = lib.lhaf_rpt_mixed(A2, g2, reps)
    assert rel(got, ref) <= tol_for(2 * sum(reps)), (reps, got, ref)


@pytest.mark.parametrize("seed", range(4))
def test_mixed_matching_search(lib, orc, seed):
    # mixed mode 3 (lhaf_rpt_mixed's default): the matching with the least estimated cancellation
    # among 16 greedy matchings of the doubled pattern (every matching gives the same
    # lhaf) -- the same value as the oracle's natural pairing and as modes 1 and 2
    rng = G.rng_for(650 + seed)
    k = int(rng.integers(3, 7))
    U = G.haar_unitary(k, rng)
    A2 = G.lossy_squeezed_A2(U, 0.8, 0.4)
    g2 = G.complex_gaussian(2 * k, 0.2, rng)
    reps = G.random_pattern(k, int(rng.integers(4, 10)), rng, max_rep=3)
    ref = orc.lhaf_mixed(A2, g2, reps)
    vals = []
    for mode in (1, 2, 3):
        job = lib.Job(A2, g2, reps, mixed=mode)
        job.reset(); job.run()
        vals.append(job.finalize()[0])
        job.close()
    for v in vals:
        assert rel(v, ref) <= tol_for(2 * sum(reps)), (reps, vals, ref)
    assert rel(lib.lhaf_rpt_mixed(A2, g2, reps), ref) <= tol_for(2 * sum(reps))


def test_cfg3_collision_heavy(lib, orc):
    cfg = G.config(3)
    ref, T, sabs = orc.lhaf_fds(cfg["A"], cfg["gamma"], cfg["reps"])   # 14400 terms, d = 16
    got = lib.lhaf_rpt(cfg["A"], cfg["gamma"], cfg["reps"])
    assert rel(got, ref) <= 1e-8, (got, ref)
    assert rel(got, ref) <= 1e-10      # measured margin: FDS kappa ~ 5e4


def test_cfg2_batch_sampled(lib, orc):
    cfg = G.config(2)
    reps = cfg["reps_batch"]
    got = lib.lhaf_rpt_batch(cfg["A"], cfg["gamma"], reps)
    assert got.shape == (4096,)
    rng = G.rng_for(77)
    for b in rng.choice(4096, 24, replace=False):
        ref = orc.lhaf(cfg["A"], cfg["gamma"], reps[b], method="et")
        assert rel(got[b], ref) <= 1e-10, (b, got[b], ref)


def test_batch_mixed_shapes(lib, orc):
    # patterns of different d / n / parity in one batch, incl. N = 0 and a single photon
    rng = G.rng_for(88)
    k = 6
    A = G.random_symmetric(k, rng)
    g = G.complex_gaussian(k, 0.7, rng)
    pats = [[0] * k, [1, 0, 0, 0, 0, 0], [2, 1, 0, 3, 0, 0], [1, 1, 1, 1, 1, 1], [5, 0, 0, 0, 0, 2],
            [1, 2, 3, 0, 1, 1], [0, 0, 0, 0, 0, 7]]
    got = lib.lhaf_rpt_batch(A, g, np.array(pats, np.int32))
    for p, v in zip(pats, got):
        ref = orc.lhaf(A, g, p)
        assert rel(v, ref) <= 1e-10, (p, v, ref)


def tree_order(pairs, eta):
    """The evaluation order of the tree variant, restated from its rule: the
    pair eliminated first (last in the list) is the one with the smallest odd eta; the others
    by descending eta (stable).  Integer bookkeeping only."""
    H = len(eta)
    odd = [h for h in range(H) if eta[h] % 2]
    root = min(odd, key=lambda h: (eta[h], h)) if odd else None
    rest = sorted([h for h in range(H) if h != root], key=lambda h: -eta[h])
    order = rest + ([root] if root is not None else [])
    return [pairs[h] for h in order], [eta[h] for h in order]


def job_order(lib, orc, job, reps, mixed):
    """The job's pair order, checked against the oracle's matching (same pairs, permuted by
    the rule above when the job runs the tree), and the oracle's (C, v) in that order."""
    reps_o = np.concatenate([reps, reps]) if mixed else reps
    pairs, eta, left = orc.matched_reps(reps_o)
    if left is not None:
        pairs, eta = pairs + [(left, -1)], eta + [1]
    if job.info.kernel == 6:
        pairs, eta = tree_order(pairs, eta)
    jp = job.plan(0)
    assert jp.pairs() == [(int(p), int(q)) for p, q in pairs] and jp.etas() == eta
    return pairs, eta, jp


@pytest.mark.parametrize("which", ["cfg4_d60", "cfg5_d48", "cfg2_d24"])
def test_per_term_parity(lib, orc, which):
    # P14: g(t) on 1024 seeded sampled t at d = 60 (cfg4), 48 (cfg5, greedy matching of the
    # doubled pattern, C11b) and 24 (a cfg2 pattern) against the oracle's explicit-power term
    # (long double), t decoded in the job's pair order (the per-term kernel, v3).  Reported:
    # median and max of |g_gpu - g_ref| / |g_ref| per term and of |g_gpu - g_ref| / max_t
    # |g_ref|; asserted: the latter <= 1e-10 for every sampled t.
    if which == "cfg4_d60":
        cfg, mixed = G.config(4), False
    elif which == "cfg5_d48":
        cfg, mixed = G.config(5), True
    else:
        c2 = G.config(2)
        cfg, mixed = dict(A=c2["A"], gamma=c2["gamma"], reps=c2["reps_batch"][0]), False
    job = lib.Job(cfg["A"], cfg["gamma"], cfg["reps"], mixed=mixed)
    pairs, eta, jp = job_order(lib, orc, job, cfg["reps"], mixed)
    C, v = orc.reduced_from_pairs(cfg["A"], cfg["gamma"], pairs)
    n = sum(eta)
    rng = G.rng_for(99)
    ts = rng.integers(0, jp.T_eval, 1024, dtype=np.uint64)
    gg = job.terms_g(ts)
    job.close()
    W = np.array([orc.decode(int(t), eta)[1] for t in ts], np.int32)
    refs = orc.fds_terms(C, v, W, n)
    scale = np.max(np.abs(refs))
    err_abs = np.abs(gg - refs)
    per_term = err_abs / np.maximum(np.abs(refs), 1e-300)
    print(f"P14 {which}: per-term rel err median {np.median(per_term):.2e} max {per_term.max():.2e}; "
          f"|err| / max|g| median {np.median(err_abs) / scale:.2e} max {err_abs.max() / scale:.2e}")
    assert err_abs.max() / scale <= 1e-10, (which, err_abs.max() / scale)


def test_determinism_and_virtual_ranks(lib):
    cfg = G.config(3)
    job = lib.Job(cfg["A"], cfg["gamma"], cfg["reps"])
    U = job.units
    job.reset(); job.run(); full = job.finalize()
    job.reset(); job.run(); again = job.finalize()
    assert full[0] == again[0]                           # bit-identical reruns
    for R in (2, 3, 8):                                   # virtual ranks on one GPU
        job.reset()
        for r in range(R):
            job.run(U * r // R, U * (r + 1) // R)
        assert job.finalize()[0] == full[0]
    job.close()


def test_edge_cases(lib, orc):
    rng = G.rng_for(1234)
    A = G.random_symmetric(3, rng)
    g = G.complex_gaussian(3, 1.0, rng)
    assert lib.lhaf_rpt(A, g, [0, 0, 0]) == 1
    assert rel(lib.lhaf_rpt(A, g, [0, 1, 0]), g[1]) <= 1e-15
    assert abs(lib.lhaf_rpt(A, np.zeros(3), [0, 1, 2])) <= 1e-13     # odd N, no loops -> 0 (|A| ~ 2)
    # diagonal of A irrelevant when reps <= 1
    A2 = A.copy()
    np.fill_diagonal(A2, 9.0 + 9j)
    assert rel(lib.lhaf_rpt(A2, g, [1, 1, 1]), lib.lhaf_rpt(A, g, [1, 1, 1])) <= 1e-13
    # N = 60 closed forms: single-mode squeezed vacuum (eta = 30) and TMSV (a = 30)
    t = 0.6 + 0.2j
    got = lib.lhaf_rpt(np.array([[t]]), np.zeros(1), [60])
    assert rel(got, dfact(59) * t ** 30) <= 1e-8
    A_t = np.array([[0, t], [t, 0]])
    got = lib.lhaf_rpt(A_t, np.zeros(2), [30, 30])
    assert rel(got, math.factorial(30) * t ** 30) <= 1e-8


RANK_ONE_PATTERNS = [[1] * 60, [2] * 30, [2, 1] * 20, [6, 5, 5, 4, 4, 4, 4, 4, 4, 4, 4, 4, 4, 4],
                     [3] * 20, [10, 10, 10, 10, 10, 10]]


@pytest.mark.parametrize("reps", RANK_ONE_PATTERNS)
def test_rank_one_N60(lib, reps):
    # P4 at N = 60: lhaf = T(N) prod a_i^{n_i}.  Parity (the north_star's 1e-8) is asserted
    # wherever the sieve's own cancellation allows FP64 to promise it: kappa * eps <= 1e-10,
    # kappa = sum|term| / |lhaf| (SURVEY 8(c) "oracle error estimate").  The heavy-collision
    # rank-one patterns reach kappa = 1e10..1e13: there the test is a labelled DIAGNOSTIC
    # (printed kappa and error, checked against the a-priori bound 4 kappa eps, not counted as
    # parity; DESIGN.md section 6 lists them as out of tolerance).
    rng = G.rng_for(sum(reps) + len(reps))
    k = len(reps)
    a = (rng.standard_normal(k) + 1j * rng.standard_normal(k)) * 0.6
    job = lib.Job(np.outer(a, a), a, reps)
    job.reset(); job.run()
    got = job.finalize()[0]
    kappa = job.abs_sum()[0] / abs(got)
    job.close()
    want = telephone(sum(reps)) * np.prod(a.astype(complex) ** np.array(reps))
    err = rel(got, want)
    parity = kappa * 2.0 ** -53 <= 1e-10
    print(f"rank-one N=60 reps={reps[:4]}..: kappa {kappa:.2e} rel err {err:.2e} "
          f"{'PARITY (1e-8 asserted)' if parity else 'DIAGNOSTIC (kappa*eps > 1e-10)'}")
    if parity:
        assert err <= 1e-8, (reps, err, kappa)
    else:
        assert err <= 4 * kappa * 2.0 ** -53, (reps, err, kappa)


def test_errors(lib):
    A = np.array([[1.0, 2.0], [3.0, 1.0]], complex)
    with pytest.raises(lib.LhafError) as e:
        lib.lhaf_rpt(A, np.ones(2), [1, 1])
    assert e.value.status == 2
    with pytest.raises(lib.LhafError) as e:
        lib.lhaf_rpt(np.eye(2), np.ones(2), [1, -1])
    assert e.value.status == 1
    with pytest.raises(lib.LhafError) as e:
        lib.lhaf_rpt(np.eye(130), np.ones(130), np.ones(130, np.int32))   # d = 130 > 64
    assert e.value.status == 3


@pytest.mark.parametrize("variant", [1, 3, 5])
def test_kernel_variants_agree_with_oracle(lib, orc, variant):
    # every kernel variant (v1 Householder baseline, v3, v5) on loop and
    # loop-free patterns with collisions, odd N (phantom) and a mixed-state pattern
    rng = G.rng_for(4242)
    k = 7
    A = G.pure_B(G.haar_unitary(k, rng), 0.85)
    g = G.complex_gaussian(k, 0.4, rng)
    cases = [([2, 1, 0, 3, 1, 0, 2], g), ([1, 1, 1, 1, 1, 1, 1], g), ([3, 0, 2, 0, 0, 1, 1], np.zeros(k)),
             ([0, 4, 0, 0, 0, 0, 1], g)]
    lib.lhaf_set_kernel(variant)
    try:
        for reps, gg in cases:
            ref = orc.lhaf(A, gg, reps)
            got = lib.lhaf_rpt(A, gg, reps)
            if abs(ref) == 0.0:   # odd N without loops: exactly 0, rounding-level output
                assert abs(got) <= 1e-14, (variant, reps, got)
            else:
                assert rel(got, ref) <= 1e-10, (variant, reps, got, ref)
        U = G.haar_unitary(4, rng)
        A2 = G.lossy_squeezed_A2(U, 0.6, 0.7)
        g2 = G.complex_gaussian(8, 0.2, rng)
        ref = orc.lhaf_mixed(A2, g2, [2, 1, 0, 2])
        assert rel(lib.lhaf_rpt_mixed(A2, g2, [2, 1, 0, 2]), ref) <= 1e-10
    finally:
        lib.lhaf_set_kernel(0)


def test_batch_mixing_dims_and_loop_flags(lib, orc):
    # one job whose patterns span reduced dimensions 2..44 and both loop flags: the kernel is
    # instantiated for the largest bordered size and every smaller pattern runs padded
    rng = G.rng_for(777)
    k = 24
    A = G.pure_B(G.haar_unitary(k, rng), 0.8)
    gam = np.stack([G.complex_gaussian(k, 0.3, rng) for _ in range(6)])
    gam[1] = 0.0
    gam[4] = 0.0
    pats = np.zeros((6, k), np.int32)
    pats[0, :2] = 1                      # d = 2
    pats[1, :6] = [2, 2, 1, 1, 0, 2]     # no loops, collisions
    pats[2, :10] = 1                     # d = 10
    pats[3, :5] = [3, 1, 1, 2, 1]
    pats[4, :16] = 1                     # no loops, d = 16
    pats[5, :22] = 1                     # d = 22 (+1 border)
    got = lib.lhaf_rpt_batch(A, gam, pats, gamma_per_pattern=True)
    for b in range(6):
        ref = orc.lhaf(A, gam[b], pats[b])
        assert rel(got[b], ref) <= 1e-10, (b, got[b], ref)


def test_block_diagonal_N40(lib, orc):
    # Fig. 5 protocol at N = 40 through the full sieve (2^19 evaluated terms, d = 40):
    # lhaf(A1 (+) A2) = lhaf(A1) lhaf(A2), rows/cols permuted so pairs straddle the blocks
    rng = G.rng_for(510)
    m = 20
    A1 = G.random_symmetric(m, rng, 0.5)
    A2 = G.random_symmetric(m, rng, 0.5)
    g1 = G.complex_gaussian(m, 0.5, rng)
    g2 = G.complex_gaussian(m, 0.5, rng)
    Z = np.zeros((m, m), complex)
    A = np.block([[A1, Z], [Z, A2]])
    g = np.concatenate([g1, g2])
    perm = rng.permutation(2 * m)
    Ap = A[np.ix_(perm, perm)]
    gp = g[perm]
    one = np.ones(m, np.int32)
    want = orc.lhaf(A1, g1, one, method="et") * orc.lhaf(A2, g2, one, method="et")
    got = lib.lhaf_rpt(Ap, gp, np.ones(2 * m, np.int32))
    assert rel(got, want) <= 1e-8, (got, want)


@pytest.mark.parametrize("mult", [[2, 1, 2, 1, 2, 1, 2, 1, 1, 1], [3, 2, 3, 1, 2, 2, 3, 2],
                                  [1] * 12, [2, 1, 1, 2, 1, 1, 1, 1, 2]])
def test_pure_mixed_factorisation_full_size(lib, mult):
    # P:104-107 / P:332 at config-5 scale (pure limit eta = 1, m = 100): lhaf_mixed(B (+) B*)
    # over the doubled pattern equals |lhaf(B, 0, n)|^2.  Parity (1e-8) is asserted where
    # kappa * eps <= 1e-10 (kappa = sum|term| / |lhaf| of the mixed sieve); heavier
    # cancellation makes the case a labelled DIAGNOSTIC (a-priori bound 64 kappa eps only).
    rng = G.rng_for(1005)
    U = G.haar_unitary(100, rng)
    A2 = G.lossy_squeezed_A2(U, 0.9, 1.0)
    B = G.pure_B(U, 0.9)
    reps = np.zeros(100, np.int32)
    reps[rng.choice(100, len(mult), replace=False)] = mult
    job = lib.Job(A2, np.zeros(200), reps, mixed=True)
    job.reset(); job.run()
    mixed = job.finalize()[0]
    kappa = job.abs_sum()[0] / abs(mixed)
    job.close()
    pure = lib.lhaf_rpt(B, np.zeros(100), reps)
    err = rel(mixed, abs(pure) ** 2)
    parity = kappa * 2.0 ** -53 <= 1e-10
    print(f"pure/mixed factorisation mult={mult}: kappa {kappa:.2e} rel err {err:.2e} "
          f"{'PARITY (1e-8 asserted)' if parity else 'DIAGNOSTIC (kappa*eps > 1e-10)'}")
    if parity:
        assert err <= 1e-8, (mult, err, kappa)
    else:
        assert err <= 64 * kappa * 2.0 ** -53, (mult, err, kappa)


def test_cutoff_batched_chain_rule(lib, orc):
    # App. B.5: one mode takes 0..n_cut with the others fixed; every value equals
    # the individually computed lhaf (oracle), including odd counts (phantom) and n = 0
    rng = G.rng_for(523)
    k = 8
    A = G.pure_B(G.haar_unitary(k, rng), 0.8)
    g = G.complex_gaussian(k, 0.3, rng)
    fixed = np.array([1, 2, 0, 1, 0, 1, 0, 0], np.int32)
    vals = lib.lhaf_rpt_cutoff(A, g, fixed, 2, 8)
    assert vals.shape == (9,)
    for j in range(9):
        reps = fixed.copy()
        reps[2] = j
        ref = orc.lhaf(A, g, reps)
        assert rel(vals[j], ref) <= 1e-10, (j, vals[j], ref)
    # n_cut = 0 equals the plain call; bad arguments are rejected
    assert rel(lib.lhaf_rpt_cutoff(A, g, fixed, 2, 0)[0], lib.lhaf_rpt(A, g, fixed)) <= 1e-15
    with pytest.raises(lib.LhafError):
        lib.lhaf_rpt_cutoff(A, g, fixed, k, 3)


@pytest.mark.parametrize("fixed,mode,n_cut,loops", [
    ([1, 2, 0, 1, 0, 1, 0, 0], 2, 9, True),     # odd N_f: the leftover photon pairs with mode 2
    ([2, 0, 1, 1, 0, 0, 2, 0], 5, 12, True),    # even N_f: the odd counts get a phantom pair
    ([1, 1, 0, 1, 0, 0, 0, 1], 0, 10, False),   # no loops: odd totals vanish
    ([0] * 8, 3, 7, True),                      # nothing fixed: single-mode counts 0..7
])
def test_cutoff_shared_vs_oracle(lib, orc, fixed, mode, n_cut, loops):
    # App. B.5 shared evaluation (one reduction per (fixed term, w_b) serving every count)
    # against the oracle for each count, and against the per-count sieves
    rng = G.rng_for(5230 + n_cut)
    k = 8
    A = G.pure_B(G.haar_unitary(k, rng), 0.75)
    g = G.complex_gaussian(k, 0.35, rng) if loops else np.zeros(k, complex)
    fixed = np.array(fixed, np.int32)
    vals = lib.lhaf_rpt_cutoff(A, g, fixed, mode, n_cut)
    os.environ["LHAF_CUTOFF_SEPARATE"] = "1"
    try:
        sep = lib.lhaf_rpt_cutoff(A, g, fixed, mode, n_cut)
    finally:
        del os.environ["LHAF_CUTOFF_SEPARATE"]
    for c in range(n_cut + 1):
        reps = fixed.copy()
        reps[mode] = c
        ref = orc.lhaf(A, g, reps)
        if abs(ref) == 0.0:
            assert abs(vals[c]) <= 1e-13 * max(1.0, max(abs(x) for x in sep)), (c, vals[c])
            continue
        assert rel(vals[c], ref) <= 1e-10, (c, vals[c], ref)
        assert rel(vals[c], sep[c]) <= 1e-11, (c, vals[c], sep[c])


def test_et_inclusion_exclusion_vs_oracle(lib, orc):
    # the same loop hafnian by inclusion/exclusion over pair copies
    # (P:403-415), with repeats, odd N (phantom), no loops, and against the sieve at N = 32
    rng = G.rng_for(403)
    k = 7
    A = G.random_symmetric(k, rng, 0.6)
    g = G.complex_gaussian(k, 0.5, rng)
    for reps in ([2, 1, 0, 3, 0, 1, 0], [1, 1, 1, 1, 1, 0, 0], [4, 0, 0, 0, 0, 0, 3], [0, 2, 2, 0, 1, 0, 2]):
        ref = orc.lhaf(A, g, reps)
        assert rel(lib.lhaf_rpt_et(A, g, reps), ref) <= 1e-10, reps
    assert abs(lib.lhaf_rpt_et(A, np.zeros(k), [1, 1, 1, 0, 0, 0, 0])) <= 1e-14   # odd N, no loops
    cfg = G.config(1)
    assert rel(lib.lhaf_rpt_et(cfg["A"], cfg["gamma"], cfg["reps"]),
               orc.lhaf(cfg["A"], cfg["gamma"], cfg["reps"], method="brute")) <= 1e-10
    m = 32
    A2 = G.random_symmetric(m, rng, 0.4)
    g2 = G.complex_gaussian(m, 0.4, rng)
    one = np.ones(m, np.int32)
    assert rel(lib.lhaf_rpt_et(A2, g2, one), lib.lhaf_rpt(A2, g2, one)) <= 1e-9


@pytest.mark.parametrize("c,last", [(4, True), (4, False), (5, True), (5, False)])
def test_full_size_sieve_unit_vs_oracle(lib, orc, c, last):
    # The bench's own launch (the default path: the tree's level kernels, work-unit layout and
    # finalize) at the BASELINE config's full size, on one work unit: 2^{1-n} times the
    # oracle's long-double sum of the same terms (halving C6).  A unit is a contiguous
    # range of T_eval / units terms in the job's pair order (for the tree: one subtree, the
    # top digits fixed).  Tolerance: 1e-12 of the unit's sum |term|.  cfg5 (mixed) is planned
    # by the greedy matching of the doubled pattern (C11b).
    cfg = G.config(c)
    job = lib.Job(cfg["A"], cfg["gamma"], cfg["reps"], mixed=cfg["mixed"])
    pairs, eta, jp = job_order(lib, orc, job, cfg["reps"], cfg["mixed"])
    U = job.units
    chunk = jp.T_eval // U
    assert chunk * U == jp.T_eval
    u = U - 1 if last else 0
    t0, t1 = u * chunk, (u + 1) * chunk
    job.reset()
    job.run(u, u + 1)
    got = job.finalize()[0]
    sabs = job.abs_sum()[0]
    job.close()
    C, v = orc.reduced_from_pairs(cfg["A"], cfg["gamma"], pairs)
    n = sum(eta)
    s, oabs = orc.fds_sum(C, v, eta, n, t0, t1)
    want = s * 2.0 ** (1 - n)
    assert abs(sabs - oabs * 2.0 ** (1 - n)) <= 1e-10 * sabs
    assert abs(got - want) <= 1e-12 * sabs, (c, u, got, want, sabs)


def test_cutoff_limits_single_mode_closed_form(lib):
    # one photon-number-resolved mode alone: lhaf of c photons with pair weight a and loop g is
    # sum_m C(c, 2m) (2m-1)!! a^m g^(c-2m) (all matchings of c copies: m pairs, c-2m loops).
    # n_cut = 63 is the largest shared evaluation (eta_b = 31: one lane per count), n_cut = 64
    # falls back to per-count sieves; both must give the closed form for the low counts.
    k = 3
    A = np.zeros((k, k), complex)
    A[1, 1] = 0.45 - 0.2j
    g = np.array([0.0, 0.3 + 0.1j, 0.0])
    fixed = np.zeros(k, np.int32)

    def closed(c):
        a, gg = A[1, 1], g[1]
        return sum(math.comb(c, 2 * m) * dfact(2 * m - 1) * a ** m * gg ** (c - 2 * m) for m in range(c // 2 + 1))

    for n_cut in (63, 64):
        vals = lib.lhaf_rpt_cutoff(A, g, fixed, 1, n_cut)
        assert vals.shape == (n_cut + 1,)
        for c in range(17):
            assert rel(vals[c], closed(c)) <= 1e-9, (n_cut, c, vals[c], closed(c))


def test_multigamma_vs_oracle(lib, orc):
    # one pattern, several loop vectors incl. gamma = 0 -- the shared cubic
    # step (FLAG_MG: one reduction per term, loop vectors carried as inert rows/columns) against
    # the oracle and against the separate evaluation of each loop vector
    rng = G.rng_for(388)
    k = 6
    A = G.random_symmetric(k, rng, 0.6)
    gs = np.stack([G.complex_gaussian(k, 0.5, rng) for _ in range(4)] + [np.zeros(k, complex)])
    for reps in ([2, 1, 0, 1, 3, 1], [1, 1, 1, 1, 1, 0], [0, 3, 0, 2, 0, 0]):
        vals = lib.lhaf_rpt_multigamma(A, gs, reps)
        assert vals.shape == (5,)
        os.environ["LHAF_MULTIGAMMA_SEPARATE"] = "1"
        try:
            sep = lib.lhaf_rpt_multigamma(A, gs, reps)
        finally:
            del os.environ["LHAF_MULTIGAMMA_SEPARATE"]
        for g, v, w in zip(gs, vals, sep):
            ref = orc.lhaf(A, g, reps)
            if abs(ref) == 0.0:
                assert abs(v) <= 1e-14
                continue
            assert rel(v, ref) <= 1e-10, (reps, v, ref)
            assert rel(v, w) <= 1e-12, (reps, v, w)


def test_multigamma_shared_full_width(lib, orc):
    # d = 24 (a cfg2 pattern) with G = 16 loop vectors: d + G = 40 columns in the tile, every
    # compaction phase; sampled against the oracle's ET
    c2 = G.config(2)
    rng = G.rng_for(389)
    gs = np.stack([G.complex_gaussian(50, 0.2, rng) for _ in range(16)])
    reps = c2["reps_batch"][0]
    vals = lib.lhaf_rpt_multigamma(c2["A"], gs, reps)
    for g in (0, 7, 15):
        ref = orc.lhaf(c2["A"], gs[g], reps, method="et")
        assert rel(vals[g], ref) <= 1e-10, (g, vals[g], ref)


@pytest.mark.parametrize("reps", [[2, 2, 2, 1, 1], [4, 0, 2, 2, 1], [2, 2, 2, 2, 2]])
def test_zero_weight_deletion_v5(lib, orc, reps):
    # v5 removes zero-weight indices per term (w_h = 0 when eta_h = 2 k_h): terms of patterns
    # with even repeats run at their own size; values against the oracle, with and without loops
    rng = G.rng_for(390 + sum(reps))
    k = len(reps)
    A = G.pure_B(G.haar_unitary(k, rng), 0.8)
    lib.lhaf_set_kernel(5)
    try:
        for g in (G.complex_gaussian(k, 0.4, rng), np.zeros(k, complex)):
            ref = orc.lhaf(A, g, reps)
            got = lib.lhaf_rpt(A, g, reps)
            if abs(ref) == 0.0:
                assert abs(got) <= 1e-14
            else:
                assert rel(got, ref) <= 1e-10, (reps, got, ref)
    finally:
        lib.lhaf_set_kernel(0)


@pytest.mark.parametrize("e", [-100, -40, 60])
def test_extreme_input_scales(lib, orc, e):
    # homogeneity lhaf(4^e A, 2^e gamma) = 2^{eN} lhaf(A, gamma) at scales where the raw
    # characteristic-polynomial coefficients (~4^{e t}) or the pivots (~4^e) would leave the
    # double range: the library normalises host inputs by an exact power of two and restores the
    # scale in the finalize, so the result is the unscaled one times 2^{eN} exactly
    rng = G.rng_for(7100)
    k = 6
    A = G.pure_B(G.haar_unitary(k, rng), 0.8)
    g = G.complex_gaussian(k, 0.4, rng)
    for reps in ([2, 1, 1, 0, 1, 1], [1, 1, 1, 1, 1, 1], [3, 0, 1, 2, 0, 0]):
        N = sum(reps)
        base = lib.lhaf_rpt(A, g, reps)
        got = lib.lhaf_rpt(np.ldexp(A.real, 2 * e) + 1j * np.ldexp(A.imag, 2 * e),
                           np.ldexp(g.real, e) + 1j * np.ldexp(g.imag, e), reps)
        want = complex(np.ldexp(base.real, e * N), np.ldexp(base.imag, e * N))
        assert got == want, (e, reps, got, want)
        assert rel(base, orc.lhaf(A, g, reps)) <= 1e-10
