"""GPU parity of kernel variant 6 (the prefix-sharing tree) against the oracle,
and its work-unit invariants.

The tree evaluates the same sieve terms as the per-term kernels but shares the
Schur complements of every eliminated prefix of pairs; these tests pin it to the oracle on
the shapes where its code paths differ: collisions (several digits per level, zero weights =
deleted pairs), all-even multiplicities (no halving, FLAG_FULL), a single pair (the root is the
leaf level), odd N (phantom), loops on and off (border index), mixed states, batches whose
patterns fall into several tree shapes, and unit ranges (bit-identical results for any slicing).
Tolerances: the north_star's 1e-10 for N <= 24 (relative), absolute against sum|term| where the
exact value is 0 (reading C18).
"""
import os

import numpy as np
import pytest

import gbs_inputs as G

pytestmark = pytest.mark.gpu


def rel(a, b):
    return abs(a - b) / max(abs(b), 1e-300)


@pytest.fixture()
def tree(lib):
    lib.lhaf_set_kernel(6)
    yield lib
    lib.lhaf_set_kernel(0)


def check(got, ref, sabs, tol=1e-10):
    if abs(ref) < 1e-6 * sabs:
        assert abs(got - ref) <= 1e-12 * sabs, (got, ref, sabs)
    else:
        assert rel(got, ref) <= tol, (got, ref)


@pytest.mark.parametrize("seed", range(30))
def test_tree_random_collisions(tree, orc, seed):
    rng = G.rng_for(7000 + seed)
    k = int(rng.integers(1, 8))
    N = int(rng.integers(1, 21))
    A = G.pure_B(G.haar_unitary(k, rng), 0.8) if seed % 2 else G.random_symmetric(k, rng)
    g = np.zeros(k, complex) if seed % 3 == 0 else G.complex_gaussian(k, 0.5, rng)
    reps = G.random_pattern(k, N, rng)
    ref, T, sabs = orc.lhaf_fds(A, g, reps)
    got = tree.lhaf_rpt(A, g, reps)
    check(got, ref, sabs)


@pytest.mark.parametrize("N", list(range(2, 29, 2)) + [7, 13, 21])
def test_tree_series_length_sweep(tree, orc, N):
    # distinct modes, n = ceil(N / 2) pairs, series length L = n + 1 = 2 .. 15: every remainder
    # of tree_bc_k's product routine (chunks of TB = 8 steps + a tail of L mod 8, the block
    # triangle with fewer than TB - 1 operands when L < 8) and odd N (phantom index)
    rng = G.rng_for(7300 + N)
    A = G.pure_B(G.haar_unitary(N, rng), 0.7)
    g = G.complex_gaussian(N, 0.3, rng)
    reps = [1] * N
    ref, T, sabs = orc.lhaf_fds(A, g, reps)
    check(tree.lhaf_rpt(A, g, reps), ref, sabs, tol=1e-10 if N <= 24 else 1e-8)  # north_star tolerances


@pytest.mark.parametrize("reps", [[1], [2], [3], [4], [6], [2, 2], [4, 2], [2, 2, 2], [1, 1], [5, 1]])
def test_tree_single_and_even(tree, orc, reps):
    # one pair (the root is the leaf level), self-pairs, and all-even multiplicities (every eta
    # even after matching: no halving, the whole range is evaluated, prefactor 2^-n)
    rng = G.rng_for(7100 + sum(reps) * 10 + len(reps))
    k = len(reps)
    A = G.random_symmetric(k, rng, 0.7)
    g = G.complex_gaussian(k, 0.6, rng)
    ref, T, sabs = orc.lhaf_fds(A, g, reps)
    check(tree.lhaf_rpt(A, g, reps), ref, sabs)
    ref0, _, sabs0 = orc.lhaf_fds(A, np.zeros(k, complex), reps)
    check(tree.lhaf_rpt(A, np.zeros(k, complex), reps), ref0, sabs0)


def test_tree_vs_v3_cfg1_cfg3(lib, orc):
    for cfgn in (1, 3):
        cfg = G.config(cfgn)
        lib.lhaf_set_kernel(6)
        t = lib.lhaf_rpt(cfg["A"], cfg["gamma"], cfg["reps"])
        lib.lhaf_set_kernel(3)
        v = lib.lhaf_rpt(cfg["A"], cfg["gamma"], cfg["reps"])
        lib.lhaf_set_kernel(0)
        ref, T, sabs = orc.lhaf_fds(cfg["A"], cfg["gamma"], cfg["reps"])
        check(t, ref, sabs, 1e-10 if cfgn == 1 else 1e-8)
        assert abs(t - v) <= 1e-8 * max(abs(ref), 1e-12 * sabs)


@pytest.mark.parametrize("seed", range(6))
def test_tree_mixed(tree, orc, seed):
    rng = G.rng_for(7200 + seed)
    k = int(rng.integers(2, 6))
    A2 = G.lossy_squeezed_A2(G.haar_unitary(k, rng), 0.7, 0.5)
    g2 = np.zeros(2 * k, complex) if seed % 2 else G.complex_gaussian(2 * k, 0.3, rng)
    reps = G.random_pattern(k, int(rng.integers(1, 8)), rng)
    ref = orc.lhaf_mixed(A2, g2, reps)
    assert rel(tree.lhaf_rpt_mixed(A2, g2, reps), ref) <= 1e-10


def test_tree_batch_shapes(tree, orc):
    # a batch whose patterns fall into several tree shapes (different H, n, eta, loop flags):
    # each shape is its own group with contiguous units
    rng = G.rng_for(7300)
    k = 8
    A = G.pure_B(G.haar_unitary(k, rng), 0.8)
    g = G.complex_gaussian(k, 0.4, rng)
    pats = [G.random_pattern(k, int(rng.integers(0, 13)), rng) for _ in range(24)]
    pats[3] = np.zeros(k, np.int32)                           # N = 0
    pats[5] = np.array([2, 0, 0, 0, 0, 0, 0, 0], np.int32)   # one self-pair, eta even
    got = tree.lhaf_rpt_batch(A, g, np.array(pats))
    for i, reps in enumerate(pats):
        ref, T, sabs = orc.lhaf_fds(A, g, reps)
        check(got[i], ref, sabs)


def test_tree_unit_ranges_bit_identical(tree):
    # results do not depend on how the unit range is split (rank count, bench slices)
    cfg = G.config(40)
    rng = G.rng_for(7400)
    reps = np.zeros(100, np.int32)
    reps[rng.choice(100, 28, replace=False)] = 1
    job = tree.Job(cfg["A"], cfg["gamma"], reps)
    assert job.info.kernel == 6
    U = job.units
    job.reset(); job.run()
    whole = job.finalize()[0]
    for parts in (2, 3, 7):
        job.reset()
        cuts = [U * i // parts for i in range(parts + 1)]
        for a, b in zip(cuts[:-1], cuts[1:]):
            job.run(a, b)
        v = job.finalize()[0]
        assert v == whole, (parts, v, whole)
    job.close()


def test_tree_n28_vs_v3(lib):
    # d = 28 with loops: the tree and the per-term v3 kernel agree (two different algorithms)
    cfg = G.config(40)
    rng = G.rng_for(7500)
    reps = np.zeros(100, np.int32)
    reps[rng.choice(100, 28, replace=False)] = 1
    lib.lhaf_set_kernel(6)
    t = lib.lhaf_rpt(cfg["A"], cfg["gamma"], reps)
    lib.lhaf_set_kernel(3)
    v = lib.lhaf_rpt(cfg["A"], cfg["gamma"], reps)
    lib.lhaf_set_kernel(0)
    assert rel(t, v) <= 1e-9, (t, v)


@pytest.mark.parametrize("seed", range(8))
def test_tree_inclusion_exclusion(lib, orc, seed):
    # lhaf_rpt_et on the tree (digit k -> weight eta - k, zero weights delete the pair, no
    # halving, prefactor 1: P:403-415) against the oracle, and against the per-term
    # v5 evaluation of the same inclusion/exclusion sum
    rng = G.rng_for(7600 + seed)
    k = int(rng.integers(2, 8))
    A = G.random_symmetric(k, rng, 0.6)
    g = G.complex_gaussian(k, 0.5, rng) if seed % 2 else np.zeros(k, complex)
    reps = G.random_pattern(k, int(rng.integers(2, 15)), rng)
    ref, T, sabs = orc.lhaf_fds(A, g, reps)
    lib.lhaf_set_kernel(6)
    t = lib.lhaf_rpt_et(A, g, reps)
    lib.lhaf_set_kernel(5)
    v = lib.lhaf_rpt_et(A, g, reps)
    lib.lhaf_set_kernel(0)
    check(t, ref, sabs, 1e-9)
    assert abs(t - v) <= max(1e-9 * abs(ref), 1e-12 * sabs)



@pytest.mark.parametrize("fixed,mode,n_cut,loops", [
    ([1, 2, 0, 1, 0, 1, 0, 0], 2, 9, True),     # odd N_f: the leftover photon pairs with mode 2
    ([2, 0, 1, 1, 0, 0, 2, 0], 5, 12, True),    # even N_f: the odd counts get a phantom pair
    ([1, 1, 0, 1, 0, 0, 0, 1], 0, 10, False),   # no loops: odd totals vanish
    ([0] * 8, 3, 7, True),                      # nothing fixed: single-mode counts 0..7
    ([2, 2, 0, 2, 0, 0, 0, 0], 1, 8, True),     # every fixed eta even: no halving on the tree
])
def test_tree_cutoff_batched(lib, orc, fixed, mode, n_cut, loops):
    # App. B.5 on the tree: the batched self-pair is the leaf level, one series per
    # (fixed-pair prefix, w_b) serves every count 2m + p; against the oracle per count and the
    # per-term shared evaluation (v3)
    rng = G.rng_for(5330 + n_cut)
    k = 8
    A = G.pure_B(G.haar_unitary(k, rng), 0.75)
    g = G.complex_gaussian(k, 0.35, rng) if loops else np.zeros(k, complex)
    fixed = np.array(fixed, np.int32)
    try:
        lib.lhaf_set_kernel(6)
        vals = lib.lhaf_rpt_cutoff(A, g, fixed, mode, n_cut)
    finally:
        lib.lhaf_set_kernel(0)
    os.environ["LHAF_CUTOFF_PER_TERM"] = "1"
    try:
        per_term = lib.lhaf_rpt_cutoff(A, g, fixed, mode, n_cut)
    finally:
        del os.environ["LHAF_CUTOFF_PER_TERM"]
    for c in range(n_cut + 1):
        reps = fixed.copy()
        reps[mode] = c
        ref = orc.lhaf(A, g, reps)
        if abs(ref) == 0.0:
            assert abs(vals[c]) <= 1e-13 * max(1.0, max(abs(x) for x in per_term)), (c, vals[c])
            continue
        assert rel(vals[c], ref) <= 1e-10, (c, vals[c], ref)
        assert rel(vals[c], per_term[c]) <= 1e-11, (c, vals[c], per_term[c])
