"""Host-side logic of the product (no GPU): the C-ABI library loads and exports every symbol
include/lhaf.h declares; planning (greedy matching, phantom, term counts) and the mixed-radix
decode are bit-exact against the oracle's independent implementation; compute calls fail
loudly (LHAF_E_CUDA) when no device is present -- there is no CPU path."""
import os
import re
import subprocess

import numpy as np
import pytest

import gbs_inputs as G

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "lhaf.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(lhaf_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.check_output(["nm", "-D", "--defined-only", lib.LIB_PATH], text=True)
    exported = set(ln.split()[-1] for ln in out.splitlines() if ln.strip())
    declared = header_symbols()
    assert len(declared) >= 20
    missing = [s for s in declared if s not in exported]
    assert not missing, missing
    assert set(lib.EXPORTED) == set(declared)


def test_library_is_sm100a_only(lib):
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lib.LIB_PATH], text=True)
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_no_cpu_fallback_without_gpu(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(lib.LhafError) as e:
        lib.lhaf_rpt(np.eye(2), np.ones(2), [1, 1])
    assert e.value.status == 4


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2108_01622_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"(#|//).*", "", txt).lower().replace("oracle/", ""), f


def test_plan_paper_example(lib, orc):
    info = lib.lhaf_plan([2, 1, 0, 3])
    assert info.T == 6 and info.T_eval == 3 and info.H == 2 and info.n == 3 and info.d == 4
    pairs, eta, left = orc.matched_reps([2, 1, 0, 3])
    assert info.pairs() == pairs and info.etas() == eta and left is None
    # config 1 (reading C19: BASELINE's "108 terms" does not follow from the paper's rule)
    info = lib.lhaf_plan([2, 2, 2, 1, 1, 1, 1, 2])
    assert info.etas() == [2, 2, 1, 1] and info.T == 36 and info.T_eval == 18


def test_plan_matches_oracle_random(lib, orc):
    rng = G.rng_for(21)
    for _ in range(1000):
        k = int(rng.integers(1, 12))
        reps = rng.integers(0, 7, k).astype(np.int32)
        info = lib.lhaf_plan(reps)
        pairs, eta, left = orc.matched_reps(reps)
        if left is not None:
            pairs = pairs + [(left, -1)]
            eta = eta + [1]
        assert info.pairs() == pairs and info.etas() == eta
        assert info.leftover == (left if left is not None else -1)
        assert info.N == int(reps.sum()) and info.n == sum(eta) and info.d == 2 * len(eta)
        assert info.T == int(np.prod([e + 1 for e in eta])) if eta else info.T == 1
        assert info.T_eval == (info.T // 2 if eta else 0)


def test_plan_mixed_natural_pairing(lib):
    info = lib.lhaf_plan([2, 0, 3, 1], mixed=2)   # the paper's natural pairing (C11)
    assert info.pairs() == [(0, 4), (2, 6), (3, 7)] and info.etas() == [2, 3, 1]
    assert info.T == 3 * 4 * 2 and info.n == 6 and info.N == 12
    # the default mixed plan is the greedy matching of the doubled pattern (C11b)
    g = lib.lhaf_plan([2, 0, 3, 1, 2, 0, 3, 1])
    m = lib.lhaf_plan([2, 0, 3, 1], mixed=1)
    assert m.pairs() == g.pairs() and m.etas() == g.etas() and m.N == 12 and m.n == 6


def test_decode_bit_exact(lib, orc):
    rng = G.rng_for(22)
    for _ in range(200):
        k = int(rng.integers(1, 8))
        reps = rng.integers(0, 9, k).astype(np.int32)
        info = lib.lhaf_plan(reps)
        if info.H == 0:
            continue
        C, v, eta, n = orc.reduced_system(np.eye(k), np.ones(k), reps)
        for t in rng.integers(0, info.T, 10):
            kk, w, sign, weight = lib.lhaf_decode(info, int(t))
            ok, ow, osign, oweight = orc.decode(int(t), eta)
            assert (kk, w, sign, weight) == (ok, ow, osign, oweight)


def test_term_count_bounds_and_strictness(lib):
    # P:452-466 bounds, P:485 strictness; reading C7 adds the phantom factor for odd N
    import math
    rng = G.rng_for(23)
    for _ in range(1000):
        k = int(rng.integers(1, 10))
        reps = rng.integers(0, 6, k).astype(np.int32)
        info = lib.lhaf_plan(reps)
        N = int(reps.sum())
        lower = float(np.prod([math.sqrt(c + 1) for c in reps]))
        assert lower <= info.T * (1 + 1e-12)
        assert info.T <= 2 ** ((N + 1) // 2)
        if N % 2 == 0 and (sum(c > 1 for c in reps) >= 2 or any(c >= 4 for c in reps)):
            assert info.T < 2 ** (N // 2)


def test_errors_before_device(lib):
    with pytest.raises(lib.LhafError) as e:
        lib.lhaf_plan([1, -1])
    assert e.value.status == 1
    with pytest.raises(lib.LhafError) as e:
        lib.lhaf_plan(np.ones(130, np.int32))
    assert e.value.status == 3
