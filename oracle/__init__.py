"""TEST INFRASTRUCTURE ONLY -- the CPU oracle for the loop hafnian with repeated rows/columns.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product
(``paper_2108_01622_b200``) never imports it, and this package never imports the
product: the two share no code ("Oracle").

The arithmetic lives in ``oracle.c`` (x87 long double, OpenMP).  This module is a thin
ctypes marshaller plus ``build()``.  Every function cites the paper passage it follows
(``P:nnn`` = line of PAPER.md of arXiv 2108.01622).

Parity status per function:
  lhaf_brute        pinned: telephone numbers, (N-1)!!, 2x2 closed form, rank-one, TMSV,
                    coherent, involution counts          (tests/test_oracle_pins.py)
  lhaf_et           pinned: agreement with lhaf_brute (N <= 12) + closed forms to N = 40
  matched_reps      pinned: the paper's worked example n = (2,1,0,3) -> 6 terms
  fds_term          pinned: 2x2 closed form; full-sum agreement with lhaf_brute/lhaf_et
  fds_terms         the same routine over a batch (pinned: equality with fds_term)
  fds_sum           signed, binomially weighted fds_terms over a term range in a given pair
                    order (pinned: whole range = lhaf_fds for a permuted pair order)
  fds_range         pinned: fds_range(0, T) 2^{-n} = lhaf_fds = lhaf_brute, additivity over a
                    split of [0, T), halving 2 sum_{t < T/2} = sum_{t < T}  (test_oracle_pins.py)
  lhaf_fds          pinned: agreement with lhaf_brute / lhaf_et, closed forms
  gbs_prob          pinned: squeezed-vacuum, coherent (Poisson) and thermal (geometric)
                    photon statistics, the sum rule sum_n P(n) = 1   (tests/test_gbs_pins.py)
  ips_prob          pinned: single-mode Poisson convolution closed form, sum rule
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so with gcc (-O2 -fopenmp, long double)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(
            ["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", _LIB, _SRC, "-lm"]
        )
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        dp = ctypes.POINTER(ctypes.c_double)
        ip = ctypes.POINTER(ctypes.c_int32)
        lib.orc_expand.argtypes = [dp, dp, ip, ctypes.c_int32, dp]
        lib.orc_expand.restype = ctypes.c_int
        lib.orc_lhaf_brute.argtypes = [ctypes.c_int32, dp, dp]
        lib.orc_lhaf_brute.restype = None
        lib.orc_count_matchings.argtypes = [ctypes.c_int32]
        lib.orc_count_matchings.restype = ctypes.c_uint64
        lib.orc_lhaf_et.argtypes = [ctypes.c_int32, dp, dp, dp]
        lib.orc_lhaf_et.restype = None
        lib.orc_matched_reps.argtypes = [ip, ctypes.c_int32, ip, ip, ip, ctypes.c_int32, ip]
        lib.orc_matched_reps.restype = ctypes.c_int32
        lib.orc_fds_term.argtypes = [ctypes.c_int32, dp, dp, ip, ctypes.c_int32, dp]
        lib.orc_fds_term.restype = None
        lib.orc_fds_terms.argtypes = [ctypes.c_int32, dp, dp, ip, ctypes.c_int32, ctypes.c_int32, dp]
        lib.orc_fds_terms.restype = None
        lib.orc_lhaf_fds.argtypes = [dp, dp, ip, ctypes.c_int32, ctypes.c_int32, dp, dp]
        lib.orc_lhaf_fds.restype = ctypes.c_uint64
        _lib = lib
    return _lib


def _cplx(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.complex128))


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _iptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))


def expand(A, gamma, reps) -> np.ndarray:
    """A_n: repeat row/col i reps[i] times, diagonal replaced by gamma_n."""
    A = _cplx(A)
    gamma = _cplx(gamma)
    reps = np.ascontiguousarray(np.asarray(reps, dtype=np.int32))
    k = reps.shape[0]
    N = int(reps.sum())
    out = np.zeros((N, N), dtype=np.complex128)
    _load().orc_expand(_dptr(A), _dptr(gamma), _iptr(reps), k, _dptr(out))
    return out


def lhaf_brute(Ahat) -> complex:
    """Sum over single-pair matchings of the (already expanded) matrix."""
    Ahat = _cplx(Ahat)
    N = Ahat.shape[0]
    out = np.zeros(2)
    _load().orc_lhaf_brute(N, _dptr(Ahat), _dptr(out))
    return complex(out[0], out[1])


def count_matchings(N: int) -> int:
    """Number of single-pair matchings the brute force visits (telephone number T(N))."""
    return int(_load().orc_count_matchings(N))


def lhaf_et(Ahat) -> complex:
    """Eigenvalue-trace inclusion/exclusion, Eq. ET_loop/ET_poly, explicit powers."""
    return lhaf_et_kappa(Ahat)[0]


def lhaf_et_kappa(Ahat):
    """(value, sum_Z |f(A_Z)|): the second number over |value| is the cancellation factor
    kappa; the oracle's rounding error is bounded by ~ kappa * 5.4e-20 * (small factor)."""
    Ahat = _cplx(Ahat)
    N = Ahat.shape[0]
    out = np.zeros(2)
    sabs = np.zeros(1)
    _load().orc_lhaf_et(N, _dptr(Ahat), _dptr(out), _dptr(sabs))
    return complex(out[0], out[1]), float(sabs[0])


EPS_LD = 2.0 ** -64   # unit roundoff of x87 long double


def lhaf(A, gamma, reps, method: str = "auto") -> complex:
    """lhaf of the expanded matrix A_n: brute force for N <= 14, else ET."""
    Ahat = expand(A, gamma, reps)
    N = Ahat.shape[0]
    if method == "brute" or (method == "auto" and N <= 14):
        return lhaf_brute(Ahat)
    return lhaf_et(Ahat)


def lhaf_mixed(A2, gamma2, reps) -> complex:
    """Mixed-state lhaf: A2 (2k x 2k) expanded with the doubled pattern (reps, reps)."""
    reps = np.asarray(reps, dtype=np.int32)
    return lhaf(A2, gamma2, np.concatenate([reps, reps]))


def matched_reps(reps):
    """Greedy pair matching. Returns (pairs [(p,q)], eta [..], leftover or None)."""
    reps = np.ascontiguousarray(np.asarray(reps, dtype=np.int32))
    k = reps.shape[0]
    cap = max(1, int(reps.sum()))
    p = np.zeros(cap, np.int32)
    q = np.zeros(cap, np.int32)
    eta = np.zeros(cap, np.int32)
    left = np.zeros(1, np.int32)
    H = _load().orc_matched_reps(_iptr(reps), k, _iptr(p), _iptr(q), _iptr(eta), cap, _iptr(left))
    if H < 0:
        raise RuntimeError("matched_reps capacity exceeded")
    pairs = [(int(p[i]), int(q[i])) for i in range(H)]
    return pairs, [int(e) for e in eta[:H]], (int(left[0]) if left[0] >= 0 else None)


def fds_term(C, v, w, n: int) -> complex:
    """One repeated-pair sieve term g(w), explicit powers."""
    C = _cplx(C)
    v = _cplx(v)
    w = np.ascontiguousarray(np.asarray(w, dtype=np.int32))
    h = w.shape[0]
    assert C.shape == (2 * h, 2 * h) and v.shape == (2 * h,)
    out = np.zeros(2)
    _load().orc_fds_term(h, _dptr(C), _dptr(v), _iptr(w), n, _dptr(out))
    return complex(out[0], out[1])


def fds_terms(C, v, W, n: int) -> np.ndarray:
    """A batch of sieve terms g(w), one per row of W (nt x h), by the same explicit-power
    routine as fds_term (OpenMP over the rows).  Parity status: pinned through fds_term."""
    C = _cplx(C)
    v = _cplx(v)
    W = np.ascontiguousarray(np.atleast_2d(np.asarray(W, dtype=np.int32)))
    nt, h = W.shape
    assert C.shape == (2 * h, 2 * h) and v.shape == (2 * h,)
    out = np.zeros(2 * nt)
    _load().orc_fds_terms(h, _dptr(C), _dptr(v), _iptr(W), nt, n, _dptr(out))
    return out[0::2] + 1j * out[1::2]


def lhaf_fds(A, gamma, reps, mixed: bool = False):
    """Full repeated-pair sieve, no halving. Returns (value, T, sum|term| 2^-n)."""
    A = _cplx(A)
    gamma = _cplx(gamma)
    reps = np.ascontiguousarray(np.asarray(reps, dtype=np.int32))
    out = np.zeros(2)
    sabs = np.zeros(1)
    T = _load().orc_lhaf_fds(_dptr(A), _dptr(gamma), _iptr(reps), reps.shape[0], int(mixed),
                             _dptr(out), _dptr(sabs))
    return complex(out[0], out[1]), int(T), float(sabs[0])


def reduced_system(A, gamma, reps, mixed: bool = False):
    """Oracle-side reduced matrix for per-term parity: (C, v, eta, n) following reading C8
    (index list (p_1..p_H, q_1..q_H), C_ab = A_{r_a r_b} incl. diagonal, v = gamma_r,
    phantom row/col zero with loop 1).  Pure Python indexing, no arithmetic."""
    reps = np.asarray(reps, dtype=np.int32)
    if mixed:
        k = reps.shape[0]
        pairs = [(i, i + k) for i in range(k) if reps[i] > 0]
        eta = [int(reps[i]) for i in range(k) if reps[i] > 0]
        left = None
    else:
        pairs, eta, left = matched_reps(reps)
    if left is not None:
        pairs = pairs + [(left, -1)]
        eta = eta + [1]
    C, v = reduced_from_pairs(A, gamma, pairs)
    return C, v, eta, int(sum(eta))


def reduced_from_pairs(A, gamma, pairs):
    """(C, v) over the index list (p_1..p_H, q_1..q_H) of the given pairs (q = -1: the phantom,
    reading C7): C_ab = A_{r_a r_b} (incl. the diagonal, reading C8), v = gamma_r (1 for the
    phantom).  Pure Python indexing, no arithmetic."""
    A = _cplx(A)
    gamma = _cplx(gamma)
    idx = [p for p, _ in pairs] + [q for _, q in pairs]
    d = len(idx)
    C = np.zeros((d, d), np.complex128)
    v = np.zeros(d, np.complex128)
    for a in range(d):
        v[a] = 1.0 if idx[a] < 0 else gamma[idx[a]]
        for b in range(d):
            if idx[a] >= 0 and idx[b] >= 0:
                C[a, b] = A[idx[a], idx[b]]
    return C, v


def fds_sum(C, v, eta, n: int, t0: int, t1: int, batch: int = 8192):
    """sum_{t0 <= t < t1} (-1)^{sum k} prod C(eta_h, k_h) g(w(t)) (reading C5) over the
    pair order of (C, v, eta): each term by fds_terms (explicit powers, long double), the
    digits by decode.  Returns (sum, sum |term|), without the 2^{-n} prefactor."""
    tot = 0j
    tabs = 0.0
    for b0 in range(t0, t1, batch):
        ts = range(b0, min(t1, b0 + batch))
        dec = [decode(t, eta) for t in ts]
        W = np.array([x[1] for x in dec], np.int32)
        g = fds_terms(C, v, W, n)
        f = np.array([x[2] * x[3] for x in dec], np.float64)
        tot += complex(np.sum(f * g))
        tabs += float(np.sum(np.abs(f) * np.abs(g)))
    return tot, tabs


def decode(t: int, eta):
    """Mixed-radix decode of term index t (lowest pair fastest): digits k_h, w = eta - 2k,
    sign (-1)^{sum k}, weight prod C(eta_h, k_h) (reading C5).  Integers only."""
    from math import comb
    ks = []
    rem = int(t)
    for e in eta:
        ks.append(rem % (e + 1))
        rem //= e + 1
    w = [e - 2 * kk for e, kk in zip(eta, ks)]
    sign = -1 if sum(ks) % 2 else 1
    weight = 1
    for e, kk in zip(eta, ks):
        weight *= comb(e, kk)
    return ks, w, sign, weight


def fds_range(A, gamma, reps, t0: int, t1: int, mixed: bool = False):
    """Timing helper for bench.py's CPU baseline: sum of sieve terms [t0, t1) (no prefactor).
    Returns (partial sum, number of terms evaluated)."""
    lib = _load()
    if not hasattr(lib, "_range_ready"):
        dp = ctypes.POINTER(ctypes.c_double)
        ip = ctypes.POINTER(ctypes.c_int32)
        lib.orc_fds_range.argtypes = [dp, dp, ip, ctypes.c_int32, ctypes.c_int32, ctypes.c_uint64,
                                      ctypes.c_uint64, dp]
        lib.orc_fds_range.restype = ctypes.c_uint64
        lib.orc_num_threads.restype = ctypes.c_int
        lib._range_ready = True
    A = _cplx(A)
    gamma = _cplx(gamma)
    reps = np.ascontiguousarray(np.asarray(reps, dtype=np.int32))
    out = np.zeros(2)
    cnt = lib.orc_fds_range(_dptr(A), _dptr(gamma), _iptr(reps), reps.shape[0], int(mixed),
                            t0, t1, _dptr(out))
    return complex(out[0], out[1]), int(cnt)


def num_threads() -> int:
    fds_range(np.zeros((1, 1)), np.zeros(1), [0], 0, 0)
    return int(_load().orc_num_threads())


def gbs_prob(sigma, alpha, n) -> complex:
    """P(n | sigma, alpha) of a Gaussian state, App. A step by step:
    sigma_Q = sigma + I/2, O = I - sigma_Q^{-1}, A = X O, gamma = alpha^dag sigma_Q^{-1}
    (P:308-312); A_n by repeating rows/cols i and i+M n_i times, its diagonal replaced by the
    repeated gamma; P = exp(-alpha^dag sigma_Q^{-1} alpha / 2) / (sqrt(det sigma_Q)
    prod n_i!) lhaf(A_n) (Eq. mixed_prob) with lhaf by brute force (<= 16 indices, else
    the ET tier)."""
    import math
    sigma = np.asarray(sigma, complex)
    alpha = np.asarray(alpha, complex)
    M = alpha.shape[0] // 2
    sq = sigma + 0.5 * np.eye(2 * M)
    qi = np.linalg.inv(sq)
    O = np.eye(2 * M) - qi
    X = np.block([[np.zeros((M, M)), np.eye(M)], [np.eye(M), np.zeros((M, M))]])
    A = X @ O
    gamma = alpha.conj() @ qi
    idx = [i for i in range(M) for _ in range(n[i])] + [i + M for i in range(M) for _ in range(n[i])]
    An = A[np.ix_(idx, idx)].copy()
    np.fill_diagonal(An, gamma[idx])
    lh = (lhaf_brute(An) if len(idx) <= 16 else lhaf_et(An)) if idx else 1.0
    pref = np.exp(-0.5 * (alpha.conj() @ qi @ alpha)) / np.sqrt(np.linalg.det(sq))
    return complex(pref * lh / np.prod([math.factorial(int(k)) for k in n]))


def ips_prob(B, alpha, n) -> float:
    """MIS proposal probability: Q(n) = exp(-sum |alpha_j|^2 - sum_{j,k} |B_jk|^2 / 2)
    / prod n_i! lhaf(C_n), C_n = |B_n|^2 with its diagonal replaced by |alpha_n|^2, formed
    explicitly (B_n repeats row/col i n_i times) and summed by brute force / ET."""
    import math
    B = np.asarray(B, complex)
    alpha = np.asarray(alpha, complex)
    M = alpha.shape[0]
    idx = [i for i in range(M) for _ in range(n[i])]
    Cn = np.abs(B[np.ix_(idx, idx)]) ** 2 + 0j
    np.fill_diagonal(Cn, np.abs(alpha[idx]) ** 2)
    lh = (lhaf_brute(Cn) if len(idx) <= 16 else lhaf_et(Cn)) if idx else 1.0
    pref = math.exp(-np.sum(np.abs(alpha) ** 2) - 0.5 * np.sum(np.abs(B) ** 2))
    return float((pref * lh).real / np.prod([math.factorial(int(k)) for k in n]))
