"""Design exploration (not product, not oracle): the shared-prefix (tree) evaluation of sieve
terms by symmetric block Schur complements with truncated power series.

For one term w, det(I - lam C X_w) and the loop term follow from the symmetric matrix
Y = W^{-1} X - lam K (K = C at the root) bordered by the loop vector; pairs are eliminated one
at a time with 2x2 block pivots (constant part [[0, 1/w], [1/w, 0]], always invertible as a
series), so a prefix of eliminated pairs is shared by every term with the same prefix weights.
This script checks the per-term accuracy of that route in FP64 against the long-double oracle
term (explicit powers) on sampled terms of the BASELINE configs.
usage: python tests/diag/tree_series.py [cfg] [nsample]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def smul(a, b, L):
    return np.convolve(a, b)[:L]


def shift(a, L):  # lam * a
    out = np.zeros(L, complex)
    out[1:] = a[:L - 1]
    return out


def sinv(D, L):
    R = np.zeros(L, complex)
    R[0] = 1.0 / D[0]
    for t in range(1, L):
        R[t] = -np.dot(D[1:t + 1], R[t - 1::-1][:t]) * R[0]
    return R


def sexp(a, L):  # exp of a series with a[0] = 0
    E = np.zeros(L, complex)
    E[0] = 1.0
    ja = np.arange(L) * a
    for m in range(1, L):
        E[m] = np.dot(ja[1:m + 1], E[m - 1::-1][:m]) / m
    return E


def term_path(C, v, w, n, order=None):
    H = len(w)
    d = 2 * H
    L = n + 1
    idx = list(range(d)) + [d]  # live indices, border last
    K = np.zeros((d + 1, d + 1, L), complex)
    K[:d, :d, 0] = C
    K[d, :d, 0] = -v
    K[:d, d, 0] = -v
    logc = np.zeros(L, complex)
    order = range(H) if order is None else order
    for p in order:
        a, b = p, p + H
        wp = float(w[p])
        live = [i for i in idx if i != a and i != b]
        if wp == 0.0:
            idx = live
            continue
        Kaa, Kbb, Kab = K[a, a], K[b, b], K[a, b]
        one_m = -wp * shift(Kab, L)
        one_m[0] += 1.0
        D = smul(one_m, one_m, L) - wp * wp * shift(shift(smul(Kaa, Kbb, L), L), L)
        R = sinv(D, L)
        dD = np.zeros(L, complex)
        dD[:L - 1] = np.arange(1, L) * D[1:]
        q = smul(dD, R, L)
        lg = np.zeros(L, complex)
        lg[1:] = q[:L - 1] / np.arange(1, L)
        logc += lg
        q11 = wp * wp * shift(smul(Kbb, R, L), L)
        q22 = wp * wp * shift(smul(Kaa, R, L), L)
        q12 = smul(wp * one_m, R, L)
        U = {j: K[j, a] for j in live}
        X = {j: K[j, b] for j in live}
        T1 = {j: smul(q11, U[j], L) + smul(q12, X[j], L) for j in live}
        T2 = {j: smul(q12, U[j], L) + smul(q22, X[j], L) for j in live}
        Kn = K.copy()
        for ii, i in enumerate(live):
            for j in live[ii:]:
                val = K[i, j] + shift(smul(U[i], T1[j], L) + smul(X[i], T2[j], L), L)
                Kn[i, j] = val
                Kn[j, i] = val
        K = Kn
        idx = live
    F = sexp(0.5 * K[d, d] - 0.5 * logc, L)
    return F[n]


def main():
    import gbs_inputs as G
    import oracle as O

    cfgn = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    ns = int(sys.argv[2]) if len(sys.argv) > 2 else 16
    cfg = G.config(cfgn)
    C, v, eta, n = O.reduced_system(cfg['A'], cfg['gamma'], cfg['reps'], mixed=cfg['mixed'])
    rng = np.random.default_rng(5)
    T = int(np.prod([e + 1 for e in eta]))
    ts = rng.integers(0, T, ns)
    W = np.array([O.decode(int(t), eta)[1] for t in ts], np.int32)
    ref = O.fds_terms(C, v, W, n)
    errs = []
    for i in range(ns):
        g = term_path(C, v, W[i], n)
        errs.append(abs(g - ref[i]) / abs(ref[i]))
    errs = np.array(errs)
    print(f"cfg{cfgn} d={2 * len(eta)} n={n}: tree-series per-term rel err median {np.median(errs):.2e} "
          f"max {errs.max():.2e}")


if __name__ == "__main__":
    main()
