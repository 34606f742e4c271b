"""Which stage of the tree's per-term arithmetic dominates its FP64 error:
the term's path evaluated with one stage in FP64 and the rest in x87 long double, against the
all-long-double path (and the oracle term).  Stages: K = the Schur-complement updates
(T = Q (u, x)^T, K' = K + lam (u T1 + x T2)), P = the pivot series (D, 1/D, log D, Q),
E = the final exp series and its lam^n coefficient; finer pivot stages: D = the pivot
determinant D_w, R = 1/D_w, G = log D_w and its sum log c, Q = the 2x2 Q block; L = only the
last eliminated pair's pivot in FP64, U = every pivot but the last.
usage: python tests/diag/tree_stage_errors.py [cfg] [nsample]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
LD = np.clongdouble


def smul(a, b, L):
    return np.convolve(a, b)[:L]


def shift(a, L):
    out = np.zeros(L, a.dtype)
    out[1:] = a[:L - 1]
    return out


def sinv(D, L):
    R = np.zeros(L, D.dtype)
    R[0] = 1.0
    for t in range(1, L):
        R[t] = -np.dot(D[1:t + 1], R[t - 1::-1][:t])
    return R


def sexp(a, L):
    E = np.zeros(L, a.dtype)
    E[0] = 1.0
    ja = np.arange(L) * a
    for m in range(1, L):
        E[m] = np.dot(ja[1:m + 1], E[m - 1::-1][:m]) / m
    return E


def term_path(C, v, w, n, fp64=""):
    tK = np.complex128 if "K" in fp64 else LD
    tP = np.complex128 if "P" in fp64 else LD
    tE = np.complex128 if "E" in fp64 else LD
    H = len(w)
    d = 2 * H
    L = n + 1
    idx = list(range(d)) + [d]
    K = np.zeros((d + 1, d + 1, L), LD)
    K[:d, :d, 0] = C
    K[d, :d, 0] = -v
    K[:d, d, 0] = -v
    logc = np.zeros(L, LD)
    last = max([q for q in range(H) if float(w[q]) != 0.0], default=-1)
    for p in range(H):
        a, b = p, p + H
        wp = float(w[p])
        if "L" in fp64 or "U" in fp64:  # L: only the last pair's pivot in FP64; U: all but the last
            is_last = p == last
            tP = np.complex128 if (("L" in fp64 and is_last) or ("U" in fp64 and not is_last)) else LD
        live = [i for i in idx if i != a and i != b]
        if wp == 0.0:
            idx = live
            continue
        tD = np.complex128 if "D" in fp64 else tP
        tR = np.complex128 if "R" in fp64 else tP
        tG = np.complex128 if "G" in fp64 else tP
        tQ = np.complex128 if "Q" in fp64 else tP
        Kaa, Kbb, Kab = (K[a, a].astype(tD), K[b, b].astype(tD), K[a, b].astype(tD))
        one_m = -wp * shift(Kab, L)
        one_m[0] += 1.0
        D = smul(one_m, one_m, L) - wp * wp * shift(shift(smul(Kaa, Kbb, L), L), L)
        R = sinv(D.astype(tR), L)
        dD = np.zeros(L, tG)
        dD[:L - 1] = np.arange(1, L) * D[1:]
        q = smul(dD, R.astype(tG), L)
        lg = np.zeros(L, tG)
        lg[1:] = q[:L - 1] / np.arange(1, L)
        logc = (logc.astype(tG) + lg).astype(LD)
        Rq = R.astype(tQ)
        q11 = (wp * wp * shift(smul(Kbb.astype(tQ), Rq, L), L)).astype(tK)
        q22 = (wp * wp * shift(smul(Kaa.astype(tQ), Rq, L), L)).astype(tK)
        q12 = smul((wp * one_m).astype(tQ), Rq, L).astype(tK)
        U = {j: K[j, a].astype(tK) for j in live}
        X = {j: K[j, b].astype(tK) for j in live}
        T1 = {j: smul(q11, U[j], L) + smul(q12, X[j], L) for j in live}
        T2 = {j: smul(q12, U[j], L) + smul(q22, X[j], L) for j in live}
        Kn = K.copy()
        for ii, i in enumerate(live):
            for j in live[ii:]:
                val = K[i, j].astype(tK) + shift(smul(U[i], T1[j], L) + smul(X[i], T2[j], L), L)
                Kn[i, j] = val
                Kn[j, i] = val
        K = Kn
        idx = live
    phi = (0.5 * K[d, d] - 0.5 * logc).astype(tE)
    F = sexp(phi, L)
    return complex(F[n])


def main():
    import gbs_inputs as G
    import oracle as O
    cfgn = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    ns = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    cfg = G.config(cfgn)
    C, v, eta, n = O.reduced_system(cfg['A'], cfg['gamma'], cfg['reps'], mixed=cfg['mixed'])
    rng = np.random.default_rng(5)
    T = int(np.prod([e + 1 for e in eta]))
    ts = rng.integers(0, T, ns)
    W = np.array([O.decode(int(t), eta)[1] for t in ts], np.int32)
    ref_o = O.fds_terms(C, v, W, n)
    res = {k: [] for k in ["", "K", "P", "E", "KPE", "L", "U"]}
    for i in range(ns):
        ref = term_path(C, v, W[i], n, "")
        for k in res:
            g = ref if k == "" else term_path(C, v, W[i], n, k)
            res[k].append(abs(g - (ref if k else ref_o[i])) / abs(ref))
        print(i, {k: f"{res[k][-1]:.1e}" for k in res}, flush=True)
    print(f"cfg{cfgn} d={2 * len(eta)} n={n}; column '' = long-double path vs oracle; others: that stage in FP64")
    for k in res:
        a = np.array(res[k])
        print(f"  {k or 'LD-vs-oracle':>13}: median {np.median(a):.2e} max {a.max():.2e}")


if __name__ == "__main__":
    main()
