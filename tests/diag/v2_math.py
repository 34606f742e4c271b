"""Design exploration (not product, not oracle): numpy emulation of the v2 per-term pipeline
before writing it in CUDA.  Bordered matrix B = [[0, z^T], [y, M]], Gauss-transform
Hessenberg reduction with partial pivoting keeping index 0 fixed, trailing La Budde truncated
to the top n+2 coefficients, then the series g = [lam^n] c_M^{-1/2} exp(S/2) with
lam S = (c_M - c_B) / c_M.  Compared with the long-double oracle term."""
import sys

import numpy as np

import os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import gbs_inputs as G  # noqa: E402
import oracle as O  # noqa: E402


def bordered(C, v, w, loops):
    d = C.shape[0]
    H = d // 2
    ww = np.concatenate([w, w]).astype(float)
    part = np.concatenate([np.arange(H, d), np.arange(0, H)])
    M = C[:, part] * ww[None, :]
    if not loops:
        return M
    z = v[part] * ww
    B = np.zeros((d + 1, d + 1), complex)
    B[0, 1:] = z
    B[1:, 0] = v
    B[1:, 1:] = M
    return B


def gauss_hessenberg(B):
    A = B.copy()
    E = A.shape[0]
    for k in range(E - 2):
        col = np.abs(A[k + 1:, k])
        p = k + 1 + int(np.argmax(col))
        if col.max() == 0:
            continue
        # eliminate with pivot row p (pre-swap labels), then swap k+1 <-> p
        piv = A[p, k]
        rows = [r for r in range(k + 1, E) if r != p]
        m = A[rows, k] / piv
        A[rows, :] -= np.outer(m, A[p, :])     # left (done columns of row p are 0)
        A[rows, k] = 0
        A[:, p] += A[:, rows] @ m               # right
        A[[k + 1, p], :] = A[[p, k + 1], :]
        A[:, [k + 1, p]] = A[:, [p, k + 1]]
    return A


def labudde_top(Hm, ntop):
    """q_j^top[t], t = 0..ntop-1, for j = E..0 (q_j = det(xI - H[j:, j:]))."""
    E = Hm.shape[0]
    Q = np.zeros((E + 1, ntop), complex)
    Q[E, 0] = 1
    sub = np.array([Hm[i, i - 1] for i in range(1, E)])
    for j in range(E - 1, -1, -1):
        F = np.zeros(ntop, complex)
        pi = 1.0 + 0j
        for m in range(1, min(ntop, E - j)):
            pi *= Hm[j + m, j + m - 1]
            F[m] = Hm[j, j + m] * pi
        for t in range(ntop):
            if t > E - j:
                continue
            val = Q[j + 1, t] if t <= E - j - 1 else 0
            if t >= 1:
                val -= Hm[j, j] * Q[j + 1, t - 1]
            for m in range(1, min(t - 1, E - 1 - j) + 1):
                val -= F[m] * Q[j + m + 1, t - m - 1]
            Q[j, t] = val
    return Q


def series(cM, cB, n, loops):
    Qs = np.zeros(n + 1, complex)
    Qs[0] = 1
    for m in range(1, n + 1):
        Qs[m] = -sum((m - i / 2) * cM[i] * Qs[m - i] for i in range(1, m + 1)) / m
    if not loops:
        return Qs[n]
    R = np.zeros(n + 2, complex)
    for m in range(n + 2):
        R[m] = (cM[m] - cB[m]) - sum(cM[i] * R[m - i] for i in range(1, m + 1))
    S = np.zeros(n + 1, complex)
    S[1:] = R[2:n + 2]
    Ee = np.zeros(n + 1, complex)
    Ee[0] = 1
    for m in range(1, n + 1):
        Ee[m] = 0.5 * sum(j * S[j] * Ee[m - j] for j in range(1, m + 1)) / m
    return sum(Qs[m] * Ee[n - m] for m in range(n + 1))


def term_v2(C, v, w, n):
    loops = np.any(v != 0)
    B = bordered(C, v, np.array(w), loops)
    Hm = gauss_hessenberg(B)
    ntop = n + 2
    Q = labudde_top(Hm, ntop)
    if loops:
        cB, cM = Q[0], Q[1]
    else:
        cM = Q[0]
        cB = cM
    return series(cM, cB, n, loops)


if __name__ == '__main__':
    rng = G.rng_for(5)
    for cfgn in [1, 3, 2, 4, 5]:
        cfg = G.config(cfgn)
        reps = cfg.get('reps_batch', [cfg.get('reps')])[0] if cfgn == 2 else cfg['reps']
        C, v, eta, n = O.reduced_system(cfg['A'], cfg['gamma'], reps, mixed=cfg['mixed'])
        errs = []
        for trial in range(3):
            ks = [int(rng.integers(0, e + 1)) for e in eta]
            w = [e - 2 * k for e, k in zip(eta, ks)]
            ref = O.fds_term(C, v, w, n)
            g = term_v2(C, v, w, n)
            errs.append(abs(g - ref) / max(abs(ref), 1e-300))
        print('cfg', cfgn, 'd', C.shape[0], 'n', n, ['%.2e' % e for e in errs], flush=True)
