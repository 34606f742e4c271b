"""Design exploration (not product, not oracle): accuracy of candidate per-term pipelines in
fp64 vs the long-double oracle term, on config-4-like matrices.  Pipelines:
  H: Householder Hessenberg (e1 fixed after a P0 reflector mapping v -> beta e1)
  E: Gaussian-elimination Hessenberg with partial pivoting (same P0 trick via a Gauss transform)
  S: complex-symmetric tridiagonalisation with complex-orthogonal reflectors
all followed by trailing La Budde + first-row loop correction + det^{-1/2} / exp series."""
import sys, numpy as np
import os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import oracle as O, gbs_inputs as G

def series_g(c, Dt, beta, n, d):
    # c: coeffs of det(I - lam H), len d+1 ; Dt: len d (coeffs of D~) ; g = [lam^n] c^{-1/2} exp(beta lam Dt/c / 2)
    cc = np.zeros(n + 1, complex); cc[:min(n, d) + 1] = c[:min(n, d) + 1]
    Q = np.zeros(n + 1, complex); Q[0] = 1
    for m in range(1, n + 1):
        s = 0
        for i in range(1, min(m, d) + 1):
            s += (m - i / 2) * cc[i] * Q[m - i]
        Q[m] = -s / m
    R = np.zeros(n, complex)
    Dz = np.zeros(n, complex); Dz[:min(n, d)] = Dt[:min(n, d)]
    for m in range(n):
        s = Dz[m]
        for i in range(1, min(m, d) + 1):
            s -= cc[i] * R[m - i]
        R[m] = s
    r = np.zeros(n + 1, complex); r[1:] = beta * R
    E = np.zeros(n + 1, complex); E[0] = 1
    for m in range(1, n + 1):
        E[m] = 0.5 * sum(j * r[j] * E[m - j] for j in range(1, m + 1)) / m
    return sum(Q[m] * E[n - m] for m in range(n + 1))

def labudde_trailing(Hm):
    d = Hm.shape[0]
    q = [None] * (d + 1); q[d] = np.array([1.0 + 0j])   # coeffs low->high, monic
    for j in range(d - 1, -1, -1):
        L = d - j + 1
        p = np.zeros(L, complex)
        p[1:] += q[j + 1]
        p[:L - 1] -= Hm[j, j] * q[j + 1]
        pi = 1.0 + 0j
        for m in range(1, d - j):
            pi *= Hm[j + m, j + m - 1]
            qq = q[j + m + 1]
            p[:len(qq)] -= Hm[j, j + m] * pi * qq
        q[j] = p
    return q

def finish(Hm, z, beta, n):
    d = Hm.shape[0]
    q = labudde_trailing(Hm)
    c = q[0][::-1]                      # c_m = q0[d-m]
    D = np.zeros(d, complex)           # degree d-1
    D[:len(q[1])] += z[0] * q[1]
    pi = 1.0 + 0j
    for m in range(1, d):
        pi *= Hm[m, m - 1]
        D[:len(q[m + 1])] += z[m] * pi * q[m + 1]
    Dt = D[::-1]                        # Dt_m = D[d-1-m]
    return series_g(c, Dt, beta, n, d)

def build_M(C, v, w):
    d = C.shape[0]; Hh = d // 2
    Xw = np.zeros((d, d)); 
    for h in range(Hh):
        Xw[h, h + Hh] = Xw[h + Hh, h] = w[h]
    M = C @ Xw
    z = v @ Xw
    return M, z

def pipeline_H(C, v, w, n):
    M, z = build_M(C, v, w); y = v.copy(); d = M.shape[0]
    # P0: Householder mapping y -> beta e1
    nrm = np.linalg.norm(y)
    if nrm > 0:
        ph = y[0] / abs(y[0]) if y[0] != 0 else 1
        alpha = -ph * nrm
        u = y.copy(); u[0] -= alpha
        s = 1 / (nrm * (nrm + abs(y[0])))
        P = np.eye(d) - s * np.outer(u, u.conj())
        M = P @ M @ P; z = z @ P; beta = alpha
    else:
        beta = 0
    A = M.copy()
    for k in range(d - 2):
        x = A[k + 1:, k].copy()
        nx = np.linalg.norm(x)
        if nx == 0: continue
        ph = x[0] / abs(x[0]) if x[0] != 0 else 1
        alpha = -ph * nx
        u = x.copy(); u[0] -= alpha
        s = 1 / (nx * (nx + abs(x[0])))
        # left
        A[k + 1:, :] -= s * np.outer(u, u.conj() @ A[k + 1:, :])
        A[:, k + 1:] -= s * np.outer(A[:, k + 1:] @ u, u.conj())
        z[k + 1:] -= s * (z[k + 1:] @ u) * u.conj()
    return finish(A, z, beta, n)

def pipeline_E(C, v, w, n):
    M, z = build_M(C, v, w); y = v.copy(); d = M.shape[0]
    A = M.copy(); z = z.copy()
    beta = 0
    if np.linalg.norm(y) > 0:
        p = int(np.argmax(np.abs(y)))
        perm = list(range(d)); perm[0], perm[p] = perm[p], perm[0]
        A = A[np.ix_(perm, perm)]; z = z[perm]; y = y[perm]
        m = y / y[0]; m[0] = 0
        # L = I - m e1^T ; A <- L A L^{-1}, L^{-1} = I + m e1^T ; z^T <- z^T L^{-1}; y <- L y = y0 e1
        A = A - np.outer(m, A[0, :])
        A[:, 0] += A @ m
        z[0] += z @ m
        beta = y[0]
    for k in range(d - 2):
        col = A[k + 1:, k]
        p = k + 1 + int(np.argmax(np.abs(col)))
        if A[p, k] == 0: continue
        if p != k + 1:
            A[[k + 1, p], :] = A[[p, k + 1], :]
            A[:, [k + 1, p]] = A[:, [p, k + 1]]
            z[[k + 1, p]] = z[[p, k + 1]]
        m = np.zeros(d, complex)
        m[k + 2:] = A[k + 2:, k] / A[k + 1, k]
        A[k + 2:, :] -= np.outer(m[k + 2:], A[k + 1, :])
        A[:, k + 1] += A @ m
        z[k + 1] += z @ m
    return finish(A, z, beta, n)

rng = G.rng_for(11)
cfg = G.config(4)
C, v, eta, n = O.reduced_system(cfg['A'], cfg['gamma'], cfg['reps'])
d = C.shape[0]; H = d // 2
print("d", d, "n", n)
errs = {'H': [], 'E': []}
for trial in range(int(sys.argv[1]) if len(sys.argv) > 1 else 6):
    w = rng.choice([-1, 1], H)
    ref = O.fds_term(C, v, w, n)
    for name, f in [('H', pipeline_H), ('E', pipeline_E)]:
        g = f(C, v, w, n)
        errs[name].append(abs(g - ref) / abs(ref))
    print(trial, abs(ref), {k: '%.2e' % e[-1] for k, e in errs.items()}, flush=True)

def pipeline_S(C, v, w, n):
    d = C.shape[0]; Hh = d // 2
    K = np.zeros((d, d), complex)
    for h in range(Hh):
        sp, sm = np.sqrt(complex(w[h])), np.sqrt(complex(-w[h]))
        a, b = (sp + sm) / 2, (sp - sm) / 2
        K[h, h] = K[h + Hh, h + Hh] = a; K[h, h + Hh] = K[h + Hh, h] = b
    S = K @ C @ K; u = K @ v
    A = S.copy()
    def refl(x):
        a2 = x @ x; al = np.sqrt(a2)
        if abs(al - x[0]) < abs(-al - x[0]): al = -al
        p = x.copy(); p[0] -= al
        return p, 2 / (p @ p), al
    beta2 = u @ u
    p, s, al = refl(u)
    P = np.eye(d) - s * np.outer(p, p)
    A = P @ A @ P
    for k in range(d - 2):
        x = A[k + 1:, k].copy()
        if np.all(x[1:] == 0): continue
        p, s, al = refl(x)
        P = np.eye(d, dtype=complex); P[k + 1:, k + 1:] -= s * np.outer(p, p)
        A = P @ A @ P
    a = np.diag(A).copy(); b = np.diag(A, 1).copy()
    # trailing q_j
    q = [None] * (d + 2); q[d] = np.array([1 + 0j]); q[d + 1] = np.array([0j])
    for j in range(d - 1, -1, -1):
        L = d - j + 1; pp = np.zeros(L, complex)
        pp[1:] += q[j + 1]; pp[:L - 1] -= a[j] * q[j + 1]
        if j + 2 <= d and j < d - 1:
            qq = q[j + 2]; pp[:len(qq)] -= b[j] ** 2 * qq
        q[j] = pp
    c = q[0][::-1]
    Dt = np.zeros(d, complex); Dt[:d] = q[1][::-1][:d]   # det(I - lam T_{2:}) coeffs, degree d-1
    return series_g(c, Dt, beta2, n, d)

for cfgn in [4, 5]:
    cfg = G.config(cfgn)
    C, v, eta, n = O.reduced_system(cfg['A'], cfg['gamma'], cfg['reps'], mixed=cfg['mixed'])
    d = C.shape[0]; H = d // 2
    print("cfg", cfgn, "d", d, "n", n)
    for trial in range(4):
        ks = [int(rng.integers(0, e + 1)) for e in eta]
        w = [e - 2 * k for e, k in zip(eta, ks)]
        if 0 in w: w = [x if x != 0 else 1 for x in w]  # avoid w=0 for S (needs deletion)
        ref = O.fds_term(C, v, w, n)
        out = {}
        for name, f in [('H', pipeline_H), ('E', pipeline_E), ('S', pipeline_S)]:
            g = f(C, v, w, n); out[name] = '%.2e' % (abs(g - ref) / abs(ref))
        print(trial, abs(ref), out, flush=True)
