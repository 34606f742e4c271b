"""Seeded synthetic inputs for the loop-hafnian hot path (shared by tests, bench and the
oracle legs).  Holds NO arithmetic of the method itself (no matching, no sieve, no
characteristic polynomials): only Haar unitaries, squeezing/loss constructions of the GBS
matrix and photon patterns.  Both the oracle and the product read what this returns.

Recipe (BASELINE.json configs):
  numpy.random.Generator(PCG64(seed)), seed = 1000 + cfg, draws in this order:
    1. U  : complex Ginibre (randn + i randn)/sqrt(2) -> QR -> R-diagonal phase fix (Haar)
    2. gamma : Re, Im iid N(0, sigma^2)           (reading C15)
    3. pattern modes : rng.choice(m, K, replace=False)
    4. multiplicities : rng.integers(lo, hi+1, K), then +-1 steps on seeded modes within
       [lo, hi] until the sum matches (reading C17)
  Pure matrices: B = U diag(t) U^T (t = tanh r), complex symmetric, ||B|| <= t.
  Mixed (config 5): A2 of App. A.5 built from P:301-313 (sigma_Q, O = I - sigma_Q^{-1},
  A = X O) for single-mode squeezing t, uniform loss eta, then the interferometer.
"""
from __future__ import annotations

import numpy as np


def rng_for(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def haar_unitary(m: int, rng: np.random.Generator) -> np.ndarray:
    """Haar-random m x m unitary: QR of a complex Ginibre matrix with the phase fix."""
    z = (rng.standard_normal((m, m)) + 1j * rng.standard_normal((m, m))) / np.sqrt(2.0)
    q, r = np.linalg.qr(z)
    ph = np.diagonal(r) / np.abs(np.diagonal(r))
    return q * ph[None, :]


def pure_B(U: np.ndarray, t) -> np.ndarray:
    """B = U diag(t) U^T (P:326 pure block; t = tanh r per mode)."""
    t = np.broadcast_to(np.asarray(t, dtype=float), (U.shape[0],))
    B = (U * t[None, :]) @ U.T
    return 0.5 * (B + B.T)          # exact symmetry (removes rounding asymmetry)


def complex_gaussian(m: int, sigma: float, rng: np.random.Generator) -> np.ndarray:
    return sigma * rng.standard_normal(m) + 1j * sigma * rng.standard_normal(m)


def adjusted_multiplicities(K: int, lo: int, hi: int, total: int, rng: np.random.Generator):
    """Uniform draws in [lo, hi], then seeded +-1 steps within bounds until sum == total."""
    n = rng.integers(lo, hi + 1, K).astype(np.int64)
    assert K * lo <= total <= K * hi
    while n.sum() != total:
        i = int(rng.integers(0, K))
        if n.sum() < total and n[i] < hi:
            n[i] += 1
        elif n.sum() > total and n[i] > lo:
            n[i] -= 1
    return n.astype(np.int32)


def lossy_squeezed_A2(U: np.ndarray, t: float, eta: float) -> np.ndarray:
    """Mixed-state GBS matrix (2m x 2m) for single-mode squeezing tanh r = t in every mode,
    uniform pure loss eta, zero displacement, then the interferometer U (App. A.5 of SURVEY,
    from P:301-313).  Per mode after loss: nu = eta sinh^2 r, mu = eta sinh r cosh r;
    sigma_Q = [[nu+1, mu], [mu, nu+1]] in the (a, a^dagger) basis, D = (nu+1)^2 - mu^2,
    A0 = X (I - sigma_Q^{-1}) = [[mu/D, c], [c, mu/D]], c = 1 - (nu+1)/D.
    Block order B-first: [[U diag(mu/D) U^T, U diag(c) U^dag],
                                  [U* diag(c) U^T,  U* diag(mu/D) U^dag]]."""
    r = np.arctanh(t)
    nu = eta * np.sinh(r) ** 2
    mu = eta * np.sinh(r) * np.cosh(r)
    D = (nu + 1.0) ** 2 - mu ** 2
    c = 1.0 - (nu + 1.0) / D
    m = U.shape[0]
    b = np.full(m, mu / D)
    cc = np.full(m, c)
    B = (U * b[None, :]) @ U.T
    Cx = (U * cc[None, :]) @ U.conj().T
    A2 = np.block([[B, Cx], [Cx.T, B.conj()]])
    return 0.5 * (A2 + A2.T)


def lossy_vacuum_prob(t: float, eta: float, m: int) -> float:
    """P_0 = 1/sqrt(det sigma_Q) = D^{-m/2} for the construction above (alpha = 0)."""
    r = np.arctanh(t)
    nu = eta * np.sinh(r) ** 2
    mu = eta * np.sinh(r) * np.cosh(r)
    D = (nu + 1.0) ** 2 - mu ** 2
    return float(D ** (-m / 2.0))


def config(cfg: int) -> dict:
    """The five BASELINE.json configs.  Returns a dict with
    A (k x k, or 2k x 2k for mixed), gamma, reps (k,) or reps_batch (batch, k), mixed flag."""
    rng = rng_for(1000 + cfg)
    if cfg == 1:
        U = haar_unitary(24, rng)
        A = pure_B(U, 0.7)
        gamma = complex_gaussian(24, 0.3, rng)
        reps = np.zeros(24, np.int32)
        reps[:8] = [2, 2, 2, 1, 1, 1, 1, 2]
        return dict(name="cfg1_N12_repeats", A=A, gamma=gamma, reps=reps, mixed=False)
    if cfg == 2:
        U = haar_unitary(50, rng)
        A = pure_B(U, 0.8)
        gamma = complex_gaussian(50, 0.2, rng)
        batch = 4096
        reps = np.zeros((batch, 50), np.int32)
        for b in range(batch):
            reps[b, rng.choice(50, 24, replace=False)] = 1
        return dict(name="cfg2_batch4096_N24", A=A, gamma=gamma, reps_batch=reps, mixed=False)
    if cfg == 3:
        U = haar_unitary(100, rng)
        A = pure_B(U, 0.9)
        gamma = np.zeros(100, np.complex128)
        modes = rng.choice(100, 16, replace=False)
        mult = adjusted_multiplicities(16, 1, 4, 40, rng)
        reps = np.zeros(100, np.int32)
        reps[modes] = mult
        return dict(name="cfg3_N40_collisions", A=A, gamma=gamma, reps=reps, mixed=False)
    if cfg == 4:
        U = haar_unitary(100, rng)
        A = pure_B(U, 0.9)
        gamma = complex_gaussian(100, 0.1, rng)
        reps = np.zeros(100, np.int32)
        reps[rng.choice(100, 60, replace=False)] = 1
        return dict(name="cfg4_N60", A=A, gamma=gamma, reps=reps, mixed=False)
    if cfg == 5:
        U = haar_unitary(100, rng)
        A2 = lossy_squeezed_A2(U, 0.9, 0.3)
        gamma2 = np.zeros(200, np.complex128)
        modes = rng.choice(100, 24, replace=False)
        mult = adjusted_multiplicities(24, 1, 3, 36, rng)
        reps = np.zeros(100, np.int32)
        reps[modes] = mult
        return dict(name="cfg5_mixed_N36", A=A2, gamma=gamma2, reps=reps, mixed=True)
    if cfg == 40:
        # supplementary N = 40 collision-free point: cfg4's construction with
        # 40 distinct modes (d = 40, 2^19 evaluated terms)
        U = haar_unitary(100, rng)
        A = pure_B(U, 0.9)
        gamma = complex_gaussian(100, 0.1, rng)
        reps = np.zeros(100, np.int32)
        reps[rng.choice(100, 40, replace=False)] = 1
        return dict(name="n40_distinct", A=A, gamma=gamma, reps=reps, mixed=False)
    raise ValueError(cfg)


def random_symmetric(N: int, rng: np.random.Generator, scale: float = 1.0) -> np.ndarray:
    """iid standard-normal Re/Im, symmetrised (Fig. 5 halves, reading C18)."""
    X = rng.standard_normal((N, N)) + 1j * rng.standard_normal((N, N))
    return scale * 0.5 * (X + X.T)


def random_pattern(k: int, N: int, rng: np.random.Generator, max_rep: int | None = None):
    """N photons dropped uniformly on k modes (collisions allowed), optional cap per mode."""
    reps = np.zeros(k, np.int32)
    placed = 0
    while placed < N:
        i = int(rng.integers(0, k))
        if max_rep is None or reps[i] < max_rep:
            reps[i] += 1
            placed += 1
    return reps


def gaussian_state(U: np.ndarray, r, eta=1.0, beta=None, nbar=None):
    """Covariance sigma (2m x 2m) and mean alpha (2m) in the (a_1..a_m, a_1^dag..a_m^dag) basis
    (sigma_ij = <a_i a_j^dag + a_j^dag a_i>/2 - alpha_i alpha_j^*) of: single-mode
    squeezed (r_i) or thermal (nbar_i) inputs, per-mode transmission eta_i (pure loss), the
    interferometer U (a -> U a), then a displacement beta (<a> = beta).  Input construction for
    tests (the probability formula itself is the method)."""
    m = U.shape[0]
    r = np.broadcast_to(np.asarray(r, float), (m,))
    eta = np.broadcast_to(np.asarray(eta, float), (m,))
    ch, sh = np.cosh(r), np.sinh(r)
    sig = np.zeros((2 * m, 2 * m), complex)
    for i in range(m):
        sig[i, i] = sig[i + m, i + m] = sh[i] ** 2 + 0.5
        sig[i, i + m] = sig[i + m, i] = -ch[i] * sh[i]
    if nbar is not None:
        sig = sig + np.diag(np.concatenate([nbar, nbar]).astype(complex))
    e2 = np.concatenate([eta, eta])
    sig = np.sqrt(e2)[:, None] * sig * np.sqrt(e2)[None, :] + np.diag((1.0 - e2) / 2.0)
    S = np.block([[U, np.zeros((m, m))], [np.zeros((m, m)), U.conj()]])
    sig = S @ sig @ S.conj().T
    b = np.zeros(m, complex) if beta is None else np.asarray(beta, complex)
    alpha = np.concatenate([b, b.conj()])
    return sig, alpha
