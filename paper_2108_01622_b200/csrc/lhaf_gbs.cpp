// lhaf_gbs.cpp -- photon-number probabilities of Gaussian states on top of the loop hafnian
// (App. A of the paper, Eq. (mixed_prob); pure block form
// P:322-334), and the MIS proposal probability Q(n | B, alpha).  Host arithmetic on the 2M x 2M covariance (one LU per state: sigma_Q^{-1} and
// det sigma_Q), then ONE device loop hafnian through the C-ABI (lhaf_rpt_mixed, or lhaf_rpt on
// the half-size B_n for pure states).  Product code: shares nothing with oracle/.
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdio>
#include <vector>

#include "../../include/lhaf.h"
#include "lhaf_internal.h"

namespace {

using cd = std::complex<double>;

// In-place LU with partial pivoting of the n x n row-major matrix a; returns false if a
// pivot is exactly zero.  det = product of the pivots with the permutation sign.
bool lu(std::vector<cd> &a, int n, std::vector<int> &piv, cd &det) {
  piv.resize(n);
  det = 1.0;
  for (int k = 0; k < n; ++k) {
    int p = k;
    for (int i = k + 1; i < n; ++i)
      if (std::abs(a[(size_t)i * n + k]) > std::abs(a[(size_t)p * n + k])) p = i;
    piv[k] = p;
    if (a[(size_t)p * n + k] == cd(0.0)) return false;
    if (p != k) {
      for (int c = 0; c < n; ++c) std::swap(a[(size_t)k * n + c], a[(size_t)p * n + c]);
      det = -det;
    }
    const cd d = a[(size_t)k * n + k];
    det *= d;
    for (int i = k + 1; i < n; ++i) {
      const cd m = a[(size_t)i * n + k] / d;
      a[(size_t)i * n + k] = m;
      for (int c = k + 1; c < n; ++c) a[(size_t)i * n + c] -= m * a[(size_t)k * n + c];
    }
  }
  return true;
}

// inverse from the LU factors (column by column)
std::vector<cd> lu_inverse(const std::vector<cd> &lu_, const std::vector<int> &piv, int n) {
  std::vector<cd> inv((size_t)n * n), x(n);
  for (int col = 0; col < n; ++col) {
    for (int i = 0; i < n; ++i) x[i] = (i == col) ? 1.0 : 0.0;
    for (int k = 0; k < n; ++k) std::swap(x[k], x[piv[k]]);
    for (int i = 0; i < n; ++i)
      for (int k = 0; k < i; ++k) x[i] -= lu_[(size_t)i * n + k] * x[k];
    for (int i = n - 1; i >= 0; --i) {
      for (int k = i + 1; k < n; ++k) x[i] -= lu_[(size_t)i * n + k] * x[k];
      x[i] /= lu_[(size_t)i * n + i];
    }
    for (int i = 0; i < n; ++i) inv[(size_t)i * n + col] = x[i];
  }
  return inv;
}

// A = X (I - sigma_Q^{-1}), gamma = alpha^dag sigma_Q^{-1}, prefactor
// exp(-1/2 alpha^dag sigma_Q^{-1} alpha) / sqrt(det sigma_Q)
lhaf_status gbs_matrices(const double *sigma, const double *alpha, int M, std::vector<cd> &A,
                         std::vector<cd> &gamma, cd &pref) {
  const int n = 2 * M;
  std::vector<cd> sq((size_t)n * n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j)
      sq[(size_t)i * n + j] = cd(sigma[2 * ((size_t)i * n + j)], sigma[2 * ((size_t)i * n + j) + 1]) +
                              ((i == j) ? cd(0.5) : cd(0.0));
  std::vector<int> piv;
  cd det;
  if (!lu(sq, n, piv, det))
    return (lhaf_status)lhaf::set_error(LHAF_E_ARG, "sigma + I/2 is singular");
  if (!(det.real() > 0.0))
    return (lhaf_status)lhaf::set_error(LHAF_E_ARG, "det(sigma + I/2) is not positive: not a covariance matrix");
  const std::vector<cd> qi = lu_inverse(sq, piv, n);
  A.assign((size_t)n * n, 0.0);
  for (int i = 0; i < n; ++i) {
    const int xi = (i < M) ? i + M : i - M;  // (X O)_{ij} = O_{xi, j}
    for (int j = 0; j < n; ++j)
      A[(size_t)i * n + j] = ((xi == j) ? cd(1.0) : cd(0.0)) - qi[(size_t)xi * n + j];
  }
  gamma.assign(n, 0.0);
  cd quad = 0.0;
  for (int j = 0; j < n; ++j) {
    cd g = 0.0;
    for (int i = 0; i < n; ++i) g += std::conj(cd(alpha[2 * i], alpha[2 * i + 1])) * qi[(size_t)i * n + j];
    gamma[j] = g;
    quad += g * cd(alpha[2 * j], alpha[2 * j + 1]);
  }
  pref = std::exp(-0.5 * quad) / std::sqrt(det);
  return LHAF_OK;
}

// Covariance and mean of the Gaussian state prepared by M single-mode squeezers (r_i), pure loss
// per input mode (transmission eta_i), the interferometer a -> U a and a displacement beta of the
// output modes (App. A of SURVEY; reading C12 for the basis and sign conventions):
//   input  sigma_0 = [[(sinh^2 r + 1/2) I, -cosh r sinh r], [-cosh r sinh r, (sinh^2 r + 1/2) I]]
//          per mode in the basis (a_1..a_M, a_1^dag..a_M^dag) (sigma_ij = <a_i a_j^dag + a_j^dag a_i>/2);
//   loss   sigma <- sqrt(E) sigma sqrt(E) + (I - E)/2,  E = diag(eta, eta);
//   U      sigma <- S sigma S^dag,  S = diag(U, U*);   mean alpha = (beta, conj(beta)).
void gbs_state(const double *U, const double *r, const double *eta, const double *beta, int M,
               std::vector<cd> &sig, std::vector<cd> &alpha) {
  const int n = 2 * M;
  std::vector<cd> s0((size_t)n * n, 0.0);
  for (int i = 0; i < M; ++i) {
    const double ch = std::cosh(r[i]), sh = std::sinh(r[i]);
    const double e = eta ? eta[i] : 1.0, se = std::sqrt(e);
    s0[(size_t)i * n + i] = s0[(size_t)(i + M) * n + i + M] = e * (sh * sh + 0.5) + 0.5 * (1.0 - e);
    s0[(size_t)i * n + i + M] = s0[(size_t)(i + M) * n + i] = -se * se * ch * sh;
  }
  // S sigma_0 S^dag with S = diag(U, U*)
  auto Sij = [&](int a, int b) -> cd {  // S[a][b]
    if (a < M && b < M) return cd(U[2 * ((size_t)a * M + b)], U[2 * ((size_t)a * M + b) + 1]);
    if (a >= M && b >= M) return std::conj(cd(U[2 * ((size_t)(a - M) * M + b - M)], U[2 * ((size_t)(a - M) * M + b - M) + 1]));
    return cd(0.0);
  };
  std::vector<cd> t((size_t)n * n, 0.0);  // S sigma_0
  for (int a = 0; a < n; ++a)
    for (int b = 0; b < n; ++b) {
      cd acc = 0.0;
      for (int c = 0; c < n; ++c) acc += Sij(a, c) * s0[(size_t)c * n + b];
      t[(size_t)a * n + b] = acc;
    }
  sig.assign((size_t)n * n, 0.0);
  for (int a = 0; a < n; ++a)
    for (int b = 0; b < n; ++b) {
      cd acc = 0.0;
      for (int c = 0; c < n; ++c) acc += t[(size_t)a * n + c] * std::conj(Sij(b, c));
      sig[(size_t)a * n + b] = acc;
    }
  alpha.assign(n, 0.0);
  for (int i = 0; i < M; ++i) {
    const cd b = beta ? cd(beta[2 * i], beta[2 * i + 1]) : cd(0.0);
    alpha[i] = b;
    alpha[i + M] = std::conj(b);
  }
}

}  // namespace

extern "C" {

lhaf_status lhaf_gbs_state(const double *U, const double *r, const double *eta, const double *beta,
                           int32_t M, double *sigma, double *alpha) {
  if (!U || !r || !sigma || !alpha) return (lhaf_status)lhaf::set_error(LHAF_E_ARG, "null pointer");
  if (M < 1 || M > 2048) return (lhaf_status)lhaf::set_error(LHAF_E_ARG, "bad mode count");
  for (int i = 0; i < M; ++i) {
    if (!std::isfinite(r[i])) return (lhaf_status)lhaf::set_error(LHAF_E_ARG, "squeezing not finite");
    if (eta && !(eta[i] >= 0.0 && eta[i] <= 1.0))
      return (lhaf_status)lhaf::set_error(LHAF_E_ARG, "transmission outside [0, 1]");
  }
  // U must be unitary (to 1e-10): the constructor describes a lossless interferometer
  double dev = 0.0;
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < M; ++j) {
      cd acc = 0.0;
      for (int c = 0; c < M; ++c)
        acc += cd(U[2 * ((size_t)i * M + c)], U[2 * ((size_t)i * M + c) + 1]) *
               std::conj(cd(U[2 * ((size_t)j * M + c)], U[2 * ((size_t)j * M + c) + 1]));
      dev = std::max(dev, std::abs(acc - ((i == j) ? cd(1.0) : cd(0.0))));
    }
  if (dev > 1e-10) return (lhaf_status)lhaf::set_error(LHAF_E_ARG, "U is not unitary");
  std::vector<cd> sg, al;
  gbs_state(U, r, eta, beta, M, sg, al);
  for (size_t i = 0; i < sg.size(); ++i) { sigma[2 * i] = sg[i].real(); sigma[2 * i + 1] = sg[i].imag(); }
  for (size_t i = 0; i < al.size(); ++i) { alpha[2 * i] = al[i].real(); alpha[2 * i + 1] = al[i].imag(); }
  return LHAF_OK;
}

lhaf_status lhaf_gbs_prob_state(const double *U, const double *r, const double *eta,
                                const double *beta, int32_t M, const int32_t *n, double out[2]) {
  if (!n || !out) return (lhaf_status)lhaf::set_error(LHAF_E_ARG, "null pointer");
  if (M < 1 || M > 2048) return (lhaf_status)lhaf::set_error(LHAF_E_ARG, "bad mode count");
  std::vector<double> sg((size_t)8 * M * M), al((size_t)4 * M);
  lhaf_status s = lhaf_gbs_state(U, r, eta, beta, M, sg.data(), al.data());
  if (s != LHAF_OK) return s;
  bool pure = true;  // no loss: a pure state, the half-size |lhaf(B_n)|^2 form applies
  for (int i = 0; eta && i < M; ++i) pure = pure && eta[i] == 1.0;
  return lhaf_gbs_prob(sg.data(), al.data(), M, n, pure ? 1 : 0, out);
}

lhaf_status lhaf_gbs_matrices(const double *sigma, const double *alpha, int32_t M, double *A,
                              double *gamma, double out_pref[2]) {
  if (!sigma || !alpha || !A || !gamma || !out_pref)
    return (lhaf_status)lhaf::set_error(LHAF_E_ARG, "null pointer");
  if (M < 1 || M > 2048) return (lhaf_status)lhaf::set_error(LHAF_E_ARG, "bad mode count");
  std::vector<cd> a, g;
  cd pref;
  const lhaf_status s = gbs_matrices(sigma, alpha, M, a, g, pref);
  if (s != LHAF_OK) return s;
  for (size_t i = 0; i < a.size(); ++i) { A[2 * i] = a[i].real(); A[2 * i + 1] = a[i].imag(); }
  for (size_t i = 0; i < g.size(); ++i) { gamma[2 * i] = g[i].real(); gamma[2 * i + 1] = g[i].imag(); }
  out_pref[0] = pref.real();
  out_pref[1] = pref.imag();
  return LHAF_OK;
}

lhaf_status lhaf_gbs_prob(const double *sigma, const double *alpha, int32_t M, const int32_t *n,
                          int32_t pure, double out[2]) {
  if (!sigma || !alpha || !n || !out) return (lhaf_status)lhaf::set_error(LHAF_E_ARG, "null pointer");
  if (M < 1 || M > 2048) return (lhaf_status)lhaf::set_error(LHAF_E_ARG, "bad mode count");
  double fact = 1.0;
  for (int i = 0; i < M; ++i) {
    if (n[i] < 0) return (lhaf_status)lhaf::set_error(LHAF_E_ARG, "negative photon count");
    for (int c = 2; c <= n[i]; ++c) fact *= (double)c;
  }
  std::vector<cd> A, g;
  cd pref;
  lhaf_status s = gbs_matrices(sigma, alpha, M, A, g, pref);
  if (s != LHAF_OK) return s;
  double lh[2];
  cd val;
  if (pure) {
    // A = B (+) B*: lhaf(A_n) = |lhaf(B_n)|^2 with the loops of the first M entries
    std::vector<double> B((size_t)2 * M * M), gb((size_t)2 * M);
    for (int i = 0; i < M; ++i) {
      for (int j = 0; j < M; ++j) {
        const cd b = A[(size_t)i * 2 * M + j];
        B[2 * ((size_t)i * M + j)] = b.real();
        B[2 * ((size_t)i * M + j) + 1] = b.imag();
      }
      gb[2 * i] = g[i].real();
      gb[2 * i + 1] = g[i].imag();
    }
    s = lhaf_rpt(B.data(), gb.data(), n, M, lh);
    if (s != LHAF_OK) return s;
    val = std::norm(cd(lh[0], lh[1]));
  } else {
    std::vector<double> A2(A.size() * 2), g2(g.size() * 2);
    for (size_t i = 0; i < A.size(); ++i) { A2[2 * i] = A[i].real(); A2[2 * i + 1] = A[i].imag(); }
    for (size_t i = 0; i < g.size(); ++i) { g2[2 * i] = g[i].real(); g2[2 * i + 1] = g[i].imag(); }
    s = lhaf_rpt_mixed(A2.data(), g2.data(), n, M, lh);
    if (s != LHAF_OK) return s;
    val = cd(lh[0], lh[1]);
  }
  const cd p = pref * val / fact;
  out[0] = p.real();
  out[1] = p.imag();
  return LHAF_OK;
}

lhaf_status lhaf_ips_prob(const double *B, const double *alpha, int32_t M, const int32_t *n,
                          double out[2]) {
  if (!B || !alpha || !n || !out) return (lhaf_status)lhaf::set_error(LHAF_E_ARG, "null pointer");
  if (M < 1 || M > 4096) return (lhaf_status)lhaf::set_error(LHAF_E_ARG, "bad mode count");
  double fact = 1.0, expo = 0.0;
  for (int i = 0; i < M; ++i) {
    if (n[i] < 0) return (lhaf_status)lhaf::set_error(LHAF_E_ARG, "negative photon count");
    for (int c = 2; c <= n[i]; ++c) fact *= (double)c;
  }
  // C = |B|^2 elementwise (its diagonal: the within-mode pair weight), loops |alpha|^2
  std::vector<double> C((size_t)2 * M * M, 0.0), g((size_t)2 * M, 0.0);
  for (size_t i = 0; i < (size_t)M * M; ++i) {
    const double a = B[2 * i] * B[2 * i] + B[2 * i + 1] * B[2 * i + 1];
    C[2 * i] = a;
    expo += 0.5 * a;
  }
  for (int i = 0; i < M; ++i) {
    const double a = alpha[2 * i] * alpha[2 * i] + alpha[2 * i + 1] * alpha[2 * i + 1];
    g[2 * i] = a;
    expo += a;
  }
  double lh[2];
  const lhaf_status s = lhaf_rpt(C.data(), g.data(), n, M, lh);
  if (s != LHAF_OK) return s;
  out[0] = std::exp(-expo) * lh[0] / fact;
  out[1] = std::exp(-expo) * lh[1] / fact;
  return LHAF_OK;
}

}  // extern "C"
