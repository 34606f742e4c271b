// lhaf_tree.cu -- kernel variant 6: the sieve terms of a pattern as the leaves of a tree that
// shares every prefix of eliminated pairs.  Product code only.
//
// One sieve term (P:431-435 with X -> X_w, reading C4):
//   F_w(lam) = det(I - lam C X_w)^{-1/2} exp(1/2 lam z^T (I - lam C X_w)^{-1} v),  g(w) = [lam^n] F_w,
// z^T = v^T X_w.  With W = diag(w) (a pair's two indices carry the same weight) and X the pair
// swap, I - lam C X W = (W^{-1}X - lam C) X W, so with the complex-symmetric Y = W^{-1}X - lam C
//   det(I - lam C X_w) = det(X) det(W) det(Y),   z^T (I - lam C X_w)^{-1} v = v^T Y^{-1} v.
// Y's constant part couples only the two indices of a pair: pairs are eliminated one at a time
// with 2x2 block pivots whose constant part [[0, 1/w], [1/w, 0]] is invertible (no pivoting,
// no division by anything but a series with constant term 1).  Writing the live part as
// Y = W^{-1}X - lam K (K = C at the root), eliminating pair (a, b) with weight w gives
//   D  = -w^2 det(Y_pp) = 1 - 2 w lam K_ab + w^2 lam^2 (K_ab^2 - K_aa K_bb)       (D(0) = 1)
//   Q  = D^{-1} [[lam w^2 K_bb, w - lam w^2 K_ab], [w - lam w^2 K_ab, lam w^2 K_aa]]
//   K' = K_rr + lam (u, x) Q (u, x)^T          (u = K_{r,a}, x = K_{r,b})
// and det(I - lam C X_w) = prod D over the eliminated pairs.  A weight of 0 (an even eta with
// k = eta/2) gives D = 1, Q = 0: the pair is deleted.  The loop vector is a border index
// 0 (K_00 = 0, K_0j = -v_j at the root); after the last pair K_00 = lam v^T Y^{-1} v, so
//   F_w = exp(1/2 (K_00 - sum_p log D_p)).
// A pair's weight enters only when that pair is eliminated, so all terms that share the weights
// of the first k eliminated pairs share the first k Schur complements: depth k of the tree
// eliminates pair H-1-k (tree order) once per digit, and the leaves are the sieve terms.  Every
// series is truncated at lam^n (L = n + 1 coefficients).  Halving (term(t) = term(T-1-t),
// reading C6) keeps the first (eta+1)/2 digits of the root pair (odd eta).
//
// Layout (HBM): a level buffer holds the nodes of one depth, structure-of-arrays with the node
// index fastest -- K[(s * NE + e) * cap + node] (coefficient s, packed lower-triangle entry
// e = i(i+1)/2 + j, j <= i), logc[s * cap + node], coef[node] -- so that threads working on
// consecutive nodes (or consecutive children of one parent) read consecutive addresses.  Index
// layout inside a node: [border] p_0 q_0 p_1 q_1 ...: the pair eliminated next is the last two
// indices, and a child's matrix is the leading block of its parent's (the same packed prefix).
#include <algorithm>
#include <cmath>
#include <vector>

#include "lhaf_device.cuh"

namespace lhaf {
namespace tree {

constexpr int TB = 8;  // output block of the blocked truncated series products

struct SR {  // series view: element s at p[s * st]
  const double2 *p;
  int64_t st;
};
__device__ __forceinline__ double2 at(const SR &r, int i) { return r.p[(int64_t)i * r.st]; }
__device__ __forceinline__ int tri(int i, int j) { return i * (i + 1) / 2 + j; }

// acc[k] += sum_{s + q = t0 + k - sh} a[s] b[q]   (0 <= s < La, 0 <= q < Lb; k < TB)
// The b operand streams through a TB-slot window in registers (one new value per step, slot
// indices resolved at compile time by unrolling the steps by TB): two loads per TB complex MACs.
__device__ __forceinline__ void conv_acc(double2 (&acc)[TB], int t0, int sh, SR a, int La, SR b, int Lb) {
  const int base = t0 - sh;
  const int s_lo = max(0, base - (Lb - 1));
  const int s_hi = min(La - 1, base + TB - 1);
  if (s_lo > s_hi) return;
  const int Q0 = base - s_lo;  // q of output k = 0 at step 0
  double2 w[TB];
#pragma unroll
  for (int k = 0; k < TB; ++k) {
    const int q = Q0 + k;
    w[k] = (q >= 0 && q < Lb) ? at(b, q) : c0();
  }
  const int nsteps = s_hi - s_lo + 1;
  for (int r0 = 0; r0 < nsteps; r0 += TB) {
#pragma unroll
    for (int rho = 0; rho < TB; ++rho) {
      const int r = r0 + rho;
      if (r < nsteps) {
        if (r > 0) {  // the value output 0 needs now; output k reads slot (k - r) mod TB
          const int q = Q0 - r;
          w[(TB - rho) % TB] = (q >= 0 && q < Lb) ? at(b, q) : c0();
        }
        const double2 av = at(a, s_lo + r);
#pragma unroll
        for (int k = 0; k < TB; ++k) acc[k] = cfma(av, w[(k - rho + TB) % TB], acc[k]);
      }
    }
  }
}

// R = 1/D for D_0 = 1: R_t = -sum_{s=1}^{t} D_s R_{t-s}, blocked by TB (earlier blocks by
// conv_acc, the block itself by forward substitution)
__device__ __forceinline__ void ser_recip(double2 *R, int64_t st, const double2 *D, int L) {
  double2 dl[TB];
#pragma unroll
  for (int k = 0; k < TB; ++k) dl[k] = (k >= 1 && k < L) ? D[(int64_t)k * st] : c0();
  for (int t0 = 0; t0 < L; t0 += TB) {
    double2 acc[TB];
#pragma unroll
    for (int k = 0; k < TB; ++k) acc[k] = c0();
    if (t0 > 0) conv_acc(acc, t0, 1, SR{D + st, st}, L - 1, SR{R, st}, t0);
    double2 r[TB];
#pragma unroll
    for (int k = 0; k < TB; ++k) {
      double2 x = (t0 + k == 0) ? c1() : make_double2(-acc[k].x, -acc[k].y);
#pragma unroll
      for (int q = 0; q < k; ++q) x = cfms(dl[k - q], r[q], x);
      r[k] = x;
    }
#pragma unroll
    for (int k = 0; k < TB; ++k)
      if (t0 + k < L) R[(int64_t)(t0 + k) * st] = r[k];
  }
}

// E = exp(phi) for phi_0 = 0 from Psi_j = j phi_j:  m E_m = sum_{j=1}^{m} Psi_j E_{m-j}
__device__ __forceinline__ void ser_exp(double2 *Ev, int64_t st, const double2 *Psi, int L) {
  double2 pl[TB];
#pragma unroll
  for (int k = 0; k < TB; ++k) pl[k] = (k >= 1 && k < L) ? Psi[(int64_t)k * st] : c0();
  for (int t0 = 0; t0 < L; t0 += TB) {
    double2 acc[TB];
#pragma unroll
    for (int k = 0; k < TB; ++k) acc[k] = c0();
    if (t0 > 0) conv_acc(acc, t0, 1, SR{Psi + st, st}, L - 1, SR{Ev, st}, t0);
    double2 e[TB];
#pragma unroll
    for (int k = 0; k < TB; ++k) {
      double2 x = acc[k];
#pragma unroll
      for (int q = 0; q < k; ++q) x = cfma(pl[k - q], e[q], x);
      const int m = t0 + k;
      e[k] = (m == 0) ? c1() : cscale(x, 1.0 / m);
    }
#pragma unroll
    for (int k = 0; k < TB; ++k)
      if (t0 + k < L) Ev[(int64_t)(t0 + k) * st] = e[k];
  }
}

__device__ __forceinline__ double binom_d(int e, int k) {
  double c = 1.0;
  for (int i = 1; i <= k; ++i) c = c * (double)(e - k + i) / (double)i;
  return c;
}

// The pivot of one child: D, R = 1/D, log D (added to the parent's log c), Q.
// S: scratch [3][L] at stride st (D, R, s*D_s); Qo: [3][L] at stride st (q11, q12, q22).
__device__ __forceinline__ void pivot(const SR &Kaa, const SR &Kbb, const SR &Kab, int L, int w,
                                      double2 *S, double2 *Qo, int64_t st, const SR &logc_par,
                                      double2 *logc_out, int64_t lst, double2 *psi_out, double2 *Rcopy) {
  double2 *Dp = S, *Rp = S + (int64_t)L * st, *D2p = S + 2 * (int64_t)L * st;
  const double wd = (double)w, w2 = wd * wd;
  for (int t0 = 0; t0 < L; t0 += TB) {
    double2 p1[TB], p2[TB];
#pragma unroll
    for (int k = 0; k < TB; ++k) p1[k] = p2[k] = c0();
    if (w != 0) {
      conv_acc(p1, t0, 2, Kab, L, Kab, L);
      conv_acc(p2, t0, 2, Kaa, L, Kbb, L);
    }
#pragma unroll
    for (int k = 0; k < TB; ++k) {
      const int t = t0 + k;
      if (t < L) {
        double2 d = cscale(csub(p1[k], p2[k]), w2);
        if (t >= 1 && w != 0) {
          const double2 kab = at(Kab, t - 1);
          d.x -= 2.0 * wd * kab.x;
          d.y -= 2.0 * wd * kab.y;
        }
        if (t == 0) d = c1();
        Dp[(int64_t)t * st] = d;
        D2p[(int64_t)t * st] = cscale(d, (double)t);
      }
    }
  }
  ser_recip(Rp, st, Dp, L);
  // t log D_t = sum_s (s D_s) R_{t-s}
  for (int t0 = 0; t0 < L; t0 += TB) {
    double2 acc[TB];
#pragma unroll
    for (int k = 0; k < TB; ++k) acc[k] = c0();
    conv_acc(acc, t0, 0, SR{D2p, st}, L, SR{Rp, st}, L);
#pragma unroll
    for (int k = 0; k < TB; ++k) {
      const int t = t0 + k;
      if (t < L) {
        if (logc_out) {
          const double2 lg = t > 0 ? cscale(acc[k], 1.0 / t) : c0();
          logc_out[(int64_t)t * lst] = cadd(at(logc_par, t), lg);
        }
        if (psi_out) psi_out[(int64_t)t * st] = acc[k];  // t log D_t
      }
    }
  }
  if (!Qo) return;
  double2 *q11 = Qo, *q12 = Qo + (int64_t)L * st, *q22 = Qo + 2 * (int64_t)L * st;
  const SR R{Rp, st};
  for (int t0 = 0; t0 < L; t0 += TB) {
    double2 a1[TB], a2[TB], a3[TB];
#pragma unroll
    for (int k = 0; k < TB; ++k) a1[k] = a2[k] = a3[k] = c0();
    if (w != 0) {
      conv_acc(a1, t0, 1, Kbb, L, R, L);
      conv_acc(a2, t0, 1, Kaa, L, R, L);
      conv_acc(a3, t0, 1, Kab, L, R, L);
    }
#pragma unroll
    for (int k = 0; k < TB; ++k) {
      const int t = t0 + k;
      if (t < L) {
        const double2 r = at(R, t);
        q11[(int64_t)t * st] = cscale(a1[k], w2);
        q22[(int64_t)t * st] = cscale(a2[k], w2);
        q12[(int64_t)t * st] = make_double2(wd * r.x - w2 * a3[k].x, wd * r.y - w2 * a3[k].y);
      }
    }
  }
  (void)Rcopy;
}

struct TStep {  // parent depth k -> children at depth k + 1, one chunk of children
  TLevel par, ch;
  uint64_t pbase;  // global index of the parent buffer's slot 0
  uint64_t c0;     // global index of the first child (slot 0 of the child buffer)
  uint64_t nc;     // children in the chunk
  int L, E, b, dmin, eta;
  double2 *Q;  // [3][L][nc]
  double2 *T;  // [2][L][E-2][nc]
  double2 *S;  // [3][L][nc]
};

__global__ void __launch_bounds__(128) tree_pivot_k(TStep P) {
  const uint64_t i = (uint64_t)blockIdx.x * 128 + threadIdx.x;
  if (i >= P.nc) return;
  const uint64_t c = P.c0 + i, pg = c / P.b, ps = pg - P.pbase;
  const int kh = P.dmin + (int)(c - pg * P.b), w = P.eta - 2 * kh;
  const int L = P.L, E = P.E, NE = E * (E + 1) / 2, a = E - 2, b = E - 1;
  const int64_t kst = (int64_t)NE * P.par.cap;
  const SR Kaa{P.par.K + (int64_t)tri(a, a) * P.par.cap + ps, kst};
  const SR Kbb{P.par.K + (int64_t)tri(b, b) * P.par.cap + ps, kst};
  const SR Kab{P.par.K + (int64_t)tri(b, a) * P.par.cap + ps, kst};
  const int64_t st = (int64_t)P.nc;
  pivot(Kaa, Kbb, Kab, L, w, P.S + i, P.Q + i, st, SR{P.par.logc + ps, (int64_t)P.par.cap},
        P.ch.logc + i, (int64_t)P.ch.cap, nullptr, nullptr);
  P.ch.coef[i] = P.par.coef[ps] * ((kh & 1) ? -1.0 : 1.0) * binom_d(P.eta, kh);
}

// T_j = Q (u_j, x_j)^T for every live index j of every child (thread per (j, child))
__global__ void __launch_bounds__(128) tree_tmat_k(TStep P) {
  const int Ep = P.E - 2;
  const uint64_t i = (uint64_t)blockIdx.x * 128 + threadIdx.x;
  if (i >= P.nc * (uint64_t)Ep) return;
  const uint64_t ci = i % P.nc;
  const int j = (int)(i / P.nc);
  const uint64_t ps = (P.c0 + ci) / P.b - P.pbase;
  const int L = P.L, E = P.E, NE = E * (E + 1) / 2, a = E - 2, b = E - 1;
  const int64_t kst = (int64_t)NE * P.par.cap, st = (int64_t)P.nc;
  const SR u{P.par.K + (int64_t)tri(a, j) * P.par.cap + ps, kst};
  const SR x{P.par.K + (int64_t)tri(b, j) * P.par.cap + ps, kst};
  const SR q11{P.Q + ci, st}, q12{P.Q + (int64_t)L * st + ci, st}, q22{P.Q + 2 * (int64_t)L * st + ci, st};
  double2 *T1 = P.T + (int64_t)j * st + ci, *T2 = P.T + ((int64_t)L * Ep + j) * st + ci;
  const int64_t tst = (int64_t)Ep * st;
  const int Lo = L - 1;  // T enters K' at lam^1: degrees <= L - 2
  for (int t0 = 0; t0 < Lo; t0 += TB) {
    double2 a1[TB], a2[TB];
#pragma unroll
    for (int k = 0; k < TB; ++k) a1[k] = a2[k] = c0();
    conv_acc(a1, t0, 0, q11, Lo, u, Lo);
    conv_acc(a1, t0, 0, q12, Lo, x, Lo);
    conv_acc(a2, t0, 0, q12, Lo, u, Lo);
    conv_acc(a2, t0, 0, q22, Lo, x, Lo);
#pragma unroll
    for (int k = 0; k < TB; ++k)
      if (t0 + k < Lo) {
        T1[(int64_t)(t0 + k) * tst] = a1[k];
        T2[(int64_t)(t0 + k) * tst] = a2[k];
      }
  }
}

// K'_ij = K_ij + lam (u_i T1_j + x_i T2_j) for the packed lower triangle of every child
__global__ void __launch_bounds__(128) tree_update_k(TStep P) {
  const int Ep = P.E - 2, NEc = Ep * (Ep + 1) / 2;
  const uint64_t i = (uint64_t)blockIdx.x * 128 + threadIdx.x;
  if (i >= P.nc * (uint64_t)NEc) return;
  const uint64_t ci = i % P.nc;
  const int e = (int)(i / P.nc);
  int ii = (int)((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);
  while (tri(ii + 1, 0) <= e) ++ii;
  while (tri(ii, 0) > e) --ii;
  const int jj = e - tri(ii, 0);
  const uint64_t ps = (P.c0 + ci) / P.b - P.pbase;
  const int L = P.L, E = P.E, NE = E * (E + 1) / 2, a = E - 2, b = E - 1;
  const int64_t kst = (int64_t)NE * P.par.cap, st = (int64_t)P.nc, tst = (int64_t)Ep * st;
  const SR u{P.par.K + (int64_t)tri(a, ii) * P.par.cap + ps, kst};
  const SR x{P.par.K + (int64_t)tri(b, ii) * P.par.cap + ps, kst};
  const SR K{P.par.K + (int64_t)e * P.par.cap + ps, kst};
  const SR T1{P.T + (int64_t)jj * st + ci, tst}, T2{P.T + ((int64_t)L * Ep + jj) * st + ci, tst};
  double2 *out = P.ch.K + (int64_t)e * P.ch.cap + ci;
  const int64_t ost = (int64_t)NEc * P.ch.cap;
  for (int t0 = 0; t0 < L; t0 += TB) {
    double2 acc[TB];
#pragma unroll
    for (int k = 0; k < TB; ++k) acc[k] = (t0 + k < L) ? at(K, t0 + k) : c0();
    conv_acc(acc, t0, 1, u, L - 1, T1, L - 1);
    conv_acc(acc, t0, 1, x, L - 1, T2, L - 1);
#pragma unroll
    for (int k = 0; k < TB; ++k)
      if (t0 + k < L) out[(int64_t)(t0 + k) * ost] = acc[k];
  }
}

struct TLeaf {
  TLevel par;      // nodes at depth H-1 (one pair left, plus the border)
  uint64_t pbase;  // global index of slot 0 (= first node of the chunk)
  uint64_t np;     // nodes in the chunk
  int L, E, bord, b, dmin, eta;
  double2 *S;      // scratch [9][L][np]
  double2 *val;    // [np]: sum over the node's leaves of sign * prod C * g
  double *absv;    // [np]: the same sum of |.|
};

// The last pair of every node: its (eta + 1) leaves (or the halved root digits when H = 1).
__global__ void __launch_bounds__(128) tree_leaf_k(TLeaf P) {
  const uint64_t i = (uint64_t)blockIdx.x * 128 + threadIdx.x;
  if (i >= P.np) return;
  const int L = P.L, E = P.E, NE = E * (E + 1) / 2, a = E - 2, b = E - 1;
  const int64_t kst = (int64_t)NE * P.par.cap, st = (int64_t)P.np;
  const SR Kaa{P.par.K + (int64_t)tri(a, a) * P.par.cap + i, kst};
  const SR Kbb{P.par.K + (int64_t)tri(b, b) * P.par.cap + i, kst};
  const SR Kab{P.par.K + (int64_t)tri(b, a) * P.par.cap + i, kst};
  const SR logc{P.par.logc + i, (int64_t)P.par.cap};
  double2 *S = P.S + i;                                   // D, R, sD
  double2 *Qo = P.S + 3 * (int64_t)L * st + i;            // q11, q12, q22
  double2 *Psi = P.S + 6 * (int64_t)L * st + i;           // t log D_t, then Psi
  double2 *T1 = P.S + 7 * (int64_t)L * st + i, *T2 = P.S + 8 * (int64_t)L * st + i;
  const double coef = P.par.coef[i];
  double2 vsum = c0();
  double asum = 0.0;
  for (int d = 0; d < P.b; ++d) {
    const int kh = P.dmin + d, w = P.eta - 2 * kh;
    pivot(Kaa, Kbb, Kab, L, w, S, P.bord ? Qo : nullptr, st, logc, nullptr, 0, Psi, nullptr);
    // Psi_t = t phi_t, phi = 1/2 (K'_00 - log c - log D)
    if (P.bord) {
      const SR u{P.par.K + (int64_t)tri(a, 0) * P.par.cap + i, kst};
      const SR x{P.par.K + (int64_t)tri(b, 0) * P.par.cap + i, kst};
      const SR q11{Qo, st}, q12{Qo + (int64_t)L * st, st}, q22{Qo + 2 * (int64_t)L * st, st};
      const int Lo = L - 1;
      for (int t0 = 0; t0 < Lo; t0 += TB) {
        double2 a1[TB], a2[TB];
#pragma unroll
        for (int k = 0; k < TB; ++k) a1[k] = a2[k] = c0();
        conv_acc(a1, t0, 0, q11, Lo, u, Lo);
        conv_acc(a1, t0, 0, q12, Lo, x, Lo);
        conv_acc(a2, t0, 0, q12, Lo, u, Lo);
        conv_acc(a2, t0, 0, q22, Lo, x, Lo);
#pragma unroll
        for (int k = 0; k < TB; ++k)
          if (t0 + k < Lo) {
            T1[(int64_t)(t0 + k) * st] = a1[k];
            T2[(int64_t)(t0 + k) * st] = a2[k];
          }
      }
      const SR K00{P.par.K + i, kst};
      for (int t0 = 0; t0 < L; t0 += TB) {
        double2 acc[TB];
#pragma unroll
        for (int k = 0; k < TB; ++k) acc[k] = (t0 + k < L) ? at(K00, t0 + k) : c0();
        conv_acc(acc, t0, 1, u, Lo, SR{T1, st}, Lo);
        conv_acc(acc, t0, 1, x, Lo, SR{T2, st}, Lo);
#pragma unroll
        for (int k = 0; k < TB; ++k) {
          const int t = t0 + k;
          if (t < L) {
            const double2 k00 = acc[k], lc = at(logc, t), tl = Psi[(int64_t)t * st];
            Psi[(int64_t)t * st] = make_double2(0.5 * (t * (k00.x - lc.x) - tl.x), 0.5 * (t * (k00.y - lc.y) - tl.y));
          }
        }
      }
    } else {
      for (int t = 0; t < L; ++t) {
        const double2 lc = at(logc, t), tl = Psi[(int64_t)t * st];
        Psi[(int64_t)t * st] = make_double2(-0.5 * (t * lc.x + tl.x), -0.5 * (t * lc.y + tl.y));
      }
    }
    double2 *Ev = S;  // reuse D's slots
    ser_exp(Ev, st, Psi, L);
    const double2 g = Ev[(int64_t)(L - 1) * st];
    const double f = coef * ((kh & 1) ? -1.0 : 1.0) * binom_d(P.eta, kh);
    vsum.x = fma(f, g.x, vsum.x);
    vsum.y = fma(f, g.y, vsum.y);
    asum += fabs(f) * hypot(g.x, g.y);
  }
  P.val[i] = vsum;
  P.absv[i] = asum;
}

// Whole units of the chunk: one warp per unit sums its per-node values in a fixed order
// (double-double) and writes the unit's partial.
__global__ void __launch_bounds__(128) tree_reduce_k(const double2 *val, const double *absv,
                                                     uint64_t units, uint64_t per_unit, uint64_t unit0,
                                                     Partial *partials) {
  const uint64_t u = (uint64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (u >= units) return;
  double rh = 0, rl = 0, ih = 0, il = 0, ah = 0, al = 0;
  for (uint64_t m = lane; m < per_unit; m += 32) {
    const double2 v = val[u * per_unit + m];
    dd_add(rh, rl, v.x);
    dd_add(ih, il, v.y);
    dd_add(ah, al, absv[u * per_unit + m]);
  }
#pragma unroll
  for (int s = 16; s; s >>= 1) {
    const double orh = __shfl_xor_sync(LHAF_FULL, rh, s), orl = __shfl_xor_sync(LHAF_FULL, rl, s);
    const double oih = __shfl_xor_sync(LHAF_FULL, ih, s), oil = __shfl_xor_sync(LHAF_FULL, il, s);
    const double oah = __shfl_xor_sync(LHAF_FULL, ah, s), oal = __shfl_xor_sync(LHAF_FULL, al, s);
    // combine in a lane-order-independent way: the lower lane's value first
    if (lane & s) {
      double th = orh, tl = orl; dd_add_dd(th, tl, rh, rl); rh = th; rl = tl;
      th = oih; tl = oil; dd_add_dd(th, tl, ih, il); ih = th; il = tl;
      th = oah; tl = oal; dd_add_dd(th, tl, ah, al); ah = th; al = tl;
    } else {
      dd_add_dd(rh, rl, orh, orl);
      dd_add_dd(ih, il, oih, oil);
      dd_add_dd(ah, al, oah, oal);
    }
  }
  if (lane == 0) {
    Partial q;
    q.re_hi = rh; q.re_lo = rl; q.im_hi = ih; q.im_lo = il; q.abs_hi = ah; q.abs_lo = al;
    q.pad0 = q.pad1 = 0.0;
    partials[unit0 + u] = q;
  }
}

// Root nodes of patterns pats[g0 .. g0 + n): K = C (tree index order, border first), degree 0.
__global__ void __launch_bounds__(128) tree_root_k(JobDev J, const int32_t *pats, uint64_t g0, uint64_t n,
                                                   TLevel out, int L, int E, int bord) {
  const int NE = E * (E + 1) / 2;
  const uint64_t i = (uint64_t)blockIdx.x * 128 + threadIdx.x;
  if (i >= n * (uint64_t)NE) return;
  const uint64_t slot = i % n;
  const int e = (int)(i / n);
  int ii = (int)((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);
  while (tri(ii + 1, 0) <= e) ++ii;
  while (tri(ii, 0) > e) --ii;
  const int jj = e - tri(ii, 0);
  const PatDesc P = J.descs[pats[g0 + slot]];
  const int H = P.H;
  const int32_t *r = J.ipool + P.idx_off;
  auto mode = [&](int t) {  // tree index -> mode of A (-1: phantom)
    const int h = (t - bord) >> 1, side = (t - bord) & 1;
    return r[side * H + h];
  };
  double2 v = c0();
  if (bord && jj == 0) {
    if (ii > 0) {
      const int m = mode(ii);
      const double2 gm = m < 0 ? c1() : J.gamma[P.gamma_off + m];
      v = make_double2(-gm.x, -gm.y);
    }
  } else {
    const int mi = mode(ii), mj = mode(jj);
    if (mi >= 0 && mj >= 0) v = J.A[(int64_t)mi * J.kdim + mj];
  }
  const int64_t st = (int64_t)NE * out.cap;
  double2 *o = out.K + (int64_t)e * out.cap + slot;
  o[0] = v;
  for (int s = 1; s < L; ++s) o[(int64_t)s * st] = c0();
  if (e == 0) {
    for (int s = 0; s < L; ++s) out.logc[(int64_t)s * out.cap + slot] = c0();
    out.coef[slot] = 1.0;
  }
}

// ------------------------------------------------------------------ host driver

static cudaError_t grow(void **p, size_t &have, size_t need) {
  if (need <= have) return cudaSuccess;
  if (*p) cudaFree(*p);
  *p = nullptr;
  have = 0;
  cudaError_t e = cudaMalloc(p, need);
  if (e == cudaSuccess) have = need;
  return e;
}

static inline unsigned blocks_for(uint64_t n) { return (unsigned)((n + 127) / 128); }

struct Runner {
  const JobDev &J;
  TreeGroup &g;
  TreeWork &w;
  cudaStream_t st;
  uint64_t U0, U1;  // requested group-local units
  int L, H;
  std::vector<int> E, b, dmin, eta;   // per depth k: dimension, branches, first digit, eta
  std::vector<uint64_t> cap, Pk;      // per depth: node capacity; nodes per unit (k >= k_u)

  uint64_t desc_to_ku(int k) const {  // nodes at depth k_u per node at depth k (k <= k_u)
    uint64_t q = 1;
    for (int l = k; l < g.k_u; ++l) q *= (uint64_t)b[l];
    return q;
  }

  cudaError_t level_alloc(int k) {
    const int NE = E[k] * (E[k] + 1) / 2;
    TLevel &T = w.lv[k];
    T.cap = cap[k];
    cudaError_t e = grow((void **)&T.K, w.kbytes[k], (size_t)L * NE * cap[k] * sizeof(double2));
    if (e == cudaSuccess) e = grow((void **)&T.logc, w.lbytes[k], (size_t)L * cap[k] * sizeof(double2));
    if (e == cudaSuccess) e = grow((void **)&T.coef, w.cbytes[k], (size_t)cap[k] * sizeof(double));
    return e;
  }

  cudaError_t leaf(uint64_t gs, uint64_t cnt) {
    const int k = H - 1;
    TLeaf P;
    P.par = w.lv[k];
    P.pbase = gs;
    P.np = cnt;
    P.L = L; P.E = E[k]; P.bord = g.bord; P.b = b[k]; P.dmin = dmin[k]; P.eta = eta[k];
    P.S = (double2 *)w.scratch;
    P.val = (double2 *)w.val;
    P.absv = (double *)w.absv;
    tree_leaf_k<<<blocks_for(cnt), 128, 0, st>>>(P);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const uint64_t per = Pk[k], units = cnt / per;
    tree_reduce_k<<<(unsigned)((units + 3) / 4), 128, 0, st>>>(P.val, P.absv, units, per,
                                                              g.unit_base + gs / per, J.partials);
    return cudaGetLastError();
  }

  cudaError_t expand(int k, uint64_t gs, uint64_t cnt) {
    if (k == H - 1) return leaf(gs, cnt);
    const uint64_t nb = (uint64_t)b[k];
    uint64_t lo = gs * nb, hi = (gs + cnt) * nb;
    if (k + 1 <= g.k_u) {
      const uint64_t q = desc_to_ku(k + 1);
      lo = std::max(lo, U0 / q);
      hi = std::min(hi, (U1 - 1) / q + 1);
    }
    uint64_t chunk = cap[k + 1];
    for (uint64_t c = lo; c < hi; c += chunk) {
      const uint64_t n = std::min(chunk, hi - c);
      TStep P;
      P.par = w.lv[k];
      P.ch = w.lv[k + 1];
      P.pbase = gs;
      P.c0 = c;
      P.nc = n;
      P.L = L; P.E = E[k]; P.b = b[k]; P.dmin = dmin[k]; P.eta = eta[k];
      const int Ep = E[k] - 2;
      P.S = (double2 *)w.scratch;
      P.Q = P.S + (size_t)3 * L * n;
      P.T = P.Q + (size_t)3 * L * n;
      tree_pivot_k<<<blocks_for(n), 128, 0, st>>>(P);
      if (Ep > 0) {
        tree_tmat_k<<<blocks_for(n * Ep), 128, 0, st>>>(P);
        tree_update_k<<<blocks_for(n * (uint64_t)(Ep * (Ep + 1) / 2)), 128, 0, st>>>(P);
      }
      cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) return e;
      e = expand(k + 1, c, n);
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  }

  cudaError_t run() {
    // roots: group patterns [U0 / units_pp, (U1 - 1) / units_pp]
    const uint64_t p0 = U0 / g.units_pp, p1 = (U1 - 1) / g.units_pp + 1;
    for (uint64_t p = p0; p < p1; p += cap[0]) {
      const uint64_t n = std::min(cap[0], p1 - p);
      const int NE = E[0] * (E[0] + 1) / 2;
      tree_root_k<<<blocks_for(n * NE), 128, 0, st>>>(J, g.d_pats, p, n, w.lv[0], L, E[0], g.bord);
      cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) return e;
      e = expand(0, p, n);
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  }
};

}  // namespace tree

// Work units of a tree group: the nodes at depth k_u.  Chunks below k_u always
// hold whole units, and a unit's partial is one fixed-order sum: results do not depend on the
// requested range (rank count, slicing).
void tree_plan_group(TreeGroup &g, uint64_t target_units) {
  const int H = g.H;
  std::vector<uint64_t> b(H);
  for (int k = 0; k < H; ++k) {
    const int e = g.eta[H - 1 - k];
    b[k] = (uint64_t)((k == 0 && g.halve) ? (e + 1) / 2 : e + 1);
  }
  const int L = g.n + 1;
  auto node_bytes = [&](int k) {
    const int E = 2 * (H - k) + g.bord;
    return (double)(E * (E + 1) / 2 + 1) * L * 16.0 + 8.0;
  };
  int ku = 0;
  uint64_t N = 1;
  while (ku < H - 1 && (uint64_t)g.npat * N < target_units) N *= b[ku++];
  // a unit's descendants must fit one level buffer at every depth below it
  for (;;) {
    bool fits = true;
    uint64_t P = 1;
    for (int k = ku + 1; k < H && fits; ++k) {
      P *= b[k - 1];
      if ((double)P * node_bytes(k) > (double)TreeWork::kLevelBudget) fits = false;
    }
    if (fits || ku >= H - 1) break;
    N *= b[ku++];
  }
  g.k_u = ku;
  g.units_pp = N;
}

double tree_cmacs_per_term(const TreeGroup &g) {
  // complex MACs of the kernels above for the whole tree of one pattern / evaluated leaves
  const int H = g.H, L = g.n + 1;
  auto conv = [](int Lo, int sh, int La, int Lb) {
    double c = 0;
    for (int t = 0; t < Lo; ++t) {
      const int base = t - sh;
      for (int s = 0; s < La; ++s)
        if (base - s >= 0 && base - s < Lb) c += 1;
    }
    return c;
  };
  const double piv = 2 * conv(L, 2, L, L) + conv(L, 1, L - 1, L) + conv(L, 0, L, L) + 3 * conv(L, 1, L, L);
  const double tm = 4 * conv(L - 1, 0, L - 1, L - 1), up = 2 * conv(L, 1, L - 1, L - 1);
  const double ex = conv(L, 1, L - 1, L);
  double nodes = 1, total = 0, leaves = 0;
  for (int k = 0; k < H; ++k) {
    const int e = g.eta[H - 1 - k];
    const double bk = (k == 0 && g.halve) ? (e + 1) / 2 : e + 1;
    const int E = 2 * (H - k) + g.bord, Ep = E - 2;
    const double ch = nodes * bk;
    if (k < H - 1) {
      total += ch * (piv + Ep * tm + (Ep * (Ep + 1) / 2.0) * up);
    } else {
      total += ch * (piv - (g.bord ? 0 : 3 * conv(L, 1, L, L)) + (g.bord ? tm + up : 0) + ex);
      leaves = ch;
    }
    nodes = ch;
  }
  return leaves > 0 ? total / leaves : 0.0;
}

cudaError_t tree_run(const JobDev &J, TreeGroup &g, TreeWork &w, uint64_t ub, uint64_t ue, cudaStream_t st) {
  if (ue <= ub) return cudaSuccess;
  tree::Runner R{J, g, w, st, ub, ue, g.n + 1, g.H, {}, {}, {}, {}, {}, {}};
  const int H = g.H, L = g.n + 1;
  R.E.resize(H); R.b.resize(H); R.dmin.resize(H); R.eta.resize(H); R.cap.resize(H); R.Pk.resize(H);
  for (int k = 0; k < H; ++k) {
    R.eta[k] = g.eta[H - 1 - k];
    R.E[k] = 2 * (H - k) + g.bord;
    R.b[k] = (k == 0 && g.halve) ? (R.eta[k] + 1) / 2 : R.eta[k] + 1;
    R.dmin[k] = 0;
  }
  uint64_t P = 1;
  size_t scratch = 0;
  for (int k = 0; k < H; ++k) {
    if (k > g.k_u) P *= (uint64_t)R.b[k - 1];
    R.Pk[k] = k >= g.k_u ? P : 1;
    const int NE = R.E[k] * (R.E[k] + 1) / 2;
    const double nbytes = (double)(NE + 1) * L * 16.0 + 8.0;
    uint64_t c = (uint64_t)std::max(1.0, (double)TreeWork::kLevelBudget / nbytes);
    if (k == 0) c = std::min<uint64_t>(c, (uint64_t)g.npat);
    if (k >= g.k_u && k > 0) c = std::max<uint64_t>(1, c / R.Pk[k]) * R.Pk[k];
    R.cap[k] = c;
    // scratch of the transition into depth k (k >= 1) / of the leaf kernel (k = H - 1)
    if (k >= 1) scratch = std::max(scratch, (size_t)L * c * (6 + 2 * (size_t)(R.E[k - 1] - 2)));
    if (k == H - 1) scratch = std::max(scratch, (size_t)9 * L * c);
  }
  if (w.lv.size() < (size_t)H) {
    w.lv.resize(H, tree::TLevel{nullptr, nullptr, nullptr, 0});
    w.kbytes.resize(H, 0); w.lbytes.resize(H, 0); w.cbytes.resize(H, 0);
  }
  cudaError_t e = cudaSuccess;
  for (int k = 0; k < H && e == cudaSuccess; ++k) e = R.level_alloc(k);
  if (e == cudaSuccess) e = tree::grow(&w.scratch, w.scratch_bytes, scratch * sizeof(double2));
  if (e == cudaSuccess) e = tree::grow(&w.val, w.val_bytes, (size_t)R.cap[H - 1] * sizeof(double2));
  if (e == cudaSuccess) e = tree::grow(&w.absv, w.abs_bytes, (size_t)R.cap[H - 1] * sizeof(double));
  if (e != cudaSuccess) return e;
  return R.run();
}

void tree_work_free(TreeWork &w) {
  for (auto &l : w.lv) {
    if (l.K) cudaFree(l.K);
    if (l.logc) cudaFree(l.logc);
    if (l.coef) cudaFree(l.coef);
  }
  w.lv.clear();
  w.kbytes.clear(); w.lbytes.clear(); w.cbytes.clear();
  if (w.scratch) cudaFree(w.scratch);
  if (w.val) cudaFree(w.val);
  if (w.absv) cudaFree(w.absv);
  w.scratch = w.val = w.absv = nullptr;
  w.scratch_bytes = w.val_bytes = w.abs_bytes = 0;
}

}  // namespace lhaf
