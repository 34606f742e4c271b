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
// Layout (HBM): a level buffer holds the nodes of one depth, node-major with each series
// contiguous -- K[(node * NE + e) * L + s] (packed lower-triangle entry e = i(i+1)/2 + j, j <= i,
// coefficient s), logc[node * L + s], coef[node].  Index layout inside a node: [border] p_0 q_0
// p_1 q_1 ...: the pair eliminated next is the last two indices, so a child's matrix is the
// leading block of its parent's (the same packed prefix), and the two columns (u, x) of the
// eliminated pair restricted to the live indices are the first Ep entries of the parent's last
// two packed rows -- two contiguous runs of Ep * L coefficients.
//
// Kernels per depth transition: tree_pivot (thread per child: D, 1/D, log D, Q; series in
// registers for L <= 40), tree_bc (a block per group of children: the parent's (u, x) rows and
// the children's Q staged in shared memory, then T = Q (u, x)^T and the update K' = K + lam (u T1
// + x T2) from shared memory); the last pair: tree_leaf (thread per node, both leaves, the
// exp-series coefficient); tree_reduce (one block per work unit).
#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <vector>

#include "lhaf_device.cuh"

namespace lhaf {
namespace tree {

#ifndef LHAF_TREE_TB
#define LHAF_TREE_TB 8
#endif
constexpr int TB = LHAF_TREE_TB;  // output block of the blocked truncated series products

struct SR {  // series view: element s at p[s * st]
  const double2 *p;
  int64_t st;
};
__device__ __forceinline__ double2 at(const SR &r, int i) { return r.p[(int64_t)i * r.st]; }
__device__ __forceinline__ int tri(int i, int j) { return i * (i + 1) / 2 + j; }
// 16-byte global -> shared copies that bypass the registers (and L1)
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// acc[k] += sum_{s + q = t0 + k - sh} a[s] b[q]   (0 <= s < La, 0 <= q < Lb; k < TB)
// The b operand streams through a TB-slot window in registers (one new value per step, slot
// indices resolved at compile time by unrolling the steps by TB): two loads per TB complex MACs.
// acc[k] += av * w[(k - rho) mod TB] for the TB outputs, the first FMA of every output issued
// before the second (the two FMAs of one complex component are dependent: this order keeps
// 2 TB independent chains between them)
#ifndef LHAF_TWOPASS
#define LHAF_TWOPASS 1
#endif
#ifndef LHAF_RS_PREFETCH
#define LHAF_RS_PREFETCH 0
#endif
#ifndef LHAF_LEAF_PREFETCH
#define LHAF_LEAF_PREFETCH 0
#endif
#ifndef LHAF_PIVOT_TWO
#define LHAF_PIVOT_TWO 0
#endif
__device__ __forceinline__ void cfma_row(double2 (&acc)[TB], double2 av, const double2 (&w)[TB], const int RHO) {
  if (!LHAF_TWOPASS) {
#pragma unroll
    for (int k = 0; k < TB; ++k) acc[k] = cfma(av, w[(k - RHO + TB) % TB], acc[k]);
    return;
  }
  double2 t[TB];
#pragma unroll
  for (int k = 0; k < TB; ++k) {
    const double2 b = w[(k - RHO + TB) % TB];
    t[k].x = fma(av.x, b.x, acc[k].x);
    t[k].y = fma(av.x, b.y, acc[k].y);
  }
#pragma unroll
  for (int k = 0; k < TB; ++k) {
    const double2 b = w[(k - RHO + TB) % TB];
    acc[k].x = fma(-av.y, b.y, t[k].x);
    acc[k].y = fma(av.y, b.x, t[k].y);
  }
}

// Steps s <= base feed every output of the block (the windowed loop); the last steps s = base + j
// (j = 1 .. TB-1) feed only outputs k >= j with q = k - j (the triangle of the block, unrolled on
// b[0 .. TB-2] in registers, so that no MAC is spent on a zero).
__device__ __forceinline__ void conv_acc(double2 (&acc)[TB], int t0, int sh, SR a, int La, SR b, int Lb) {
  const int base = t0 - sh;
  const int s_lo = max(0, base - (Lb - 1));
  const int s_hi = min(La - 1, base + TB - 1);
  if (s_lo > s_hi) return;
  const int s_top = min(s_hi, base);
  if (s_lo <= s_top) {
    // window: output k reads b[Q0 + k - r] at step r; for s <= base every index the steps load
    // lies in [0, Lb) (q = base - s >= 0 and q <= Q0 <= Lb - 1): only the first fill checks
    const int Q0 = base - s_lo;  // q of output k = 0 at step 0
    double2 w[TB];
#pragma unroll
    for (int k = 0; k < TB; ++k) {
      const int q = Q0 + k;
      w[k] = (q < Lb) ? at(b, q) : c0();
    }
    const int nsteps = s_top - s_lo + 1;
    const double2 *ap = a.p + (int64_t)s_lo * a.st, *bp = b.p + (int64_t)Q0 * b.st;
    for (int r0 = 0; r0 < nsteps; r0 += TB) {
#pragma unroll
      for (int rho = 0; rho < TB; ++rho) {
        const int r = r0 + rho;
        if (r < nsteps) {
          if (r > 0) w[(TB - rho) % TB] = bp[-(int64_t)r * b.st];
          cfma_row(acc, ap[(int64_t)r * a.st], w, rho);
        }
      }
    }
  }
  {  // triangle
    const int jlo = max(1, -base), jhi = s_hi - base;
    if (jlo <= jhi) {
      double2 bq[TB - 1];
#pragma unroll
      for (int q = 0; q < TB - 1; ++q) bq[q] = (q < Lb && q <= TB - 1 - jlo) ? at(b, q) : c0();
      const double2 *ap = a.p + (int64_t)base * a.st;
#pragma unroll
      for (int j = 1; j < TB; ++j) {
        if (j >= jlo && j <= jhi) {
          const double2 av = ap[(int64_t)j * a.st];
#pragma unroll
          for (int k = j; k < TB; ++k) acc[k] = cfma(av, bq[k - j], acc[k]);
        }
      }
    }
  }
}

// conv_acc for unit-stride operands in shared memory, written for ONE inlined instance per kernel
// (tree_bc_k): full chunks of TB steps run without per-step guards, so ptxas hoists the two
// shared-memory loads of a step over the FMAs of the steps before it (with a guard per step a
// third of the loop's cycles were short-scoreboard stalls on the first FMA after the loads,
// profiles/r02/s5/ncu_bc_order1.json); the last nsteps mod TB steps leave by one forward branch.
__device__ __forceinline__ void conv_acc1(double2 (&acc)[TB], int t0, int sh, const double2 *a, int La,
                                          const double2 *b, int Lb) {
  const int base = t0 - sh;
  const int s_lo = max(0, base - (Lb - 1));
  const int s_hi = min(La - 1, base + TB - 1);
  if (s_lo > s_hi) return;
  const int s_top = min(s_hi, base);
  if (s_lo <= s_top) {
    const int Q0 = base - s_lo;
    double2 w[TB];
#pragma unroll
    for (int k = 0; k < TB; ++k) {
      const int q = Q0 + k;
      w[k] = (q < Lb) ? b[q] : c0();
    }
    const int nsteps = s_top - s_lo + 1;
    const double2 *ap = a + s_lo, *bp = b + Q0;
    int r0 = 0;
    for (; r0 + TB <= nsteps; r0 += TB) {
#pragma unroll
      for (int rho = 0; rho < TB; ++rho) {
        w[(TB - rho) % TB] = bp[-(r0 + rho)];  // step 0 reloads w[0] = b[Q0]
        cfma_row(acc, ap[r0 + rho], w, rho);
      }
    }
    const int rem = nsteps - r0;
#pragma unroll
    for (int rho = 0; rho < TB - 1; ++rho) {
      if (rho >= rem) break;
      w[(TB - rho) % TB] = bp[-(r0 + rho)];
      cfma_row(acc, ap[r0 + rho], w, rho);
    }
  }
  {  // triangle
    const int jlo = max(1, -base), jhi = s_hi - base;
    if (jlo == 1 && jhi == TB - 1 && Lb >= TB - 1) {
      double2 bq[TB - 1];
#pragma unroll
      for (int q = 0; q < TB - 1; ++q) bq[q] = b[q];
      const double2 *ap = a + base;
#pragma unroll
      for (int j = 1; j < TB; ++j) {
        const double2 av = ap[j];
#pragma unroll
        for (int k = j; k < TB; ++k) acc[k] = cfma(av, bq[k - j], acc[k]);
      }
    } else if (jlo <= jhi) {
      double2 bq[TB - 1];
#pragma unroll
      for (int q = 0; q < TB - 1; ++q) bq[q] = (q < Lb && q <= TB - 1 - jlo) ? b[q] : c0();
      const double2 *ap = a + base;
#pragma unroll
      for (int j = 1; j < TB; ++j) {
        if (j >= jlo && j <= jhi) {
          const double2 av = ap[j];
#pragma unroll
          for (int k = j; k < TB; ++k) acc[k] = cfma(av, bq[k - j], acc[k]);
        }
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


// ================================================================ register-array series (L <= LM)
// Series of length L <= LM held in registers (compile-time indices, fully unrolled loops with
// uniform early exits at runtime L).  One operand may stream from memory (a[s], contiguous).

template <int LM>
__device__ __forceinline__ void rz(double2 (&A)[LM]) {
#pragma unroll
  for (int t = 0; t < LM; ++t) A[t] = c0();
}
template <int LM>
__device__ __forceinline__ void rload(double2 (&A)[LM], const double2 *p, int L) {
#pragma unroll
  for (int t = 0; t < LM; ++t) A[t] = (t < L) ? p[t] : c0();
}
template <int LM>
__device__ __forceinline__ void rstore(double2 *p, const double2 (&A)[LM], int L) {
#pragma unroll
  for (int t = 0; t < LM; ++t)
    if (t < L) p[t] = A[t];
}
// Request a per-thread series (global memory) into L1: one prefetch per 32-byte sector, no
// scoreboard.  The streamed operand of the product that follows then hits L1 instead of taking one
// L2 round trip per sector, serialised by the product's steps (tree_leaf_r: long-scoreboard stalls).
__device__ __forceinline__ void rprefetch(const double2 *p, int L) {
#if LHAF_LEAF_PREFETCH
  for (int s = 0; s < L; s += 2) asm volatile("prefetch.global.L1 [%0];" ::"l"(p + s));
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p + L - 1));
#endif
}
// acc[t] (+/-)= sum_{s + q + SH = t} a[s] B[q]  for t < L  (a streamed, B in registers).
// Entries t >= L are never read: computing them (zero-padded operands) is harmless, so the
// inner loops run to LM - 1 - s - SH with one uniform guard per s.
template <int LM, int SH, bool NEG>
__device__ __forceinline__ void rs_acc(double2 (&acc)[LM], const double2 *__restrict__ a, const double2 (&B)[LM],
                                       int L) {
#pragma unroll
  for (int s = 0; s + SH < LM; ++s) {
    if (s + SH < L) {
      double2 av = a[s];
      if (NEG) av = make_double2(-av.x, -av.y);
#pragma unroll
      for (int q = 0; q + s + SH < LM; ++q) acc[q + s + SH] = cfma(av, B[q], acc[q + s + SH]);
    }
  }
}
// acc[t] += sum_{s + q = t} A[s] B[q] (both in registers; zero beyond L)
template <int LM>
__device__ __forceinline__ void rr_acc(double2 (&acc)[LM], const double2 (&A)[LM], const double2 (&B)[LM], int L) {
#pragma unroll
  for (int s = 0; s < LM; ++s) {
    if (s < L) {
#pragma unroll
      for (int q = 0; q + s < LM; ++q) acc[q + s] = cfma(A[s], B[q], acc[q + s]);
    }
  }
}
// R = 1/D (D[0] = 1; D zero beyond L)
template <int LM>
__device__ __forceinline__ void rrecip(double2 (&R)[LM], const double2 (&D)[LM], int L) {
  R[0] = c1();
#pragma unroll
  for (int t = 1; t < LM; ++t) {
    double2 x = c0();
    if (t < L) {
#pragma unroll
      for (int s = 1; s <= t; ++s) x = cfma(D[s], R[t - s], x);
    }
    R[t] = make_double2(-x.x, -x.y);
  }
}
// D <- t log D_t = sum_{s=1}^{t} s D_s R_{t-s}, in place (descending t), D[0] <- 0
template <int LM>
__device__ __forceinline__ void rtlog_inplace(double2 (&D)[LM], const double2 (&R)[LM], int L) {
#pragma unroll
  for (int s = 1; s < LM; ++s) D[s] = cscale(D[s], (double)s);
#pragma unroll
  for (int t = LM - 1; t >= 1; --t) {
    double2 x = c0();
    if (t < L) {
#pragma unroll
      for (int s = 1; s <= t; ++s) x = cfma(D[s], R[t - s], x);
    }
    D[t] = x;
  }
  D[0] = c0();
}
// E = exp(phi) from Psi_j = j phi_j (Psi[0] ignored): m E_m = sum_{j=1}^{m} Psi_j E_{m-j}
template <int LM>
__device__ __forceinline__ void rexp(double2 (&E)[LM], const double2 (&Psi)[LM], int L) {
  E[0] = c1();
#pragma unroll
  for (int m = 1; m < LM; ++m) {
    double2 x = c0();
    if (m < L) {
#pragma unroll
      for (int j = 1; j <= m; ++j) x = cfma(Psi[j], E[m - j], x);
    }
    E[m] = cscale(x, 1.0 / m);
  }
}
// A = D_w = 1 - 2 w lam Kab + w^2 lam^2 Delta (Kab, Delta streamed; zero beyond L)
template <int LM>
__device__ __forceinline__ void rdet(double2 (&A)[LM], const double2 *Kab, const double2 *Dl, int w, int L) {
  const double wd = (double)w, w2 = wd * wd;
#pragma unroll
  for (int t = 0; t < LM; ++t) {
    double2 d = (t == 0) ? c1() : c0();
    if (t < L && w != 0) {
      if (t >= 1) { const double2 k = Kab[t - 1]; d.x -= 2.0 * wd * k.x; d.y -= 2.0 * wd * k.y; }
      if (t >= 2) { const double2 q = Dl[t - 2]; d.x += w2 * q.x; d.y += w2 * q.y; }
    }
    A[t] = d;
  }
}

// The three recursions of the method in one routine (one code instance per kernel):
//   X[t] = alpha_t (gamma t P[t] + beta sum_{s=1}^{t} P[s] X[t-s]),  X[0] = x0
//   1/P:       x0 = 1, gamma = 0, beta = -1, alpha = 1
//   t log P_t: x0 = 0, gamma = 1, beta = -1, alpha = 1   (t l_t = t P_t - sum_s P_s (t-s) l_{t-s}, P_0 = 1)
//   exp(phi):  x0 = 1, gamma = 0, beta = 1,  alpha = 1/t  (P = Psi, Psi_t = t phi_t)
template <int LM>
__device__ __forceinline__ void rrec(double2 (&X)[LM], const double2 (&P)[LM], int L, double x0, double gamma,
                                     double beta, bool inv_t) {
  X[0] = make_double2(x0, 0.0);
#pragma unroll
  for (int t = 1; t < LM; ++t) {
    double2 x = c0();
    if (t < L) {
#pragma unroll
      for (int s = 1; s <= t; ++s) x = cfma(P[s], X[t - s], x);
      x = cscale(x, beta);
      x.x = fma(gamma * t, P[t].x, x.x);
      x.y = fma(gamma * t, P[t].y, x.y);
      if (inv_t) x = cscale(x, 1.0 / t);
    }
    X[t] = x;
  }
}
// acc[t] += sgn * sum_{s + q = t} a[s] B[q] (a streamed; runtime sign: one code instance)
template <int LM>
__device__ __forceinline__ void rs_op(double2 (&acc)[LM], const double2 *__restrict__ a, const double2 (&B)[LM], int L,
                                      double sgn) {
#if LHAF_RS_PREFETCH
  // a[s + 1] (and a[s + 2]) are requested before the FMAs of step s: a is a per-thread series in
  // HBM / L2 and every step began with a long-scoreboard stall on its own load (tree_leaf_r)
  double2 n0 = a[0];
#if LHAF_RS_PREFETCH > 1
  double2 n1 = a[min(1, L - 1)];
#endif
#pragma unroll
  for (int s = 0; s < LM; ++s) {
    if (s < L) {
      const double2 av = cscale(n0, sgn);
#if LHAF_RS_PREFETCH > 1
      n0 = n1;
      n1 = a[min(s + 2, L - 1)];
#else
      n0 = a[min(s + 1, L - 1)];
#endif
#pragma unroll
      for (int q = 0; q + s < LM; ++q) acc[q + s] = cfma(av, B[q], acc[q + s]);
    }
  }
#else
#pragma unroll
  for (int s = 0; s < LM; ++s) {
    if (s < L) {
      const double2 av = cscale(a[s], sgn);
#pragma unroll
      for (int q = 0; q + s < LM; ++q) acc[q + s] = cfma(av, B[q], acc[q + s]);
    }
  }
#endif
}

// acc[t] += sum_{s + q = t} av(s) B[q] with av(s) = (a1 + b1 s) p1[max(s - o1, 0)] + (a2 + b2 s) p2[max(s - o2, 0)]
// (operands in shared memory): one code instance serves the plain products (a1 = 1, the rest 0)
// and t log D = sum_s (s D_s) R_{t-s} with s D_s = s (-2 w Kab[s-1] + w^2 Delta[s-2]) rebuilt from
// the staged series (tree_pivot_s: two unrolled triangular routines instead of three).
template <int LM>
__device__ __forceinline__ void rs_op2(double2 (&acc)[LM], const double2 *p1, int o1, double a1, double b1,
                                       const double2 *p2, int o2, double a2, double b2,
                                       const double2 (&B)[LM], int L) {
#pragma unroll
  for (int s = 0; s < LM; ++s) {
    if (s < L) {
      const double c1 = fma(b1, (double)s, a1), c2 = fma(b2, (double)s, a2);
      const double2 v1 = p1[max(s - o1, 0)], v2 = p2[max(s - o2, 0)];
      const double2 av = make_double2(fma(c2, v2.x, c1 * v1.x), fma(c2, v2.y, c1 * v1.y));
#pragma unroll
      for (int q = 0; q + s < LM; ++q) acc[q + s] = cfma(av, B[q], acc[q + s]);
    }
  }
}

// ================================================================ kernels
struct TStep {  // parent depth k -> children at depth k + 1, one chunk of children
  TLevel par, ch;
  uint64_t pbase;  // global index of the parent buffer's slot 0
  uint64_t c0;     // global index of the first child (slot 0 of the child buffer)
  uint64_t nc;     // children in the chunk
  int L, E, b, dmin, eta, wmul;
  double2 *Q;      // [nc][3][L]: q11, q12, q22 of every child
  double2 *S;      // fallback scratch
  double2 *T;      // fallback T: [nc][2][E-2][L]
  int G;           // children per block of tree_bc_k
  double2 *auxp;   // parents' Delta = K_ab^2 - K_aa K_bb at auxp[parent slot * L] (tree_delta_r)
};

__device__ __forceinline__ void child_of(const TStep &P, uint64_t i, uint64_t &ps, int &kh, int &w) {
  const uint64_t c = P.c0 + i, pg = c / P.b;
  ps = pg - P.pbase;
  kh = P.dmin + (int)(c - pg * P.b);
  w = P.eta - P.wmul * kh;
}

// Delta = K_ab^2 - K_aa K_bb of parent slots [p0, p0 + np) (shared by its children: the weight
// enters only D = 1 - 2 w lam K_ab + w^2 lam^2 Delta), into P.auxp[slot * L].  Used where no
// tree_bc_k produced it (the root depth, the fallback update kernels).
template <int LM>
__global__ void __launch_bounds__(128) tree_delta_r(TStep P, uint64_t p0, uint64_t np) {
  const uint64_t i = (uint64_t)blockIdx.x * 128 + threadIdx.x;
  if (i >= np) return;
  const uint64_t ps = p0 + i;
  LHAF_DCHECK(ps < P.par.cap);
  const int L = P.L, E = P.E, NE = E * (E + 1) / 2, a = E - 2, b = E - 1;
  const double2 *Kp = P.par.K + (int64_t)ps * NE * L;
  double2 A[LM], B[LM];
  rload(B, Kp + (int64_t)tri(b, a) * L, L);
  rz(A);
  rr_acc(A, B, B, L);
  rload(B, Kp + (int64_t)tri(a, a) * L, L);
  rs_op(A, Kp + (int64_t)tri(b, b) * L, B, L, -1.0);
  rstore(P.auxp + (int64_t)ps * L, A, L);
}

// Per child: D_w, R = 1/D_w, t log D_w (child log c), Q.  Series in two register arrays; each
// triangular routine appears once (rolled loops over the phases that share it: the unrolled
// bodies are large, and the instruction cache limited the first version).
template <int LM>
__global__ void __launch_bounds__(128) tree_pivot_r(TStep P) {
  const uint64_t i = (uint64_t)blockIdx.x * 128 + threadIdx.x;
  if (i >= P.nc) return;
  uint64_t ps; int kh, w;
  child_of(P, i, ps, kh, w);
  const int L = P.L, E = P.E, NE = E * (E + 1) / 2, a = E - 2, b = E - 1;
  const double2 *Kp = P.par.K + (int64_t)ps * NE * L;
  const double2 *Kaa = Kp + (int64_t)tri(a, a) * L, *Kbb = Kp + (int64_t)tri(b, b) * L,
                *Kab = Kp + (int64_t)tri(b, a) * L;
  const double2 *Dl = P.auxp + (int64_t)ps * L;
  const double2 *lp = P.par.logc + (int64_t)ps * L;
  double2 *lc = P.ch.logc + (int64_t)i * L;
  double2 *Q = P.Q + (int64_t)i * 3 * L;
  const double wd = (double)w, w2 = wd * wd;
  P.ch.coef[i] = P.par.coef[ps] * ((kh & 1) ? -1.0 : 1.0) * binom_d(P.eta, kh);
  if (w == 0) {  // deleted pair: D = 1, Q = 0
    for (int t = 0; t < L; ++t) { lc[t] = lp[t]; Q[t] = Q[L + t] = Q[2 * L + t] = c0(); }
    return;
  }
  double2 A[LM], B[LM];
#pragma unroll 1
  for (int ph = 0; ph < 2; ++ph) {
    rdet(A, Kab, Dl, w, L);                                   // A = D_w
    rrec(B, A, L, ph ? 0.0 : 1.0, ph ? 1.0 : 0.0, -1.0, false);  // B = 1/D (ph 0), t log D (ph 1)
    if (ph == 0) {
#pragma unroll 1
      for (int qi = 0; qi < 3; ++qi) {                        // lam K R for K = Kbb, Kaa, Kab
        rz(A);
        rs_op(A, qi == 0 ? Kbb : qi == 1 ? Kaa : Kab, B, L, 1.0);
#pragma unroll
        for (int t = 0; t < LM; ++t) {
          if (t < L) {
            const double2 m = t ? A[t - 1] : c0();
            if (qi == 0) Q[t] = cscale(m, w2);                                           // q11
            else if (qi == 1) Q[2 * L + t] = cscale(m, w2);                              // q22
            else Q[L + t] = make_double2(wd * B[t].x - w2 * m.x, wd * B[t].y - w2 * m.y);  // q12
          }
        }
      }
    } else {
#pragma unroll
      for (int t = 0; t < LM; ++t)
        if (t < L) lc[t] = t ? cadd(lp[t], cscale(B[t], 1.0 / t)) : lp[t];
    }
  }
}

// The same pivot with the operands staged in shared memory: the parents' K_ab, Delta, K_aa (then
// K_bb in Delta's place) are copied by the whole block with coalesced 16-byte copies, so the
// register-array products read shared memory instead of issuing one L2 load per coefficient.
// Children of a block span at most (PV_THREADS - 1) / b + 2 parents (b >= 2, host-checked); a
// parent's series sits at an odd stride (in 16-byte units) so that the lanes of a quarter-warp
// hit distinct banks.  t log D is the in-place product sum_s s D_s R_{t-s} (no recursion).
constexpr int PV_THREADS = 128;
__host__ __device__ __forceinline__ int pv_stride(int L) { return L | 1; }
__host__ __device__ __forceinline__ int pv_parents(int b) { return (PV_THREADS - 1) / b + 2; }
template <int LM>
__global__ void __launch_bounds__(PV_THREADS, 2) tree_pivot_s(TStep P) {
  extern __shared__ double2 sv[];
  const int L = P.L, E = P.E, NE = E * (E + 1) / 2, a = E - 2, b = E - 1;
  const int SP = pv_stride(L), NPM = pv_parents(P.b);
  double2 *bKab = sv, *bX = sv + (int64_t)NPM * SP, *bKaa = sv + 2 * (int64_t)NPM * SP;
  const uint64_t i0 = (uint64_t)blockIdx.x * PV_THREADS, i = i0 + threadIdx.x;
  const bool active = i < P.nc;
  uint64_t psf, psl; int kh, w;
  child_of(P, min(i0 + PV_THREADS - 1, P.nc - 1), psl, kh, w);
  child_of(P, i0, psf, kh, w);
  const int NP = (int)(psl - psf) + 1;
  LHAF_DCHECK(NP >= 1 && NP <= NPM);
  LHAF_DCHECK(psl < P.par.cap && min(i0 + PV_THREADS, P.nc) <= P.ch.cap);
#ifdef LHAF_CHECK
  {
    unsigned sbytes;
    asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(sbytes));
    LHAF_DCHECK((size_t)3 * NPM * SP * sizeof(double2) <= sbytes);
  }
#endif
  for (int c = threadIdx.x; c < NP * L; c += PV_THREADS) {
    const int p = c / L, s = c - p * L;
    const double2 *Kp = P.par.K + (int64_t)(psf + p) * NE * L;
    cp_async16(bKab + p * SP + s, Kp + (int64_t)tri(b, a) * L + s);
    cp_async16(bKaa + p * SP + s, Kp + (int64_t)tri(a, a) * L + s);
    cp_async16(bX + p * SP + s, P.auxp + (int64_t)(psf + p) * L + s);
  }
  cp_async_wait_all();
  __syncthreads();
  uint64_t ps = 0;
  if (active) child_of(P, i, ps, kh, w);
  const int pl = (int)(ps - psf);
  const double wd = (double)w, w2 = wd * wd;
  double2 A[LM], B[LM];
#if LHAF_PIVOT_TWO
  const bool live = active && w != 0;
  if (live) {
    rdet(A, bKab + pl * SP, bX + pl * SP, w, L);                // A = D_w
    rrec(B, A, L, 1.0, 0.0, -1.0, false);                     // B = 1/D
  } else if (active) {  // deleted pair: D = 1, Q = 0
    const double2 *lp = P.par.logc + (int64_t)ps * L;
    double2 *lc = P.ch.logc + (int64_t)i * L, *Q = P.Q + (int64_t)i * 3 * L;
    for (int t = 0; t < L; ++t) { lc[t] = lp[t]; Q[t] = Q[L + t] = Q[2 * L + t] = c0(); }
  }
  if (active) P.ch.coef[i] = P.par.coef[ps] * ((kh & 1) ? -1.0 : 1.0) * binom_d(P.eta, kh);
  double2 *Q = P.Q + (int64_t)i * 3 * L;
  // qi = 0: A = t log D = sum_s (s D_s) R_{t-s};  qi = 1..3: lam K R for K = Kbb, Kaa, Kab
#pragma unroll 1
  for (int qi = 0; qi < 4; ++qi) {
    if (live) {
      rz(A);
      const double2 *p1 = (qi == 0 ? bKab : qi == 1 ? bX : qi == 2 ? bKaa : bKab) + pl * SP;
      const double2 *p2 = (qi == 0 ? bX : p1) + (qi == 0 ? pl * SP : 0);
      // s D_s = s (-2 w Kab[s-1] + w^2 Delta[s-2]): the clamped index at s < offset meets a zero
      // coefficient for s = 0 only; s = 1 of the Delta term must vanish too: D_1 has no Delta part
      rs_op2(A, p1, qi == 0 ? 1 : 0, qi == 0 ? 0.0 : 1.0, qi == 0 ? -2.0 * wd : 0.0,
             p2, qi == 0 ? 2 : 0, 0.0, qi == 0 ? w2 : 0.0, B, L);
      if (qi == 0) {
        // the s = 1 step took Delta[max(1 - 2, 0)] = Delta[0] with coefficient w^2: remove it
        const double2 d0 = (bX + pl * SP)[0];
        const double2 av = make_double2(-w2 * d0.x, -w2 * d0.y);
#pragma unroll
        for (int q = 0; q + 1 < LM; ++q) A[q + 1] = cfma(av, B[q], A[q + 1]);
        const double2 *lp = P.par.logc + (int64_t)ps * L;
        double2 *lc = P.ch.logc + (int64_t)i * L;
#pragma unroll
        for (int t = 0; t < LM; ++t)
          if (t < L) lc[t] = t ? cadd(lp[t], cscale(A[t], 1.0 / t)) : lp[t];
      } else {
#pragma unroll
        for (int t = 0; t < LM; ++t) {
          if (t < L) {
            const double2 m = t ? A[t - 1] : c0();
            if (qi == 1) Q[t] = cscale(m, w2);                                           // q11
            else if (qi == 2) Q[2 * L + t] = cscale(m, w2);                              // q22
            else Q[L + t] = make_double2(wd * B[t].x - w2 * m.x, wd * B[t].y - w2 * m.y);  // q12
          }
        }
      }
    }
    if (qi == 0) {
      __syncthreads();  // Delta consumed: K_bb takes its buffer
      for (int c = threadIdx.x; c < NP * L; c += PV_THREADS) {
        const int p = c / L, sx = c - p * L;
        cp_async16(bX + p * SP + sx, P.par.K + ((int64_t)(psf + p) * NE + tri(b, b)) * L + sx);
      }
      cp_async_wait_all();
      __syncthreads();
    }
  }
}
#else
  if (active && w != 0) {
    rdet(A, bKab + pl * SP, bX + pl * SP, w, L);                // A = D_w
    rrec(B, A, L, 1.0, 0.0, -1.0, false);                     // B = 1/D
    rtlog_inplace(A, B, L);                                   // A = t log D_t
    const double2 *lp = P.par.logc + (int64_t)ps * L;
    double2 *lc = P.ch.logc + (int64_t)i * L;
#pragma unroll
    for (int t = 0; t < LM; ++t)
      if (t < L) lc[t] = t ? cadd(lp[t], cscale(A[t], 1.0 / t)) : lp[t];
  } else if (active) {  // deleted pair: D = 1, Q = 0
    const double2 *lp = P.par.logc + (int64_t)ps * L;
    double2 *lc = P.ch.logc + (int64_t)i * L, *Q = P.Q + (int64_t)i * 3 * L;
    for (int t = 0; t < L; ++t) { lc[t] = lp[t]; Q[t] = Q[L + t] = Q[2 * L + t] = c0(); }
  }
  if (active) P.ch.coef[i] = P.par.coef[ps] * ((kh & 1) ? -1.0 : 1.0) * binom_d(P.eta, kh);
  __syncthreads();  // Delta consumed: K_bb takes its buffer
  for (int c = threadIdx.x; c < NP * L; c += PV_THREADS) {
    const int p = c / L, s = c - p * L;
    cp_async16(bX + p * SP + s, P.par.K + ((int64_t)(psf + p) * NE + tri(b, b)) * L + s);
  }
  cp_async_wait_all();
  __syncthreads();
  if (!active || w == 0) return;
  double2 *Q = P.Q + (int64_t)i * 3 * L;
#pragma unroll 1
  for (int qi = 0; qi < 3; ++qi) {                            // lam K R for K = Kbb, Kaa, Kab
    rz(A);
    rs_op(A, (qi == 0 ? bX : qi == 1 ? bKaa : bKab) + pl * SP, B, L, 1.0);
#pragma unroll
    for (int t = 0; t < LM; ++t) {
      if (t < L) {
        const double2 m = t ? A[t - 1] : c0();
        if (qi == 0) Q[t] = cscale(m, w2);                                           // q11
        else if (qi == 1) Q[2 * L + t] = cscale(m, w2);                              // q22
        else Q[L + t] = make_double2(wd * B[t].x - w2 * m.x, wd * B[t].y - w2 * m.y);  // q12
      }
    }
  }
}
#endif

// generic pivot (any L): the blocked series routines above with per-child scratch in HBM
__global__ void __launch_bounds__(128) tree_pivot_g(TStep P) {
  const uint64_t i = (uint64_t)blockIdx.x * 128 + threadIdx.x;
  if (i >= P.nc) return;
  uint64_t ps; int kh, w;
  child_of(P, i, ps, kh, w);
  const int L = P.L, E = P.E, NE = E * (E + 1) / 2, a = E - 2, b = E - 1;
  const double2 *Kp = P.par.K + (int64_t)ps * NE * L;
  pivot(SR{Kp + (int64_t)tri(a, a) * L, 1}, SR{Kp + (int64_t)tri(b, b) * L, 1}, SR{Kp + (int64_t)tri(b, a) * L, 1},
        L, w, P.S + (int64_t)i * 3 * L, P.Q + (int64_t)i * 3 * L, 1, SR{P.par.logc + (int64_t)ps * L, 1},
        P.ch.logc + (int64_t)i * L, 1, nullptr, nullptr);
  P.ch.coef[i] = P.par.coef[ps] * ((kh & 1) ? -1.0 : 1.0) * binom_d(P.eta, kh);
}

// T_j = Q (u_j, x_j)^T and K'_ij = K_ij + lam (u_i T1_j + x_i T2_j) for a group of G children:
// the parent rows (u, x) -- once per parent, shared by its children in the group -- and the
// children's Q in shared memory, T written there, then the packed lower triangle of every child.
// Shared layout: parents U[Ep][L] X[Ep][L] (bc_smem_parents of them), then per child Q[3][L]
// T1[Ep][L] T2[Ep][L].  The block size (blockDim.x <= BC_THREADS) and G come from bc_choose.
#ifndef LHAF_BC_THREADS
#define LHAF_BC_THREADS 128
#endif
#ifndef LHAF_BC_MINB
#define LHAF_BC_MINB 4
#endif
#ifndef LHAF_BC_SMEM_KB
#define LHAF_BC_SMEM_KB 72
#endif
// Task order inside a phase: 1 = part-major (the lanes of a warp work on the same pair of output
// blocks, so the windowed loops of a warp have one trip count); 0 = part fastest (lanes 2i, 2i+1
// take the short and the long pair: the warp runs max(trip counts) per block, ~25 % idle lanes).
#ifndef LHAF_BC_ORDER
#define LHAF_BC_ORDER 1
#endif
#ifndef LHAF_BC_UNIFIED
#define LHAF_BC_UNIFIED 1
#endif
constexpr int BC_THREADS = LHAF_BC_THREADS;
// parents a group of G consecutive children can span (b children per parent)
__host__ __device__ __forceinline__ int bc_smem_parents(int G, int b) { return min(G, (G - 1) / b + 2); }
__global__ void __launch_bounds__(BC_THREADS, LHAF_BC_MINB) tree_bc_k(TStep P) {
  extern __shared__ double2 sm[];
  const int L = P.L, E = P.E, NE = E * (E + 1) / 2, a = E - 2, b = E - 1, Ep = E - 2;
  const int NEc = Ep * (Ep + 1) / 2;
  const int per = (2 * Ep + 3) * L;
  const uint64_t g0 = (uint64_t)blockIdx.x * P.G;
  const int G = (int)min((uint64_t)P.G, P.nc - g0);
  const int tid = threadIdx.x, nth = blockDim.x;
  uint64_t ps0; int kh0, w0;
  child_of(P, g0, ps0, kh0, w0);
  uint64_t psl; int khl, wl;
  child_of(P, g0 + G - 1, psl, khl, wl);
  const int NP = (int)(psl - ps0) + 1;
  double2 *cbase = sm + (int64_t)bc_smem_parents(P.G, P.b) * 2 * Ep * L;
  LHAF_DCHECK(NP >= 1 && NP <= bc_smem_parents(P.G, P.b));
  LHAF_DCHECK(g0 + G <= P.ch.cap && G >= 1);
  LHAF_DCHECK(psl < P.par.cap);
#ifdef LHAF_CHECK
  {
    unsigned sbytes;
    asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(sbytes));
    LHAF_DCHECK((size_t)((int64_t)bc_smem_parents(P.G, P.b) * 2 * Ep * L + (int64_t)P.G * per) * sizeof(double2) <= sbytes);
  }
#endif
  // stage: parent rows, then the children's Q
  for (int p = 0; p < NP; ++p) {
    const double2 *Kp = P.par.K + (int64_t)(ps0 + p) * NE * L;
    const double2 *ur = Kp + (int64_t)tri(a, 0) * L, *xr = Kp + (int64_t)tri(b, 0) * L;
    double2 *pb = sm + (int64_t)p * 2 * Ep * L;
    for (int t = tid; t < Ep * L; t += nth) {
      cp_async16(pb + t, ur + t);
      cp_async16(pb + Ep * L + t, xr + t);
    }
  }
  for (int g = 0; g < G; ++g) {
    const double2 *qr = P.Q + (int64_t)(g0 + g) * 3 * L;
    for (int t = tid; t < 3 * L; t += nth) cp_async16(cbase + (int64_t)g * per + t, qr + t);
  }
  cp_async_wait_all();
  __syncthreads();
#if LHAF_BC_UNIFIED
  // Both phases -- T = Q (u, x)^T into shared memory, then K' = K + lam (u T1 + x T2) -- run through
  // one task loop with one inlined conv_acc1 (the two products of a task in a rolled loop): the
  // kernel's code is a quarter of the four-instance version (tree_bc_k was 54 KB of SASS and
  // stalled on instruction fetch).  Tasks are output blocks paired (p, nb - 1 - p) so that every
  // task does about the same work; part-major order (LHAF_BC_ORDER).
  const int Lo = L - 1;
  const int nbB = (Lo + TB - 1) / TB, PB = (nbB + 1) / 2;
  const int nbC = (L + TB - 1) / TB, PC = (nbC + 1) / 2;
#pragma unroll 1
  for (int phase = 0; phase < 2; ++phase) {
    const int NT = phase ? G * NEc : G * 2 * Ep, NPt = phase ? PC : PB, nb = phase ? nbC : nbB;
    const int Lout = phase ? L : Lo;
#pragma unroll 1
    for (int task = tid; task < NT * NPt; task += nth) {
      const int part = LHAF_BC_ORDER ? task / NT : task % NPt, tk = LHAF_BC_ORDER ? task - part * NT : task / NPt;
      int g, a0o, a1o, b0o, b1o, oo = 0;   // operand / output offsets in sm (double2 units)
      const double2 *K = nullptr;
      double2 *out = nullptr;
      uint64_t ps; int kh, w;
      if (!phase) {
        g = tk / (2 * Ep);
        const int r = tk - g * 2 * Ep, j = r >> 1, which = r & 1;
        child_of(P, g0 + g, ps, kh, w);
        if (w == 0) continue;  // deleted pair: the child is the parent's leading block
        const int Uo = (int)(ps - ps0) * 2 * Ep * L, Co = (int)(cbase - sm) + g * per;
        // T1 = q11 u + q12 x ; T2 = q12 u + q22 x
        a0o = Co + (which ? L : 0); a1o = Co + (which ? 2 * L : L);
        b0o = Uo + j * L; b1o = Uo + Ep * L + j * L;
        oo = Co + 3 * L + which * Ep * L + j * L;
      } else {
        g = tk / NEc;
        const int e = tk - g * NEc;
        int ii = (int)((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);
        while (tri(ii + 1, 0) <= e) ++ii;
        while (tri(ii, 0) > e) --ii;
        const int jj = e - tri(ii, 0);
        child_of(P, g0 + g, ps, kh, w);
        const int Uo = (int)(ps - ps0) * 2 * Ep * L, Co = (int)(cbase - sm) + g * per;
        a0o = Uo + ii * L; a1o = Uo + Ep * L + ii * L;
        b0o = Co + 3 * L + jj * L; b1o = Co + 3 * L + Ep * L + jj * L;
        K = P.par.K + ((int64_t)ps * NE + e) * L;
        out = P.ch.K + ((int64_t)(g0 + g) * NEc + e) * L;
      }
#pragma unroll 1
      for (int bi = 0; bi < 2; ++bi) {
        const int blk = bi ? nb - 1 - part : part;
        if (bi && blk == part) break;
        const int t0 = blk * TB;
        if (phase && w == 0) {
          for (int t = t0; t < t0 + TB && t < L; ++t) out[t] = K[t];
          continue;
        }
        double2 acc[TB];
#pragma unroll
        for (int k = 0; k < TB; ++k) acc[k] = (phase && t0 + k < L) ? K[t0 + k] : c0();
#pragma unroll 1
        for (int op = 0; op < 2; ++op) conv_acc1(acc, t0, phase, sm + (op ? a1o : a0o), Lo, sm + (op ? b1o : b0o), Lo);
        if (phase) {
#pragma unroll
          for (int k = 0; k < TB; ++k)
            if (t0 + k < Lout) out[t0 + k] = acc[k];
        } else {
#pragma unroll
          for (int k = 0; k < TB; ++k)
            if (t0 + k < Lout) sm[oo + t0 + k] = acc[k];
        }
      }
    }
    __syncthreads();
  }
}
#else
  const int Lo = L - 1;
  // tasks are split by output blocks, paired (p, nb - 1 - p) so that every task does about the
  // same work (the products are triangular): PB parts per series
  const int nbB = (Lo + TB - 1) / TB, PB = (nbB + 1) / 2;
  const int NT1 = G * 2 * Ep;
  for (int task = tid; task < NT1 * PB; task += nth) {
    const int part = LHAF_BC_ORDER ? task / NT1 : task % PB, tk = LHAF_BC_ORDER ? task - part * NT1 : task / PB;
    const int g = tk / (2 * Ep), r = tk - g * 2 * Ep, j = r >> 1, which = r & 1;
    uint64_t ps; int kh, w;
    child_of(P, g0 + g, ps, kh, w);
    if (w == 0) continue;  // deleted pair: the child is the parent's leading block
    const double2 *U = sm + (int64_t)(ps - ps0) * 2 * Ep * L, *X = U + Ep * L;
    double2 *base = cbase + (int64_t)g * per;
    const double2 *Qs = base;
    double2 *T = base + 3 * L + (int64_t)which * Ep * L + (int64_t)j * L;
    // T1 = q11 u + q12 x ; T2 = q12 u + q22 x
    const SR qa{Qs + (which ? L : 0), 1}, qb{Qs + (which ? 2 * L : L), 1};
    for (int bi = 0; bi < 2; ++bi) {
      const int blk = bi ? nbB - 1 - part : part;
      if (bi && blk == part) break;
      const int t0 = blk * TB;
      double2 acc[TB];
#pragma unroll
      for (int k = 0; k < TB; ++k) acc[k] = c0();
      conv_acc(acc, t0, 0, qa, Lo, SR{U + (int64_t)j * L, 1}, Lo);
      conv_acc(acc, t0, 0, qb, Lo, SR{X + (int64_t)j * L, 1}, Lo);
#pragma unroll
      for (int k = 0; k < TB; ++k)
        if (t0 + k < Lo) T[t0 + k] = acc[k];
    }
  }
  __syncthreads();
  const int nbC = (L + TB - 1) / TB, PC = (nbC + 1) / 2;
  const int NT2 = G * NEc;
  for (int task = tid; task < NT2 * PC; task += nth) {
    const int part = LHAF_BC_ORDER ? task / NT2 : task % PC, tk = LHAF_BC_ORDER ? task - part * NT2 : task / PC;
    const int g = tk / NEc, e = tk - g * NEc;
    int ii = (int)((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);
    while (tri(ii + 1, 0) <= e) ++ii;
    while (tri(ii, 0) > e) --ii;
    const int jj = e - tri(ii, 0);
    uint64_t ps; int kh, w;
    child_of(P, g0 + g, ps, kh, w);
    const double2 *U = sm + (int64_t)(ps - ps0) * 2 * Ep * L, *X = U + Ep * L;
    const double2 *T1 = cbase + (int64_t)g * per + 3 * L, *T2 = T1 + Ep * L;
    const double2 *K = P.par.K + ((int64_t)ps * NE + e) * L;
    double2 *out = P.ch.K + ((int64_t)(g0 + g) * NEc + e) * L;
    for (int bi = 0; bi < 2; ++bi) {
      const int blk = bi ? nbC - 1 - part : part;
      if (bi && blk == part) break;
      const int t0 = blk * TB;
      if (w == 0) {
        for (int t = t0; t < t0 + TB && t < L; ++t) out[t] = K[t];
        continue;
      }
      double2 acc[TB];
#pragma unroll
      for (int k = 0; k < TB; ++k) acc[k] = (t0 + k < L) ? K[t0 + k] : c0();
      conv_acc(acc, t0, 1, SR{U + (int64_t)ii * L, 1}, Lo, SR{T1 + (int64_t)jj * L, 1}, Lo);
      conv_acc(acc, t0, 1, SR{X + (int64_t)ii * L, 1}, Lo, SR{T2 + (int64_t)jj * L, 1}, Lo);
#pragma unroll
      for (int k = 0; k < TB; ++k)
        if (t0 + k < L) out[t0 + k] = acc[k];
    }
  }
}
#endif

// fallback when a child group's rows do not fit shared memory: T in HBM, then the update
__global__ void __launch_bounds__(128) tree_tmat_g(TStep P) {
  const int Ep = P.E - 2;
  const uint64_t i = (uint64_t)blockIdx.x * 128 + threadIdx.x;
  if (i >= P.nc * (uint64_t)Ep) return;
  const uint64_t ci = i / Ep;
  const int j = (int)(i - ci * Ep);
  uint64_t ps; int kh, w;
  child_of(P, ci, ps, kh, w);
  const int L = P.L, E = P.E, NE = E * (E + 1) / 2, a = E - 2, b = E - 1, Lo = L - 1;
  const double2 *Kp = P.par.K + (int64_t)ps * NE * L;
  const SR u{Kp + (int64_t)tri(a, j) * L, 1}, x{Kp + (int64_t)tri(b, j) * L, 1};
  const double2 *Qs = P.Q + (int64_t)ci * 3 * L;
  double2 *T1 = P.T + ((int64_t)ci * 2 * Ep + j) * L, *T2 = T1 + (int64_t)Ep * L;
  for (int t0 = 0; t0 < Lo; t0 += TB) {
    double2 a1[TB], a2[TB];
#pragma unroll
    for (int k = 0; k < TB; ++k) a1[k] = a2[k] = c0();
    conv_acc(a1, t0, 0, SR{Qs, 1}, Lo, u, Lo);
    conv_acc(a1, t0, 0, SR{Qs + L, 1}, Lo, x, Lo);
    conv_acc(a2, t0, 0, SR{Qs + L, 1}, Lo, u, Lo);
    conv_acc(a2, t0, 0, SR{Qs + 2 * L, 1}, Lo, x, Lo);
#pragma unroll
    for (int k = 0; k < TB; ++k)
      if (t0 + k < Lo) { T1[t0 + k] = a1[k]; T2[t0 + k] = a2[k]; }
  }
}
__global__ void __launch_bounds__(128) tree_update_g(TStep P) {
  const int Ep = P.E - 2, NEc = Ep * (Ep + 1) / 2;
  const uint64_t i = (uint64_t)blockIdx.x * 128 + threadIdx.x;
  if (i >= P.nc * (uint64_t)NEc) return;
  const uint64_t ci = i / NEc;
  const int e = (int)(i - ci * NEc);
  int ii = (int)((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);
  while (tri(ii + 1, 0) <= e) ++ii;
  while (tri(ii, 0) > e) --ii;
  const int jj = e - tri(ii, 0);
  uint64_t ps; int kh, w;
  child_of(P, ci, ps, kh, w);
  const int L = P.L, E = P.E, NE = E * (E + 1) / 2, a = E - 2, b = E - 1, Lo = L - 1;
  const double2 *Kp = P.par.K + (int64_t)ps * NE * L;
  const SR u{Kp + (int64_t)tri(a, ii) * L, 1}, x{Kp + (int64_t)tri(b, ii) * L, 1};
  const double2 *T1 = P.T + ((int64_t)ci * 2 * Ep + jj) * L, *T2 = T1 + (int64_t)Ep * L;
  const double2 *K = Kp + (int64_t)e * L;
  double2 *out = P.ch.K + ((int64_t)ci * NEc + e) * L;
  for (int t0 = 0; t0 < L; t0 += TB) {
    double2 acc[TB];
#pragma unroll
    for (int k = 0; k < TB; ++k) acc[k] = (t0 + k < L) ? K[t0 + k] : c0();
    conv_acc(acc, t0, 1, u, Lo, SR{T1, 1}, Lo);
    conv_acc(acc, t0, 1, x, Lo, SR{T2, 1}, Lo);
#pragma unroll
    for (int k = 0; k < TB; ++k)
      if (t0 + k < L) out[t0 + k] = acc[k];
  }
}

struct TLeaf {
  TLevel par;      // nodes at depth H-1 (one pair left, plus the border)
  uint64_t np;     // nodes in the chunk
  int L, E, bord, b, dmin, eta, wmul;
  double2 *S;      // scratch [np][9][L]
  double2 *val;    // [np]: sum over the node's leaves of sign * prod C * g
  double *absv;    // [np]: the same sum of |.|
  int cut_eb, nf;  // cutoff group (cut_eb >= 0): per count m, val / absv at [m * vstride + node]
  uint64_t vstride;
};

// The last pair of every node, both (all) digits; the node-level products shared by the leaves:
// Delta = K_ab^2 - K_aa K_bb, and with the border P = u (K_bb u - K_ab x) + x (K_aa x - K_ab u)
// and N0 = u x, so that the leaf's border entry is K'_00 = K_00 + lam R_w (lam w^2 P + 2 w N0).
// Scratch per node (HBM, L1-resident while the thread works): S0 Delta, S1 P, S2 N0, S3.
template <int LM>
__global__ void __launch_bounds__(128) tree_leaf_r(TLeaf P) {
  const uint64_t i = (uint64_t)blockIdx.x * 128 + threadIdx.x;
  if (i >= P.np) return;
  LHAF_DCHECK(i < P.par.cap);
  const int L = P.L, E = P.E, NE = E * (E + 1) / 2, a = E - 2, b = E - 1;
  const double2 *Kp = P.par.K + (int64_t)i * NE * L;
  const double2 *Kaa = Kp + (int64_t)tri(a, a) * L, *Kbb = Kp + (int64_t)tri(b, b) * L,
                *Kab = Kp + (int64_t)tri(b, a) * L;
  const double2 *u = Kp + (int64_t)tri(a, 0) * L, *x = Kp + (int64_t)tri(b, 0) * L;
  const double2 *lc = P.par.logc + (int64_t)i * L;
  double2 *S0 = P.S + (int64_t)i * 4 * L, *S1 = S0 + L, *S2 = S1 + L, *S3 = S2 + L;
  double2 A[LM], B[LM];
  rload(B, Kab, L);
  rz(A);
  rr_acc(A, B, B, L);                       // A = Kab^2
  // node-level ops on (acc A, operand B):
  //  0: B=Kaa  A -= Kbb B -> S0 (Delta)       [no border: stop here]
  //  1: B=u    A  = Kbb B                      2: B=x  A -= Kab B -> S1 (P1)
  //  3:        A  = Kaa B                      4: B=u  A -= Kab B -> S2 (P2)
  //  5:        A  = S1 B                       6: B=x  A += S2 B -> S1 (P)
  //  7:        A  = u B -> S2 (N0)
  const int nops = P.bord ? 8 : 1;
#pragma unroll 1
  for (int op = 0; op < nops; ++op) {
    const double2 *ld = (op == 0) ? Kaa : (op == 1 || op == 4) ? u : (op == 2 || op == 6) ? x : nullptr;
    const double2 *src = (op == 0 || op == 1) ? Kbb : (op == 2 || op == 4) ? Kab : (op == 3) ? Kaa
                       : (op == 5) ? S1 : (op == 6) ? S2 : u;
    rprefetch(src, L);
    if (ld) rload(B, ld, L);
    if (op == 1 || op == 3 || op == 5 || op == 7) rz(A);
    const double sg = (op == 0 || op == 2 || op == 4) ? -1.0 : 1.0;
    rs_op(A, src, B, L, sg);
    double2 *st = (op == 0) ? S0 : (op == 2 || op == 6) ? S1 : (op == 4 || op == 7) ? S2 : nullptr;
    if (st) rstore(st, A, L);
  }
  const double coef = P.par.coef[i];
  double2 vsum = c0();
  double asum = 0.0;
  const bool cut = P.cut_eb >= 0;
  if (cut)
    for (int m = 0; m <= P.cut_eb; ++m) { P.val[m * P.vstride + i] = c0(); P.absv[m * P.vstride + i] = 0.0; }
#pragma unroll 1
  for (int d = 0; d < P.b; ++d) {
    // cutoff groups: the leaf pair is the batched self-pair, weight w_b = (eta - 2 k) / 2
    const int kh = P.dmin + d, w = cut ? (P.eta - P.wmul * kh) / 2 : P.eta - P.wmul * kh;
    const double wd = (double)w, w2 = wd * wd;
    // phases sharing one recursion instance: 0: R = 1/D; 1: t log D; 2: exp(phi)
#pragma unroll 1
    for (int ph = 0; ph < 3; ++ph) {
      if (ph < 2) rdet(A, Kab, S0, w, L);   // A = D_w
      rrec(B, A, L, ph == 1 ? 0.0 : 1.0, ph == 1 ? 1.0 : 0.0, ph == 2 ? 1.0 : -1.0, ph == 2);
      if (ph == 0) {
        if (P.bord) {
          // S3 = N_w = lam w^2 P + 2 w N0;  A = R_w N_w;  S3 = A (lam M enters K'_00)
#pragma unroll
          for (int t = 0; t < LM; ++t)
            if (t < L) {
              double2 nv = cscale(S2[t], 2.0 * wd);
              if (t >= 1) { const double2 pv = S1[t - 1]; nv.x += w2 * pv.x; nv.y += w2 * pv.y; }
              S3[t] = nv;
            }
          rz(A);
          rprefetch(S3, L);
          rs_op(A, S3, B, L, 1.0);
          rstore(S3, A, L);
        }
      } else if (ph == 1) {
        // A = Psi_t = t phi_t, phi = 1/2 (K00 + lam M - log c - log D)   (B = t log D)
#pragma unroll
        for (int t = 0; t < LM; ++t) {
          double2 ps = c0();
          if (t >= 1 && t < L) {
            const double2 l0 = lc[t], tl = B[t];
            if (P.bord) {
              const double2 k0 = Kp[t], m = S3[t - 1];
              ps = make_double2(0.5 * (t * (k0.x + m.x - l0.x) - tl.x), 0.5 * (t * (k0.y + m.y - l0.y) - tl.y));
            } else {
              ps = make_double2(-0.5 * (t * l0.x + tl.x), -0.5 * (t * l0.y + tl.y));
            }
          }
          A[t] = ps;
        }
      }
    }
    if (cut) {
      // every count 2m + p with m >= |w_b|, m = w_b (mod 2): (-1)^{k_b} C(m, k_b) [lam^{nf + m}] F,
      // k_b = (m - w_b) / 2 (App. B.5)
#pragma unroll 1
      for (int m = abs(w); m <= P.cut_eb; m += 2) {
        const int deg = P.nf + m;
        double2 g = c0();
#pragma unroll
        for (int t = 0; t < LM; ++t)
          if (t == deg) g = B[t];
        const int kb = (m - w) / 2;
        const double cb = binom_d(m, kb), f = coef * ((kb & 1) ? -cb : cb);
        double2 *vp = P.val + m * P.vstride + i;
        *vp = make_double2(fma(f, g.x, vp->x), fma(f, g.y, vp->y));
        P.absv[m * P.vstride + i] += fabs(f) * hypot(g.x, g.y);
      }
      continue;
    }
    double2 g = c0();
#pragma unroll
    for (int t = 0; t < LM; ++t)
      if (t == L - 1) g = B[t];
    const double f = coef * ((kh & 1) ? -1.0 : 1.0) * binom_d(P.eta, kh);
    vsum.x = fma(f, g.x, vsum.x);
    vsum.y = fma(f, g.y, vsum.y);
    asum += fabs(f) * hypot(g.x, g.y);
  }
  if (cut) return;
  P.val[i] = vsum;
  P.absv[i] = asum;
}

// generic leaf (any L): the blocked series routines with scratch in HBM
__global__ void __launch_bounds__(128) tree_leaf_g(TLeaf P) {
  const uint64_t i = (uint64_t)blockIdx.x * 128 + threadIdx.x;
  if (i >= P.np) return;
  const int L = P.L, E = P.E, NE = E * (E + 1) / 2, a = E - 2, b = E - 1;
  const double2 *Kp = P.par.K + (int64_t)i * NE * L;
  const SR Kaa{Kp + (int64_t)tri(a, a) * L, 1}, Kbb{Kp + (int64_t)tri(b, b) * L, 1}, Kab{Kp + (int64_t)tri(b, a) * L, 1};
  const SR logc{P.par.logc + (int64_t)i * L, 1};
  double2 *S = P.S + (int64_t)i * 9 * L;
  double2 *Qo = S + 3 * L, *Psi = S + 6 * L, *T1 = S + 7 * L, *T2 = S + 8 * L;
  const double coef = P.par.coef[i];
  double2 vsum = c0();
  double asum = 0.0;
  for (int d = 0; d < P.b; ++d) {
    const int kh = P.dmin + d, w = P.eta - P.wmul * kh;
    pivot(Kaa, Kbb, Kab, L, w, S, P.bord ? Qo : nullptr, 1, logc, nullptr, 0, Psi, nullptr);
    if (P.bord) {
      const SR u{Kp + (int64_t)tri(a, 0) * L, 1}, x{Kp + (int64_t)tri(b, 0) * L, 1};
      const int Lo = L - 1;
      for (int t0 = 0; t0 < Lo; t0 += TB) {
        double2 a1[TB], a2[TB];
#pragma unroll
        for (int k = 0; k < TB; ++k) a1[k] = a2[k] = c0();
        conv_acc(a1, t0, 0, SR{Qo, 1}, Lo, u, Lo);
        conv_acc(a1, t0, 0, SR{Qo + L, 1}, Lo, x, Lo);
        conv_acc(a2, t0, 0, SR{Qo + L, 1}, Lo, u, Lo);
        conv_acc(a2, t0, 0, SR{Qo + 2 * L, 1}, Lo, x, Lo);
#pragma unroll
        for (int k = 0; k < TB; ++k)
          if (t0 + k < Lo) { T1[t0 + k] = a1[k]; T2[t0 + k] = a2[k]; }
      }
      for (int t0 = 0; t0 < L; t0 += TB) {
        double2 acc[TB];
#pragma unroll
        for (int k = 0; k < TB; ++k) acc[k] = (t0 + k < L) ? Kp[t0 + k] : c0();
        conv_acc(acc, t0, 1, u, Lo, SR{T1, 1}, Lo);
        conv_acc(acc, t0, 1, x, Lo, SR{T2, 1}, Lo);
#pragma unroll
        for (int k = 0; k < TB; ++k) {
          const int t = t0 + k;
          if (t < L) {
            const double2 k00 = acc[k], lc = at(logc, t), tl = Psi[t];
            Psi[t] = make_double2(0.5 * (t * (k00.x - lc.x) - tl.x), 0.5 * (t * (k00.y - lc.y) - tl.y));
          }
        }
      }
    } else {
      for (int t = 0; t < L; ++t) {
        const double2 lc = at(logc, t), tl = Psi[t];
        Psi[t] = make_double2(-0.5 * (t * lc.x + tl.x), -0.5 * (t * lc.y + tl.y));
      }
    }
    ser_exp(S, 1, Psi, L);
    const double2 g = S[L - 1];
    const double f = coef * ((kh & 1) ? -1.0 : 1.0) * binom_d(P.eta, kh);
    vsum.x = fma(f, g.x, vsum.x);
    vsum.y = fma(f, g.y, vsum.y);
    asum += fabs(f) * hypot(g.x, g.y);
  }
  P.val[i] = vsum;
  P.absv[i] = asum;
}

// Whole units of the chunk: one block per unit sums its per-node values (thread t: nodes
// t, t + 256, ... in double-double; then a fixed-shape tree over the threads) and writes the
// unit's partial.  The order depends only on the unit's size: results are independent of the
// chunking and of the rank count.
__global__ void __launch_bounds__(256) tree_reduce_k(const double2 *val, const double *absv,
                                                     uint64_t per_unit, uint64_t unit0, Partial *partials) {
  __shared__ double sh[6][256];
  const uint64_t u = blockIdx.x;
  const int t = threadIdx.x;
  double rh = 0, rl = 0, ih = 0, il = 0, ah = 0, al = 0;
  for (uint64_t m = t; m < per_unit; m += 256) {
    const double2 v = val[u * per_unit + m];
    dd_add(rh, rl, v.x);
    dd_add(ih, il, v.y);
    dd_add(ah, al, absv[u * per_unit + m]);
  }
  sh[0][t] = rh; sh[1][t] = rl; sh[2][t] = ih; sh[3][t] = il; sh[4][t] = ah; sh[5][t] = al;
  __syncthreads();
  for (int s = 128; s; s >>= 1) {
    if (t < s) {
      dd_add_dd(sh[0][t], sh[1][t], sh[0][t + s], sh[1][t + s]);
      dd_add_dd(sh[2][t], sh[3][t], sh[2][t + s], sh[3][t + s]);
      dd_add_dd(sh[4][t], sh[5][t], sh[4][t + s], sh[5][t + s]);
    }
    __syncthreads();
  }
  if (t == 0) {
    Partial q;
    q.re_hi = sh[0][0]; q.re_lo = sh[1][0]; q.im_hi = sh[2][0]; q.im_lo = sh[3][0];
    q.abs_hi = sh[4][0]; q.abs_lo = sh[5][0];
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
  const uint64_t slot = i / NE;
  const int e = (int)(i - slot * NE);
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
  double2 *o = out.K + ((int64_t)slot * NE + e) * L;
  o[0] = v;
  for (int s = 1; s < L; ++s) o[s] = c0();
  if (e == 0) {
    for (int s = 0; s < L; ++s) out.logc[(int64_t)slot * L + s] = c0();
    out.coef[slot] = 1.0;
  }
}

// ------------------------------------------------------------------ host driver

// Buffers come from the device's stream-ordered pool (its release threshold is kept at the
// maximum, lhaf_host.cpp): a new job reuses the memory of the jobs destroyed before it.
static cudaError_t grow(void **p, size_t &have, size_t need, cudaStream_t st) {
  if (need <= have) return cudaSuccess;
  if (*p) cudaFreeAsync(*p, st);
  *p = nullptr;
  have = 0;
  cudaError_t e = cudaMallocAsync(p, need, st);
  if (e == cudaSuccess) have = need;
  return e;
}

static inline unsigned blocks_for(uint64_t n) { return (unsigned)((n + 127) / 128); }

// Bytes per depth for the run's level buffers (the chunk capacity): bigger chunks mean fewer,
// larger launches (measured: 512 MB -> 1-2 GB per depth +5-7 % at cfg4, smaller -25 % and
// worse, profiles/r02/ab_s3_level.txt); default 32 GB / H clamped to [512 MB, 2 GB] so that all
// depths together stay within 32 GB of the 180 GB.  LHAF_TREE_LEVEL_MB overrides.  The unit
// plan always uses TreeWork::kLevelBudget: results do not depend on this choice.
static size_t run_budget(int H) {
  static const long env_mb = [] {
    const char *e = getenv("LHAF_TREE_LEVEL_MB");
    return e ? atol(e) : 0L;
  }();
  if (env_mb > 0) return (size_t)env_mb << 20;
  const size_t b = ((size_t)32 << 30) / (size_t)std::max(1, H);
  return std::min(std::max(b, TreeWork::kLevelBudget), (size_t)2 << 30);
}

static int reg_limit() {  // LHAF_TREE_REGL: largest L for the register-array kernels (default 40)
  static const int v = [] {
    const char *e = getenv("LHAF_TREE_REGL");
    return e ? atoi(e) : 40;
  }();
  return v;
}

static size_t bc_smem(int Ep, int b, int L, int G) {
  return ((size_t)bc_smem_parents(G, b) * 2 * Ep + (size_t)G * (2 * Ep + 3)) * L * sizeof(double2);
}
// Children per block G and threads per block for tree_bc_k: the choice that maximises a model
// of the block's task rounds (each phase's tasks are spread over the block's threads; a round
// = one task per thread): the lane utilisation of the rounds (idle lanes of a partial round
// still hold the DFMA pipe) x the saturation of resident warps (14 per SM).  A/B knob
// LHAF_BC_MODEL: 2 (default) this; 1 children per round-time x blocks; 0 the
// fixed heuristic (128 threads, about two tasks each).
static size_t bc_choose(int Ep, int NEc, int b, int L, int &Gbest, int &nbest) {
  static int regs = 0;
  if (!regs) {
    cudaFuncAttributes fa;
    regs = (cudaFuncGetAttributes(&fa, tree_bc_k) == cudaSuccess && fa.numRegs > 0) ? fa.numRegs : 168;
    regs = (regs + 7) / 8 * 8;
  }
  const int Lo = L - 1, PB = ((Lo + TB - 1) / TB + 1) / 2, PC = ((L + TB - 1) / TB + 1) / 2;
  const size_t cap = (size_t)LHAF_BC_SMEM_KB << 10;
  static const int model = [] {
    const char *e = getenv("LHAF_BC_MODEL");
    return e ? atoi(e) : 2;
  }();
  if (!model) {
    int G = std::max(1, 2 * 128 / (2 * Ep + NEc) + 1);
    while (G > 1 && bc_smem(Ep, b, L, G) > cap) --G;
    Gbest = G; nbest = 128;
    return bc_smem(Ep, b, L, G);
  }
  double best = -1.0;
  size_t bestb = bc_smem(Ep, b, L, 1);
  Gbest = 1; nbest = 128;
  for (int nth = 64; nth <= BC_THREADS; nth += 32)
    for (int G = 1; G <= 64; ++G) {
      const size_t sb = bc_smem(Ep, b, L, G);
      if (sb > (size_t)(220 << 10)) break;
      if (G > 1 && sb > cap) break;
      auto rounds = [&](long t) { return (double)((t + nth - 1) / nth); };
      const double r = rounds((long)G * 2 * Ep * PB) + rounds((long)G * NEc * PC);
      const int bl_smem = (int)((228u << 10) / (sb + 1024)), bl_reg = 65536 / (regs * nth);
      const int blocks = std::max(1, std::min(std::min(bl_smem, bl_reg), std::min(32, 64 / (nth / 32))));
      const double warps = (double)blocks * nth / 32.0;
      // model 1: children per round-time; model 2: lane utilisation of the block's task rounds
      // (idle lanes of a partial round still occupy the DFMA pipe) x resident-warp saturation
      const double util = (double)((long)G * 2 * Ep * PB + (long)G * NEc * PC) / (r * nth);
      const double score = model == 2 ? util * std::min(1.0, warps / 14.0) + 1e-3 * G
                                      : (double)blocks * G / r * std::min(1.0, warps / 12.0);
      if (score > best) { best = score; Gbest = G; nbest = nth; bestb = sb; }
    }
  return bestb;
}

static bool pivot_staged() {  // LHAF_TREE_PIVOT=0: the register kernel reading HBM (A/B knob)
  static const bool v = [] {
    const char *e = getenv("LHAF_TREE_PIVOT");
    return e ? atoi(e) != 0 : true;
  }();
  return v;
}

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
    cudaError_t e = grow((void **)&T.K, w.kbytes[k], (size_t)L * NE * cap[k] * sizeof(double2), st);
    if (e == cudaSuccess) e = grow((void **)&T.logc, w.lbytes[k], (size_t)L * cap[k] * sizeof(double2), st);
    if (e == cudaSuccess) e = grow((void **)&T.coef, w.cbytes[k], (size_t)cap[k] * sizeof(double), st);
    if (e == cudaSuccess) e = grow(&w.aux[k], w.abytes[k], (size_t)L * cap[k] * sizeof(double2), st);
    return e;
  }

  cudaError_t leaf(uint64_t gs, uint64_t cnt) {
    const int k = H - 1;
    TLeaf P;
    P.par = w.lv[k];
    P.np = cnt;
    P.L = L; P.E = E[k]; P.bord = g.bord; P.b = b[k]; P.dmin = dmin[k]; P.eta = eta[k]; P.wmul = g.wmul;
    P.S = (double2 *)w.scratch;
    P.val = (double2 *)w.val;
    P.absv = (double *)w.absv;
    P.cut_eb = g.cut_eb; P.nf = g.nf; P.vstride = cap[k];
    ++lhaf::g_launches;
    const int rl = reg_limit();
    if (g.cut_eb >= 0) {  // cutoff group: register-array leaf only (the host keeps L <= 40 here)
      const uint64_t per = Pk[k], units = cnt / per;
      if (L <= 16) tree_leaf_r<16><<<blocks_for(cnt), 128, 0, st>>>(P);
      else if (L <= 24) tree_leaf_r<24><<<blocks_for(cnt), 128, 0, st>>>(P);
      else if (L <= 32) tree_leaf_r<32><<<blocks_for(cnt), 128, 0, st>>>(P);
      else tree_leaf_r<40><<<blocks_for(cnt), 128, 0, st>>>(P);
      cudaError_t e = cudaGetLastError();
      for (int m = 0; m <= g.cut_eb && e == cudaSuccess; ++m) {
        ++lhaf::g_launches;
        tree_reduce_k<<<(unsigned)units, 256, 0, st>>>(P.val + m * cap[k], P.absv + m * cap[k], per,
                                                       g.part_base + (uint64_t)m * g.units_pp + gs / per, J.partials);
        e = cudaGetLastError();
      }
      return e;
    }
    if (L <= 16 && L <= rl) tree_leaf_r<16><<<blocks_for(cnt), 128, 0, st>>>(P);
    else if (L <= 24 && L <= rl) tree_leaf_r<24><<<blocks_for(cnt), 128, 0, st>>>(P);
    else if (L <= 32 && L <= rl) tree_leaf_r<32><<<blocks_for(cnt), 128, 0, st>>>(P);
    else if (L <= 40 && L <= rl) tree_leaf_r<40><<<blocks_for(cnt), 128, 0, st>>>(P);
    else tree_leaf_g<<<blocks_for(cnt), 128, 0, st>>>(P);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    const uint64_t per = Pk[k], units = cnt / per;
    ++lhaf::g_launches;
    tree_reduce_k<<<(unsigned)units, 256, 0, st>>>(P.val, P.absv, per, g.unit_base + gs / per, J.partials);
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
    const int rl = reg_limit();
    const bool regk = L <= 40 && L <= rl;
    if (regk) {  // Delta of the parents of this expansion (shared by their children's pivots)
      const uint64_t p0 = lo / nb - gs, np = (hi - 1) / nb - gs - p0 + 1;
      TStep D;
      D.par = w.lv[k]; D.L = L; D.E = E[k]; D.auxp = (double2 *)w.aux[k];
      ++lhaf::g_launches;
      if (L <= 16) tree_delta_r<16><<<blocks_for(np), 128, 0, st>>>(D, p0, np);
      else if (L <= 24) tree_delta_r<24><<<blocks_for(np), 128, 0, st>>>(D, p0, np);
      else if (L <= 32) tree_delta_r<32><<<blocks_for(np), 128, 0, st>>>(D, p0, np);
      else tree_delta_r<40><<<blocks_for(np), 128, 0, st>>>(D, p0, np);
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
      P.L = L; P.E = E[k]; P.b = b[k]; P.dmin = dmin[k]; P.eta = eta[k]; P.wmul = g.wmul;
      P.auxp = (double2 *)w.aux[k];
      const int Ep = E[k] - 2, NEc = Ep * (Ep + 1) / 2;
      P.Q = (double2 *)w.scratch;
      P.S = P.Q + (size_t)3 * L * n;
      P.T = P.S + (size_t)3 * L * n;
      ++lhaf::g_launches;
      const bool staged = pivot_staged() && nb >= 2;
      const size_t pv_smem = (size_t)3 * pv_parents((int)nb) * pv_stride(L) * sizeof(double2);
#define LHAF_PIVOT(LMV)                                                                         \
  do {                                                                                          \
    if (staged) {                                                                               \
      static bool set = false;                                                                  \
      if (!set) {                                                                               \
        cudaFuncSetAttribute(tree_pivot_s<LMV>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 << 10); \
        set = true;                                                                             \
      }                                                                                         \
      tree_pivot_s<LMV><<<(unsigned)((n + PV_THREADS - 1) / PV_THREADS), PV_THREADS, pv_smem, st>>>(P); \
    } else {                                                                                    \
      tree_pivot_r<LMV><<<blocks_for(n), 128, 0, st>>>(P);                                      \
    }                                                                                           \
  } while (0)
      if (L <= 16 && regk) LHAF_PIVOT(16);
      else if (L <= 24 && regk) LHAF_PIVOT(24);
      else if (L <= 32 && regk) LHAF_PIVOT(32);
      else if (regk) LHAF_PIVOT(40);
      else tree_pivot_g<<<blocks_for(n), 128, 0, st>>>(P);
#undef LHAF_PIVOT
      if (Ep > 0) {
        int G = 1, nth = 128;  // children and threads per block (bc_choose)
        const size_t sbytes = bc_choose(Ep, NEc, (int)nb, L, G, nth);
        if (sbytes <= (size_t)(220 << 10)) {
          P.G = G;
          ++lhaf::g_launches;
          tree_bc_k<<<(unsigned)((n + G - 1) / G), nth, sbytes, st>>>(P);
        } else {
          lhaf::g_launches += 2;
          tree_tmat_g<<<blocks_for(n * Ep), 128, 0, st>>>(P);
          tree_update_g<<<blocks_for(n * (uint64_t)NEc), 128, 0, st>>>(P);
        }
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
      ++lhaf::g_launches;
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
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(tree::tree_bc_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 << 10);
    if (e != cudaSuccess) return e;
    attr = true;
  }
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
    uint64_t c = (uint64_t)std::max(1.0, (double)tree::run_budget(H) / nbytes);
    // never more than the forest has at this depth (small jobs keep small buffers)
    double forest = (double)g.npat;
    for (int l = 0; l < k; ++l) forest *= (double)R.b[l];
    if ((double)c > forest) c = (uint64_t)forest;
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
  if (w.aux.size() < (size_t)H) { w.aux.resize(H, nullptr); w.abytes.resize(H, 0); }
  cudaError_t e = cudaSuccess;
  for (int k = 0; k < H && e == cudaSuccess; ++k) e = R.level_alloc(k);
  if (e == cudaSuccess) e = tree::grow(&w.scratch, w.scratch_bytes, scratch * sizeof(double2), st);
  const size_t nvals = (size_t)R.cap[H - 1] * (size_t)(g.cut_eb >= 0 ? g.cut_eb + 1 : 1);
  if (e == cudaSuccess) e = tree::grow(&w.val, w.val_bytes, nvals * sizeof(double2), st);
  if (e == cudaSuccess) e = tree::grow(&w.absv, w.abs_bytes, nvals * sizeof(double), st);
  if (e != cudaSuccess) return e;
  return R.run();
}

void tree_work_free(TreeWork &w) {
  for (auto &l : w.lv) {
    if (l.K) cudaFreeAsync(l.K, 0);
    if (l.logc) cudaFreeAsync(l.logc, 0);
    if (l.coef) cudaFreeAsync(l.coef, 0);
  }
  w.lv.clear();
  w.kbytes.clear(); w.lbytes.clear(); w.cbytes.clear();
  for (auto &a : w.aux)
    if (a) cudaFreeAsync(a, 0);
  w.aux.clear(); w.abytes.clear();
  if (w.scratch) cudaFreeAsync(w.scratch, 0);
  if (w.val) cudaFreeAsync(w.val, 0);
  if (w.absv) cudaFreeAsync(w.absv, 0);
  w.scratch = w.val = w.absv = nullptr;
  w.scratch_bytes = w.val_bytes = w.abs_bytes = 0;
}

}  // namespace lhaf
