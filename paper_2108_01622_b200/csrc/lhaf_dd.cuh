// lhaf_dd.cuh -- the precise per-term tail (precision mode 1): trailing La Budde and the power
// series of a7-a9 in complex double-double arithmetic (~106-bit significands), on the FP64
// Hessenberg band.  DESIGN.md section 6 "Precise mode".  Product code only.
//
// Why these two stages: the per-term rounding error of the FP64 pipeline at the BASELINE sizes
// is dominated by La Budde (the coefficient recursion cancels) and, for the natural pairing of
// mixed states, by the series; the Hessenberg reduction itself contributes ~1e-15..1e-14
// (tests/diag/stage_errors.py: each stage swapped to long double in turn).  Carrying the
// characteristic-polynomial coefficients and the series in double-double leaves the FP64
// reduction as the only per-term error source.
#pragma once
#include <cuda_runtime.h>
#include "lhaf_device.cuh"
#include "lhaf_tail.cuh"

namespace lhaf {
namespace dd {

// complex double-double: value = h + l componentwise (re = h.x + l.x, im = h.y + l.y)
struct C {
  double2 h, l;
};

__device__ __forceinline__ C zero() { return {make_double2(0.0, 0.0), make_double2(0.0, 0.0)}; }
__device__ __forceinline__ C one() { return {make_double2(1.0, 0.0), make_double2(0.0, 0.0)}; }
__device__ __forceinline__ C from(double2 x) { return {x, make_double2(0.0, 0.0)}; }

__device__ __forceinline__ void qts(double a, double b, double &s, double &e) {
  s = a + b;
  e = b - (s - a);
}
__device__ __forceinline__ void ts(double a, double b, double &s, double &e) {
  s = a + b;
  const double bb = s - a;
  e = (a - (s - bb)) + (b - bb);
}
// real double-double sum (sloppy add: absolute error ~2^-104 max(|a|, |b|))
__device__ __forceinline__ void add1(double ah, double al, double bh, double bl, double &sh, double &sl) {
  double s, e;
  ts(ah, bh, s, e);
  e += al + bl;
  qts(s, e, sh, sl);
}
__device__ __forceinline__ C add(const C &a, const C &b) {
  C r;
  add1(a.h.x, a.l.x, b.h.x, b.l.x, r.h.x, r.l.x);
  add1(a.h.y, a.l.y, b.h.y, b.l.y, r.h.y, r.l.y);
  return r;
}
__device__ __forceinline__ C neg(const C &a) {
  return {make_double2(-a.h.x, -a.h.y), make_double2(-a.l.x, -a.l.y)};
}
__device__ __forceinline__ C norm(const C &a) {
  C r;
  qts(a.h.x, a.l.x, r.h.x, r.l.x);
  qts(a.h.y, a.l.y, r.h.y, r.l.y);
  return r;
}

// Unnormalised accumulator (Dot2-style): acc.h collects the rounded products by error-free
// sums, acc.l the product errors and the sum errors; norm() at the end.
// acc += f * q   (f: complex double, q: complex double-double)
__device__ __forceinline__ void acc_fq(C &acc, double2 f, const C &q) {
  // re += f.x q.re - f.y q.im ; im += f.x q.im + f.y q.re
  double p, e, s, err;
  p = f.x * q.h.x; e = fma(f.x, q.l.x, fma(f.x, q.h.x, -p));
  ts(acc.h.x, p, s, err); acc.h.x = s; acc.l.x += err + e;
  p = -f.y * q.h.y; e = fma(-f.y, q.l.y, fma(-f.y, q.h.y, -p));
  ts(acc.h.x, p, s, err); acc.h.x = s; acc.l.x += err + e;
  p = f.x * q.h.y; e = fma(f.x, q.l.y, fma(f.x, q.h.y, -p));
  ts(acc.h.y, p, s, err); acc.h.y = s; acc.l.y += err + e;
  p = f.y * q.h.x; e = fma(f.y, q.l.x, fma(f.y, q.h.x, -p));
  ts(acc.h.y, p, s, err); acc.h.y = s; acc.l.y += err + e;
}
// acc += a * b   (both complex double-double)
__device__ __forceinline__ void acc_qq(C &acc, const C &a, const C &b) {
  double p, e, s, err;
#define LHAF_DD_TERM(SIGN, AH, AL, BH, BL, DH, DL)                      \
  p = SIGN (AH) * (BH);                                                 \
  e = fma(SIGN (AH), (BH), -p) + (SIGN (AH) * (BL) + SIGN (AL) * (BH)); \
  ts(DH, p, s, err);                                                    \
  DH = s;                                                               \
  DL += err + e;
  LHAF_DD_TERM(+, a.h.x, a.l.x, b.h.x, b.l.x, acc.h.x, acc.l.x)
  LHAF_DD_TERM(-, a.h.y, a.l.y, b.h.y, b.l.y, acc.h.x, acc.l.x)
  LHAF_DD_TERM(+, a.h.x, a.l.x, b.h.y, b.l.y, acc.h.y, acc.l.y)
  LHAF_DD_TERM(+, a.h.y, a.l.y, b.h.x, b.l.x, acc.h.y, acc.l.y)
#undef LHAF_DD_TERM
}
// x * s for a double s (each component a double-double times a double)
__device__ __forceinline__ C scale(const C &x, double s) {
  C r;
  double p, e;
  p = x.h.x * s; e = fma(x.l.x, s, fma(x.h.x, s, -p)); qts(p, e, r.h.x, r.l.x);
  p = x.h.y * s; e = fma(x.l.y, s, fma(x.h.y, s, -p)); qts(p, e, r.h.y, r.l.y);
  return r;
}
// x / m for a small positive integer m (quotient of the high part, exact remainder by fma)
__device__ __forceinline__ C div_int(const C &x, double m) {
  C r;
  double q, rem;
  q = x.h.x / m; rem = fma(-q, m, x.h.x); qts(q, (rem + x.l.x) / m, r.h.x, r.l.x);
  q = x.h.y / m; rem = fma(-q, m, x.h.y); qts(q, (rem + x.l.y) / m, r.h.y, r.l.y);
  return r;
}
__device__ __forceinline__ C shfl(const C &v, int src) {
  return {shfl2(v.h, src), shfl2(v.l, src)};
}
__device__ __forceinline__ C shfl_xor(const C &v, int m) {
  return {shfl2_xor(v.h, m), shfl2_xor(v.l, m)};
}
__device__ __forceinline__ C shfl_down(const C &v, int d) {
  return {shfl2_down(v.h, d), shfl2_down(v.l, d)};
}
__device__ __forceinline__ C ld(const double2 *H, const double2 *Lo, int i) { return {H[i], Lo[i]}; }
__device__ __forceinline__ void st(double2 *H, double2 *Lo, int i, const C &v) {
  H[i] = v.h;
  Lo[i] = v.l;
}

// Level-by-level team La Budde (tail::labudde_levels_team) in double-double: the band F is the
// FP64 Hessenberg band; q coefficients, the level ring and the warp totals are double-double.
// Qh/Ql: [E + 1][BS]; Lh/Ll: [2][64]; Th/Tl: [2][NW].
template <int NW, int TEAMS, int NTLMAX>
__device__ __forceinline__ void labudde_levels_team(const double2 *hb, double2 *Qh, double2 *Ql,
                                                    double2 *Lh, double2 *Ll, double2 *Th,
                                                    double2 *Tl, int E, int NTL, int BS, int warp,
                                                    int lane, int team) {
  constexpr int MT = NTLMAX / 2;
  const int i = warp * 16 + (lane >> 1), h = lane & 1;
  const bool ri = i < E;
  const int ci = min(i, E);
  const int mx = ri ? E - 1 - i : 0;
  const double2 *F = hb + ci * BS + 1;
  const double2 hii = (ri && h == 0) ? F[0] : c0();
  const double2 mhii = make_double2(-hii.x, -hii.y);
  if (h == 0 && i <= E) st(Qh, Ql, i * BS, one());
  if (warp == 0 && lane == 0 && E >= NW * 16) st(Qh, Ql, E * BS, one());
  tail::team_sync<NW, TEAMS>(team);
  for (int t = 1; t <= NTL; ++t) {
    const int pb = (t - 1) & 1, cb = t & 1;
    if (t - 1 >= 1) {  // finalise level t-1 of my rows
      C Cw = zero();
#pragma unroll
      for (int w = NW - 1; w > 0; --w)
        if (w > warp) Cw = add(Cw, ld(Th, Tl, pb * NW + w));
      if (h == 0 && i <= E)
        st(Qh, Ql, i * BS + t - 1, (i < E && t - 1 <= E - i) ? add(ld(Lh, Ll, pb * 64 + i), Cw) : zero());
    }
    if (t == NTL) break;
    C a = zero(), b = zero();
    if (h == 0) {
      const int s = i + 1;
      C q;
      if (t - 1 == 0) q = (s <= E) ? one() : zero();
      else if (s >= E || s >= NW * 16) q = zero();
      else {
        C Cs = zero();
        const int ws = s >> 4;
#pragma unroll
        for (int w = NW - 1; w > 0; --w)
          if (w > ws) Cs = add(Cs, ld(Th, Tl, pb * NW + w));
        q = add(ld(Lh, Ll, pb * 64 + s), Cs);
      }
      acc_fq(a, mhii, q);
    }
#pragma unroll
    for (int x = 0; x < MT; ++x) {
      const int m = 1 + h + 2 * x;
      if (2 * x + 1 > NTLMAX - 2) break;
      const bool ok = m <= t - 1 && m <= mx;
      const double2 f = ok ? F[m] : c0();
      const int qi = min(i + m + 1, E) * BS + max(t - m - 1, 0);
      const double2 mf = make_double2(-f.x, -f.y);
      if (x & 1) acc_fq(b, mf, ld(Qh, Ql, qi));
      else acc_fq(a, mf, ld(Qh, Ql, qi));
    }
    C u = add(norm(a), norm(b));
    u = add(u, shfl_xor(u, 1));
    if (!ri) u = zero();
#pragma unroll
    for (int off = 2; off < 32; off <<= 1) {
      const C x = shfl_down(u, off);
      if (lane + off < 32) u = add(u, x);
    }
    if (h == 0 && i < 64) st(Lh, Ll, cb * 64 + i, u);
    if (lane == 0) st(Th, Tl, cb * NW + warp, u);
    tail::team_sync<NW, TEAMS>(team);
  }
  if (warp == 0 && lane == 0 && E >= NW * 16)
    for (int tt = 1; tt < NTL; ++tt) st(Qh, Ql, E * BS + tt, zero());
  tail::team_sync<NW, TEAMS>(team);
}

// g = [lam^n] c_M^{-1/2} exp(S/2) (tail::series) in double-double, one warp, n + 2 <= 64:
// column sweeps, lane m (and m + 32) accumulates coefficient m.  cM, cB: coefficient arrays
// (hi / lo, stride 1); scratch: 6 (n + 2) double2.  Returns g rounded to complex double.
__device__ __forceinline__ double2 series(const double2 *cMh, const double2 *cMl, const double2 *cBh,
                                          const double2 *cBl, int n, int NTL, bool loops,
                                          double2 *scr, int lane) {
  constexpr int NR = 2;
  double2 *Qsh = scr, *Qsl = Qsh + (n + 2), *Rsh = Qsl + (n + 2), *Rsl = Rsh + (n + 2);
  double2 *Esh = Rsl + (n + 2), *Esl = Esh + (n + 2);
  C qa[NR], ra[NR];
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    const int m = lane + 32 * r;
    qa[r] = zero();
    ra[r] = (loops && m <= n + 1 && m < NTL) ? add(ld(cMh, cMl, m), neg(ld(cBh, cBl, m))) : zero();
  }
  const int jmax = loops ? n + 1 : n;
  for (int j = 0; j <= jmax; ++j) {
    const int lj = j & 31, rj = j >> 5;
    C qs = rj ? qa[1] : qa[0], rs = rj ? ra[1] : ra[0];
    C qj = (j == 0) ? one() : neg(div_int(norm(qs), (double)j));
    qj = shfl(qj, lj);
    const C rv = shfl(norm(rs), lj);
    if (lane == lj) { st(Qsh, Qsl, j, qj); st(Rsh, Rsl, j, rv); }
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      const int m = lane + 32 * r;
      if (m > j && m <= jmax && m - j < NTL) {
        const C c = ld(cMh, cMl, m - j);
        if (m <= n) acc_qq(qa[r], scale(c, 0.5 * (double)(m + j)), qj);
        if (loops) acc_qq(ra[r], neg(c), rv);
      }
    }
  }
  __syncwarp();
  if (!loops) {
    const C g = ld(Qsh, Qsl, n);
    return make_double2(g.h.x + g.l.x, g.h.y + g.l.y);
  }
  C ea[NR];
#pragma unroll
  for (int r = 0; r < NR; ++r) ea[r] = zero();
  for (int i = 0; i <= n; ++i) {
    const int li = i & 31, ri = i >> 5;
    const C es = ri ? ea[1] : ea[0];
    C ei = (i == 0) ? one() : div_int(norm(es), (double)i);
    ei = shfl(ei, li);
    if (lane == li) st(Esh, Esl, i, ei);
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      const int m = lane + 32 * r;
      if (m > i && m <= n) acc_qq(ea[r], scale(ld(Rsh, Rsl, m - i + 1), 0.5 * (double)(m - i)), ei);
    }
  }
  __syncwarp();
  C gp = zero();
  for (int m = lane; m <= n; m += 32) acc_qq(gp, ld(Qsh, Qsl, m), ld(Esh, Esl, n - m));
  gp = norm(gp);
#pragma unroll
  for (int off = 16; off; off >>= 1) gp = add(gp, shfl_xor(gp, off));
  return make_double2(gp.h.x + gp.l.x, gp.h.y + gp.l.y);
}

}  // namespace dd
}  // namespace lhaf
