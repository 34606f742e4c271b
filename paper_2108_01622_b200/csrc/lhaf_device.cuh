// lhaf_device.cuh -- device helpers shared by the sm_100a kernels (complex FP64 arithmetic,
// double-double accumulation, warp reductions, term decode).  Product code only.
#pragma once
#include <cuda_runtime.h>
#include <cstdio>
#include "lhaf_internal.h"

namespace lhaf {

#define LHAF_FULL 0xffffffffu

// Device-side bounds checks of a diagnostic build (-DLHAF_CHECK, tools/build_variant.py; the
// pool's compute-sanitizer is unavailable): a failed check prints its site and traps.
#ifdef LHAF_CHECK
#define LHAF_DCHECK(cond)                                                                   \
  do {                                                                                      \
    if (!(cond)) {                                                                          \
      printf("LHAF_CHECK failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__, __LINE__, \
             (int)blockIdx.x, (int)threadIdx.x);                                            \
      __trap();                                                                             \
    }                                                                                       \
  } while (0)
#else
#define LHAF_DCHECK(cond) ((void)0)
#endif

__device__ __forceinline__ double2 c0() { return make_double2(0.0, 0.0); }
__device__ __forceinline__ double2 c1() { return make_double2(1.0, 0.0); }
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// acc + a*b
__device__ __forceinline__ double2 cfma(double2 a, double2 b, double2 acc) {
  acc.x = fma(a.x, b.x, acc.x); acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y); acc.y = fma(a.y, b.x, acc.y);
  return acc;
}
// acc - a*b
__device__ __forceinline__ double2 cfms(double2 a, double2 b, double2 acc) {
  acc.x = fma(-a.x, b.x, acc.x); acc.x = fma(a.y, b.y, acc.x);
  acc.y = fma(-a.x, b.y, acc.y); acc.y = fma(-a.y, b.x, acc.y);
  return acc;
}
// acc + conj(a)*b
__device__ __forceinline__ double2 cfma_cj(double2 a, double2 b, double2 acc) {
  acc.x = fma(a.x, b.x, acc.x); acc.x = fma(a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y); acc.y = fma(-a.y, b.x, acc.y);
  return acc;
}
// acc - a*conj(b)
__device__ __forceinline__ double2 cfms_jc(double2 a, double2 b, double2 acc) {
  acc.x = fma(-a.x, b.x, acc.x); acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y); acc.y = fma(-a.y, b.x, acc.y);
  return acc;
}
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
// 1/x for x > 0 normal: the MUFU approximation refined by two Newton steps (quadratic:
// ~2^-20 -> 2^-40 -> full precision, within an ulp or two; no IEEE division slow path)
__device__ __forceinline__ double rcp_nr(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}
// 1/a = conj(b) / |b|^2 * s with b = a s, s = 2^-floor(log2 max(|re|, |im|)) (exact): scale-free,
// so a pivot anywhere in the normal range (1e-300 as well as 1e300) has a finite reciprocal
__device__ __forceinline__ double2 crecip(double2 a) {
  const double m = fmax(fabs(a.x), fabs(a.y));
  const int e = min((__double2hiint(m) >> 20) & 0x7ff, 2045);  // biased exponent of m
  const double s = __hiloint2double((2046 - e) << 20, 0);      // 2^{-(e - 1023)}
  const double bx = a.x * s, by = a.y * s;                      // max(|bx|, |by|) in [1, 2)
  const double r = rcp_nr(fma(bx, bx, by * by)) * s;
  return make_double2(bx * r, -by * r);
}

__device__ __forceinline__ double2 shfl2(double2 v, int src) {
  return make_double2(__shfl_sync(LHAF_FULL, v.x, src), __shfl_sync(LHAF_FULL, v.y, src));
}
__device__ __forceinline__ double2 shfl2_down(double2 v, int d) {
  return make_double2(__shfl_down_sync(LHAF_FULL, v.x, d), __shfl_down_sync(LHAF_FULL, v.y, d));
}
__device__ __forceinline__ double2 shfl2_xor(double2 v, int m) {
  return make_double2(__shfl_xor_sync(LHAF_FULL, v.x, m), __shfl_xor_sync(LHAF_FULL, v.y, m));
}

// xor-butterfly sums: every lane ends with bit-identical values (IEEE + is commutative).
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int m = 16; m; m >>= 1) v += __shfl_xor_sync(LHAF_FULL, v, m);
  return v;
}
__device__ __forceinline__ double2 warp_sum2(double2 v) {
#pragma unroll
  for (int m = 16; m; m >>= 1) {
    v.x += __shfl_xor_sync(LHAF_FULL, v.x, m);
    v.y += __shfl_xor_sync(LHAF_FULL, v.y, m);
  }
  return v;
}

// Pivot key of a candidate row (partial pivoting by |re| + |im|): the high word of the
// double |re| + |im| (monotone for non-negative doubles; 11 exponent + 14 mantissa bits kept,
// so the comparison is scale-free down to the smallest normal doubles -- a float conversion
// would flush candidates below ~1e-38 to "zero"), plus 1 so that only an exact zero (or a
// subnormal below 2^-1036) keeps the high part at 1 ("no pivot"), and the low 6 bits
// = 63 - label so that ties go to the smallest label.  One REDUX.MAX per warp finds the pivot.
__device__ __forceinline__ unsigned pivot_key(double2 v, int label) {
  const unsigned hi = (unsigned)__double2hiint(fabs(v.x) + fabs(v.y));
  return (((hi >> 6) + 1u) << 6) | (unsigned)(63 - label);
}

// ---------------------------------------------------------------- double-double
__device__ __forceinline__ void two_sum(double a, double b, double &s, double &e) {
  s = a + b;
  double bb = s - a;
  e = (a - (s - bb)) + (b - bb);
}
__device__ __forceinline__ void dd_add(double &hi, double &lo, double x) {
  double s, e;
  two_sum(hi, x, s, e);
  e += lo;
  hi = s + e;
  lo = e - (hi - s);
}
__device__ __forceinline__ void dd_add_dd(double &hi, double &lo, double xh, double xl) {
  double s, e;
  two_sum(hi, xh, s, e);
  e += lo + xl;
  hi = s + e;
  lo = e - (hi - s);
}

// ---------------------------------------------------------------- plan helpers
__device__ __forceinline__ int find_pattern(const JobDev &J, uint64_t u) {
  int lo = 0, hi = J.npat - 1;
  while (lo < hi) {  // largest p with unit_begin <= u
    int mid = (lo + hi + 1) >> 1;
    if (J.descs[mid].unit_begin <= u) lo = mid; else hi = mid - 1;
  }
  return lo;
}

// S8(a) a4: mixed-radix decode of term t on lanes h < H of one warp (pair 0 fastest).
// Writes w_h = eta_h - 2 k_h to w_s[h]; returns the sign (-1)^{sum k}; `weight` gets
// prod_h C(eta_h, k_h) (bit-identical on every lane).  Integer work except the binomial
// product, which is exact while it stays below 2^53.
__device__ __forceinline__ int decode_term(const PatDesc &P, const JobDev &J, uint64_t t, int lane,
                                           int *w_s, double &weight) {
  const int H = P.H;
  int kd = 0;
  double fac = 1.0;
  if (lane < H) {
    const int e = J.ipool[P.eta_off + lane];
    const uint64_t R = J.upool[P.radix_off + lane];
    kd = (int)((t / R) % (uint64_t)(e + 1));
    if ((P.flags & FLAG_CUT) && lane == H - 1) {
      w_s[lane] = kd - P.eta_b;  // batched self-pair: w in [-eta_b, eta_b], sign and binomial
      kd = 0;                    // belong to each count (applied by the caller)
    } else {
      w_s[lane] = (P.flags & FLAG_ET) ? e - kd : e - 2 * kd;
      fac = J.dpool[P.bin_off + J.ipool[P.eta_off + H + lane] + kd];
    }
  }
  const unsigned odd = __ballot_sync(LHAF_FULL, (lane < H) && (kd & 1));
#pragma unroll
  for (int m = 16; m; m >>= 1) fac *= __shfl_xor_sync(LHAF_FULL, fac, m);
  weight = fac;
  return (__popc(odd) & 1) ? -1 : 1;
}

}  // namespace lhaf
