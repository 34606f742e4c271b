// lhaf_kernels.cu -- sm_100a kernels of the repeated-pair finite-difference sieve.
//
// Per term t:
//   a4  decode t -> digits k_h (mixed radix, pair 0 fastest), w = eta - 2k, sign, weight
//   a5  M = P0 C X_w P0 (P0: the fixed reflector with P0 v = beta e1, folded into Ct = P0 C
//       by the prep kernel); loop row vector z^T = v X_w P0
//   a6  Householder Hessenberg reduction of M keeping e1 fixed (z transformed alongside)
//   a7  trailing La Budde: q_j(x) = det(xI - H[j:, j:]), j = d..0; c(lam) = det(I - lam H)
//   a8  loop terms: det(xI - H - beta e1 z'^T) = q_0 - beta D(x) (first-row expansion), so
//       sum_j s_j lam^j = beta lam D~(lam) / c(lam)
//   a9  g = [lam^n] c(lam)^{-1/2} exp(beta lam D~ / (2 c))    (= the paper's f, P:409-415,
//       with X -> X_w, reading C4)
//   a10 term = (-1)^{sum k} prod C(eta_h, k_h) g, accumulated in double-double.
// Variants: 1 = generic warp-per-term, matrix in shared memory (this file, "v1").
#include <cstdio>
#include <cuda_runtime.h>
#include "lhaf_device.cuh"

namespace lhaf {

std::atomic<unsigned long long> g_launches{0};

#define FULL LHAF_FULL

// ================================================================ variant 1 (generic)
struct V1Smem {
  double2 *A, *poly, *piA, *piB, *f, *u, *z, *tv, *c, *Dt, *Qs, *R, *r, *E;
  int *w;
};

__host__ __device__ inline int v1_words(int d, int nmax) {  // in double2 units, per warp
  const int ld = d + 1;
  return d * ld + (d + 1) * (d + 2) / 2 + 2 * d + 5 * d + (d + 1) + d + 4 * (nmax + 1) + 16;
}

__device__ inline V1Smem v1_carve(double2 *base, int d, int nmax) {
  V1Smem S;
  const int ld = d + 1;
  double2 *p = base;
  S.A = p; p += d * ld;
  S.poly = p; p += (d + 1) * (d + 2) / 2;
  S.piA = p; p += d;
  S.piB = p; p += d;
  S.f = p; p += d;
  S.u = p; p += d;
  S.z = p; p += d;
  S.tv = p; p += d;
  p += d;  // spare
  S.c = p; p += d + 1;
  S.Dt = p; p += d;
  S.Qs = p; p += nmax + 1;
  S.R = p; p += nmax + 1;
  S.r = p; p += nmax + 1;
  S.E = p; p += nmax + 1;
  S.w = reinterpret_cast<int *>(p);
  return S;
}

// g(w) for the term whose weights are already in S.w.  Warp-cooperative; all lanes return g.
__device__ double2 v1_g(const PatDesc &P, const JobDev &J, V1Smem &S, int lane) {
  const int d = P.d, H = P.H, n = P.n, ld = d + 1;
  const double2 *Ct = J.cpool + P.mat_off;
  const double2 *uh = Ct + (size_t)d * d;
  const double2 *vv = uh + d;
  const double2 beta = vv[d];
  const bool loop = vv[d + 1].x != 0.0;
  double2 *A = S.A;

  // ---- a5: M1 = Ct X_w  (column j of M1 = w_{j mod H} * column partner(j) of Ct)
  for (int idx = lane; idx < d * d; idx += 32) {
    const int i = idx / d, j = idx - i * d;
    const int h = j < H ? j : j - H;
    const int pj = j < H ? j + H : j - H;
    A[i * ld + j] = cscale(Ct[i * d + pj], (double)S.w[h]);
  }
  for (int j = lane; j < d; j += 32) {
    const int h = j < H ? j : j - H;
    const int pj = j < H ? j + H : j - H;
    S.z[j] = cscale(vv[pj], (double)S.w[h]);
  }
  __syncwarp();
  if (loop) {  // M' = M1 P0 = M1 - (M1 uh) uh^H ;  z'^T = z^T P0
    for (int i = lane; i < d; i += 32) {
      double2 acc = c0();
      for (int j = 0; j < d; ++j) acc = cfma(A[i * ld + j], uh[j], acc);
      S.tv[i] = acc;
    }
    double2 zu = c0();
    for (int j = lane; j < d; j += 32) zu = cfma(S.z[j], uh[j], zu);
    zu = warp_sum2(zu);
    __syncwarp();
    for (int idx = lane; idx < d * d; idx += 32) {
      const int i = idx / d, j = idx - i * d;
      A[i * ld + j] = cfms_jc(S.tv[i], uh[j], A[i * ld + j]);
    }
    for (int j = lane; j < d; j += 32) S.z[j] = cfms_jc(zu, uh[j], S.z[j]);
    __syncwarp();
  }

  // ---- a6: Householder Hessenberg, e1 fixed
  for (int k = 0; k < d - 2; ++k) {
    const int len = d - k - 1;
    double s2 = 0.0;
    for (int i = lane + 1; i < len; i += 32) {
      const double2 x = A[(k + 1 + i) * ld + k];
      s2 = fma(x.x, x.x, fma(x.y, x.y, s2));
    }
    s2 = warp_sum(s2);
    if (s2 == 0.0) continue;  // column already reduced
    const double2 x0 = A[(k + 1) * ld + k];
    const double ax0 = hypot(x0.x, x0.y);
    const double nx = sqrt(fma(ax0, ax0, s2));
    const double2 ph = ax0 > 0.0 ? make_double2(x0.x / ax0, x0.y / ax0) : make_double2(1.0, 0.0);
    const double2 alpha = make_double2(-ph.x * nx, -ph.y * nx);
    const double sc = 1.0 / (nx * (nx + ax0));
    for (int i = lane; i < len; i += 32) {
      const double2 x = A[(k + 1 + i) * ld + k];
      S.u[i] = (i == 0) ? csub(x, alpha) : x;
      A[(k + 1 + i) * ld + k] = (i == 0) ? alpha : c0();
    }
    __syncwarp();
    // left: rows k+1.., columns k+1..d-1
    for (int j = k + 1 + lane; j < d; j += 32) {
      double2 wj = c0();
      for (int i = 0; i < len; ++i) wj = cfma_cj(S.u[i], A[(k + 1 + i) * ld + j], wj);
      wj = cscale(wj, sc);
      for (int i = 0; i < len; ++i) A[(k + 1 + i) * ld + j] = cfms(S.u[i], wj, A[(k + 1 + i) * ld + j]);
    }
    __syncwarp();
    // right: all rows, columns k+1..d-1
    for (int i = lane; i < d; i += 32) {
      double2 yi = c0();
      for (int j = 0; j < len; ++j) yi = cfma(A[i * ld + k + 1 + j], S.u[j], yi);
      yi = cscale(yi, sc);
      for (int j = 0; j < len; ++j) A[i * ld + k + 1 + j] = cfms_jc(yi, S.u[j], A[i * ld + k + 1 + j]);
    }
    if (loop) {
      double2 zu = c0();
      for (int j = lane; j < len; j += 32) zu = cfma(S.z[k + 1 + j], S.u[j], zu);
      zu = cscale(warp_sum2(zu), sc);
      for (int j = lane; j < len; j += 32) S.z[k + 1 + j] = cfms_jc(zu, S.u[j], S.z[k + 1 + j]);
    }
    __syncwarp();
  }

  // ---- a7: trailing La Budde.  q_j stored at poly + (d-j)(d-j+1)/2, d-j+1 coeffs (low->high)
  double2 *poly = S.poly;
  if (lane == 0) poly[0] = make_double2(1.0, 0.0);  // q_d = 1
  double2 *piPrev = S.piA, *piCur = S.piB;
  __syncwarp();
  for (int j = d - 1; j >= 0; --j) {
    const int mmax = d - 1 - j;
    const double2 sub = (j + 1 < d) ? A[(j + 1) * ld + j] : c0();
    for (int m = lane; m <= mmax; m += 32) {
      const double2 pim = (m == 0) ? make_double2(1.0, 0.0) : cmul(sub, piPrev[m - 1]);
      piCur[m] = pim;
      if (m >= 1) S.f[m] = cmul(A[j * ld + j + m], pim);
    }
    __syncwarp();
    const int L = d - j + 1;
    const double2 *q1 = poly + (d - j - 1) * (d - j) / 2;   // q_{j+1}, length d-j
    double2 *qj = poly + (d - j) * (d - j + 1) / 2;
    const double2 hjj = A[j * ld + j];
    for (int i = lane; i < L; i += 32) {
      double2 val = (i >= 1) ? q1[i - 1] : c0();
      if (i <= L - 2) val = cfms(hjj, q1[i], val);
      for (int m = 1; m <= mmax; ++m) {
        const int lenq = d - j - m;  // length of q_{j+m+1}
        if (i >= lenq) break;
        const double2 *qm = poly + (d - j - m - 1) * (d - j - m) / 2;
        val = cfms(S.f[m], qm[i], val);
      }
      qj[i] = val;
    }
    double2 *tmp = piPrev; piPrev = piCur; piCur = tmp;
    __syncwarp();
  }
  // c_m = q_0[d-m]
  const double2 *q0 = poly + d * (d + 1) / 2;
  for (int m = lane; m <= d; m += 32) S.c[m] = q0[d - m];

  // ---- a8: D(x) = sum_{m=0}^{d-1} z'_m pi_{0,m} q_{m+1}(x); Dt_m = D[d-1-m]
  if (loop) {
    for (int m = lane; m < d; m += 32) S.f[m] = cmul(S.z[m], piPrev[m]);  // piPrev = pi_{0,.}
    __syncwarp();
    for (int i = lane; i < d; i += 32) {
      double2 val = c0();
      for (int m = 0; m < d; ++m) {
        const int lenq = d - m;  // length of q_{m+1}
        if (i >= lenq) break;
        const double2 *qm = poly + (d - m - 1) * (d - m) / 2;
        val = cfma(S.f[m], qm[i], val);
      }
      S.Dt[d - 1 - i] = val;
    }
  }
  __syncwarp();

  // ---- a9: series.  Qs = c^{-1/2}: m Qs_m = -sum_{i=1}^{min(m,d)} (m - i/2) c_i Qs_{m-i}
  if (lane == 0) S.Qs[0] = make_double2(1.0, 0.0);
  __syncwarp();
  for (int m = 1; m <= n; ++m) {
    double2 acc = c0();
    const int im = m < d ? m : d;
    for (int i = 1 + lane; i <= im; i += 32) acc = cfma(cscale(S.c[i], (double)m - 0.5 * i), S.Qs[m - i], acc);
    acc = warp_sum2(acc);
    if (lane == 0) S.Qs[m] = cscale(acc, -1.0 / m);
    __syncwarp();
  }
  if (!loop) return S.Qs[n];
  // R = Dt / c (power series), r_m = beta R_{m-1}; E = exp(r/2): m E_m = 1/2 sum_j j r_j E_{m-j}
  for (int m = 0; m < n; ++m) {
    double2 acc = c0();
    const int im = m < d ? m : d;
    for (int i = 1 + lane; i <= im; i += 32) acc = cfma(S.c[i], S.R[m - i], acc);
    acc = warp_sum2(acc);
    if (lane == 0) S.R[m] = csub(m < d ? S.Dt[m] : c0(), acc);
    __syncwarp();
  }
  for (int m = lane; m <= n; m += 32) S.r[m] = (m == 0) ? c0() : cmul(beta, S.R[m - 1]);
  if (lane == 0) S.E[0] = make_double2(1.0, 0.0);
  __syncwarp();
  for (int m = 1; m <= n; ++m) {
    double2 acc = c0();
    for (int jj = 1 + lane; jj <= m; jj += 32) acc = cfma(cscale(S.r[jj], (double)jj), S.E[m - jj], acc);
    acc = warp_sum2(acc);
    if (lane == 0) S.E[m] = cscale(acc, 0.5 / m);
    __syncwarp();
  }
  double2 g = c0();
  for (int m = lane; m <= n; m += 32) g = cfma(S.Qs[m], S.E[n - m], g);
  return warp_sum2(g);
}

__global__ void __launch_bounds__(128) sieve_v1(JobDev J, uint64_t ubeg, uint64_t uend, int dmax,
                                                int nmax, int per_warp) {
  extern __shared__ double2 smem[];
  __shared__ unsigned long long s_unit;
  __shared__ double s_acc[4][6];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, W = blockDim.x >> 5;
  V1Smem S = v1_carve(smem + (size_t)warp * per_warp, dmax, nmax);
  for (;;) {
    if (threadIdx.x == 0) s_unit = ubeg + atomicAdd(J.counter, 1ull);
    __syncthreads();
    const uint64_t u = s_unit;
    if (u >= uend) break;
    const PatDesc P = J.descs[find_pattern(J, u)];
    const uint64_t tb = (u - P.unit_begin) * P.chunk;
    const uint64_t te = min(tb + P.chunk, P.T_eval);
    double rh = 0, rl = 0, ih = 0, il = 0, ah = 0, al = 0;
    for (uint64_t t = tb + warp; t < te; t += W) {
      double weight;
      const int sign = decode_term(P, J, t, lane, S.w, weight);
      const double2 g = v1_g(P, J, S, lane);
      const double sw = sign * weight;
      dd_add(rh, rl, sw * g.x);
      dd_add(ih, il, sw * g.y);
      dd_add(ah, al, weight * hypot(g.x, g.y));
      __syncwarp();
    }
    if (lane == 0) {
      s_acc[warp][0] = rh; s_acc[warp][1] = rl; s_acc[warp][2] = ih;
      s_acc[warp][3] = il; s_acc[warp][4] = ah; s_acc[warp][5] = al;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double a0 = 0, a1 = 0, a2 = 0, a3 = 0, a4 = 0, a5 = 0;
      for (int w = 0; w < W; ++w) {
        dd_add_dd(a0, a1, s_acc[w][0], s_acc[w][1]);
        dd_add_dd(a2, a3, s_acc[w][2], s_acc[w][3]);
        dd_add_dd(a4, a5, s_acc[w][4], s_acc[w][5]);
      }
      Partial q;
      q.re_hi = a0; q.re_lo = a1; q.im_hi = a2; q.im_lo = a3; q.abs_hi = a4; q.abs_lo = a5;
      q.pad0 = 0; q.pad1 = 0;
      J.partials[u] = q;
    }
  }
}

// Diagnostic: g(t) (unweighted) of pattern 0 for a list of term indices; one warp per index.
__global__ void __launch_bounds__(32) terms_v1(JobDev J, const uint64_t *ts, int nt, double2 *g_out,
                                               int dmax, int nmax) {
  extern __shared__ double2 smem[];
  const int lane = threadIdx.x & 31;
  V1Smem S = v1_carve(smem, dmax, nmax);
  const PatDesc P = J.descs[0];
  for (int i = blockIdx.x; i < nt; i += gridDim.x) {
    double weight;
    decode_term(P, J, ts[i], lane, S.w, weight);
    const double2 g = v1_g(P, J, S, lane);
    if (lane == 0) g_out[i] = g;
    __syncwarp();
  }
}

// ================================================================ prep (a3): gather + P0
// One warp per pattern: C_ab = A[r_a][r_b] (phantom rows/cols zero), v_a = gamma[r_a] (phantom 1);
// P0 = I - uh uh^H with P0 v = beta e1 (Householder, beta = -e^{i arg v0} |v|); Ct = P0 C.
__global__ void __launch_bounds__(128) prep_kernel(JobDev J) {
  const int lane = threadIdx.x & 31;
  const int p = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (p >= J.npat) return;
  const PatDesc P = J.descs[p];
  const int d = P.d;
  if (d == 0) return;
  const int *r = J.ipool + P.idx_off;
  double2 *Ct = J.cpool + P.mat_off;
  double2 *uh = Ct + (size_t)d * d;
  double2 *vv = uh + d;
  const double2 *g = J.gamma + P.gamma_off;
  for (int idx = lane; idx < d * d; idx += 32) {
    const int a = idx / d, b = idx - a * d;
    Ct[idx] = (r[a] < 0 || r[b] < 0) ? c0() : J.A[(size_t)r[a] * J.kdim + r[b]];
  }
  double s2 = 0.0;
  for (int a = lane; a < d; a += 32) {
    const double2 x = (r[a] < 0) ? make_double2(1.0, 0.0) : g[r[a]];
    vv[a] = x;
    if (a > 0) s2 = fma(x.x, x.x, fma(x.y, x.y, s2));
  }
  s2 = warp_sum(s2);
  __syncwarp();
  const double2 x0 = vv[0];
  const double ax0 = hypot(x0.x, x0.y);
  if (s2 == 0.0 && ax0 == 0.0) {  // no loops at all
    for (int a = lane; a < d; a += 32) uh[a] = c0();
    if (lane == 0) { vv[d] = c0(); vv[d + 1] = c0(); }
    return;
  }
  const double nx = sqrt(fma(ax0, ax0, s2));
  const double2 ph = ax0 > 0.0 ? make_double2(x0.x / ax0, x0.y / ax0) : make_double2(1.0, 0.0);
  const double2 alpha = make_double2(-ph.x * nx, -ph.y * nx);
  const double rs = sqrt(1.0 / (nx * (nx + ax0)));
  for (int a = lane; a < d; a += 32) {
    const double2 x = vv[a];
    uh[a] = cscale(a == 0 ? csub(x, alpha) : x, rs);
  }
  if (lane == 0) { vv[d] = alpha; vv[d + 1] = make_double2(1.0, 0.0); }
  __syncwarp();
  // Ct <- C - uh (uh^H C), column by column (lane per column)
  for (int b = lane; b < d; b += 32) {
    double2 wb = c0();
    for (int a = 0; a < d; ++a) wb = cfma_cj(uh[a], Ct[a * d + b], wb);
    for (int a = 0; a < d; ++a) Ct[a * d + b] = cfms(uh[a], wb, Ct[a * d + b]);
  }
}

// ================================================================ prep of the bordered matrix (a3)
// One warp per pattern.  Reduced system (reading C8): C_ab = A[r_a][r_b] (phantom rows and
// columns zero), v_a = gamma[r_a] (phantom 1).  Stores the column-swapped bordered matrix
// B0 = [[0, (v X)^T], [v, C X]] (E = d + 1) when loop terms are present, else B0 = C X
// (E = d); X swaps the two halves of the index list.  Per term B = B0 diag(1, w, w).
__global__ void __launch_bounds__(128) prep_bordered(JobDev J) {
  const int lane = threadIdx.x & 31;
  const int p = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (p >= J.npat) return;
  const PatDesc P = J.descs[p];
  const int d = P.d;
  if (d == 0) return;
  const int H = P.H;
  const int o = (P.flags & FLAG_LOOP) ? 1 : 0;
  const int E = d + o;
  const int *r = J.ipool + P.idx_off;
  double2 *B0 = J.cpool + P.mat_off;
  const double2 *g = J.gamma + P.gamma_off;
  for (int idx = lane; idx < E * E; idx += 32) {
    const int a = idx / E - o, c = idx % E - o;          // reduced indices, -1 = border
    const int b = c < 0 ? -1 : (c < H ? c + H : c - H);  // partner column
    double2 x = c0();
    if (a >= 0 && c >= 0) {
      x = (r[a] < 0 || r[b] < 0) ? c0() : J.A[(size_t)r[a] * J.kdim + r[b]];
    } else if (a < 0 && c >= 0) {
      x = (r[b] < 0) ? c1() : g[r[b]];
    } else if (a >= 0 && c < 0) {
      x = (r[a] < 0) ? c1() : g[r[a]];
    }
    B0[idx] = x;
  }
}

// ================================================================ finalize (a11-a12)
// One block per pattern: thread i double-double-sums the contiguous unit range
// [i c, (i+1) c) in order, then thread 0 adds the 128 thread sums in order.  The order
// depends only on the unit count, never on the rank count, so results are bit-identical for
// any number of ranks.
__global__ void __launch_bounds__(128) finalize_kernel(JobDev J, double2 *out, double *abs_out) {
  __shared__ double s[128][6];
  const int p = blockIdx.x;
  const PatDesc P = J.descs[p];
  if (P.d == 0) {  // N = 0
    if (threadIdx.x == 0) {
      out[p] = make_double2(1.0, 0.0);
      if (abs_out) abs_out[p] = 1.0;
    }
    return;
  }
  const uint64_t c = (P.units + 127) / 128;
  const uint64_t ub = min(P.units, c * threadIdx.x), ue = min(P.units, ub + c);
  double a0 = 0, a1 = 0, a2 = 0, a3 = 0, a4 = 0, a5 = 0;
  for (uint64_t u = ub; u < ue; ++u) {
    const Partial q = J.partials[P.unit_begin + u];
    dd_add_dd(a0, a1, q.re_hi, q.re_lo);
    dd_add_dd(a2, a3, q.im_hi, q.im_lo);
    dd_add_dd(a4, a5, q.abs_hi, q.abs_lo);
  }
  s[threadIdx.x][0] = a0; s[threadIdx.x][1] = a1; s[threadIdx.x][2] = a2;
  s[threadIdx.x][3] = a3; s[threadIdx.x][4] = a4; s[threadIdx.x][5] = a5;
  __syncthreads();
  if (threadIdx.x != 0) return;
  a0 = a1 = a2 = a3 = a4 = a5 = 0;
  for (int i = 0; i < 128; ++i) {
    dd_add_dd(a0, a1, s[i][0], s[i][1]);
    dd_add_dd(a2, a3, s[i][2], s[i][3]);
    dd_add_dd(a4, a5, s[i][4], s[i][5]);
  }
  // 2^{1-n}: halving (x2) and the 2^{-n} prefactor, exact; 2^{-n} without halving (FLAG_FULL);
  // 1 for inclusion/exclusion
  const int e = ((P.flags & FLAG_ET) ? 0 : (P.flags & FLAG_FULL) ? -P.n : 1 - P.n) + P.out_exp;
  out[p] = make_double2(ldexp(a0 + a1, e), ldexp(a2 + a3, e));
  if (abs_out) abs_out[p] = ldexp(a4 + a5, e);
}

// ================================================================ launchers
cudaError_t launch_prep(const JobDev &job, int, cudaStream_t s) {
  if (job.npat == 0) return cudaSuccess;
  const int blocks = (job.npat + 3) / 4;
  ++lhaf::g_launches;
  prep_kernel<<<blocks, 128, 0, s>>>(job);
  return cudaGetLastError();
}

static int v1_warps(int dmax, int nmax) {
  const size_t per = (size_t)v1_words(dmax, nmax) * sizeof(double2);
  int w = (int)((200u * 1024u) / per);
  if (w > 4) w = 4;
  if (w < 1) w = 1;
  return w;
}

cudaError_t launch_sieve(const JobDev &job, int variant, int dmax, int nmax, uint64_t ubeg,
                         uint64_t uend, int num_sms, cudaStream_t s) {
  if (uend <= ubeg) return cudaSuccess;
  (void)variant;
  const int per = v1_words(dmax, nmax);
  const int W = v1_warps(dmax, nmax);
  const size_t smem = (size_t)per * W * sizeof(double2);
  cudaError_t e = cudaFuncSetAttribute(sieve_v1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sieve_v1, 32 * W, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  const uint64_t units = uend - ubeg;
  uint64_t grid = (uint64_t)num_sms * per_sm;
  if (grid > units) grid = units;
  e = cudaMemsetAsync(job.counter, 0, sizeof(unsigned long long), s);
  if (e != cudaSuccess) return e;
  ++lhaf::g_launches;
  sieve_v1<<<(unsigned)grid, 32 * W, smem, s>>>(job, ubeg, uend, dmax, nmax, per);
  return cudaGetLastError();
}

cudaError_t launch_prep_bordered(const JobDev &job, cudaStream_t s) {
  if (job.npat == 0) return cudaSuccess;
  ++lhaf::g_launches;
  prep_bordered<<<(job.npat + 3) / 4, 128, 0, s>>>(job);
  return cudaGetLastError();
}

cudaError_t launch_finalize(const JobDev &job, double2 *out, double *abs_out, cudaStream_t s) {
  if (job.npat == 0) return cudaSuccess;
  ++lhaf::g_launches;
  finalize_kernel<<<job.npat, 128, 0, s>>>(job, out, abs_out);
  return cudaGetLastError();
}

cudaError_t launch_terms(const JobDev &job, int, int dmax, int nmax, const uint64_t *t, int nt,
                         double2 *g_out, cudaStream_t s) {
  if (nt <= 0) return cudaSuccess;
  const size_t smem = (size_t)v1_words(dmax, nmax) * sizeof(double2);
  cudaError_t e = cudaFuncSetAttribute(terms_v1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  ++lhaf::g_launches;
  terms_v1<<<nt < 1024 ? nt : 1024, 32, smem, s>>>(job, t, nt, g_out, dmax, nmax);
  return cudaGetLastError();
}

// Algorithmic FP64 flops per term (real flops; 1 complex MAC = 8).  Counts the arithmetic
// the variant's algorithm performs for one term.
double flops_per_term(int variant, int d, int n, bool loops) {
  (void)variant;
  double cmac = 0.0;
  if (loops) cmac += 2.0 * d * d;                        // M1 P0 (matvec + rank-1)
  for (int k = 0; k < d - 2; ++k) {                       // Householder Hessenberg
    const double len = d - k - 1;
    cmac += 2.0 * len * len + 2.0 * d * len + (loops ? 2.0 * len : 0.0);
  }
  for (int j = d - 1; j >= 0; --j) {                      // trailing La Budde
    const double L = d - j;
    cmac += L * (L + 1) / 2.0 + 2.0 * L;
  }
  if (loops) cmac += d * (d + 1) / 2.0 + d;              // D(x)
  const double mn = n < d ? n : d;
  cmac += n * mn;                                         // c^{-1/2}
  if (loops) cmac += n * mn + n * (n + 1) / 2.0 + n + 1; // D~/c, exp, final product
  else cmac += 0;
  return 8.0 * cmac;
}

int bordered_supported(int e_max, int n_max) { return e_max <= 64 && n_max + 2 <= 255; }
// automatic choice: v3 (measured fastest at every size); v1 beyond its
// limits.  v5 (a second data layout) is selected explicitly (lhaf_set_kernel(5)) and by the
// precise mode.
int choose_variant(int e_max, int n_max) { return bordered_supported(e_max, n_max) ? 3 : 1; }

}  // namespace lhaf
