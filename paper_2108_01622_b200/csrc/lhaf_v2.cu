// lhaf_v2.cu -- variant 2 of the sieve kernel: register-resident rows, Gauss-transform
// Hessenberg reduction of the bordered matrix, La Budde and power series on an auxiliary warp.
// DESIGN.md "Kernel v2" has the derivation; SURVEY 8(a) rows a4-a11.
//
// A CTA holds MT "groups" of 32*NW matrix threads (one sieve term each) plus one auxiliary
// warp; all warps advance in lockstep, one CTA barrier per Hessenberg column.  Per term t:
//   a4  (aux) decode t -> w_h = eta_h - 2 k_h, sign (-1)^{sum k}, weight prod C(eta_h, k_h)
//   a5  (matrix) B = [[0, z^T], [y, M]] with M = C X_w, y = v, z^T = v X_w (loops present),
//       else B = M.  Row r of B lives in the registers of S threads (columns interleaved).
//   a6  (matrix) Hessenberg reduction of B by Gauss transforms with partial pivoting, index 0
//       fixed: B <- L B L^{-1} one column k at a time.  Rows never move (a row's final
//       position is a label); live columns stay contiguous in the register slots because the
//       lowest live column moves into the slot the pivot column frees (compaction), so every
//       per-slot loop runs over a slot suffix entered by a computed jump.  The new pivot
//       column produced by the right update is carried in registers, never written back.
//       Keeping index 0 fixed makes the first step map y -> beta e1 and carry
//       z^T -> z^T L^{-1} along (the "bordered" loop trick).
//   a7  (aux) leading La Budde recursions advance one step per finished column k:
//       P_{k+1}(x) = det(x I - H[:k+1, :k+1]) and Pm_{k+1} = det(x I - H[1:k+1, 1:k+1]),
//       top n+2 coefficients only (coefficient t of x^{deg-t} needs only t' <= t).
//       c_B(lam) = det(I - lam B) = P_E^top, c_M(lam) = det(I - lam M) = Pm_E^top.
//   a8  (aux) loop terms: lam S(lam) = 1 - c_B / c_M, S = sum_j s_j lam^j, s_j = z^T M^{j-1} y.
//   a9  (aux) g = [lam^n] c_M^{-1/2} exp(S/2)  (the paper's f with X -> X_w, P:409-415,
//       reading C4), computed for the previous batch of terms while the matrix warps reduce
//       the current one (software pipeline).
//   a10 (aux) term = (-1)^{sum k} prod C(eta_h, k_h) g, double-double sum per work unit.
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdint>
#include "lhaf_device.cuh"

namespace lhaf {
namespace v2 {

// 1/m for the series recursions (m <= 255)
__constant__ double c_inv[256];
static bool g_inv_ready = false;

// ---------------------------------------------------------------- dynamic slot access
// Warp-uniform slot index -> one register of the row (a switch; a few times per column,
// never inside the per-slot loops).
#define LHAF_CASES32(X)                                                                      \
  X(0) X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) X(14) X(15)      \
  X(16) X(17) X(18) X(19) X(20) X(21) X(22) X(23) X(24) X(25) X(26) X(27) X(28) X(29) X(30) \
  X(31)

template <int CS>
__device__ __forceinline__ double2 rd_slot(const double2 (&A)[CS], int s) {
  double2 v = c0();
  switch (s) {
#define LHAF_RD(i)                  \
  case i:                           \
    if constexpr (i < CS) v = A[i]; \
    break;
    LHAF_CASES32(LHAF_RD)
#undef LHAF_RD
    default: break;
  }
  return v;
}
template <int CS>
__device__ __forceinline__ void wr_slot(double2 (&A)[CS], int s, double2 v) {
  switch (s) {
#define LHAF_WR(i)                  \
  case i:                           \
    if constexpr (i < CS) A[i] = v; \
    break;
    LHAF_CASES32(LHAF_WR)
#undef LHAF_WR
    default: break;
  }
}
// value at column position q (uniform) of this thread's row, on all S lanes of the row
template <int S, int CS>
__device__ __forceinline__ double2 read_pos(const double2 (&A)[CS], int q, int lane) {
  double2 v = rd_slot<CS>(A, q / S);
  if constexpr (S > 1) v = shfl2(v, (lane & ~(S - 1)) | (q & (S - 1)));
  return v;
}

// Duff's device over the slot suffix [s0, 32): X(i) for i = s0 .. 31 (X drops i >= CS).
#define LHAF_SUFFIX(s0, X)                                                                    \
  switch (s0) {                                                                               \
    case 0: X(0) [[fallthrough]];                                                             \
    case 1: X(1) [[fallthrough]];                                                             \
    case 2: X(2) [[fallthrough]];                                                             \
    case 3: X(3) [[fallthrough]];                                                             \
    case 4: X(4) [[fallthrough]];                                                             \
    case 5: X(5) [[fallthrough]];                                                             \
    case 6: X(6) [[fallthrough]];                                                             \
    case 7: X(7) [[fallthrough]];                                                             \
    case 8: X(8) [[fallthrough]];                                                             \
    case 9: X(9) [[fallthrough]];                                                             \
    case 10: X(10) [[fallthrough]];                                                           \
    case 11: X(11) [[fallthrough]];                                                           \
    case 12: X(12) [[fallthrough]];                                                           \
    case 13: X(13) [[fallthrough]];                                                           \
    case 14: X(14) [[fallthrough]];                                                           \
    case 15: X(15) [[fallthrough]];                                                           \
    case 16: X(16) [[fallthrough]];                                                           \
    case 17: X(17) [[fallthrough]];                                                           \
    case 18: X(18) [[fallthrough]];                                                           \
    case 19: X(19) [[fallthrough]];                                                           \
    case 20: X(20) [[fallthrough]];                                                           \
    case 21: X(21) [[fallthrough]];                                                           \
    case 22: X(22) [[fallthrough]];                                                           \
    case 23: X(23) [[fallthrough]];                                                           \
    case 24: X(24) [[fallthrough]];                                                           \
    case 25: X(25) [[fallthrough]];                                                           \
    case 26: X(26) [[fallthrough]];                                                           \
    case 27: X(27) [[fallthrough]];                                                           \
    case 28: X(28) [[fallthrough]];                                                           \
    case 29: X(29) [[fallthrough]];                                                           \
    case 30: X(30) [[fallthrough]];                                                           \
    case 31: X(31) [[fallthrough]];                                                           \
    default: break;                                                                           \
  }

// Hides a value from loop-invariant code motion: per-pattern quantities are re-derived for
// every unit instead of being hoisted out of the loops into (many) live registers.
__device__ __forceinline__ int opaque(int x) {
  asm volatile("mov.b32 %0, %0;" : "+r"(x));
  return x;
}

struct Dims {  // per pattern
  int d, H, n, E, o, NTL, jmax, nss;
  bool loops;
};

__device__ __forceinline__ Dims dims_of(const PatDesc &P) {
  Dims D;
  D.d = opaque(P.d);
  D.H = opaque(P.H);
  D.n = opaque(P.n);
  D.loops = (P.flags & FLAG_LOOP) != 0;
  D.o = D.loops ? 1 : 0;
  D.E = D.d + D.o;
  const int nt = D.n + (D.loops ? 2 : 1);
  D.NTL = nt < D.E + 1 ? nt : D.E + 1;
  D.jmax = D.loops ? D.n + 1 : D.n;
  D.nss = D.jmax + 1 + (D.loops ? D.n + 1 : 0) + 1;  // series program length
  return D;
}

// Shared memory of one group (one term in flight), in double2 words:
//   cand [2][NW][CC]   each matrix warp's best row, by column position
//   kb   [2][RC]       pivot column by position (zero outside live positions)
//   keys [2][NW][3]    (key, code), pivot value, (column position of the pivot index)
//   fb   [2][NTL+1]    F_k[m] = H[k-m][k] prod_{j=k-m+1..k} H[j][j-1] (m = 0: H[k][k]);
//                      [NTL] = H[k+1][k] as published by the row labelled k+1
//   rb   [NTL+1][NTL]  ring of P_i^top;  rm: the same for Pm_i           (aux only)
//   ww   CC doubles    column weights of the current term
//   w    64 ints       w_h of the current term                            (aux only)
//   cin  [2][NTL]      c_M, c_B of the previous batch's term (series input)
//   ser  [3][n+2]      series accumulators Q, R, E                        (aux only)
//   sw   [2]           (sign * weight, weight) and (valid, term id) of the current / previous term
template <int S, int CS, int NW>
struct Shape {
  static constexpr int TS = 32 * NW, RC = TS / S, CC = S * CS;
  static constexpr int EMAX = RC < CC ? RC : CC;
  __host__ __device__ static int words(int NTL, int n) {
    return 2 * NW * CC + 2 * RC + 6 * NW + 2 * (NTL + 1) + 2 * (NTL + 1) * NTL + CC / 2 + 1 +
           32 + 2 * NTL + 3 * (n + 2) + 4;
  }
};

struct GroupMem {
  double2 *cand, *kb, *keys, *fb, *rb, *rm, *cin, *ser, *sw;
  double *ww;
  int *w;
};

template <int S, int CS, int NW>
__device__ __forceinline__ GroupMem carve(double2 *b, int NTL, int n) {
  using Sh = Shape<S, CS, NW>;
  GroupMem G;
  G.cand = b; b += 2 * NW * Sh::CC;
  G.kb = b; b += 2 * Sh::RC;
  G.keys = b; b += 6 * NW;
  G.fb = b; b += 2 * (NTL + 1);
  G.rb = b; b += (NTL + 1) * NTL;
  G.rm = b; b += (NTL + 1) * NTL;
  G.ww = reinterpret_cast<double *>(b); b += Sh::CC / 2 + 1;
  G.w = reinterpret_cast<int *>(b); b += 32;
  G.cin = b; b += 2 * NTL;
  G.ser = b; b += 3 * (n + 2);
  G.sw = b;
  return G;
}

// ---------------------------------------------------------------- aux: La Budde
// One step of both leading La Budde recursions on the top coefficients (one warp):
//   P_{k+1}^top[t]  = P_k^top[t]  - h P_k^top[t-1]  - sum_{m=1}^{min(t-1,k)}   F[m] P_{k-m}^top[t-m-1]
//   Pm_{k+1}^top[t] = Pm_k^top[t] - h Pm_k^top[t-1] - sum_{m=1}^{min(t-1,k-1)} F[m] Pm_{k-m}^top[t-m-1]
// h = F[0] = H[k][k]; deg P_{k+1} = k+1, deg Pm_{k+1} = k (Pm_1 = 1).  Ring row i % (NTL+1)
// holds index i; entries above the degree are written as 0.
__device__ __forceinline__ void labudde_step(double2 *rb, double2 *rm, const double2 *F, int k,
                                             bool two, int NTL, int lane) {
  const int R = NTL + 1;
  const int r0 = k % R;
  const int r1 = (r0 + 1 == R) ? 0 : r0 + 1;
  const double2 h = F[0];
  for (int t = lane; t < NTL; t += 32) {
    double2 a0 = c0(), a1 = c0(), b0 = c0(), b1 = c0();
    if (t <= k + 1) {
      a0 = rb[r0 * NTL + t];
      if (t >= 1) a1 = cmul(h, rb[r0 * NTL + t - 1]);
      const bool tm = two && t <= k;
      if (tm) {
        b0 = rm[r0 * NTL + t];
        if (t >= 1) b1 = cmul(h, rm[r0 * NTL + t - 1]);
      }
      const int mm = min(t - 1, k);
      int r = r0;
      for (int m = 1; m <= mm; ++m) {
        r = (r == 0) ? R - 1 : r - 1;  // ring row of index k - m
        const double2 f = F[m];
        const int off = r * NTL + t - m - 1;
        if (m & 1) a0 = cfms(f, rb[off], a0);
        else a1 = cfma(f, rb[off], a1);
        if (tm && m < k) {
          if (m & 1) b0 = cfms(f, rm[off], b0);
          else b1 = cfma(f, rm[off], b1);
        }
      }
    }
    rb[r1 * NTL + t] = csub(a0, a1);
    if (two) rm[r1 * NTL + t] = csub(b0, b1);
  }
}

// ---------------------------------------------------------------- aux: series
// Step s of the series program of one term (one warp; S8(a) a8/a9):
//   s <= jmax:        Q/R sweep j = s:  m Q_m = -sum_{i=1}^{m} (m - i/2) c_i Q_{m-i}  (c = c_M),
//                     R = (c_M - c_B) / c_M  (loops only)
//   next n+1 steps:   E sweep i:  m E_m = 1/2 sum_{j=1}^{m} j S_j E_{m-j},  S_j = R_{j+1}
//   last step:        g = sum_m Q_m E_{n-m}  (no loops: g = Q_n); returns true, g valid
// Accumulators turn into final values in place as the sweeps pass them.
__device__ __forceinline__ bool series_step(const Dims &D, int s, const double2 *cM,
                                            double2 *ser, int lane, double2 &g) {
  const int n = D.n, jmax = D.jmax, NTL = D.NTL;
  double2 *Qa = ser, *Ra = ser + (n + 2), *Ea = ser + 2 * (n + 2);
  if (s <= jmax) {
    const int j = s;
    const double2 qacc = Qa[j];
    const double2 rj = Ra[j];
    const double2 qj = (j == 0) ? c1() : cscale(qacc, -c_inv[j]);
    __syncwarp();
    if (lane == (j & 31)) Qa[j] = qj;
    for (int m = j + 1 + ((lane - j - 1) & 31); m <= jmax && m - j < NTL; m += 32) {
      const double2 c = cM[m - j];
      if (m <= n) Qa[m] = cfma(cscale(c, 0.5 * (double)(m + j)), qj, Qa[m]);
      if (D.loops) Ra[m] = cfms(c, rj, Ra[m]);
    }
    __syncwarp();
    return false;
  }
  if (D.loops && s <= jmax + 1 + n) {
    const int i = s - jmax - 1;
    const double2 eacc = Ea[i];
    const double2 ei = (i == 0) ? c1() : cscale(eacc, c_inv[i]);
    __syncwarp();
    if (lane == (i & 31)) Ea[i] = ei;
    for (int m = i + 1 + ((lane - i - 1) & 31); m <= n; m += 32)
      Ea[m] = cfma(cscale(Ra[m - i + 1], 0.5 * (double)(m - i)), ei, Ea[m]);
    __syncwarp();
    return false;
  }
  if (!D.loops) {
    g = Qa[n];
  } else {
    double2 gp = c0();
    for (int m = lane; m <= n; m += 32) gp = cfma(Qa[m], Ea[n - m], gp);
    g = warp_sum2(gp);
  }
  __syncwarp();
  return true;
}

// ================================================================ matrix warps: one term
// Reduces group `G`'s term (B0 diag(ww)) column by column, publishing La Budde inputs in fb.
// Executes exactly E CTA barriers (matching the aux warp).
template <int S, int CS, int NW>
__device__ __forceinline__ void matrix_term(const PatDesc &P, const Dims &D, const JobDev &J,
                                            const GroupMem &G, int tid) {
  using Sh = Shape<S, CS, NW>;
  constexpr int RC = Sh::RC, CC = Sh::CC;
  const int lane = tid & 31, warp = tid >> 5;
  const int rr = tid / S, par = tid % S;
  const int E = D.E, NTL = D.NTL;

  // ---- a5: rows of B = B0 diag(ww); slot s holds column position S*s + par
  double2 A[CS];
  {
    const double2 *row = J.cpool + P.mat_off + (size_t)(rr < E ? rr : 0) * E + par;
    const double *ww = G.ww + par;
#pragma unroll
    for (int s = 0; s < CS; ++s) {
      double2 val = c0();
      if (rr < E && S * s + par < E) val = cscale(row[S * s], ww[S * s]);
      A[s] = val;
    }
  }

  // ---- a6: iteration k finishes column k (label k)
  int label = rr;      // final Hessenberg position of index rr
  int mypos = rr;      // column position of index rr while its column is live, else -1
  int lo = 1;          // live column positions are [lo, E)
  double2 colv = (S == 1) ? A[0] : shfl2(A[0], lane & ~(S - 1));  // this row's entry of column k
  double2 pr = c1();   // prod_{j=label+1..k} H[j][j-1]
  double2 sub = c0();  // H[k][k-1]
  int buf = 0;
  for (int k = 0; k < E; ++k) {
    double2 *cb = G.cand + buf * NW * CC;
    double2 *kb = G.kb + buf * RC;
    double2 *yb = G.keys + buf * NW * 3;
    double2 *fb = G.fb + buf * (NTL + 1);
    buf ^= 1;
    const bool reduce = k + 2 < E;
    // La Budde inputs: F_k[k - label] for labels in [k-NTL+2, k]; H[k+1][k] in fb[NTL]
    if (k >= 1 && label < k) pr = cmul(pr, sub);
    const int mF = k - label;
    if (par == 0 && mF >= -1 && mF <= NTL - 2)
      fb[mF < 0 ? NTL : mF] = (mF <= 0) ? colv : cmul(colv, pr);
    const bool candr = reduce && label > k && label < E;
    const int slo = lo / S;
    if (reduce) {
      double key = candr ? fabs(colv.x) + fabs(colv.y) : -1.0;
      int code = label * 128 + rr;  // ties: smallest label wins
#pragma unroll
      for (int m = S; m < 32; m <<= 1) {
        const double k2 = __shfl_xor_sync(LHAF_FULL, key, m);
        const int c2 = __shfl_xor_sync(LHAF_FULL, code, m);
        if (k2 > key || (k2 == key && c2 < code)) { key = k2; code = c2; }
      }
      if (par == 0 && mypos >= 0) kb[mypos] = candr ? colv : c0();
      if (tid < lo - S * slo) kb[S * slo + tid] = c0();  // dead head of the first live slot
      if (key >= 0.0 && code == label * 128 + rr) {  // this warp's best row publishes itself
        double2 *dst = cb + warp * CC + par;
#define LHAF_W(i) \
  if constexpr (i < CS) dst[S * (i)] = A[i];
        LHAF_SUFFIX(slo, LHAF_W)
#undef LHAF_W
        if (par == 0) {
          yb[3 * warp] = make_double2(key, (double)code);
          yb[3 * warp + 1] = colv;
          yb[3 * warp + 2] = make_double2((double)mypos, 0.0);
        }
      }
      if (lane == 0 && key < 0.0) yb[3 * warp] = make_double2(-1.0, 1e9);
    }
    __syncthreads();
    if (!reduce) {
      if (k + 1 < E) {
        sub = fb[NTL];                        // published by the row labelled k+1
        colv = read_pos<S, CS>(A, lo, lane);  // the last live column: label k+1
        lo += 1;
      }
      continue;
    }

    // pivot = best of the warps' best rows
    double bk = -1.0, bc = 2e9;
    int wb = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      const double2 kk = yb[3 * w];
      if (kk.x > bk || (kk.x == bk && kk.y < bc)) { bk = kk.x; bc = kk.y; wb = w; }
    }
    const int pcode = (int)bc;
    const int p = pcode & 127, plabel = pcode >> 7;  // pivot: physical index and label
    const int qp = (int)yb[3 * wb + 2].x;            // its column position
    const double2 piv = yb[3 * wb + 1];
    if (bk > 0.0) {
      const double2 *rowp = cb + wb * CC + par;
      const double2 ip = crecip(piv);
      // left: row r -= (B[r][k] / piv) row p for the remaining rows r != p (m = 0 elsewhere)
      const double2 m = (candr && rr != p) ? cmul(colv, ip) : c0();
#define LHAF_L(i) \
  if constexpr (i < CS) A[i] = cfms(m, rowp[S * (i)], A[i]);
      LHAF_SUFFIX(slo, LHAF_L)
#undef LHAF_L
      // right: new column p = sum over live positions q (incl. p's own, whose multiplier is
      // piv / piv) of column q * B[q][k] / piv.  Carried as the next pivot column.
      const double2 *kq = kb + par;
      double2 ac0 = c0(), ac1 = c0(), ac2 = c0(), ac3 = c0();
#define LHAF_R(i)                                                         \
  if constexpr (i < CS) {                                                 \
    if constexpr ((i & 3) == 0) ac0 = cfma(A[i], kq[S * (i)], ac0);       \
    else if constexpr ((i & 3) == 1) ac1 = cfma(A[i], kq[S * (i)], ac1);  \
    else if constexpr ((i & 3) == 2) ac2 = cfma(A[i], kq[S * (i)], ac2);  \
    else ac3 = cfma(A[i], kq[S * (i)], ac3);                              \
  }
      LHAF_SUFFIX(slo, LHAF_R)
#undef LHAF_R
      double2 a = cadd(cadd(ac0, ac1), cadd(ac2, ac3));
#pragma unroll
      for (int x = 1; x < S; x <<= 1) a = cadd(a, shfl2_xor(a, x));
      colv = cmul(a, ip);
      sub = piv;
    } else {
      colv = read_pos<S, CS>(A, qp, lane);  // nothing to eliminate: column p as it stands
      sub = c0();
    }
    // compaction: the column at position lo moves into the pivot column's position
    if (qp != lo) {
      const double2 x = read_pos<S, CS>(A, lo, lane);
      if (par == qp % S) wr_slot<CS>(A, qp / S, x);
      if (mypos == lo) mypos = qp;
    }
    if (rr == p) mypos = -1;
    lo += 1;
    label = (rr == p) ? k + 1 : (label == k + 1 ? plabel : label);
  }
}

// ================================================================ the kernel
// Unit fetch shared by the two roles: every thread of the CTA executes it (2 barriers).
// DIAG = false: the next work unit of [ubeg, uend) from the job's atomic counter.
// DIAG = true: one pass over the list slice [c * MT * 64, (c + 1) * MT * 64) of CTA c.
template <int MT, bool DIAG>
__device__ __forceinline__ bool next_unit(const JobDev &J, uint64_t ubeg, uint64_t uend, int dn,
                                          bool &first, unsigned long long *s_unit, uint64_t &u,
                                          int &pidx, uint64_t &tb, uint64_t &te) {
  __syncthreads();
  if (threadIdx.x == 0) *s_unit = DIAG ? (first ? 0ull : ~0ull) : ubeg + atomicAdd(J.counter, 1ull);
  __syncthreads();
  first = false;
  u = *s_unit;
  if (DIAG) {
    if (u != 0) return false;
    tb = (uint64_t)blockIdx.x * MT * 64;
    te = min(tb + (uint64_t)MT * 64, (uint64_t)dn);
    pidx = 0;
    return tb < te;
  }
  if (u >= uend) return false;
  pidx = find_pattern(J, u);
  const PatDesc &P = J.descs[pidx];
  tb = (u - P.unit_begin) * P.chunk;
  te = min(tb + P.chunk, P.T_eval);
  return true;
}

// Matrix warps: one group = one term per batch; per batch one barrier (A) + E column barriers.
template <int S, int CS, int NW, int MT, bool DIAG>
__device__ __noinline__ void run_matrix(const JobDev &J, uint64_t ubeg, uint64_t uend, int gwords,
                                        int dn, unsigned long long *s_unit) {
  constexpr int TS = 32 * NW;
  extern __shared__ double2 smem[];
  const int grp = threadIdx.x / TS, tid = threadIdx.x % TS;
  bool first = true;
  uint64_t u, tb, te;
  int pidx;
  while (next_unit<MT, DIAG>(J, ubeg, uend, dn, first, s_unit, u, pidx, tb, te)) {
    const PatDesc P = J.descs[pidx];
    const Dims D = dims_of(P);
    const int nb = (int)((te - tb + MT - 1) / MT);
    const GroupMem G = carve<S, CS, NW>(smem + (size_t)grp * gwords, D.NTL, D.n);
    for (int b = 0; b < nb; ++b) {
      __syncthreads();  // (A) the aux warp has decoded batch b
      matrix_term<S, CS, NW>(P, D, J, G, tid);
    }
  }
}

// Aux warp: decode, La Budde (lockstep with the columns), pipelined series, unit partials.
template <int S, int CS, int NW, int MT, bool DIAG>
__device__ __noinline__ void run_aux(const JobDev &J, uint64_t ubeg, uint64_t uend, int gwords,
                                     const uint64_t *dt, int dn, double2 *dout,
                                     unsigned long long *s_unit) {
  using Sh = Shape<S, CS, NW>;
  extern __shared__ double2 smem[];
  const int lane = threadIdx.x & 31;
  bool first = true;
  uint64_t u, tb, te;
  int pidx;
  while (next_unit<MT, DIAG>(J, ubeg, uend, dn, first, s_unit, u, pidx, tb, te)) {
    const PatDesc P = J.descs[pidx];
    const Dims D = dims_of(P);
    const int E = D.E, NTL = D.NTL, R = NTL + 1;
    const int nb = (int)((te - tb + MT - 1) / MT);
    const int per_k = (D.nss + E - 1) / E;
    double rh = 0, rl = 0, ih = 0, il = 0, ah = 0, al = 0;  // lane 0: unit sums
    auto finish = [&](const GroupMem &G, const double2 &g) {
      if (lane == 0 && G.sw[3].x != 0.0) {
        if (DIAG) {
          dout[(uint64_t)G.sw[3].y] = g;
        } else {
          const double sw = G.sw[1].x, w = G.sw[1].y;
          dd_add(rh, rl, sw * g.x);
          dd_add(ih, il, sw * g.y);
          dd_add(ah, al, w * hypot(g.x, g.y));
        }
      }
    };
    for (int b = 0; b <= nb; ++b) {
      // the previous batch's polynomials become series inputs (its series runs during this
      // batch; the one of the batch before has completed during the previous batch)
      if (b >= 1) {
#pragma unroll
        for (int q = 0; q < MT; ++q) {
          const GroupMem G = carve<S, CS, NW>(smem + (size_t)q * gwords, NTL, D.n);
          const double2 *cB = G.rb + (E % R) * NTL;
          const double2 *cM = D.loops ? G.rm + (E % R) * NTL : cB;
          for (int t = lane; t < NTL; t += 32) {
            G.cin[t] = cM[t];
            G.cin[NTL + t] = cB[t];
          }
          __syncwarp();
          double2 *Qa = G.ser, *Ra = G.ser + (D.n + 2), *Ea = G.ser + 2 * (D.n + 2);
          for (int m = lane; m < D.n + 2; m += 32) {
            Qa[m] = c0();
            Ea[m] = c0();
            Ra[m] = (D.loops && m < NTL) ? csub(G.cin[m], G.cin[NTL + m]) : c0();
          }
          if (lane == 0) { G.sw[1] = G.sw[0]; G.sw[3] = G.sw[2]; }
        }
        __syncwarp();
      }
      if (b == nb) {  // drain: the last batch's series (matrix warps wait for the next unit)
        if (nb >= 1)
          for (int s = 0; s < D.nss; ++s) {
#pragma unroll
            for (int q = 0; q < MT; ++q) {
              const GroupMem G = carve<S, CS, NW>(smem + (size_t)q * gwords, NTL, D.n);
              double2 g;
              if (series_step(D, s, G.cin, G.ser, lane, g)) finish(G, g);
            }
          }
        break;
      }
      // decode batch b: w, column weights, ring init, (sign * weight, weight), (valid, id)
#pragma unroll
      for (int q = 0; q < MT; ++q) {
        const GroupMem G = carve<S, CS, NW>(smem + (size_t)q * gwords, NTL, D.n);
        const uint64_t idx = tb + (uint64_t)b * MT + q;
        const bool valid = idx < te;
        const uint64_t t = DIAG ? dt[valid ? idx : tb] : (valid ? idx : tb);
        double weight;
        const int sign = decode_term(P, J, t, lane, G.w, weight);
        __syncwarp();
        for (int c = lane; c < Sh::CC; c += 32) {
          const int j = c - D.o;
          G.ww[c] = (c >= E) ? 0.0 : (j < 0) ? 1.0 : (double)G.w[j < D.H ? j : j - D.H];
        }
        for (int t2 = lane; t2 < NTL; t2 += 32) {
          G.rb[t2] = (t2 == 0) ? c1() : c0();                  // P_0 = 1
          G.rm[(1 % R) * NTL + t2] = (t2 == 0) ? c1() : c0();  // Pm_1 = 1
        }
        if (lane == 0) {
          G.sw[0] = make_double2(sign * weight, weight);
          G.sw[2] = make_double2(valid ? 1.0 : 0.0, (double)idx);
        }
      }
      __syncthreads();  // (A)
      int ss = (b >= 1) ? 0 : D.nss;  // series step of the previous batch
      for (int k = 0; k < E; ++k) {
        __syncthreads();  // column k of every group is published
#pragma unroll
        for (int q = 0; q < MT; ++q) {
          const GroupMem G = carve<S, CS, NW>(smem + (size_t)q * gwords, NTL, D.n);
          labudde_step(G.rb, G.rm, G.fb + (k & 1) * (NTL + 1), k, D.loops && k >= 1, NTL, lane);
        }
        for (int x = 0; x < per_k && ss < D.nss; ++x, ++ss) {
#pragma unroll
          for (int q = 0; q < MT; ++q) {
            const GroupMem G = carve<S, CS, NW>(smem + (size_t)q * gwords, NTL, D.n);
            double2 g;
            if (series_step(D, ss, G.cin, G.ser, lane, g)) finish(G, g);
          }
        }
        __syncwarp();
      }
    }
    if (!DIAG && lane == 0) {
      Partial q;
      q.re_hi = rh; q.re_lo = rl; q.im_hi = ih; q.im_lo = il; q.abs_hi = ah; q.abs_lo = al;
      q.pad0 = 0; q.pad1 = 0;
      J.partials[u] = q;
    }
  }
}

// DIAG = false: the sieve over work units [ubeg, uend) of the job, one double-double partial
// per unit.  DIAG = true: g(t) (unweighted) of pattern 0 for the term list dt[0..dn).
template <int S, int CS, int NW, int MT, int REGS, bool DIAG>
__global__ void __maxnreg__(REGS)
sieve_v2(JobDev J, uint64_t ubeg, uint64_t uend, int gwords, const uint64_t *dt, int dn,
         double2 *dout) {
  extern __shared__ double2 smem[];
  __shared__ unsigned long long s_unit;
  for (int i = threadIdx.x; i < gwords * MT; i += blockDim.x) smem[i] = c0();
  if (threadIdx.x >= 32 * NW * MT)
    run_aux<S, CS, NW, MT, DIAG>(J, ubeg, uend, gwords, dt, dn, dout, &s_unit);
  else
    run_matrix<S, CS, NW, MT, DIAG>(J, ubeg, uend, gwords, dn, &s_unit);
}

// ================================================================ prep (a3)
// One warp per pattern.  Reduced system (reading C8): C_ab = A[r_a][r_b] (phantom rows and
// columns zero), v_a = gamma[r_a] (phantom 1).  Stores the column-swapped bordered matrix
// B0 = [[0, (v X)^T], [v, C X]] (E = d + 1) when loop terms are present, else B0 = C X
// (E = d); X swaps the two halves of the index list.  Per term B = B0 diag(1, w, w).
__global__ void __launch_bounds__(128) prep_v2(JobDev J) {
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

// ================================================================ host side
template <int S, int CS, int NW, int MT, int REGS>
struct Inst {
  using Sh = Shape<S, CS, NW>;
  static constexpr int EMAX = Sh::EMAX;
  static constexpr int THREADS = 32 * NW * MT + 32;
  static cudaError_t sieve(const JobDev &job, int NTL, int n, uint64_t ubeg, uint64_t uend,
                           int num_sms, cudaStream_t s) {
    const int gw = Sh::words(NTL, n);
    const size_t smem = (size_t)gw * MT * sizeof(double2);
    auto *kern = sieve_v2<S, CS, NW, MT, REGS, false>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, THREADS, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    const uint64_t units = uend - ubeg;
    uint64_t grid = (uint64_t)num_sms * per_sm;
    if (grid > units) grid = units;
    e = cudaMemsetAsync(job.counter, 0, sizeof(unsigned long long), s);
    if (e != cudaSuccess) return e;
    kern<<<(unsigned)grid, THREADS, smem, s>>>(job, ubeg, uend, gw, nullptr, 0, nullptr);
    return cudaGetLastError();
  }
  static cudaError_t terms(const JobDev &job, int NTL, int n, const uint64_t *t, int nt,
                           double2 *g_out, cudaStream_t s) {
    const int gw = Sh::words(NTL, n);
    const size_t smem = (size_t)gw * MT * sizeof(double2);
    auto *kern = sieve_v2<S, CS, NW, MT, REGS, true>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int grid = (nt + MT * 64 - 1) / (MT * 64);
    kern<<<grid, THREADS, smem, s>>>(job, 0, 0, gw, t, nt, g_out);
    return cudaGetLastError();
  }
};

// <S, CS, NW, MT, registers per thread>  (CTAs per SM = 65536 / (threads * registers))
using I9 = Inst<1, 9, 1, 3, 128>;    // 128 threads: 4 CTAs
using I17 = Inst<1, 17, 1, 3, 128>;  // 128 threads: 4 CTAs
using I25 = Inst<1, 25, 1, 2, 168>;  //  96 threads: 4 CTAs
using I32 = Inst<1, 32, 1, 2, 168>;  //  96 threads: 4 CTAs
using I48 = Inst<2, 24, 3, 1, 168>;  // 128 threads: 3 CTAs
using I64 = Inst<2, 32, 4, 1, 200>;  // 160 threads: 2 CTAs

static cudaError_t ensure_inv() {
  if (g_inv_ready) return cudaSuccess;
  double h[256];
  h[0] = 0.0;
  for (int i = 1; i < 256; ++i) h[i] = 1.0 / (double)i;
  cudaError_t e = cudaMemcpyToSymbol(c_inv, h, sizeof h);
  if (e == cudaSuccess) g_inv_ready = true;
  return e;
}

}  // namespace v2

int v2_supported(int e_max, int n_max) { return e_max <= 64 && n_max + 2 <= 255; }

cudaError_t launch_prep_v2(const JobDev &job, cudaStream_t s) {
  if (job.npat == 0) return cudaSuccess;
  cudaError_t e = v2::ensure_inv();
  if (e != cudaSuccess) return e;
  v2::prep_v2<<<(job.npat + 3) / 4, 128, 0, s>>>(job);
  return cudaGetLastError();
}

#define LHAF_V2_DISPATCH(CALL)                \
  if (E <= v2::I9::EMAX) return v2::I9::CALL;   \
  if (E <= v2::I17::EMAX) return v2::I17::CALL; \
  if (E <= v2::I25::EMAX) return v2::I25::CALL; \
  if (E <= v2::I32::EMAX) return v2::I32::CALL; \
  if (E <= v2::I48::EMAX) return v2::I48::CALL; \
  if (E <= v2::I64::EMAX) return v2::I64::CALL; \
  return cudaErrorInvalidValue;

cudaError_t launch_sieve_v2(const JobDev &job, int e_max, int ntl_max, int n_max, uint64_t ubeg,
                            uint64_t uend, int num_sms, cudaStream_t s) {
  if (uend <= ubeg) return cudaSuccess;
  const int E = e_max;
  LHAF_V2_DISPATCH(sieve(job, ntl_max, n_max, ubeg, uend, num_sms, s))
}

cudaError_t launch_terms_v2(const JobDev &job, int e, int ntl, int n, const uint64_t *t, int nt,
                            double2 *g_out, cudaStream_t s) {
  if (nt <= 0) return cudaSuccess;
  const int E = e;
  LHAF_V2_DISPATCH(terms(job, ntl, n, t, nt, g_out, s))
}

// Algorithmic FP64 flops of one v2 term (real flops; complex MAC = 8, complex mul = 6):
// Gauss-transform Hessenberg of the E x E (bordered) matrix, La Budde recursions on the top
// NTL coefficients, the series recursions and the final product.
double v2_flops_per_term(int d, int n, bool loops) {
  const int E = d + (loops ? 1 : 0);
  const int NTL = std::min(n + (loops ? 2 : 1), E + 1);
  double cmac = 0.0, cmul_ = 0.0;
  for (int k = 0; k + 2 < E; ++k) {
    const double rem = E - k - 2;  // rows eliminated
    cmac += rem * (E - k - 1);     // left
    cmac += (double)E * rem;       // right
    cmul_ += rem;                  // multipliers
  }
  for (int k = 0; k < E; ++k) {
    cmul_ += std::min(k, NTL - 2);  // F_k
    for (int t = 0; t < NTL && t <= k + 1; ++t) cmac += (t >= 1 ? 1 : 0) + std::min(t - 1 < 0 ? 0 : t - 1, k);
    if (loops && k >= 1)
      for (int t = 0; t < NTL && t <= k; ++t) cmac += (t >= 1 ? 1 : 0) + std::min(t - 1 < 0 ? 0 : t - 1, k - 1);
  }
  const double nn = n;
  cmac += nn * (nn + 1) / 2.0;                                                  // c_M^{-1/2}
  if (loops) cmac += (nn + 2) * (nn + 1) / 2.0 + nn * (nn + 1) / 2.0 + nn + 1;  // R, exp, g
  return 8.0 * cmac + 6.0 * cmul_;
}

}  // namespace lhaf
