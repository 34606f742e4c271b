// lhaf_v3.cu -- variant 3 of the sieve kernel (the default): register-resident rows,
// Gauss-transform Hessenberg reduction of the bordered matrix with a branch-free per-column
// body, a team-parallel trailing La Budde on the band of H, and the power series of each term
// pipelined into the next term's reduction.  DESIGN.md "Kernel v3"; SURVEY 8(a) rows a4-a11.
//
// One "team" of 32*NW threads evaluates one sieve term at a time; a CTA holds TEAMS teams.
//   a4  decode t -> w_h = eta_h - 2 k_h, sign (-1)^{sum k}, weight prod C(eta_h, k_h)
//   a5  B = [[0, z^T], [y, M]] with M = C X_w, y = v, z^T = v X_w (loops present), else B = M.
//       Row r of B lives in the registers of S threads; slot s of thread (r, par) holds column
//       S*s + par.
//   a6  Hessenberg reduction of B by Gauss transforms with partial pivoting, index 0 fixed
//       (so the first step maps y -> beta e1 and carries z^T -> z^T L^{-1}: the "bordered"
//       loop trick).  Rows and columns never move: index i gets its final Hessenberg position
//       as a label.  Per column k one team barrier:
//         pivot = warp REDUX-max of a packed (|B[r][k]|_1, label) key, then across warps;
//         each warp's best row is published to smem; every row then does, in ONE fused pass
//         over all its slots,
//             left   A[r][c] -= m_r A[p][c]          (m_r = B[r][k] / piv, 0 if r is done)
//             right  acc     += A[r][c] B[c][k]      (B[c][k] = 0 unless c is remaining)
//         and the new pivot column p = acc / piv is carried in registers (never stored).
//       Columns of finished indices are left as garbage (they are multiplied by zero).
//       Finished columns go to the band hb (H[j][j-1 .. j+NTL-2]).
//   a7  F_j[m] = H[j][j+m] prod_{i=1..m} H[j+i][j+i-1]; trailing La Budde on the top
//       NTL = n+2 coefficients of q_j(x) = det(x I - H[j:, j:]) (c_B = q_0, c_M = q_1), the
//       m-sums split across the team's warps (one barrier per j).
//   a8  loop terms: lam S(lam) = 1 - c_B / c_M, S = sum_j s_j lam^j, s_j = z^T M^{j-1} y.
//   a9  g = [lam^n] c_M^{-1/2} exp(S/2)   (the paper's f with X -> X_w, reading C4):
//       a column-sweep series program of ~2n steps, run by the team's last warp one or two
//       steps per column of the NEXT term's reduction (drained at the end of a work unit).
//   a10 term = (-1)^{sum k} prod C(eta_h, k_h) g, double-double accumulation per work unit.
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include "lhaf_device.cuh"

namespace lhaf {
namespace v3 {

__constant__ double c_inv[256];  // 1/m for the series recursions
static bool g_inv_ready = false;

// Phase timing (diagnostic builds only, -DLHAF_PHASE_TIMING): cycles of thread 0 of every
// team spent in decode/build, reduction, band -> F, La Budde, hand-off, end barrier.
#ifdef LHAF_PHASE_TIMING
__device__ unsigned long long g_phase[8];
#define LHAF_PHASE(i)                                             \
  if (tid == 0) {                                                 \
    const long long now_ = clock64();                             \
    atomicAdd(&g_phase[i], (unsigned long long)(now_ - t_last_)); \
    t_last_ = now_;                                               \
  }
#else
#define LHAF_PHASE(i)
#endif

// Warp-uniform slot index -> one register of the row (off the per-column hot path).
template <int CS>
__device__ __forceinline__ double2 rd_slot(const double2 (&A)[CS], int s) {
  double2 v = c0();
#pragma unroll
  for (int i = 0; i < CS; ++i)
    if (i == s) v = A[i];
  return v;
}
// value of column c (uniform) of this thread's row, on all S lanes of the row
template <int S, int CS>
__device__ __forceinline__ double2 read_col(const double2 (&A)[CS], int c, int lane) {
  double2 v = rd_slot<CS>(A, c / S);
  if constexpr (S > 1) v = shfl2(v, (lane & ~(S - 1)) | (c & (S - 1)));
  return v;
}

// Hides a value from loop-invariant code motion (per-pattern quantities are re-derived for
// every term instead of being hoisted out of the term loop into live registers).
__device__ __forceinline__ int opaque(int x) {
  asm volatile("mov.b32 %0, %0;" : "+r"(x));
  return x;
}

template <int NW, int TEAMS>
__device__ __forceinline__ void team_sync(int team) {
  if constexpr (NW == 1) {
    __syncwarp();
  } else if constexpr (TEAMS == 1) {
    __syncthreads();
  } else {
    asm volatile("bar.sync %0, %1;" ::"r"(team + 1), "r"(32 * NW) : "memory");
  }
}

// Shared memory of one team (double2 words), for a pattern with (E, NTL, n):
//   hb   [E][NTL]       band of H: [j][0] = H[j][j-1], [j][1] = H[j][j], [j][1+m] = H[j][j+m]
//   u1   union { cand [2][NW][CC] | kb [2][RC] | keys [2][NW] | piv [2][NW] } (reduction)
//        union { Q [E+1][NTL] | part [2][NW][NTL] | base [2][NTL] } (La Budde)
//   cin  [2][NTL]      c_M, c_B of the term whose series is pending
//   ser  [3][n+2]      series accumulators Q, R, E of that term
//   psw  [2]           (sign * weight, weight), (valid, output index) of that term
//   csw  [1]           (sign * weight, weight) of the term being reduced
//   w    64 ints, then 64 doubles of column weights
template <int S, int CS, int NW>
struct Shape {
  static constexpr int TS = 32 * NW, RC = TS / S, CC = S * CS;
  static constexpr int EMAX = RC < CC ? RC : CC;
  __host__ __device__ static int red_words() { return 2 * NW * CC + 2 * RC + 4 * NW; }
  __host__ __device__ static int u1_words(int E, int NTL) {
    const int lab = (E + 1) * NTL + 2 * NW * NTL + 2 * NTL;
    return red_words() > lab ? red_words() : lab;
  }
  __host__ __device__ static int words(int E, int NTL, int n) {
    return E * NTL + u1_words(E, NTL) + 2 * NTL + 3 * (n + 2) + 3 + 32 + 32;
  }
};

struct TeamMem {
  double2 *hb, *u1, *cin, *ser, *psw, *csw;
  int *wv;
  double *ww;
};

template <int S, int CS, int NW>
__device__ __forceinline__ TeamMem carve(double2 *b, int E, int NTL, int n) {
  using Sh = Shape<S, CS, NW>;
  TeamMem T;
  T.hb = b; b += E * NTL;
  T.u1 = b; b += Sh::u1_words(E, NTL);
  T.cin = b; b += 2 * NTL;
  T.ser = b; b += 3 * (n + 2);
  T.psw = b; b += 2;
  T.csw = b; b += 1;
  T.wv = reinterpret_cast<int *>(b); b += 32;
  T.ww = reinterpret_cast<double *>(b);
  return T;
}

struct Pattern {  // per-pattern sizes (kept opaque to loop-invariant motion)
  int H, n, E, o, NTL, nss;
  bool loops;
};

__device__ __forceinline__ Pattern pattern_of(const PatDesc &P) {
  Pattern D;
  D.loops = (P.flags & FLAG_LOOP) != 0;
  D.o = opaque(D.loops ? 1 : 0);
  D.H = opaque(P.H);
  D.n = opaque(P.n);
  D.E = opaque(P.d) + D.o;
  D.NTL = min(D.n + 1 + D.o, D.E + 1);
  const int jmax = D.loops ? D.n + 1 : D.n;
  D.nss = jmax + 1 + (D.loops ? D.n + 1 : 0) + 1;
  return D;
}

// ---------------------------------------------------------------- series program (one warp)
// Step s of the series of one term; the accumulators in ser turn into final values in place:
//   s <= jmax:      Q/R sweep j = s:  m Q_m = -sum_{i=1}^{m} (m - i/2) c_i Q_{m-i}  (c = c_M),
//                   R = (c_M - c_B) / c_M  (loops only)
//   next n+1 steps: E sweep i:  m E_m = 1/2 sum_{j=1}^{m} j S_j E_{m-j},  S_j = R_{j+1}
//   last step:      g = sum_m Q_m E_{n-m}  (no loops: g = Q_n); returns true with g
__device__ __forceinline__ bool series_step(const Pattern &D, int s, const double2 *cM,
                                            double2 *ser, int lane, double2 &g) {
  const int n = D.n, NTL = D.NTL;
  const int jmax = D.loops ? n + 1 : n;
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

// Accumulation of finished terms (lane 0 of the series warp): double-double sums of
// sign * weight * g and of weight * |g|, or g itself into the diagnostic output.
struct Sums {
  double rh = 0, rl = 0, ih = 0, il = 0, ah = 0, al = 0;
};

__device__ __forceinline__ void finish_term(const TeamMem &T, const double2 &g, Sums &acc,
                                            double2 *g_out, int lane) {
  if (lane != 0 || T.psw[1].x == 0.0) return;
  if (g_out) {
    g_out[(uint64_t)T.psw[1].y] = g;
  } else {
    const double sw = T.psw[0].x, w = T.psw[0].y;
    dd_add(acc.rh, acc.rl, sw * g.x);
    dd_add(acc.ih, acc.il, sw * g.y);
    dd_add(acc.ah, acc.al, w * hypot(g.x, g.y));
  }
}

// ================================================================ one term, one team
// Reduces term t (valid == false: a duplicate term whose result is discarded) and hands its
// characteristic polynomials to the series pipeline.  ss = next series step of the pending
// term (== nss: nothing pending).
template <int S, int CS, int NW, int TEAMS>
__device__ void team_term(const PatDesc &P, const Pattern &D, const JobDev &J, uint64_t t,
                          bool valid, uint64_t out_idx, const TeamMem &T, int tid, int team,
                          int &ss, Sums &acc, double2 *g_out) {
  using Sh = Shape<S, CS, NW>;
  constexpr int RC = Sh::RC, CC = Sh::CC;
  constexpr int SW = NW - 1;  // the series warp
  const int lane = tid & 31, warp = tid >> 5;
  const int H = D.H, n = D.n, E = D.E, o = D.o, NTL = D.NTL;
  const bool loops = D.loops;
  double2 *hb = T.hb;

#ifdef LHAF_PHASE_TIMING
  long long t_last_ = clock64();
#endif
  // ---- a4: decode; ww[c] = weight of column c of B (1 for the border column)
  if (warp == 0) {
    double weight;
    const int sign = decode_term(P, J, t, lane, T.wv, weight);
    __syncwarp();
    for (int c = lane; c < CC; c += 32) {
      const int j = c - o;
      T.ww[c] = (c >= E) ? 0.0 : (j < 0) ? 1.0 : (double)T.wv[j < H ? j : j - H];
    }
    if (lane == 0) T.csw[0] = make_double2(sign * weight, weight);
  }
  team_sync<NW, TEAMS>(team);

  // ---- a5: rows of B = B0 diag(ww), B0 = the prep kernel's bordered column-swapped matrix
  const int rr = tid / S, par = tid % S;
  double2 A[CS];
  {
    const double2 *row = J.cpool + P.mat_off + (size_t)(rr < E ? rr : 0) * E + par;
    const double *wp = T.ww + par;
#pragma unroll
    for (int s = 0; s < CS; ++s) {
      double2 val = c0();
      if (rr < E && S * s + par < E) val = cscale(row[S * s], wp[S * s]);
      A[s] = val;
    }
  }
  LHAF_PHASE(0)

  // ---- a6: Gauss-transform Hessenberg reduction, one barrier per column
  double2 *cand = T.u1;                                       // [2][NW][CC]
  double2 *kbuf = cand + 2 * NW * CC;                         // [2][RC]
  unsigned *keys = reinterpret_cast<unsigned *>(kbuf + 2 * RC);  // [2][NW][4] (key, phys)
  int label = rr;
  uint64_t live = (E >= 64 ? ~0ull : ((1ull << E) - 1ull)) & ~1ull;  // indices with label > k
  double2 colv = (S == 1) ? A[0] : shfl2(A[0], lane & ~(S - 1));    // this row's B[.][k]
  int buf = 0;
  const int kend = E >= 2 ? E - 2 : 0;
  const int per_k = kend > 0 ? (D.nss + kend - 1) / kend : D.nss;
  for (int k = 0; k < kend; ++k) {
    double2 *cb = cand + buf * NW * CC;
    double2 *kb = kbuf + buf * RC;
    unsigned *yk = keys + buf * NW * 4;
    double2 *yv = reinterpret_cast<double2 *>(keys + 2 * NW * 4) + buf * NW;  // pivot values
    buf ^= 1;
    const bool candr = label > k && label < E;
    // pivot key: |re| + |im| as a float (monotone bits), low 6 bits = 63 - label so that ties
    // go to the smallest label; non-candidates 0; one REDUX per warp
    unsigned key = 0u;
    if (candr) {
      const unsigned fbits = __float_as_uint((float)(fabs(colv.x) + fabs(colv.y)));
      key = (((fbits >> 6) + 1u) << 6) | (unsigned)(63 - label);
    }
    const unsigned wkey = __reduce_max_sync(LHAF_FULL, key);
    if (par == 0) kb[rr] = candr ? colv : c0();
    if (candr && key == wkey) {  // this warp's best row publishes itself
      double2 *dst = cb + warp * CC + par;
#pragma unroll
      for (int s = 0; s < CS; ++s) dst[S * s] = A[s];
      if (par == 0) {
        yv[warp] = colv;
        yk[4 * warp + 1] = (unsigned)rr;
      }
    }
    if (lane == 0) yk[4 * warp] = wkey;
    // the pending term's series advances in the shadow of this column
    if (warp == SW) {
      for (int x = 0; x < per_k && ss < D.nss; ++x, ++ss) {
        double2 g;
        if (series_step(D, ss, T.cin, T.ser, lane, g)) finish_term(T, g, acc, g_out, lane);
      }
    }
    team_sync<NW, TEAMS>(team);

    unsigned bkey = 0u;
    int wb = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      const unsigned kw = yk[4 * w];
      if (kw > bkey) { bkey = kw; wb = w; }
    }
    const int plabel = 63 - (int)(bkey & 63u);
    const int p = (int)yk[4 * wb + 1];  // pivot: physical index
    const int newlabel = (rr == p) ? k + 1 : (label == k + 1 ? plabel : label);
    // finished column k: H[label][k] for rows with label <= k + 1
    if (par == 0 && newlabel <= k + 1 && k + 1 - newlabel < NTL) hb[newlabel * NTL + k + 1 - newlabel] = colv;
    live &= ~(1ull << p);
    if ((bkey >> 6) > 1u) {  // nonzero pivot
      const double2 piv = yv[wb];
      const double2 ip = crecip(piv);
      const double2 m = (candr && rr != p) ? cmul(colv, ip) : c0();
      const double2 *rp = cb + wb * CC + par;
      const double2 *kq = kb + par;
      // fused left + right pass; right accumulators split by component for ILP
      double xr0 = 0, xi0 = 0, yr0 = 0, yi0 = 0, xr1 = 0, xi1 = 0, yr1 = 0, yi1 = 0;
#pragma unroll
      for (int s = 0; s < CS; ++s) {
        const double2 r = rp[S * s];
        const double2 q = kq[S * s];
        double2 a = cfms(m, r, A[s]);
        A[s] = a;
        if (s & 1) {
          xr1 = fma(a.x, q.x, xr1); xi1 = fma(a.y, q.y, xi1);
          yr1 = fma(a.x, q.y, yr1); yi1 = fma(a.y, q.x, yi1);
        } else {
          xr0 = fma(a.x, q.x, xr0); xi0 = fma(a.y, q.y, xi0);
          yr0 = fma(a.x, q.y, yr0); yi0 = fma(a.y, q.x, yi0);
        }
      }
      double2 sum = make_double2((xr0 + xr1) - (xi0 + xi1), (yr0 + yr1) + (yi0 + yi1));
#pragma unroll
      for (int x = 1; x < S; x <<= 1) sum = cadd(sum, shfl2_xor(sum, x));
      colv = cmul(sum, ip);
    } else {
      colv = read_col<S, CS>(A, p, lane);  // nothing to eliminate: column p as it stands
    }
    label = newlabel;
  }
  // the last two columns: the carried one (label kend) and the remaining live index
  if (E >= 1) {
    if (par == 0 && label < E && kend + 1 - label < NTL) hb[label * NTL + kend + 1 - label] = colv;
    if (E >= 2) {
      const int pl = __ffsll((long long)live) - 1;  // label E-1
      const double2 cl = read_col<S, CS>(A, pl, lane);
      if (par == 0 && label < E && E - label < NTL) hb[label * NTL + E - label] = cl;
    }
  }
  // the pending series must be complete before its buffers are reused (E tiny)
  if (warp == SW) {
    for (; ss < D.nss; ++ss) {
      double2 g;
      if (series_step(D, ss, T.cin, T.ser, lane, g)) finish_term(T, g, acc, g_out, lane);
    }
  }
  team_sync<NW, TEAMS>(team);
  LHAF_PHASE(1)

  // ---- a7: F_j[m] = H[j][j+m] prod_{i=1..m} H[j+i][j+i-1] in place
  if (par == 0 && label < E) {
    double2 pi = c1();
    const int mmax = min(NTL - 2, E - 1 - label);
    for (int m = 1; m <= mmax; ++m) {
      pi = cmul(pi, hb[(label + m) * NTL]);
      hb[label * NTL + 1 + m] = cmul(hb[label * NTL + 1 + m], pi);
    }
  }
  double2 *Q = T.u1;                    // [E+1][NTL]: Q[j][t] = coefficient of x^{deg q_j - t}
  double2 *part = Q + (E + 1) * NTL;    // [2][NW][NTL] partial m-sums
  double2 *base = part + 2 * NW * NTL;  // [2][NTL] q_{j+1}[t] - H[j][j] q_{j+1}[t-1]
  if (warp == 0)
    for (int tt = lane; tt < NTL; tt += 32) Q[E * NTL + tt] = (tt == 0) ? c1() : c0();
  team_sync<NW, TEAMS>(team);
  LHAF_PHASE(2)

  // trailing La Budde: q_j = base_j - sum_w part_j[w]; warp w sums the m = 1 + w (mod NW)
  // terms of q_j[t] = q_{j+1}[t] - h_jj q_{j+1}[t-1] - sum_{m=1}^{min(t-1, E-1-j)} F_j[m]
  // q_{j+m+1}[t-m-1]; warp 0 finalizes row j+1 at the start of iteration j.
  for (int j = E - 1; j >= 0; --j) {
    const double2 *Fj = hb + j * NTL;
    if (warp == 0) {
      if (j + 1 < E) {
        const double2 *bp = base + ((j + 1) & 1) * NTL;
        const double2 *pp = part + ((j + 1) & 1) * NW * NTL;
        for (int tt = lane; tt < NTL; tt += 32) {
          double2 v = bp[tt];
#pragma unroll
          for (int w = 0; w < NW; ++w) v = csub(v, pp[w * NTL + tt]);
          Q[(j + 1) * NTL + tt] = v;
        }
        __syncwarp();
      }
      const double2 *q1 = Q + (j + 1) * NTL;
      const double2 hjj = Fj[1];
      for (int tt = lane; tt < NTL; tt += 32) {
        double2 v = c0();
        if (tt <= E - j) {
          v = q1[tt];  // zero above the degree of q_{j+1}
          if (tt >= 1) v = cfms(hjj, q1[tt - 1], v);
        }
        base[(j & 1) * NTL + tt] = v;
      }
    }
    double2 *pw = part + ((j & 1) * NW + warp) * NTL;
    for (int tt = lane; tt < NTL; tt += 32) {
      double2 v0 = c0(), v1 = c0();
      if (tt <= E - j) {
        const int mm = min(tt - 1, E - 1 - j);
        int m = 1 + warp;
        const double2 *qd = Q + (j + 1 + m) * NTL + tt - m - 1;  // q_{j+m+1}[tt-m-1]
        for (; m + NW <= mm; m += 2 * NW) {
          v0 = cfma(Fj[1 + m], qd[0], v0);
          v1 = cfma(Fj[1 + m + NW], qd[NW * (NTL - 1)], v1);
          qd += 2 * NW * (NTL - 1);
        }
        if (m <= mm) v0 = cfma(Fj[1 + m], qd[0], v0);
      }
      pw[tt] = cadd(v0, v1);
    }
    team_sync<NW, TEAMS>(team);
  }
  LHAF_PHASE(3)

  // ---- hand the polynomials to the series pipeline: c_M = q_1, c_B = q_0
  if (warp == SW) {
    const double2 *bp = base;  // j = 0 wrote parity 0
    const double2 *pp = part;
    const double2 *cM = Q + NTL;
    for (int tt = lane; tt < NTL; tt += 32) {
      double2 q0 = bp[tt];
#pragma unroll
      for (int w = 0; w < NW; ++w) q0 = csub(q0, pp[w * NTL + tt]);
      T.cin[NTL + tt] = q0;                  // c_B
      T.cin[tt] = loops ? cM[tt] : q0;       // c_M
    }
    __syncwarp();
    double2 *Qa = T.ser, *Ra = T.ser + (n + 2), *Ea = T.ser + 2 * (n + 2);
    for (int m = lane; m < n + 2; m += 32) {
      Qa[m] = c0();
      Ea[m] = c0();
      Ra[m] = (loops && m < NTL) ? csub(T.cin[m], T.cin[NTL + m]) : c0();
    }
    if (lane == 0) {
      T.psw[0] = T.csw[0];
      T.psw[1] = make_double2(valid ? 1.0 : 0.0, (double)out_idx);
    }
    __syncwarp();
    ss = 0;
  }
  LHAF_PHASE(4)
  team_sync<NW, TEAMS>(team);  // smem reused by the next term
  LHAF_PHASE(5)
}

// the series of the last term of a work unit (series warp only)
__device__ __forceinline__ void drain_series(const Pattern &D, const TeamMem &T, int &ss,
                                             Sums &acc, double2 *g_out, int lane) {
  for (; ss < D.nss; ++ss) {
    double2 g;
    if (series_step(D, ss, T.cin, T.ser, lane, g)) finish_term(T, g, acc, g_out, lane);
  }
}

// ================================================================ kernels
template <int S, int CS, int NW, int TEAMS, int REGS>
__global__ void __maxnreg__(REGS)
sieve_v3(JobDev J, uint64_t ubeg, uint64_t uend, int team_words) {
  extern __shared__ double2 smem[];
  __shared__ unsigned long long s_unit;
  __shared__ double s_acc[TEAMS][6];
  constexpr int TS = 32 * NW;
  const int team = threadIdx.x / TS, tid = threadIdx.x % TS;
  const int lane = tid & 31, warp = tid >> 5;
  double2 *tbase = smem + (size_t)team * team_words;
  for (int i = tid; i < team_words; i += TS) tbase[i] = c0();
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) s_unit = ubeg + atomicAdd(J.counter, 1ull);
    __syncthreads();
    const uint64_t u = s_unit;
    if (u >= uend) break;
    const PatDesc P = J.descs[find_pattern(J, u)];
    const Pattern D = pattern_of(P);
    const TeamMem T = carve<S, CS, NW>(tbase, D.E, D.NTL, D.n);
    const uint64_t tb = (u - P.unit_begin) * P.chunk;
    const uint64_t te = min(tb + P.chunk, P.T_eval);
    Sums acc;
    int ss = D.nss;  // nothing pending
    // every team runs the same number of terms (duplicates of tb are discarded)
    const uint64_t per_team = (te - tb + TEAMS - 1) / TEAMS;
    for (uint64_t i = 0; i < per_team; ++i) {
      const uint64_t t = tb + i * TEAMS + team;
      const bool valid = t < te;
      team_term<S, CS, NW, TEAMS>(P, D, J, valid ? t : tb, valid, 0, T, tid, team, ss, acc,
                                  nullptr);
    }
    if (warp == NW - 1) drain_series(D, T, ss, acc, nullptr, lane);
    if (warp == NW - 1 && lane == 0) {
      s_acc[team][0] = acc.rh; s_acc[team][1] = acc.rl; s_acc[team][2] = acc.ih;
      s_acc[team][3] = acc.il; s_acc[team][4] = acc.ah; s_acc[team][5] = acc.al;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double a0 = 0, a1 = 0, a2 = 0, a3 = 0, a4 = 0, a5 = 0;
      for (int w = 0; w < TEAMS; ++w) {
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

// g(t) (unweighted) of pattern 0 for a list of term indices; each team takes a contiguous
// slice of the list.
template <int S, int CS, int NW, int TEAMS, int REGS>
__global__ void __maxnreg__(REGS)
terms_v3(JobDev J, const uint64_t *ts, int nt, double2 *g_out, int team_words) {
  extern __shared__ double2 smem[];
  constexpr int TS = 32 * NW;
  const int team = threadIdx.x / TS, tid = threadIdx.x % TS;
  const int lane = tid & 31, warp = tid >> 5;
  double2 *tbase = smem + (size_t)team * team_words;
  for (int i = tid; i < team_words; i += TS) tbase[i] = c0();
  __syncthreads();
  const PatDesc P = J.descs[0];
  const Pattern D = pattern_of(P);
  const TeamMem T = carve<S, CS, NW>(tbase, D.E, D.NTL, D.n);
  const int nteams = gridDim.x * TEAMS;
  const int gteam = blockIdx.x * TEAMS + team;
  const int per = (nt + nteams - 1) / nteams;
  const int b = gteam * per, e = min(nt, b + per);
  Sums acc;
  int ss = D.nss;
  for (int i = b; i < e; ++i)
    team_term<S, CS, NW, TEAMS>(P, D, J, ts[i], true, (uint64_t)i, T, tid, team, ss, acc, g_out);
  if (warp == NW - 1) drain_series(D, T, ss, acc, g_out, lane);
}

// ================================================================ host side
template <int S, int CS, int NW, int TEAMS, int REGS>
struct Inst {
  using Sh = Shape<S, CS, NW>;
  static constexpr int EMAX = Sh::EMAX;
  static constexpr int THREADS = 32 * NW * TEAMS;
  static cudaError_t sieve(const JobDev &job, int E, int NTL, int n, uint64_t ubeg, uint64_t uend,
                           int num_sms, cudaStream_t s) {
    const int tw = Sh::words(E, NTL, n);
    const size_t smem = (size_t)tw * TEAMS * sizeof(double2);
    auto *kern = sieve_v3<S, CS, NW, TEAMS, REGS>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
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
    kern<<<(unsigned)grid, THREADS, smem, s>>>(job, ubeg, uend, tw);
    return cudaGetLastError();
  }
  static cudaError_t terms(const JobDev &job, int E, int NTL, int n, const uint64_t *t, int nt,
                           double2 *g_out, cudaStream_t s) {
    const int tw = Sh::words(E, NTL, n);
    const size_t smem = (size_t)tw * TEAMS * sizeof(double2);
    auto *kern = terms_v3<S, CS, NW, TEAMS, REGS>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int grid = (nt + TEAMS - 1) / TEAMS;
    if (grid > 1024) grid = 1024;
    kern<<<grid, THREADS, smem, s>>>(job, t, nt, g_out, tw);
    return cudaGetLastError();
  }
};

// <S, CS, NW, TEAMS, registers per thread>.  Each SM sub-partition has 16K registers, so a
// warp of R registers allows floor(512 / R) warps per sub-partition.
using I9 = Inst<1, 9, 1, 4, 128>;
using I17 = Inst<1, 17, 1, 4, 128>;
using I25 = Inst<1, 25, 1, 4, 168>;
using I32 = Inst<1, 32, 1, 4, 168>;
using I48 = Inst<2, 24, 3, 1, 168>;
using I62 = Inst<2, 31, 4, 1, 200>;  // 2 CTAs / SM, no spills
using I64 = Inst<2, 32, 4, 1, 168>;
// alternatives (LHAF_V3_ALT=1): more lanes per row, fewer registers, more warps per SM
using A26 = Inst<2, 13, 2, 2, 104>;   // E <= 26: 4 warps / CTA
using A48 = Inst<4, 12, 6, 1, 104>;   // E <= 48: 6 warps / CTA
using A64 = Inst<4, 16, 8, 1, 128>;   // E <= 64: 8 warps / CTA
using B62 = Inst<2, 31, 4, 1, 200>;   // (LHAF_V3_ALT=2) E <= 62 without spills: 2 CTAs / SM
static int alt_mode() {
  static const int m = [] { const char *e = getenv("LHAF_V3_ALT"); return e ? atoi(e) : 0; }();
  return m;
}

static cudaError_t ensure_inv() {
  if (g_inv_ready) return cudaSuccess;
  double h[256];
  h[0] = 0.0;
  for (int i = 1; i < 256; ++i) h[i] = 1.0 / (double)i;
  cudaError_t e = cudaMemcpyToSymbol(c_inv, h, sizeof h);
  if (e == cudaSuccess) g_inv_ready = true;
  return e;
}

}  // namespace v3

cudaError_t v3_ensure_tables() { return v3::ensure_inv(); }

#ifdef LHAF_PHASE_TIMING
extern "C" int lhaf_debug_phase_cycles(unsigned long long *out8) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out8, v3::g_phase, 8 * sizeof(unsigned long long));
  unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  return (int)cudaMemcpyToSymbol(v3::g_phase, z, sizeof z);
}
#endif

#define LHAF_V3_DISPATCH(CALL)                  \
  if (v3::alt_mode() == 2 && E > 48 && E <= v3::B62::EMAX) return v3::B62::CALL; \
  if (v3::alt_mode() == 1) {                    \
    if (E <= v3::A26::EMAX && E > 17) return v3::A26::CALL; \
    if (E <= v3::A48::EMAX && E > 32) return v3::A48::CALL; \
    if (E <= v3::A64::EMAX && E > 48) return v3::A64::CALL; \
  }                                             \
  if (E <= v3::I9::EMAX) return v3::I9::CALL;   \
  if (E <= v3::I17::EMAX) return v3::I17::CALL; \
  if (E <= v3::I25::EMAX) return v3::I25::CALL; \
  if (E <= v3::I32::EMAX) return v3::I32::CALL; \
  if (E <= v3::I48::EMAX) return v3::I48::CALL; \
  if (E <= v3::I62::EMAX) return v3::I62::CALL; \
  if (E <= v3::I64::EMAX) return v3::I64::CALL; \
  return cudaErrorInvalidValue;

cudaError_t launch_sieve_v3(const JobDev &job, int e_max, int ntl_max, int n_max, uint64_t ubeg,
                            uint64_t uend, int num_sms, cudaStream_t s) {
  if (uend <= ubeg) return cudaSuccess;
  cudaError_t e = v3::ensure_inv();
  if (e != cudaSuccess) return e;
  const int E = e_max;
  LHAF_V3_DISPATCH(sieve(job, e_max, ntl_max, n_max, ubeg, uend, num_sms, s))
}

cudaError_t launch_terms_v3(const JobDev &job, int e_max, int ntl_max, int n_max, const uint64_t *t,
                            int nt, double2 *g_out, cudaStream_t s) {
  if (nt <= 0) return cudaSuccess;
  cudaError_t e = v3::ensure_inv();
  if (e != cudaSuccess) return e;
  const int E = e_max;
  LHAF_V3_DISPATCH(terms(job, e_max, ntl_max, n_max, t, nt, g_out, s))
}

}  // namespace lhaf

namespace lhaf {
// Algorithmic FP64 flops of one v3 term (real flops; complex MAC = 8, complex mul = 6): the
// useful work of the Gauss-transform Hessenberg reduction of the E x E bordered matrix, the
// band scaling, the trailing La Budde on the top NTL coefficients, the series recursions and
// the final product.  Work the kernel spends on finished columns is
// not counted.
double v3_flops_per_term(int d, int n, bool loops) {
  const int E = d + (loops ? 1 : 0);
  const int NTL = std::min(n + (loops ? 2 : 1), E + 1);
  double cmac = 0.0, cmul_ = 0.0;
  for (int k = 0; k + 2 < E; ++k) {
    const double rem = E - k - 2;  // rows eliminated
    cmac += rem * (E - k - 1);     // left
    cmac += (double)E * rem;       // right
    cmul_ += rem + 1;              // multipliers, new pivot column scaling
  }
  for (int j = 0; j < E; ++j) cmul_ += 2.0 * std::max(0, std::min(NTL - 2, E - 1 - j));  // F
  for (int j = E - 1; j >= 0; --j)
    for (int t = 0; t < NTL && t <= E - j; ++t)
      cmac += (t >= 1 ? 1 : 0) + std::max(0, std::min(t - 1, E - 1 - j));
  const double nn = n;
  cmac += nn * (nn + 1) / 2.0;                                                  // c_M^{-1/2}
  if (loops) cmac += (nn + 2) * (nn + 1) / 2.0 + nn * (nn + 1) / 2.0 + nn + 1;  // R, exp, g
  return 8.0 * cmac + 6.0 * cmul_;
}
}  // namespace lhaf
