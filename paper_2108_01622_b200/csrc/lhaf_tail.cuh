// lhaf_tail.cuh -- the per-term tail shared by the v3 and v5 sieve kernels: trailing La Budde on
// the top NTL coefficients of the band of H (a7), and the power series of a8/a9
// (g = [lam^n] c_M^{-1/2} exp(S/2)).  DESIGN.md section 2 steps 3-4.  Product code only.
#pragma once
#include <cuda_runtime.h>
#include "lhaf_device.cuh"

namespace lhaf {
namespace tail {

// 1/m for the series recursions (one copy per translation unit; ensure_inv() uploads it)
static __constant__ double c_inv[256];

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

// ---------------------------------------------------------------- La Budde (one warp)
// Trailing La Budde on the top NTL coefficients (t = distance from the leading coefficient):
//   q_j[t] = q_{j+1}[t] - h_jj q_{j+1}[t-1] + S_j[t],
//   S_j[t] = - sum_{m=1}^{min(t-1, E-1-j)} F_j[m] q_{j+m+1}[t-m-1]     (F_j[m] = hb[j][1+m]).
// S_j needs only rows j+2.. (already final), so iteration j computes S_{j-1} ahead of the
// short loop-carried chain q_{j+1} -> q_j (a shuffle and two FMAs).  Lane t holds q_{j+1}[t]
// in registers (NRT registers per lane: NTL <= 32 NRT); rows go to Q[j][t] for the m-sums.
template <int NRT>
__device__ __forceinline__ void labudde(const double2 *hb, double2 *Q, int E, int NTL, int lane) {
  double2 qn[NRT], S[NRT];
#pragma unroll
  for (int r = 0; r < NRT; ++r) {
    const int t = lane + 32 * r;
    qn[r] = (t == 0) ? c1() : c0();  // q_E = 1
    S[r] = c0();                     // S_{E-1} = 0
    if (t < NTL) Q[E * NTL + t] = qn[r];
  }
  __syncwarp();
  for (int j = E - 1; j >= 0; --j) {
    // S_{j-1}[t] from rows j+1 .. E (final); groups of 4 terms under a warp-uniform bound
    double2 Sn[NRT];
#pragma unroll
    for (int r = 0; r < NRT; ++r) {
      const int t = lane + 32 * r;
      double2 a0 = c0(), a1 = c0(), a2 = c0(), a3 = c0();
      const int mm = (j >= 1 && t < NTL && t <= E - j + 1) ? min(t - 1, E - j) : 0;
      const int mw = min(min(NTL, 32 * (r + 1)) - 2, E - j);  // max of mm over the warp
      if (j >= 1) {
        const double2 *F = hb + (j - 1) * NTL + 1;  // F_{j-1}[m] = F[m]
        const double2 *qd = Q + (j + 1) * NTL + t - 2;  // q_{j+m}[t-m-1] at m = 1
        for (int m = 1; m <= mw; m += 4, qd += 4 * (NTL - 1)) {
          if (m <= mm) a0 = cfma(F[m], qd[0], a0);
          if (m + 1 <= mm) a1 = cfma(F[m + 1], qd[NTL - 1], a1);
          if (m + 2 <= mm) a2 = cfma(F[m + 2], qd[2 * (NTL - 1)], a2);
          if (m + 3 <= mm) a3 = cfma(F[m + 3], qd[3 * (NTL - 1)], a3);
        }
      }
      Sn[r] = make_double2(-((a0.x + a1.x) + (a2.x + a3.x)), -((a0.y + a1.y) + (a2.y + a3.y)));
    }
    // q_j from q_{j+1} (registers) and S_j
    const double2 h = hb[j * NTL + 1];
    double2 shfl_last[NRT];  // q_{j+1}[32 r + 31], for lane 0 of register r + 1
#pragma unroll
    for (int r = 0; r < NRT; ++r) shfl_last[r] = shfl2(qn[r], 31);
    double2 up[NRT];  // q_{j+1}[t-1]
#pragma unroll
    for (int r = 0; r < NRT; ++r) {
      const double2 s = shfl2(qn[r], (lane + 31) & 31);  // all lanes shuffle (full mask)
      up[r] = (lane != 0) ? s : (r == 0 ? c0() : shfl_last[r - 1]);
    }
#pragma unroll
    for (int r = 0; r < NRT; ++r) {
      const int t = lane + 32 * r;
      double2 q = cadd(S[r], cfms(h, up[r], qn[r]));
      if (t > E - j) q = c0();  // above the degree of q_j
      qn[r] = q;
      if (t < NTL) Q[j * NTL + t] = q;
      S[r] = Sn[r];
    }
    __syncwarp();
  }
}

// Team version: warp w sums the m = 1 + w (mod NW) part of S_{j-1} into part[j&1][w][t];
// warp 0 keeps q_{j+1} in registers and forms q_j = q_{j+1} - h q_{j+1}[t-1] - sum_w part;
// one team barrier per row.
template <int NRT, int NW, int TEAMS>
__device__ __forceinline__ void labudde_team(const double2 *hb, double2 *Q, double2 *part, int E,
                                             int NTL, int warp, int lane, int team) {
  double2 qn[NRT];
#pragma unroll
  for (int r = 0; r < NRT; ++r) {
    const int t = lane + 32 * r;
    qn[r] = (t == 0) ? c1() : c0();  // q_E = 1
    if (warp == 0 && t < NTL) Q[E * NTL + t] = qn[r];
  }
  team_sync<NW, TEAMS>(team);
  for (int j = E - 1; j >= 0; --j) {
    // partial m-sums of S_{j-1} (rows j+1 .. E are final)
    double2 *pw = part + ((j & 1) * NW + warp) * NTL;
#pragma unroll
    for (int r = 0; r < NRT; ++r) {
      const int t = lane + 32 * r;
      double2 a0 = c0(), a1 = c0(), a2 = c0(), a3 = c0();
      const int mm = (j >= 1 && t < NTL && t <= E - j + 1) ? min(t - 1, E - j) : 0;
      const int mw = min(min(NTL, 32 * (r + 1)) - 2, E - j);  // max of mm over the warp
      if (j >= 1) {
        const double2 *F = hb + (j - 1) * NTL + 1;  // F_{j-1}[m] = F[m]
        int m = 1 + warp;
        const double2 *qd = Q + (j + m) * NTL + t - m - 1;  // q_{j+m}[t-m-1]
        for (; m <= mw; m += 4 * NW, qd += 4 * NW * (NTL - 1)) {  // warp-uniform bound
          if (m <= mm) a0 = cfma(F[m], qd[0], a0);
          if (m + NW <= mm) a1 = cfma(F[m + NW], qd[NW * (NTL - 1)], a1);
          if (m + 2 * NW <= mm) a2 = cfma(F[m + 2 * NW], qd[2 * NW * (NTL - 1)], a2);
          if (m + 3 * NW <= mm) a3 = cfma(F[m + 3 * NW], qd[3 * NW * (NTL - 1)], a3);
        }
      }
      a0 = cadd(a0, a2);
      a1 = cadd(a1, a3);
      if (t < NTL) pw[t] = cadd(a0, a1);
    }
    if (warp == 0) {
      // q_j = q_{j+1} - h_jj q_{j+1}[t-1] - S_j, S_j = sum of the partials written at j+1
      const double2 h = hb[j * NTL + 1];
      const double2 *pp = part + ((j + 1) & 1) * NW * NTL;
      double2 last[NRT], up[NRT];
#pragma unroll
      for (int r = 0; r < NRT; ++r) last[r] = shfl2(qn[r], 31);
#pragma unroll
      for (int r = 0; r < NRT; ++r) {
        const double2 s = shfl2(qn[r], (lane + 31) & 31);
        up[r] = (lane != 0) ? s : (r == 0 ? c0() : last[r - 1]);
      }
#pragma unroll
      for (int r = 0; r < NRT; ++r) {
        const int t = lane + 32 * r;
        double2 q = cfms(h, up[r], qn[r]);
        if (j + 1 < E && t < NTL) {
#pragma unroll
          for (int w = 0; w < NW; ++w) q = csub(q, pp[w * NTL + t]);
        }
        if (t > E - j) q = c0();  // above the degree of q_j
        qn[r] = q;
        if (t < NTL) Q[j * NTL + t] = q;
      }
    }
    team_sync<NW, TEAMS>(team);
  }
}

// out[t] = q[t - d] (0 for t < d) over the NRT registers of a warp; d warp-uniform in [1, 31]
template <int NRT>
__device__ __forceinline__ void shift_up(const double2 (&q)[NRT], int d, int lane,
                                         double2 (&out)[NRT]) {
  double2 sh[NRT];
#pragma unroll
  for (int r = 0; r < NRT; ++r) sh[r] = shfl2(q[r], (lane - d) & 31);
#pragma unroll
  for (int r = 0; r < NRT; ++r) out[r] = (lane >= d) ? sh[r] : (r == 0 ? c0() : sh[r - 1]);
}

// Team version, two rows per barrier.  Block b forms rows j = E-1-2b and j-1 in warp 0:
//   q_j     = q_{j+1} - h_j q_{j+1}[t-1]     - P_j     - F_j[1] q_{j+2}[t-2]
//   q_{j-1} = q_j     - h_{j-1} q_j[t-1]     - P_{j-1} - F_{j-1}[1] q_{j+1}[t-2]
//                                                      - F_{j-1}[2] q_{j+2}[t-3]
// with q_{j+1}, q_{j+2} (the previous block's rows) held in registers, while every warp sums,
// for the next block's rows r = j-2, j-3, the m-terms on rows >= j+1 (m >= j - r), split
// m = m0 + w (mod NW): P_r[t] = sum_m F_r[m] q_{r+m+1}[t-m-1] into part[b&1][w][r][t].
template <int NRT, int NW, int TEAMS>
__device__ __forceinline__ void labudde_team2(const double2 *hb, double2 *Q, double2 *part, int E,
                                              int NTL, int warp, int lane, int team) {
  double2 qa[NRT], qb[NRT];  // q_{j+1}, q_{j+2}
#pragma unroll
  for (int r = 0; r < NRT; ++r) {
    const int t = lane + 32 * r;
    qa[r] = (t == 0) ? c1() : c0();  // q_E = 1
    qb[r] = c0();                    // (q_{E+1}: no such row)
    if (warp == 0 && t < NTL) Q[E * NTL + t] = qa[r];
    if (t < NTL) {  // the partials of block 0 (none)
      part[(NW + warp) * 2 * NTL + t] = c0();
      part[(NW + warp) * 2 * NTL + NTL + t] = c0();
    }
  }
  team_sync<NW, TEAMS>(team);
  for (int b = 0, j = E - 1; j >= 0; ++b, j -= 2) {
    // partial m-sums for rows j-2 (slot 0) and j-3 (slot 1) from rows >= j+1 (final)
    double2 *pw = part + ((b & 1) * NW + warp) * 2 * NTL;
#pragma unroll
    for (int sl = 0; sl < 2; ++sl) {
      const int rw = j - 2 - sl, m0 = 2 + sl;
#pragma unroll
      for (int r = 0; r < NRT; ++r) {
        const int t = lane + 32 * r;
        double2 a0 = c0(), a1 = c0(), a2 = c0(), a3 = c0();
        if (rw >= 0) {
          const int mm = (t < NTL && t <= E - rw) ? min(t - 1, E - 1 - rw) : 0;
          const int mw = min(min(NTL, 32 * (r + 1)) - 2, E - 1 - rw);  // max of mm over the warp
          const double2 *F = hb + rw * NTL + 1;                        // F_r[m] = F[m]
          int m = m0 + warp;
          const double2 *qd = Q + (rw + m + 1) * NTL + t - m - 1;       // q_{r+m+1}[t-m-1]
          for (; m <= mw; m += 4 * NW, qd += 4 * NW * (NTL - 1)) {     // warp-uniform bound
            if (m <= mm) a0 = cfma(F[m], qd[0], a0);
            if (m + NW <= mm) a1 = cfma(F[m + NW], qd[NW * (NTL - 1)], a1);
            if (m + 2 * NW <= mm) a2 = cfma(F[m + 2 * NW], qd[2 * NW * (NTL - 1)], a2);
            if (m + 3 * NW <= mm) a3 = cfma(F[m + 3 * NW], qd[3 * NW * (NTL - 1)], a3);
          }
        }
        if (t < NTL) pw[sl * NTL + t] = cadd(cadd(a0, a2), cadd(a1, a3));
      }
    }
    if (warp == 0) {
      const double2 *pp = part + (((b + 1) & 1) * NW) * 2 * NTL;  // written in block b-1
      double2 u1[NRT], u2[NRT], u3[NRT];
      // row j
      {
        const double2 h = hb[j * NTL + 1];
        const double2 f1 = (E - 1 - j >= 1 && NTL > 2) ? hb[j * NTL + 2] : c0();
        shift_up<NRT>(qa, 1, lane, u1);
        shift_up<NRT>(qb, 2, lane, u2);
#pragma unroll
        for (int r = 0; r < NRT; ++r) {
          const int t = lane + 32 * r;
          double2 q = cfms(h, u1[r], qa[r]);
          q = cfms(f1, u2[r], q);
          if (t < NTL) {
#pragma unroll
            for (int w = 0; w < NW; ++w) q = csub(q, pp[w * 2 * NTL + t]);
          }
          if (t > E - j) q = c0();  // above the degree of q_j
          qb[r] = q;                // (qb <- q_j, qa stays q_{j+1} for row j-1)
          if (t < NTL) Q[j * NTL + t] = q;
        }
      }
      // row j-1: q_{j+1} = qa, q_j = qb, q_{j+2} = u2 shifted by 2 (recompute by 3)
      if (j >= 1) {
        const int i = j - 1;
        const double2 h = hb[i * NTL + 1];
        const double2 f1 = (NTL > 2) ? hb[i * NTL + 2] : c0();  // (E-1-i >= 1)
        const double2 f2 = (E - 1 - i >= 2 && NTL > 3) ? hb[i * NTL + 3] : c0();
        double2 s1[NRT];
        shift_up<NRT>(qb, 1, lane, s1);  // q_j[t-1]
        shift_up<NRT>(qa, 2, lane, u1);  // q_{j+1}[t-2]
        // q_{j+2}[t-3] = u2 (q_{j+2}[t-2]) shifted by one more
        shift_up<NRT>(u2, 1, lane, u3);
#pragma unroll
        for (int r = 0; r < NRT; ++r) {
          const int t = lane + 32 * r;
          double2 q = cfms(h, s1[r], qb[r]);
          q = cfms(f1, u1[r], q);
          q = cfms(f2, u3[r], q);
          if (t < NTL) {
#pragma unroll
            for (int w = 0; w < NW; ++w) q = csub(q, pp[w * 2 * NTL + NTL + t]);
          }
          if (t > E - i) q = c0();
          qa[r] = q;  // q_{j-1}: the next block's q_{j'+1}; qb = q_j its q_{j'+2}
          if (t < NTL) Q[i * NTL + t] = q;
        }
      }
    }
    team_sync<NW, TEAMS>(team);
  }
}

// ---------------------------------------------------------------- series (one warp)
// g = [lam^n] c_M^{-1/2} exp(S/2), lam S = 1 - c_B / c_M (loops), by column sweeps: lane m
// holds the accumulators of coefficients m, m+32, ... (NR registers, n + 2 <= 32 NR):
//   m Q_m = -sum_{i=1}^{m} (m - i/2) c_i Q_{m-i}   (c = c_M),  R = (c_M - c_B) / c_M,
//   m E_m = 1/2 sum_{j=1}^{m} j S_j E_{m-j},  S_j = R_{j+1},  g = sum_m Q_m E_{n-m}.
// Finished coefficients go to scratch (Qs, Rs, Es: 3 (n+2) words).
template <int NR>
__device__ __forceinline__ double2 series(const double2 *cM, const double2 *cB, int n, int NTL,
                                          bool loops, double2 *scratch, int lane) {
  double2 *Qs = scratch, *Rs = Qs + (n + 2), *Es = Rs + (n + 2);
  double2 qa[NR], ra[NR];
  double md[NR];
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    const int m = lane + 32 * r;
    md[r] = (double)m;
    qa[r] = c0();
    ra[r] = (loops && m <= n + 1 && m < NTL) ? csub(cM[m], cB[m]) : c0();
  }
  const int jmax = loops ? n + 1 : n;
  double jd = 0.0;
  for (int j = 0; j <= jmax; ++j, jd += 1.0) {
    const int lj = j & 31, rj = j >> 5;
    double2 qs = qa[0], rs = ra[0];
#pragma unroll
    for (int r = 1; r < NR; ++r)
      if (rj == r) { qs = qa[r]; rs = ra[r]; }
    double2 qj = (j == 0) ? c1() : cscale(qs, -c_inv[j]);
    qj = shfl2(qj, lj);
    const double2 rv = shfl2(rs, lj);
    if (lane == lj) { Qs[j] = qj; Rs[j] = rv; }
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      const int m = lane + 32 * r;
      if (m > j && m <= jmax && m - j < NTL) {
        const double2 c = cM[m - j];
        if (m <= n) qa[r] = cfma(cscale(c, 0.5 * (md[r] + jd)), qj, qa[r]);
        if (loops) ra[r] = cfms(c, rv, ra[r]);
      }
    }
  }
  __syncwarp();
  if (!loops) return Qs[n];
  double2 ea[NR];
#pragma unroll
  for (int r = 0; r < NR; ++r) ea[r] = c0();
  double id = 0.0;
  for (int i = 0; i <= n; ++i, id += 1.0) {
    const int li = i & 31, ri = i >> 5;
    double2 es = ea[0];
#pragma unroll
    for (int r = 1; r < NR; ++r)
      if (ri == r) es = ea[r];
    double2 ei = (i == 0) ? c1() : cscale(es, c_inv[i]);
    ei = shfl2(ei, li);
    if (lane == li) Es[i] = ei;
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      const int m = lane + 32 * r;
      if (m > i && m <= n) ea[r] = cfma(cscale(Rs[m - i + 1], 0.5 * (md[r] - id)), ei, ea[r]);
    }
  }
  __syncwarp();
  double2 gp = c0();
  for (int m = lane; m <= n; m += 32) gp = cfma(Qs[m], Es[n - m], gp);
  return warp_sum2(gp);
}

// The two halves of series() for many loop vectors sharing one c_M (gamma-batched evaluation):
// qhalf_coeffs writes Q = c_M^{-1/2} (degrees 0..n) to Qs once per term; exp_dot then gives, per
// loop vector, g = sum_m Q_m E_{n-m} with E = exp(S/2), S = sum_{j>=1} s_j lam^j given directly
// (s_j = z'^T H^{j-1} y' from the Krylov products).  One warp each; Es: n + 1 scratch.
template <int NR>
__device__ __forceinline__ void qhalf_coeffs(const double2 *cM, int n, int NTL, double2 *Qs, int lane) {
  double2 qa[NR];
  double md[NR];
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    md[r] = (double)(lane + 32 * r);
    qa[r] = c0();
  }
  double jd = 0.0;
  for (int j = 0; j <= n; ++j, jd += 1.0) {
    const int lj = j & 31, rj = j >> 5;
    double2 qs = qa[0];
#pragma unroll
    for (int r = 1; r < NR; ++r)
      if (rj == r) qs = qa[r];
    double2 qj = (j == 0) ? c1() : cscale(qs, -c_inv[j]);
    qj = shfl2(qj, lj);
    if (lane == lj) Qs[j] = qj;
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      const int m = lane + 32 * r;
      if (m > j && m <= n && m - j < NTL) qa[r] = cfma(cscale(cM[m - j], 0.5 * (md[r] + jd)), qj, qa[r]);
    }
  }
  __syncwarp();
}

template <int NR>
__device__ __forceinline__ double2 exp_dot(const double2 *Qs, const double2 *S, int n, double2 *Es,
                                           int lane) {
  double2 ea[NR];
  double md[NR];
#pragma unroll
  for (int r = 0; r < NR; ++r) {
    md[r] = (double)(lane + 32 * r);
    ea[r] = c0();
  }
  double id = 0.0;
  for (int i = 0; i <= n; ++i, id += 1.0) {
    const int li = i & 31, ri = i >> 5;
    double2 es = ea[0];
#pragma unroll
    for (int r = 1; r < NR; ++r)
      if (ri == r) es = ea[r];
    double2 ei = (i == 0) ? c1() : cscale(es, c_inv[i]);
    ei = shfl2(ei, li);
    if (lane == li) Es[i] = ei;
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      const int m = lane + 32 * r;
      // m E_m = 1/2 sum_{j=1}^{m} j S_j E_{m-j}: the term of E_i in lane m has j = m - i
      if (m > i && m <= n) ea[r] = cfma(cscale(S[m - i], 0.5 * (md[r] - id)), ei, ea[r]);
    }
  }
  __syncwarp();
  double2 gp = c0();
  for (int m = lane; m <= n; m += 32) gp = cfma(Qs[m], Es[n - m], gp);
  return warp_sum2(gp);
}

// Blocked team La Budde (one barrier per BK rows).  Rows are processed in blocks of BK from
// the bottom; block b = rows [jhi - BK + 1, jhi], jhi = E - 1 - b BK.  For row j of block b
// the m-sum of S_j splits by source row s = j + m + 1:
//   far  s >= jhi + BK + 1 (blocks b-2 and older): computed by warps 1 .. NW-1 during stage
//        b - 1 into fp[b & 1] (the sources are final then);
//   near s in [j + 2, jhi + BK] (blocks b - 1 and b): summed by warp 0 in stage b -- the
//        block b - 1 sources for all BK rows at once (independent accumulators), then row by
//        row the in-block sources just before the row's chain step
//        q_j = q_{j+1} - h_jj q_{j+1}[t-1] - S_j.
// So warp 0 runs the sequential chain while the other warps prepare the next block, and the
// team synchronises once per BK rows instead of once per one or two.  Lane t (+ 32 r) holds
// coefficient t; q_j is stored in Q[j] (band row j + 1, consumed by then); fp holds
// [2][BK][NTL].  NW >= 2.
template <int NRT, int NW, int BK, int TEAMS>
__device__ __forceinline__ void labudde_blocked(const double2 *hb, double2 *Q, double2 *fp, int E,
                                                int NTL, int warp, int lane, int team) {
  double2 qa[NRT];  // warp 0: q_{j+1}
#pragma unroll
  for (int r = 0; r < NRT; ++r) {
    const int t = lane + 32 * r;
    qa[r] = (t == 0) ? c1() : c0();  // q_E = 1
    if (warp == 0 && t < NTL) Q[E * NTL + t] = qa[r];
  }
  team_sync<NW, TEAMS>(team);
  for (int b = 0, jhi = E - 1; jhi >= 0; ++b, jhi -= BK) {
    const int jlo = max(0, jhi - BK + 1);
    const int top = min(E, jhi + BK);
    if (warp == 0) {
      const double2 *fpb = fp + (b & 1) * BK * NTL;
      // (1) batched, all BK rows at once: far part + sources of block b - 1 (s = jhi + 1 ..
      //     top, final since the last barrier): independent accumulators, no chain
      double2 acc[BK][NRT];
#pragma unroll
      for (int jj = 0; jj < BK; ++jj) {
        const int j = jhi - jj;
#pragma unroll
        for (int r = 0; r < NRT; ++r) {
          const int t = lane + 32 * r;
          acc[jj][r] = (b > 0 && j >= jlo && t < NTL) ? fpb[jj * NTL + t] : c0();
        }
      }
#pragma unroll
      for (int ss = 1; ss <= BK; ++ss) {
        const int s = jhi + ss;
        if (s > top) break;
        const double2 *Qs = Q + s * NTL;
#pragma unroll
        for (int jj = 0; jj < BK; ++jj) {
          const int j = jhi - jj, m = ss + jj - 1;  // s - j - 1
          if (j < jlo || m < 1 || m > NTL - 2) continue;
          const double2 f = hb[j * NTL + 1 + m];
#pragma unroll
          for (int r = 0; r < NRT; ++r) {
            const int t = lane + 32 * r;
            if (t < NTL && t >= m + 1) acc[jj][r] = cfma(f, Qs[t - m - 1], acc[jj][r]);
          }
        }
      }
      // (2) sequential: in-block sources s = j + 2 .. jhi, then the chain step
#pragma unroll
      for (int jj = 0; jj < BK; ++jj) {
        const int j = jhi - jj;
        if (j < jlo) break;
        const double2 *F = hb + j * NTL + 1;
#pragma unroll
        for (int ss = 2; ss <= jj; ++ss) {  // s = j + ss <= jhi
          const int m = ss - 1;
          if (m > NTL - 2) break;
          const double2 f = F[m];
          const double2 *Qs = Q + (j + ss) * NTL;
#pragma unroll
          for (int r = 0; r < NRT; ++r) {
            const int t = lane + 32 * r;
            if (t < NTL && t >= m + 1) acc[jj][r] = cfma(f, Qs[t - m - 1], acc[jj][r]);
          }
        }
        const double2 h = F[0];  // hb[j][1] = h_jj
        double2 up[NRT];
        shift_up<NRT>(qa, 1, lane, up);
#pragma unroll
        for (int r = 0; r < NRT; ++r) {
          const int t = lane + 32 * r;
          double2 q = csub(cfms(h, up[r], qa[r]), acc[jj][r]);
          if (t > E - j) q = c0();  // above the degree of q_j
          qa[r] = q;
          if (t < NTL) Q[j * NTL + t] = q;
        }
        __syncwarp();
      }
    } else if (jhi - BK >= 0) {
      // far parts of the next block's rows from sources s >= jhi + 1 (final)
      const int jhi2 = jhi - BK, jlo2 = max(0, jhi2 - BK + 1);
      double2 *fpn = fp + ((b + 1) & 1) * BK * NTL;
      for (int jj = warp - 1; jj < BK && jhi2 - jj >= jlo2; jj += NW - 1) {
        const int j = jhi2 - jj;
        const double2 *F = hb + j * NTL + 1;
        const int smax = min(E, j + NTL - 1);
        double2 a0[NRT], a1[NRT];
#pragma unroll
        for (int r = 0; r < NRT; ++r) { a0[r] = c0(); a1[r] = c0(); }
        int s = jhi + 1;
        for (; s + 1 <= smax; s += 2) {
          const int m = s - j - 1;
          const double2 f0 = F[m], f1 = F[m + 1];
#pragma unroll
          for (int r = 0; r < NRT; ++r) {
            const int t = lane + 32 * r;
            if (t < NTL && t >= m + 1) a0[r] = cfma(f0, Q[s * NTL + t - m - 1], a0[r]);
            if (t < NTL && t >= m + 2) a1[r] = cfma(f1, Q[(s + 1) * NTL + t - m - 2], a1[r]);
          }
        }
        if (s <= smax) {
          const int m = s - j - 1;
          const double2 f0 = F[m];
#pragma unroll
          for (int r = 0; r < NRT; ++r) {
            const int t = lane + 32 * r;
            if (t < NTL && t >= m + 1) a0[r] = cfma(f0, Q[s * NTL + t - m - 1], a0[r]);
          }
        }
#pragma unroll
        for (int r = 0; r < NRT; ++r) {
          const int t = lane + 32 * r;
          if (t < NTL) fpn[jj * NTL + t] = cadd(a0[r], a1[r]);
        }
      }
    }
    team_sync<NW, TEAMS>(team);
  }
}

// Level-by-level trailing La Budde in ONE warp, no barriers (E <= 64; lane l owns rows l and
// l + 32).  The recursion q_j[t] = q_{j+1}[t] + u_j[t] with
//   u_j[t] = - h_jj q_{j+1}[t-1] - sum_{m=1}^{min(t-1, E-1-j)} F_j[m] q_{j+m+1}[t-m-1]
// involves, besides q_{j+1}[t], only coefficients t' < t: so level t (all rows at once) is a
// parallel evaluation of u_j[t] followed by a suffix sum over j (q_E[t] = 0 for t >= 1):
//   q_j[t] = sum_{i >= j} u_i[t]      (the same terms as the row-by-row recursion, summed as
// a tree).  NTL - 1 sequential levels instead of E sequential rows, each level's work spread
// over the warp.  hb: band with row stride BS (hb[j*BS + 1 + m] = F_j[m], hb[j*BS + 1] = h_jj);
// Q: [E + 1][BS] output (Q[j*BS + t] = coefficient t of q_j).  BS = NTL + 1 (odd multiple of 16
// bytes: the lanes' row-strided reads fall in distinct banks).
__device__ __forceinline__ void labudde_levels(const double2 *hb, double2 *Q, int E, int NTL,
                                               int BS, int lane) {
  const int i0 = lane, i1 = lane + 32;
  const bool r0 = i0 < E, r1 = i1 < E;
  // branch-free: out-of-range rows and sources read a clamped in-range address with the
  // coefficient F forced to 0 (no divergent loads in the m-loop)
  const int c0r = min(i0, E), c1r = min(i1, E);
  const int mx0 = r0 ? E - 1 - i0 : 0, mx1 = r1 ? E - 1 - i1 : 0;  // largest valid m per row
  const double2 *F0 = hb + c0r * BS + 1, *F1 = hb + c1r * BS + 1;
  if (i0 <= E) Q[i0 * BS] = c1();  // monic: coefficient 0 of every q_j is 1
  if (i1 <= E) Q[i1 * BS] = c1();
  __syncwarp();
  const double2 h0 = r0 ? F0[0] : c0(), h1 = r1 ? F1[0] : c0();
  for (int t = 1; t < NTL; ++t) {
    // u_j[t] for my rows: - h_jj q_{j+1}[t-1] - sum_m F_j[m] q_{j+m+1}[t-m-1]
    double2 a0 = c0(), b0 = c0(), a1 = c0(), b1 = c0();
    {
      const double2 qa = Q[min(i0 + 1, E) * BS + t - 1], qb = Q[min(i1 + 1, E) * BS + t - 1];
      a0 = cfms(h0, qa, a0);  // (q_{j+1}[t-1] = 0 above its degree: stored zeros)
      a1 = cfms(h1, qb, a1);
    }
    int m = 1;
    for (; m + 1 <= t - 1; m += 2) {
      const double2 f0a = m <= mx0 ? F0[m] : c0(), f0b = m + 1 <= mx0 ? F0[m + 1] : c0();
      const double2 f1a = m <= mx1 ? F1[m] : c0(), f1b = m + 1 <= mx1 ? F1[m + 1] : c0();
      const double2 q0a = Q[min(i0 + m + 1, E) * BS + t - m - 1], q0b = Q[min(i0 + m + 2, E) * BS + t - m - 2];
      const double2 q1a = Q[min(i1 + m + 1, E) * BS + t - m - 1], q1b = Q[min(i1 + m + 2, E) * BS + t - m - 2];
      a0 = cfms(f0a, q0a, a0);
      b0 = cfms(f0b, q0b, b0);
      a1 = cfms(f1a, q1a, a1);
      b1 = cfms(f1b, q1b, b1);
    }
    if (m <= t - 1) {
      const double2 f0a = m <= mx0 ? F0[m] : c0(), f1a = m <= mx1 ? F1[m] : c0();
      a0 = cfms(f0a, Q[min(i0 + m + 1, E) * BS + t - m - 1], a0);
      a1 = cfms(f1a, Q[min(i1 + m + 1, E) * BS + t - m - 1], a1);
    }
    double2 v0 = cadd(a0, b0), v1 = cadd(a1, b1);
    // suffix sums over rows: first the high half (rows 32 + l), then the low half plus the
    // high half's total
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const double2 x1 = shfl2_down(v1, off), x0 = shfl2_down(v0, off);
      if (lane + off < 32) { v1 = cadd(v1, x1); v0 = cadd(v0, x0); }
    }
    v0 = cadd(v0, shfl2(v1, 0));
    // store (explicit zeros above the degree E - j, and for the row q_E = 1)
    if (i0 <= E) Q[i0 * BS + t] = (i0 < E && t <= E - i0) ? v0 : c0();
    if (i1 <= E) Q[i1 * BS + t] = (i1 < E && t <= E - i1) ? v1 : c0();
    __syncwarp();
  }
}

// The same level-by-level La Budde over a team of NW warps (NW * 16 >= E rows; two lanes per
// row split the m-sum by the parity of m; one team barrier per level).  Per level t:
//   (a) each warp finalises its rows' level t-1: Q[i][t-1] = L[i] + C_w, where L is the
//       warp-local suffix sum of level t-1 and C_w the totals of the warps holding higher rows;
//   (b) u_i[t] for its rows -- the h-term reads the freshest level through L + C directly, the
//       m-terms read finalised levels <= t-2 -- then the warp-local suffix sum of u over its 16
//       rows into L (ring [2][64]) and the warp total into tot [2][NW];
//   (c) team barrier.
// After the last level the rows are finalised once more (and synchronised) for the series.
// Q: [E + 1][BS]; L: [2][64]; tot: [2][NW]; hb, BS as labudde_levels.
// QS: row stride of Q (default BS).  zmask: bit i set if H[i][i-1] = 0 (gamma-batched evaluation
// keeps the true H: the terms of F_j[m] crossing a zero subdiagonal are dropped here instead of
// being zeroed in the band).
template <int NW, int TEAMS, int NTLMAX>
__device__ __forceinline__ void labudde_levels_team(const double2 *hb, double2 *Q, double2 *L,
                                                    double2 *tot, int E, int NTL, int BS,
                                                    int warp, int lane, int team, int QS = 0,
                                                    uint64_t zmask = 0) {
  if (QS == 0) QS = BS;
  constexpr int MT = NTLMAX / 2;  // m-terms per lane at most (m <= NTL - 2, half of them)
  const int i = warp * 16 + (lane >> 1), h = lane & 1;
  const bool ri = i < E;
  const int ci = min(i, E);
  const int mx = ri ? E - 1 - i : 0;  // largest valid m of row i
  const double2 *F = hb + ci * BS + 1;
  const double2 hii = (ri && h == 0) ? F[0] : c0();
  if (h == 0 && i <= E) Q[i * QS] = c1();  // monic
  if (warp == 0 && lane == 0 && E >= NW * 16) Q[E * QS] = c1();
  team_sync<NW, TEAMS>(team);
  for (int t = 1; t < NTL; ++t) {
    const int pb = (t - 1) & 1, cb = t & 1;
    // (a) finalise level t-1 of my rows (levels >= 1), and the correction of each warp
    double2 Cw = c0();
    if (t - 1 >= 1) {
#pragma unroll
      for (int w = NW - 1; w > 0; --w)
        if (w > warp) Cw = cadd(Cw, tot[pb * NW + w]);
      if (h == 0 && i <= E) Q[i * QS + t - 1] = (i < E && t - 1 <= E - i) ? cadd(L[pb * 64 + i], Cw) : c0();
    }
    // (b) u_i[t]: the h-term from level t-1 (fresh: L + correction of the row's warp)
    double2 a = c0(), b = c0();
    if (h == 0) {
      const int s = i + 1;
      double2 q;
      if (t - 1 == 0) q = (s <= E) ? c1() : c0();
      else if (s >= E || s >= NW * 16) q = c0();  // q_E[t-1] = 0 for t-1 >= 1
      else {
        double2 Cs = c0();
        const int ws = s >> 4;
#pragma unroll
        for (int w = NW - 1; w > 0; --w)
          if (w > ws) Cs = cadd(Cs, tot[pb * NW + w]);
        q = cadd(L[pb * 64 + s], Cs);
      }
      a = cfms(hii, q, a);
    }
    // m-terms (m = 1 + h, 3 + h, ...) from finalised levels t - m - 1 <= t - 2: unrolled to the
    // compile-time bound MT with the coefficient masked to 0 past t - 1 or the row's end (all
    // loads issued up front; four independent accumulators)
    double2 c = c0(), d = c0();
#pragma unroll
    for (int x = 0; x < MT; ++x) {
      const int m = 1 + h + 2 * x;
      if (2 * x + 1 > NTLMAX - 2) break;
      const bool ok = m <= t - 1 && m <= mx && ((zmask >> (i + 1)) & ((1ull << m) - 1ull)) == 0;
      const double2 f = ok ? F[m] : c0();
      const double2 q = Q[min(i + m + 1, E) * QS + max(t - m - 1, 0)];
      if (x % 4 == 0) a = cfms(f, q, a);
      else if (x % 4 == 1) b = cfms(f, q, b);
      else if (x % 4 == 2) c = cfms(f, q, c);
      else d = cfms(f, q, d);
    }
    double2 u = cadd(cadd(a, b), cadd(c, d));
    u = cadd(u, shfl2_xor(u, 1));  // the row's two halves
    if (!ri) u = c0();
    // warp-local suffix sum over the 16 rows (lanes 2r; the odd lanes carry the same values)
#pragma unroll
    for (int off = 2; off < 32; off <<= 1) {
      const double2 x = shfl2_down(u, off);
      if (lane + off < 32) u = cadd(u, x);
    }
    if (h == 0 && i < 64) L[cb * 64 + i] = u;
    if (lane == 0) tot[cb * NW + warp] = u;
    team_sync<NW, TEAMS>(team);
  }
  // finalise the last level
  {
    const int t = NTL, pb = (t - 1) & 1;
    if (t - 1 >= 1) {
      double2 Cw = c0();
#pragma unroll
      for (int w = NW - 1; w > 0; --w)
        if (w > warp) Cw = cadd(Cw, tot[pb * NW + w]);
      if (h == 0 && i <= E) Q[i * QS + t - 1] = (i < E && t - 1 <= E - i) ? cadd(L[pb * 64 + i], Cw) : c0();
    }
    if (warp == 0 && lane == 0 && E >= NW * 16) {
      for (int tt = 1; tt < NTL; ++tt) Q[E * QS + tt] = c0();
    }
  }
  team_sync<NW, TEAMS>(team);
}

static cudaError_t ensure_inv() {
  static bool ready = false;
  if (ready) return cudaSuccess;
  double h[256];
  h[0] = 0.0;
  for (int i = 1; i < 256; ++i) h[i] = 1.0 / (double)i;
  cudaError_t e = cudaMemcpyToSymbol(c_inv, h, sizeof h);
  if (e == cudaSuccess) ready = true;
  return e;
}

}  // namespace tail
}  // namespace lhaf
