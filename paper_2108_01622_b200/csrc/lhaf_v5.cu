// lhaf_v5.cu -- variant 5 of the sieve kernel (default for bordered sizes 33 <= E <= 64):
// the same per-term method as v3 (Gauss-transform Hessenberg reduction of the bordered matrix
// with partial pivoting, unit subdiagonal, truncated trailing La Budde, det^{-1/2} exp series;
// DESIGN.md section 2), with a different data layout for the reduction: a 2-D register tile.
// SURVEY 8(a) rows a4-a11; DESIGN.md section 3 "Kernel v5".
//
// One CTA = one team of NW warps evaluates one sieve term at a time.  Lane = (rg, cg) with
// rg = lane / 8 (row group) and cg = lane % 8 (column group); warp w holds the row slots
// rho = 8 w + 2 rg + i (i = 0, 1) and every lane holds column POSITIONS q = cg + 8 j
// (j < CJ) of its two rows: the matrix is a 2 x CJ tile of double2 registers per lane.  Rows
// never move (labels); live columns are compacted to fewer positions three times per term.
// Per column k (one team barrier):
//   - every lane of a row group holds the pivot-column entries colv of its two rows (bit-
//     identical across the 8 lanes): pivot key, REDUX-max per warp; the warp's best row is
//     published whole (its 8 lanes store CJ entries each -- coalesced, no serialized row
//     store), with its reciprocal; one lane per row writes the row's entry of the right-update
//     coefficient vector kb (indexed by column position);
//   - barrier; the team's pivot = max over the NW warp records;
//   - one fused pass over the 2 x CJ tile: left  a = A - m_i P_q,  right acc_i += a kb_q;
//   - xor-butterfly over the 8 column-group lanes (3 levels): every lane of the row group gets
//     the new pivot-column entries of its rows (= the next colv, scaled by the pivot: unit
//     subdiagonal), with no shared-memory round trip.
// Compared with v3 (a row in the registers of 2 lanes, 4 warps, 2 barriers per column, the
// pivot row stored by 2 lanes one slot at a time) the column protocol has one barrier, the
// row publication is one CJ-store burst from 8 lanes, and the right-update reduction is a
// 3-level shuffle instead of per-row dot products -- latency per column goes down and the
// team has 8 warps to hide it.
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include "lhaf_device.cuh"
#include "lhaf_tail.cuh"
#include "lhaf_dd.cuh"

namespace lhaf {
namespace v5 {
using namespace tail;

__device__ __forceinline__ int opaque(int x) {
  asm volatile("mov.b32 %0, %0;" : "+r"(x));
  return x;
}

struct Pattern {
  int H, n, E, o, NTL;
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
  return D;
}

// Shared memory of one team (double2 words):
//   hb    [E+2][NTL]                   band of H (unit subdiagonal), La Budde's q rows after it
//   u1    union { reduction: cand [2][NW][64] | kb [2][64] | rec [2][NW] | yv [2][NW][2]
//                            | cmp [NW][4][64]  (compaction, per warp: 8 lanes x up to 8 positions)
//                 tail:      series scratch 3 (n+2) | La Budde partials [2][NW][2][NTL] }
//   misc  wv (64 ints) | ww (64 doubles) | beta
template <int NW>
struct Shape {
  static constexpr int TS = 32 * NW;
  static constexpr int CAND = 0, KB = CAND + 2 * NW * 64, REC = KB + 2 * 64, YV = REC + 2 * NW,
                       CMP = YV + 4 * NW, RED_END = CMP + NW * 4 * 64;
  // band row stride BS = NTL + 1 (odd multiple of 16 B: conflict-free row-strided reads)
  // PREC (double-double tail): q rows, series scratch, level ring and totals twice (hi / lo)
  __host__ __device__ static int u1_words(int E, int NTL, int n, bool prec) {
    const int f = prec ? 2 : 1;
    const int lab = f * ((E + 1) * (NTL + 1) + 3 * (n + 2) + 128 + 2 * NW);
    return RED_END > lab ? RED_END : lab;
  }
  __host__ __device__ static int words(int E, int NTL, int n, bool prec) {
    return (E + 2) * (NTL + 1) + u1_words(E, NTL, n, prec) + 32 + 64 + 1;
  }
};

struct Mem {
  double2 *hb, *u1;
  int *wv;
  double *ww;
  double2 *beta;
};

template <int NW, bool PREC>
__device__ __forceinline__ Mem carve(double2 *b, int E, int NTL, int n) {
  Mem M;
  M.hb = b; b += (E + 2) * (NTL + 1);
  M.u1 = b; b += Shape<NW>::u1_words(E, NTL, n, PREC);
  M.wv = reinterpret_cast<int *>(b); b += 32;
  M.ww = reinterpret_cast<double *>(b); b += 64;
  M.beta = b;
  return M;
}

// Per-lane state of the reduction.  A row group's 8 lanes hold 4 tile rows; the row's
// bookkeeping lives in the two lanes cg = 2 i (real part) and 2 i + 1 (imaginary part) -- the
// lanes the reduce-scatter of the right update leaves the row's new pivot-column entry in --
// so each lane tracks ONE row ("my row", i_me = cg / 2) instead of all four.
struct St {
  int label;        // Hessenberg position label of my row
  int pos;          // column position of my row's own index (-1: column no longer live)
  double2 colv;     // my row's entry of the current pivot column (scaled: unit subdiagonal)
  double2 rs;       // my row's scale (1 / pivot if it was a pivot row)
  uint64_t live;    // indices with label > k (team-uniform)
  uint64_t livec;   // the live set at the last compaction (defines the positions)
  uint64_t inert;   // gamma-batched evaluation: the loop-vector rows / columns (never pivots)
  uint64_t zmask;   // bit k+1 set if H[k+1][k] = 0 (an exactly-zero pivot at step k)
  int Lc;           // popc(livec): positions >= Lc have no column
  int zl;           // 1 + the label after the latest zero subdiagonal (0: none)
  int buf;
};

// gamma-batched evaluation (FLAG_MG): the outputs of the reduction besides H
struct MgOut {
  double2 *Y, *Z;  // [G][YS]: y'_g = D^{-1} L y_g and z'_g = z_g L^{-1} D, indexed by label
  int YS;
  int base;        // E0: the first loop-vector index
  uint64_t zmask;  // (out) zero subdiagonals of H
};

__device__ __forceinline__ int nth_bit(uint64_t m, int q) {  // position of the q-th set bit
  const unsigned lo = (unsigned)m, hi = (unsigned)(m >> 32);
  const int c = __popc(lo);
  return q < c ? (int)__fns(lo, 0, q + 1) : 32 + (int)__fns(hi, 0, q - c + 1);
}

template <int CJ>
__device__ __forceinline__ double2 rd_j(const double2 (&a)[CJ], int j) {
  double2 v = c0();
#pragma unroll
  for (int x = 0; x < CJ; ++x)
    if (x == j) v = a[x];
  return v;
}

// my row's entry at column position q (the owner lane of q holds all 4 tile rows: one shuffle
// per tile row, keep mine)
template <int CJ, int CJF>
__device__ __forceinline__ double2 my_entry(const double2 (&A)[4][CJF], int q, int lane) {
  const int src = (lane & ~7) | (q & 7), me = (lane & 7) >> 1;
  double2 v = c0();
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const double2 x = shfl2(rd_j<CJF>(A[i], q >> 3), src);
    if (i == me) v = x;
  }
  return v;
}

__device__ __forceinline__ int row_of(int warp, int lane, int i) {
  return warp * 16 + (lane >> 3) * 4 + i;
}

// reduce-scatter over the 8 lanes of a row group: lane cg ends with the group sum of v[cg]
__device__ __forceinline__ double rs8(double (&v)[8], int cg) {
  const bool b2 = cg & 4, b1 = cg & 2, b0 = cg & 1;
  double w[4], u[2];
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const double send = b2 ? v[t] : v[t + 4];
    const double keep = b2 ? v[t + 4] : v[t];
    w[t] = keep + __shfl_xor_sync(LHAF_FULL, send, 4);
  }
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    const double send = b1 ? w[t] : w[t + 2];
    const double keep = b1 ? w[t + 2] : w[t];
    u[t] = keep + __shfl_xor_sync(LHAF_FULL, send, 2);
  }
  const double send = b0 ? u[0] : u[1];
  const double keep = b0 ? u[1] : u[0];
  return keep + __shfl_xor_sync(LHAF_FULL, send, 1);
}

// Steps k in [k0, k1) of the reduction with CJ positions per lane (the tile prefix).
template <int NW, int CJ, int CJF>
__device__ __forceinline__ void steps(double2 (&A)[4][CJF], St &st, int k0, int k1, int E,
                                      int NTL, int BS, const Mem &M, int warp, int lane,
                                      const MgOut *mg = nullptr) {
  using Sh = Shape<NW>;
  const int cg = lane & 7, me = cg >> 1, im = cg & 1;
  const int rho0 = row_of(warp, lane, 0), rho = rho0 + me;
  const int tid = warp * 32 + lane;
  double2 *hb = M.hb;
  for (int k = k0; k < k1; ++k) {
    const int b = st.buf;
    st.buf ^= 1;
    double2 *cand = M.u1 + Sh::CAND + b * NW * 64;
    double2 *kb = M.u1 + Sh::KB + b * 64;
    int4 *rec = reinterpret_cast<int4 *>(M.u1 + Sh::REC) + b * NW;
    double2 *yv = M.u1 + Sh::YV + b * NW * 2;
    const bool cd = st.label > k && st.label < E;
    const unsigned key = cd ? pivot_key(st.colv, st.label) : 0u;
    const unsigned wkey = __reduce_max_sync(LHAF_FULL, key);
    // right-update coefficients by column position (one lane per row; ownerless positions 0)
    if (!im && st.pos >= 0) kb[st.pos] = cd ? st.colv : c0();
    if (tid >= st.Lc && tid < 8 * CJ) kb[tid] = c0();
    // this warp's best row: published whole by its row group (warp-uniform choice of the
    // tile row: one burst of CJ stores from 8 lanes), plus the warp record
    const unsigned win = __ballot_sync(LHAF_FULL, key == wkey && wkey != 0u);
    if (win) {
      const int lw = __ffs(win) - 1, ib = (lw & 7) >> 1;
      if ((lane >> 3) == (lw >> 3)) {
        double2 *dst = cand + warp * 64 + cg;
        switch (ib) {
#define LHAF_V5_PUB(I)                                 \
  case I:                                              \
    _Pragma("unroll") for (int j = 0; j < CJ; ++j)     \
      dst[8 * j] = A[I][j];                            \
    break;
          LHAF_V5_PUB(0) LHAF_V5_PUB(1) LHAF_V5_PUB(2) LHAF_V5_PUB(3)
#undef LHAF_V5_PUB
          default: break;
        }
      }
      if (lane == lw) {
        rec[warp] = make_int4((int)wkey, rho, st.pos, 0);
        yv[2 * warp] = st.colv;
        yv[2 * warp + 1] = crecip(st.colv);
      }
    } else if (lane == 0) {
      rec[warp] = make_int4(0, 0, 0, 0);
    }
    __syncthreads();

    unsigned bkey = 0u;
    int wb = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      const unsigned kw = (unsigned)rec[w].x;
      if (kw > bkey) { bkey = kw; wb = w; }
    }
    const int4 rw = rec[wb];
    const int p = rw.y, qp = rw.z;
    const int plabel = 63 - (int)(bkey & 63u);
    const bool elim = (bkey >> 6) > 1u;
    const double2 ip = yv[2 * wb + 1];
    const int nl = (rho == p) ? k + 1 : (st.label == k + 1 ? plabel : st.label);
    // finished column k: H[label][k] for rows with label <= k + 1 (band of width NTL)
    if (!im && nl <= k + 1 && k + 1 - nl < NTL)
      hb[nl * BS + k + 1 - nl] = (nl < st.zl && !mg) ? c0() : cmul(st.rs, st.colv);
    st.live &= ~(1ull << p);
    const double2 mm = (elim && cd && rho != p) ? cmul(st.colv, ip) : c0();
    double2 m[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) m[i] = shfl2(mm, (lane & ~7) | (2 * i));
    // fused left + right pass over the tile (m = 0 leaves A unchanged: one code path)
    const double2 *pr = cand + wb * 64 + cg;
    const double2 *kq = kb + cg;
    double xr[4], xi[4], yr[4], yi[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) xr[i] = xi[i] = yr[i] = yi[i] = 0.0;
#pragma unroll
    for (int j = 0; j < CJ; ++j) {
      const double2 P = pr[8 * j];
      const double2 K = kq[8 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const double2 a = cfms(m[i], P, A[i][j]);
        A[i][j] = a;
        xr[i] = fma(a.x, K.x, xr[i]); xi[i] = fma(a.y, K.y, xi[i]);
        yr[i] = fma(a.x, K.y, yr[i]); yi[i] = fma(a.y, K.x, yi[i]);
      }
    }
    double v[8];
#pragma unroll
    for (int i = 0; i < 4; ++i) { v[2 * i] = xr[i] - xi[i]; v[2 * i + 1] = yr[i] + yi[i]; }
    const double mine = rs8(v, cg);  // component `im` of my row's new pivot-column entry
    const double other = __shfl_xor_sync(LHAF_FULL, mine, 1);
    if (elim) {
      st.colv = im ? make_double2(other, mine) : make_double2(mine, other);  // unit subdiagonal
      if (rho == p) st.rs = ip;
    } else {
      st.colv = my_entry<CJ, CJF>(A, qp, lane);  // nothing to eliminate: column p as it stands
      st.zl = k + 1;                             // H[k+1][k] = 0
      st.zmask |= 1ull << (k + 1);
    }
    st.label = nl;
    if (mg && !im && rho < 64 && ((st.inert >> rho) & 1ull))  // z' entry of the column labelled k+1
      mg->Z[(rho - mg->base) * mg->YS + k + 1] = st.colv;
  }
}

// Warp-local compaction of the live columns from CJA to CJB positions per lane: the columns
// of st.live move to positions 0 .. L-1 (ascending index), through this warp's slice of the
// compaction buffer, one tile row at a time.  The narrower tile is the register prefix.
template <int CJA, int CJB, int CJF>
__device__ __forceinline__ void compact(double2 (&A)[4][CJF], St &st, double2 *wbuf, int warp,
                                        int lane) {
  const int rg = lane >> 3, cg = lane & 7;
  const uint64_t lv = st.live | st.inert;  // the loop-vector columns keep their positions
  const int L = __popcll(lv);
  int np[CJA];
#pragma unroll
  for (int j = 0; j < CJA; ++j) {
    const int q = cg + 8 * j;
    const int idx = q < st.Lc ? nth_bit(st.livec, q) : -1;
    np[j] = (idx >= 0 && ((lv >> idx) & 1ull)) ? __popcll(lv & ((1ull << idx) - 1ull)) : -1;
  }
  double2 *row = wbuf + rg * (8 * CJB);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
#pragma unroll
    for (int j = 0; j < CJA; ++j)
      if (np[j] >= 0) row[np[j]] = A[i][j];
    __syncwarp();
#pragma unroll
    for (int j = 0; j < CJB; ++j) {
      const int q = cg + 8 * j;
      A[i][j] = q < L ? row[q] : c0();
    }
    __syncwarp();
  }
  const int r = row_of(warp, lane, cg >> 1);
  st.pos = ((lv >> r) & 1ull) ? __popcll(lv & ((1ull << r) - 1ull)) : -1;
  st.livec = lv;
  st.Lc = L;
}


// a4-a6 of one term: decode, build, phased Hessenberg reduction into the band M.hb.
// Widths (positions per lane) C0 > C1 > C2 > C3; a phase switches when the live columns fit.
// Zero-weight deletion: an index c whose column weight is 0 (w_h = 0: eta_h = 2 k_h in the sieve,
// an excluded pair in inclusion/exclusion) has the column e_c in I - lam B, so det(I - lam B) is
// the minor without row and column c (and the loop row z vanishes there too): such indices are
// removed before the reduction -- the term is reduced at its own size E' (the paper's "z_i = 0
// deletion").  Returns (E', NTL') of the term.
template <int NW, int C0, int C1, int C2, int C3, bool MG = false>
__device__ __forceinline__ int2 team_reduce(const PatDesc &P, const Pattern &D, const JobDev &J,
                                            uint64_t t, const Mem &M, int warp, int lane,
                                            int &sign, double &weight, MgOut *mg = nullptr) {
  using Sh = Shape<NW>;
  const int H = D.H, E0 = D.E, o = D.o;
  // MG: the band is the full H (row stride HS = E0 + 1) read through hb = Hf - 1 with BS = HS + 1
  // (hb[j BS + 1 + m] = Hf[j HS + j + m] = H[j][j+m]), so every entry is written
  const int BS = MG ? E0 + 2 : D.NTL + 1;
  const int G = MG ? P.eta_b : 0;
  const int cg = lane & 7, im = cg & 1;
  const int rho0 = row_of(warp, lane, 0), rho = rho0 + (cg >> 1);
  // ---- a4: decode; ww[c] = weight of column c of B (1 for the border column)
  if (warp == 0) {
    sign = decode_term(P, J, t, lane, M.wv, weight);
    __syncwarp();
    for (int c = lane; c < 64; c += 32) {
      const int j = c - o;
      M.ww[c] = (c >= E0) ? 0.0 : (j < 0) ? 1.0 : (double)M.wv[j < H ? j : j - H];
    }
  }
  __syncthreads();
  // kept indices (nonzero weight) and the term's own size
  const uint64_t keep = ((uint64_t)__ballot_sync(LHAF_FULL, M.ww[lane + 32] != 0.0) << 32) |
                        (uint64_t)__ballot_sync(LHAF_FULL, M.ww[lane] != 0.0);
  const int E = __popcll(keep);
  const int NTL = MG ? 64 : min(D.n + 1 + o, E + 1);  // MG: band condition always true
  const int r0 = keep ? __ffsll((long long)keep) - 1 : 0;  // label 0: the first pivot column
  // ---- a5: tile of B = B0 diag(ww); position q = column q initially
  const double2 *B0 = J.cpool + P.mat_off;
  double2 A[4][C0];
#pragma unroll
  for (int j = 0; j < C0; ++j) {
    const int c = cg + 8 * j;
    const bool cok = c < E0;
    const double w = cok ? M.ww[c] : 0.0;
#pragma unroll
    for (int i = 0; i < 4; ++i)
      A[i][j] = (cok && rho0 + i < E0) ? cscale(B0[(size_t)(rho0 + i) * E0 + c], w) : c0();
  }
  if constexpr (MG) {
    // loop vectors: y_g = v_g as column E0 + g, z_g = v_g X_w as row E0 + g (v_g[a] = gamma_g at
    // the index list entry a; the phantom's loop weight is 1)
    const int *rix = J.ipool + P.idx_off;
    const double2 *gam = J.gamma + P.gamma_off;
#pragma unroll
    for (int j = 0; j < C0; ++j) {
      const int c = cg + 8 * j;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int r = rho0 + i;
        if (r < E0 && c >= E0 && c < E0 + G) {
          const int ri = rix[r];
          A[i][j] = ri < 0 ? c1() : gam[(size_t)(c - E0) * J.kdim + ri];
        } else if (r >= E0 && r < E0 + G && c < E0) {
          const int pc = c < H ? c + H : c - H;
          const int ri = rix[pc];
          const double2 v = ri < 0 ? c1() : gam[(size_t)(r - E0) * J.kdim + ri];
          A[i][j] = cscale(v, M.ww[c]);
        }
      }
    }
  }
  St st;
  const bool kept = rho < 64 && ((keep >> rho) & 1ull);
  st.label = kept ? __popcll(keep & ((1ull << rho) - 1ull)) : 63;  // deleted rows: never pivots
  st.pos = rho < E0 ? rho : -1;
  const int r0c = (MG && rho >= E0) ? 0 : rho;  // (a loop-vector row reads its own tile below)
  st.colv = kept ? cscale(B0[(size_t)r0c * E0 + r0], M.ww[r0]) : c0();  // the first pivot column
  st.rs = c1();
  const int ET = E0 + G;
  const uint64_t all = ET >= 64 ? ~0ull : ((1ull << ET) - 1ull);
  st.inert = MG ? (all & ~(E0 >= 64 ? ~0ull : ((1ull << E0) - 1ull))) : 0ull;
  st.live = keep & ~(1ull << r0);
  st.livec = all;
  st.Lc = ET;
  st.zl = 0;
  st.zmask = 0;
  st.buf = 0;
  if constexpr (MG) {
    st.pos = rho < ET ? rho : -1;  // the loop-vector rows own (and zero) the kb entries of their columns
    // the first pivot column's entry: B[row][r0] (a loop-vector row: z_g[r0])
    const double2 e0 = my_entry<C0, C0>(A, r0, lane);
    st.colv = (kept || (rho >= E0 && rho < ET)) ? e0 : c0();
    if (!im && rho >= E0 && rho < ET) mg->Z[(rho - E0) * mg->YS] = st.colv;  // z'[label 0]
  }
  double2 *wbuf = M.u1 + Sh::CMP + warp * 4 * 64;
  if (E != E0) compact<C0, C0, C0>(A, st, wbuf, warp, lane);  // drop the deleted columns
  // ---- a6: phased reduction (the loop-vector columns occupy G positions throughout)
  const int kend = E >= 2 ? E - 2 : 0;
  const int k1 = min(kend, max(0, E - 1 + G - 8 * C1));
  const int k2 = max(k1, min(kend, max(0, E - 1 + G - 8 * C2)));
  const int k3 = max(k2, min(kend, max(0, E - 1 + G - 8 * C3)));
  const MgOut *mgp = MG ? mg : nullptr;
  steps<NW, C0, C0>(A, st, 0, k1, E, NTL, BS, M, warp, lane, mgp);
  compact<C0, C1, C0>(A, st, wbuf, warp, lane);
  steps<NW, C1, C0>(A, st, k1, k2, E, NTL, BS, M, warp, lane, mgp);
  compact<C1, C2, C0>(A, st, wbuf, warp, lane);
  steps<NW, C2, C0>(A, st, k2, k3, E, NTL, BS, M, warp, lane, mgp);
  compact<C2, C3, C0>(A, st, wbuf, warp, lane);
  steps<NW, C3, C0>(A, st, k3, kend, E, NTL, BS, M, warp, lane, mgp);
  // the last two columns: the carried one (label kend) and the last live index (label E-1)
  double2 *hb = M.hb;
  if (E >= 2) {
    const int pl = __ffsll((long long)st.live) - 1;
    const int pos = __popcll(st.livec & ((1ull << pl) - 1ull));
    const double2 cl = my_entry<C3, C0>(A, pos, lane);
    if (!im) {
      const int lb = st.label;
      if (lb < E && kend + 1 - lb < NTL) hb[lb * BS + kend + 1 - lb] = (lb < st.zl && !MG) ? c0() : cmul(st.rs, st.colv);
      if (rho == pl) *M.beta = st.colv;  // H[E-1][E-2], not yet scaled to 1
      if (lb < E && E - lb < NTL) hb[lb * BS + E - lb] = (lb < st.zl && !MG) ? c0() : cmul(st.rs, cl);
      if (MG && rho < 64 && ((st.inert >> rho) & 1ull)) mg->Z[(rho - E0) * mg->YS + E - 1] = cl;
    }
  } else if (E == 1 && !im && st.label == 0) {
    hb[1] = st.colv;  // H[0][0] (a 1 x 1 term: the first pivot column is its only entry)
  }
  if constexpr (MG) {
    // y'_g[label] = rs (L y_g)[row]: the loop-vector columns after all left updates
    if (E >= 1) {
      for (int gi = 0; gi < G; ++gi) {
        const int q = __popcll(st.livec & ((1ull << (E0 + gi)) - 1ull));
        const double2 y = my_entry<C3, C0>(A, q, lane);
        if (!im && st.label < E) mg->Y[gi * mg->YS + st.label] = cmul(st.rs, y);
      }
    }
  }
  __syncthreads();
  // the last subdiagonal: scale column E-1 by it (rows above E-1): the similarity diag(.., beta)
  const bool beta_zero = E >= 2 && M.beta->x == 0.0 && M.beta->y == 0.0;
  if (E >= 2 && !im && st.label < E - 1 && E - st.label < NTL && !(MG && beta_zero))
    hb[st.label * BS + E - st.label] = cmul(hb[st.label * BS + E - st.label], *M.beta);
  if constexpr (MG) {  // the same similarity on the loop vectors: y'[E-1] / beta, z'[E-1] * beta
    const double2 b = *M.beta;
    const bool zb = (b.x == 0.0 && b.y == 0.0);  // an exactly zero last subdiagonal: no scaling
    if (E >= 2 && threadIdx.x < G && !zb) {
      const int gi = threadIdx.x;
      mg->Y[gi * mg->YS + E - 1] = cmul(mg->Y[gi * mg->YS + E - 1], crecip(b));
      mg->Z[gi * mg->YS + E - 1] = cmul(mg->Z[gi * mg->YS + E - 1], b);
    }
    mg->zmask = st.zmask | ((E >= 2 && zb) ? (1ull << (E - 1)) : 0ull);
  }
  return make_int2(E, MG ? min(D.n + 1, E + 1) : NTL);
}

#ifdef LHAF_V5_TIMING  // diagnostic builds: cycles of thread 0 in the reduction and the tail
__device__ unsigned long long g_v5_phase[4];
#define V5_T0() const long long t0_ = clock64();
#define V5_T1() const long long t1_ = clock64();
#define V5_T2()                                                         \
  if (threadIdx.x == 0) {                                               \
    atomicAdd(&g_v5_phase[0], (unsigned long long)(t1_ - t0_));         \
    atomicAdd(&g_v5_phase[1], (unsigned long long)(clock64() - t1_));   \
    atomicAdd(&g_v5_phase[3], 0ull - (unsigned long long)t1_);          \
    atomicAdd(&g_v5_phase[2], 1ull);                                    \
  }
#else
#define V5_T0()
#define V5_T1()
#define V5_T2()
#endif

// a7-a9 of one term: level-by-level team La Budde on the band (q rows in the reduction's
// scratch, free by now), then the series in warp 0; PREC: both in double-double (lhaf_dd.cuh)
template <int NW, bool PREC>
__device__ __forceinline__ double2 team_tail(const Pattern &D, int2 en, const Mem &M, int warp,
                                             int lane) {
  const int n = D.n, E = en.x, NTL = en.y, BS = D.NTL + 1;
  double2 g = c0();
  if constexpr (!PREC) {
    double2 *Q = M.u1;
    double2 *Lr = Q + (E + 1) * BS + 3 * (n + 2);  // [2][64] level ring, then [2][NW] totals
    if (NTL <= 32) labudde_levels_team<NW, 1, 32>(M.hb, Q, Lr, Lr + 128, E, NTL, BS, warp, lane, 0);
    else labudde_levels_team<NW, 1, 65>(M.hb, Q, Lr, Lr + 128, E, NTL, BS, warp, lane, 0);
#ifdef LHAF_V5_TIMING
    if (threadIdx.x == 0) atomicAdd(&g_v5_phase[3], (unsigned long long)clock64());
#endif
    if (warp == 0) {
      const double2 *cB = Q;
      const double2 *cM = D.loops ? Q + BS : Q;
      double2 *scr = Q + (E + 1) * BS;
      if (n + 2 <= 32) g = series<1>(cM, cB, n, NTL, D.loops, scr, lane);
      else if (n + 2 <= 64) g = series<2>(cM, cB, n, NTL, D.loops, scr, lane);
      else g = series<5>(cM, cB, n, NTL, D.loops, scr, lane);
    }
  } else {
    const int QW = (E + 1) * BS;
    double2 *Qh = M.u1, *Ql = Qh + QW;
    double2 *scr = Ql + QW;                 // 6 (n + 2)
    double2 *Lh = scr + 6 * (n + 2), *Ll = Lh + 128, *Th = Ll + 128, *Tl = Th + 2 * NW;
    if (NTL <= 32) dd::labudde_levels_team<NW, 1, 32>(M.hb, Qh, Ql, Lh, Ll, Th, Tl, E, NTL, BS, warp, lane, 0);
    else dd::labudde_levels_team<NW, 1, 65>(M.hb, Qh, Ql, Lh, Ll, Th, Tl, E, NTL, BS, warp, lane, 0);
    if (warp == 0) {
      const int o = D.loops ? BS : 0;
      g = dd::series(Qh + o, Ql + o, Qh, Ql, n, NTL, D.loops, scr, lane);
    }
  }
  __syncthreads();  // shared memory is reused by the next term
  return g;
}

template <int NW, int C0, int C1, int C2, int C3, int MINB, bool PREC>
__global__ void __launch_bounds__(32 * NW, MINB)
sieve_v5(JobDev J, uint64_t ubeg, uint64_t uend, int team_words) {
  extern __shared__ double2 smem[];
  __shared__ unsigned long long s_unit;
  __shared__ double s_acc[6];  // the unit's double-double sums (thread 0; off the register file)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < team_words; i += 32 * NW) smem[i] = c0();
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) s_unit = ubeg + atomicAdd(J.counter, 1ull);
    __syncthreads();
    const uint64_t u = s_unit;
    if (u >= uend) break;
    const PatDesc P = J.descs[find_pattern(J, u)];
    const Pattern D = pattern_of(P);
    const Mem M = carve<NW, PREC>(smem, D.E, D.NTL, D.n);
    const uint64_t tb = (u - P.unit_begin) * P.chunk;
    const uint64_t te = min(tb + P.chunk, P.T_eval);
    if (threadIdx.x < 6) s_acc[threadIdx.x] = 0.0;
    for (uint64_t t = tb; t < te; ++t) {
      int sign = 1;
      double weight = 1.0;
      V5_T0()
      const int2 en = team_reduce<NW, C0, C1, C2, C3>(P, D, J, t, M, warp, lane, sign, weight);
      V5_T1()
      const double2 g = team_tail<NW, PREC>(D, en, M, warp, lane);
      V5_T2()
      if (threadIdx.x == 0) {
        const double sw = sign * weight;
        dd_add(s_acc[0], s_acc[1], sw * g.x);
        dd_add(s_acc[2], s_acc[3], sw * g.y);
        dd_add(s_acc[4], s_acc[5], weight * hypot(g.x, g.y));
      }
    }
    if (threadIdx.x == 0) {
      Partial q;
      q.re_hi = s_acc[0]; q.re_lo = s_acc[1]; q.im_hi = s_acc[2]; q.im_lo = s_acc[3];
      q.abs_hi = s_acc[4]; q.abs_lo = s_acc[5];
      q.pad0 = 0; q.pad1 = 0;
      J.partials[u] = q;
    }
  }
}

// g(t) (unweighted) of pattern 0 for a list of term indices; one CTA per index at a time.
template <int NW, int C0, int C1, int C2, int C3, int MINB, bool PREC>
__global__ void __launch_bounds__(32 * NW, MINB)
terms_v5(JobDev J, const uint64_t *ts, int nt, double2 *g_out, int team_words) {
  extern __shared__ double2 smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < team_words; i += 32 * NW) smem[i] = c0();
  __syncthreads();
  const PatDesc P = J.descs[0];
  const Pattern D = pattern_of(P);
  const Mem M = carve<NW, PREC>(smem, D.E, D.NTL, D.n);
  for (int i = blockIdx.x; i < nt; i += gridDim.x) {
    int sign;
    double weight;
    const int2 en = team_reduce<NW, C0, C1, C2, C3>(P, D, J, ts[i], M, warp, lane, sign, weight);
    const double2 g = team_tail<NW, PREC>(D, en, M, warp, lane);
    if (threadIdx.x == 0) g_out[i] = g;
  }
}

// ================================================================ gamma-batched evaluation
// (FLAG_MG; "only the diagonal entries ... change between
// sub-detectors ... this does not change the eigenvalue calculation").  Per term ONE reduction of
// the gamma-free M = C X_w (the loop vectors ride along as G inert columns y_g = v_g and G inert
// rows z_g = v_g X_w: never pivots, they receive the same left / right updates and end as
// y'_g = D^-1 L y_g, z'_g = z_g L^-1 D), ONE La Budde (c_M) and ONE c_M^{-1/2}; per loop vector
// only the loop terms s_j = z'_g^T H^{j-1} y'_g (Hessenberg matvecs on the full H) and the
// exp series.  Per-gamma cost O(n d^2) on top of one O(d^3) reduction, instead of G reductions.
struct MgMem {
  double2 *Y, *Z, *S, *Ku, *Qs, *Es, *gout;
};

template <int NW>
struct MgShape {
  // hb = full H (row stride HS = E0 + 1, at offset 1); u1 as Shape<NW> but with La Budde's q
  // rows at stride QS = n + 2; then Y, Z [G][E0], S [G][n+1], Ku [NW][64], Qs [n+2],
  // Es [NW][n+2], gout [G]
  __host__ __device__ static int u1_words(int E0, int n) {
    const int lab = (E0 + 1) * (n + 2) + 128 + 2 * NW;
    return Shape<NW>::RED_END > lab ? Shape<NW>::RED_END : lab;
  }
  __host__ __device__ static int words(int E0, int G, int n) {
    return 1 + E0 * (E0 + 1) + u1_words(E0, n) + 2 * G * E0 + G * (n + 1) + NW * 64 + (n + 2) +
           NW * (n + 2) + G + 32 + 64 + 1;
  }
};

template <int NW>
__device__ __forceinline__ Mem carve_mg(double2 *b, int E0, int G, int n, MgMem &X) {
  Mem M;
  M.hb = b; b += 1 + E0 * (E0 + 1);
  M.u1 = b; b += MgShape<NW>::u1_words(E0, n);
  X.Y = b; b += G * E0;
  X.Z = b; b += G * E0;
  X.S = b; b += G * (n + 1);
  X.Ku = b; b += NW * 64;
  X.Qs = b; b += n + 2;
  X.Es = b; b += NW * (n + 2);
  X.gout = b; b += G;
  M.wv = reinterpret_cast<int *>(b); b += 32;
  M.ww = reinterpret_cast<double *>(b); b += 64;
  M.beta = b;
  return M;
}

template <int NW>
__device__ __forceinline__ void team_tail_mg(const Pattern &D, int2 en, int E0, int G,
                                             uint64_t zmask, const Mem &M, const MgMem &X,
                                             int warp, int lane) {
  const int n = D.n, E = en.x, NTL = en.y, HS = E0 + 1, BS = E0 + 2, QS = n + 2;
  double2 *Q = M.u1;
  double2 *Lr = Q + (E0 + 1) * QS;
  if (NTL <= 32) labudde_levels_team<NW, 1, 32>(M.hb, Q, Lr, Lr + 128, E, NTL, BS, warp, lane, 0, QS, zmask);
  else labudde_levels_team<NW, 1, 65>(M.hb, Q, Lr, Lr + 128, E, NTL, BS, warp, lane, 0, QS, zmask);
  if (warp == 0) {  // c_M^{-1/2}, shared by every loop vector (c_M = q_0: no border here)
    if (n + 2 <= 32) qhalf_coeffs<1>(Q, n, NTL, X.Qs, lane);
    else qhalf_coeffs<2>(Q, n, NTL, X.Qs, lane);
  }
  const double2 *Hf = M.hb + 1;
  double2 *u = X.Ku + warp * 64;
  for (int g = warp; g < G; g += NW) {  // loop terms s_j = z'^T H^{j-1} y', j = 1..n
    const double2 *y = X.Y + g * E0, *z = X.Z + g * E0;
    const int i0 = lane, i1 = lane + 32;
    const double2 z0 = i0 < E ? z[i0] : c0(), z1 = i1 < E ? z[i1] : c0();
    double2 u0 = i0 < E ? y[i0] : c0(), u1v = i1 < E ? y[i1] : c0();
    for (int j = 1; j <= n; ++j) {
      const double2 sj = warp_sum2(cadd(cmul(z0, u0), cmul(z1, u1v)));
      if (lane == 0) X.S[g * (n + 1) + j] = sj;
      if (j == n) break;
      u[i0] = u0;
      u[i1] = u1v;
      __syncwarp();
      // (H u)_i = sub_i u_{i-1} + sum_{c >= i} H[i][c] u_c; unit subdiagonal except zero pivots
      double2 a0 = c0(), a1 = c0();
      if (i0 >= 1 && i0 < E && !((zmask >> i0) & 1ull)) a0 = u[i0 - 1];
      if (i1 < E && !((zmask >> i1) & 1ull)) a1 = u[i1 - 1];
      for (int c = 0; c < E; ++c) {
        const double2 uc = u[c];
        if (c >= i0 && i0 < E) a0 = cfma(Hf[i0 * HS + c], uc, a0);
        if (c >= i1 && i1 < E) a1 = cfma(Hf[i1 * HS + c], uc, a1);
      }
      __syncwarp();
      u0 = a0;
      u1v = a1;
    }
  }
  __syncthreads();  // Qs and every S written
  for (int g = warp; g < G; g += NW) {
    double2 gv;
    if (n + 2 <= 32) gv = exp_dot<1>(X.Qs, X.S + g * (n + 1), n, X.Es + warp * (n + 2), lane);
    else gv = exp_dot<2>(X.Qs, X.S + g * (n + 1), n, X.Es + warp * (n + 2), lane);
    if (lane == 0) X.gout[g] = gv;
  }
  __syncthreads();
}

template <int NW, int C0, int C1, int C2, int C3, int MINB>
__global__ void __launch_bounds__(32 * NW, MINB)
sieve_mg_v5(JobDev J, uint64_t ubeg, uint64_t uend, int team_words) {
  extern __shared__ double2 smem[];
  __shared__ unsigned long long s_unit;
  __shared__ double s_acc[LHAF_MAX_GAMMA][6];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < team_words; i += 32 * NW) smem[i] = c0();
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) s_unit = ubeg + atomicAdd(J.counter, 1ull);
    __syncthreads();
    const uint64_t u = s_unit;
    if (u >= uend) break;
    const PatDesc P = J.descs[find_pattern(J, u)];
    const Pattern D = pattern_of(P);
    const int G = P.eta_b, E0 = D.E;
    MgMem X;
    const Mem M = carve_mg<NW>(smem, E0, G, D.n, X);
    MgOut mg;
    mg.Y = X.Y; mg.Z = X.Z; mg.YS = E0; mg.base = E0; mg.zmask = 0;
    const uint64_t tb = (u - P.unit_begin) * P.chunk;
    const uint64_t te = min(tb + P.chunk, P.T_eval);
    if (threadIdx.x < G)
      for (int q = 0; q < 6; ++q) s_acc[threadIdx.x][q] = 0.0;
    for (uint64_t t = tb; t < te; ++t) {
      int sign = 1;
      double weight = 1.0;
      const int2 en = team_reduce<NW, C0, C1, C2, C3, true>(P, D, J, t, M, warp, lane, sign, weight, &mg);
      team_tail_mg<NW>(D, en, E0, G, mg.zmask, M, X, warp, lane);
      // (sign and weight live in warp 0, lanes hold the same values)
      const double sw = __shfl_sync(LHAF_FULL, sign * weight, 0), wt = __shfl_sync(LHAF_FULL, weight, 0);
      if (warp == 0 && lane < G) {
        const double2 gv = X.gout[lane];
        dd_add(s_acc[lane][0], s_acc[lane][1], sw * gv.x);
        dd_add(s_acc[lane][2], s_acc[lane][3], sw * gv.y);
        dd_add(s_acc[lane][4], s_acc[lane][5], wt * hypot(gv.x, gv.y));
      }
    }
    __syncthreads();
    if (threadIdx.x < G) {
      const int g = threadIdx.x;
      Partial q;
      q.re_hi = s_acc[g][0]; q.re_lo = s_acc[g][1]; q.im_hi = s_acc[g][2]; q.im_lo = s_acc[g][3];
      q.abs_hi = s_acc[g][4]; q.abs_lo = s_acc[g][5];
      q.pad0 = 0; q.pad1 = 0;
      J.partials[P.part_base + (uint64_t)g * P.units + (u - P.unit_begin)] = q;
    }
  }
}

template <int NW, int C0, int C1, int C2, int C3, int MINB>
struct Inst {
  static constexpr int EMAX = 16 * NW < 8 * C0 ? 16 * NW : 8 * C0;
  static constexpr int THREADS = 32 * NW;
  template <bool PREC>
  static cudaError_t sieve(const JobDev &job, int E, int NTL, int n, uint64_t ubeg, uint64_t uend,
                           int num_sms, cudaStream_t s) {
    const int tw = Shape<NW>::words(E, NTL, n, PREC);
    const size_t smem = (size_t)tw * sizeof(double2);
    auto *kern = sieve_v5<NW, C0, C1, C2, C3, MINB, PREC>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, THREADS, smem);
    if (e != cudaSuccess) return e;
    if (const char *c = getenv("LHAF_CTAS_PER_SM")) per_sm = std::min(per_sm, atoi(c));  // diagnostics
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    const uint64_t units = uend - ubeg;
    uint64_t grid = (uint64_t)num_sms * per_sm;
    if (grid > units) grid = units;
    e = cudaMemsetAsync(job.counter, 0, sizeof(unsigned long long), s);
    if (e != cudaSuccess) return e;
    ++lhaf::g_launches;
    kern<<<(unsigned)grid, THREADS, smem, s>>>(job, ubeg, uend, tw);
    return cudaGetLastError();
  }
  template <bool PREC>
  static cudaError_t terms(const JobDev &job, int E, int NTL, int n, const uint64_t *t, int nt,
                           double2 *g_out, cudaStream_t s) {
    const int tw = Shape<NW>::words(E, NTL, n, PREC);
    const size_t smem = (size_t)tw * sizeof(double2);
    auto *kern = terms_v5<NW, C0, C1, C2, C3, MINB, PREC>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int grid = nt < 1184 ? nt : 1184;
    ++lhaf::g_launches;
    kern<<<grid, THREADS, smem, s>>>(job, t, nt, g_out, tw);
    return cudaGetLastError();
  }
};

// <warps, positions per lane in the four phases, CTAs per SM>; 16 rows per warp
using I64 = Inst<4, 8, 6, 4, 2, 2>;  // 49 <= E <= 64 (cfg4: E = 61): 128 threads, 2 CTAs / SM
using I48 = Inst<3, 6, 4, 2, 1, 4>;  // 33 <= E <= 48 (cfg5: E = 48): 96 threads, 4 CTAs / SM
using I32 = Inst<2, 4, 3, 2, 1, 4>;  //       E <= 32 (precise mode; v3 is the fast path there)

}  // namespace v5

#ifdef LHAF_V5_TIMING
extern "C" int lhaf_debug_v5_phase(unsigned long long *out4) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out4, v5::g_v5_phase, 4 * sizeof(unsigned long long));
  unsigned long long z[4] = {0, 0, 0, 0};
  return (int)cudaMemcpyToSymbol(v5::g_v5_phase, z, sizeof z);
}
#endif

int v5_supported(int e_max) { return e_max >= 1 && e_max <= 64; }

cudaError_t launch_sieve_v5(const JobDev &job, int e_max, int ntl_max, int n_max, uint64_t ubeg,
                            uint64_t uend, int num_sms, cudaStream_t s, int prec) {
  if (uend <= ubeg) return cudaSuccess;
  cudaError_t e = v5::ensure_inv();
  if (e != cudaSuccess) return e;
#define LHAF_V5_CALL(I, CALL) \
  return prec ? v5::I::CALL<true> CALL##_ARGS : v5::I::CALL<false> CALL##_ARGS;
#define sieve_ARGS (job, e_max, ntl_max, n_max, ubeg, uend, num_sms, s)
  if (e_max <= v5::I32::EMAX) LHAF_V5_CALL(I32, sieve)
  if (e_max <= v5::I48::EMAX) LHAF_V5_CALL(I48, sieve)
  if (e_max <= v5::I64::EMAX) LHAF_V5_CALL(I64, sieve)
#undef sieve_ARGS
  return cudaErrorInvalidValue;
}

cudaError_t launch_sieve_mg_v5(const JobDev &job, int e_max, int g_max, int n_max, uint64_t ubeg,
                               uint64_t uend, int num_sms, cudaStream_t s) {
  if (uend <= ubeg) return cudaSuccess;
  cudaError_t e = v5::ensure_inv();
  if (e != cudaSuccess) return e;
  if (e_max + g_max > 64 || g_max > LHAF_MAX_GAMMA) return cudaErrorInvalidValue;
  constexpr int NW = 4;
  const int tw = v5::MgShape<NW>::words(e_max, g_max, n_max);
  const size_t smem = (size_t)tw * sizeof(double2);
  // (the G loop-vector columns keep their positions through every compaction: the narrowest
  // phase must still hold G + 1 columns, hence 3 positions per lane there, G <= 16)
  auto *kern = v5::sieve_mg_v5<NW, 8, 6, 4, 3, 2>;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * NW, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  uint64_t grid = (uint64_t)num_sms * per_sm;
  if (grid > uend - ubeg) grid = uend - ubeg;
  e = cudaMemsetAsync(job.counter, 0, sizeof(unsigned long long), s);
  if (e != cudaSuccess) return e;
  ++lhaf::g_launches;
  kern<<<(unsigned)grid, 32 * NW, smem, s>>>(job, ubeg, uend, tw);
  return cudaGetLastError();
}

cudaError_t launch_terms_v5(const JobDev &job, int e_max, int ntl_max, int n_max, const uint64_t *t,
                            int nt, double2 *g_out, cudaStream_t s, int prec) {
  if (nt <= 0) return cudaSuccess;
  cudaError_t e = v5::ensure_inv();
  if (e != cudaSuccess) return e;
#define terms_ARGS (job, e_max, ntl_max, n_max, t, nt, g_out, s)
  if (e_max <= v5::I32::EMAX) LHAF_V5_CALL(I32, terms)
  if (e_max <= v5::I48::EMAX) LHAF_V5_CALL(I48, terms)
  if (e_max <= v5::I64::EMAX) LHAF_V5_CALL(I64, terms)
#undef terms_ARGS
#undef LHAF_V5_CALL
  return cudaErrorInvalidValue;
}

}  // namespace lhaf
