// lhaf_v3.cu -- variant 3 of the sieve kernel (the default): register-resident rows,
// Gauss-transform Hessenberg reduction of the bordered matrix in four register phases of
// shrinking width, a team-parallel trailing La Budde on the band of H, and the power series.
// DESIGN.md "Kernel v3"; SURVEY 8(a) rows a4-a11.
//
// One "team" of 32*NW threads evaluates one sieve term at a time; a CTA holds TEAMS teams.
//   a4  decode t -> w_h = eta_h - 2 k_h, sign (-1)^{sum k}, weight prod C(eta_h, k_h)
//   a5  B = [[0, z^T], [y, M]] with M = C X_w, y = v, z^T = v X_w (loops present), else B = M.
//       Row r of B lives in the registers of S threads; slot s of thread (r, par) holds column
//       position S*s + par.
//   a6  Hessenberg reduction of B by Gauss transforms with partial pivoting, index 0 fixed
//       (so the first step maps y -> beta e1 and carries z^T -> z^T L^{-1}: the "bordered"
//       loop trick).  Rows and columns never move: index i gets its final Hessenberg position
//       as a label.  Per column k two team barriers (one for a one-warp team):
//         pivot = warp REDUX-max of a packed (|B[r][k]|_1, label) key; each warp's best row
//         writes a small record (and 1 / its pivot) before the first barrier, then the
//         team's pivot row alone stores its row to smem before the second; every row then
//         does, in ONE fused pass over its live slots,
//             left   A[r][c] -= m_r A[p][c]          (m_r = B[r][k] / piv, 0 if r is done)
//             right  acc     += A[r][c] B[c][k]      (B[c][k] = 0 unless c is remaining)
//         and the new pivot column p = acc (scaled by piv: unit subdiagonal) is carried in
//         registers.  At 3/4, 1/2 and 1/4 of the live columns the rows are compacted into
//         narrower register arrays (reduce_phased).  Finished columns go to the band hb.
//   a7  trailing La Budde on the top NTL = n+2 coefficients of q_j(x) = det(x I - H[j:, j:])
//       (c_B = q_0, c_M = q_1), the m-sums split across the team's warps (one barrier per j).
//   a8  loop terms: lam S(lam) = 1 - c_B / c_M, S = sum_j s_j lam^j, s_j = z^T M^{j-1} y.
//   a9  g = [lam^n] c_M^{-1/2} exp(S/2)   (the paper's f with X -> X_w, reading C4):
//       column-sweep series recursions in warp 0.
//   a10 term = (-1)^{sum k} prod C(eta_h, k_h) g, double-double accumulation per work unit.
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstdio>
#include "lhaf_device.cuh"
#include "lhaf_tail.cuh"

namespace lhaf {
namespace v3 {
using namespace tail;

// Phase timing (diagnostic builds only, -DLHAF_PHASE_TIMING): cycles of thread 0 of every
// team spent in decode/build, reduction, band -> F, La Budde, hand-off, end barrier.
// Step probes (diagnostic builds only, -DLHAF_STEP_PROBE): clock64 of each warp leader of
// block 0 at 7 points of every reduction step (the last term processed wins).
#ifdef LHAF_STEP_PROBE
__device__ long long g_probe[64][8][4];
#define LHAF_SP(i) \
  if (blockIdx.x == 0 && lane == 0 && warp < 4 && k < 64) g_probe[k][i][warp] = clock64();
#else
#define LHAF_SP(i)
#endif
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
// Switch-based (jump table) variants for the once-per-column compaction move.
#define LHAF_CASES32(X)                                                                      \
  X(0) X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8) X(9) X(10) X(11) X(12) X(13) X(14) X(15)      \
  X(16) X(17) X(18) X(19) X(20) X(21) X(22) X(23) X(24) X(25) X(26) X(27) X(28) X(29) X(30) \
  X(31)
template <int CS>
__device__ __forceinline__ double2 rd_sw(const double2 (&A)[CS], int s) {
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
__device__ __forceinline__ void wr_sw(double2 (&A)[CS], int s, double2 v) {
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
template <int S, int CS>
__device__ __forceinline__ double2 read_pos(const double2 (&A)[CS], int q, int lane) {
  double2 v = rd_sw<CS>(A, q / S);
  if constexpr (S > 1) v = shfl2(v, (lane & ~(S - 1)) | (q & (S - 1)));
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

// Shared memory of one team (double2 words), for a pattern with (E, NTL, n):
//   hb   [E][NTL]       band of H (unit subdiagonal): [j][1] = H[j][j], [j][1+m] = H[j][j+m]
//   u1   union { cand [2][NW][CC] | kb [2][RC] | keys [2][NW] | piv [2][NW] } (reduction)
//        union { Q [E+1][NTL] | Qs, Rs, Es [n+2] | part [2][NW][2][NTL] }      (La Budde, series)
//   w    64 ints, then 64 doubles of column weights
template <int S, int CS, int NW>
struct Shape {
  static constexpr int TS = 32 * NW, RC = TS / S, CC = S * CS;
  static constexpr int EMAX = RC < CC ? RC : CC;
  __host__ __device__ static int red_words() { return 2 * NW * CC + 2 * RC + 6 * NW; }
  // warps whose rows share the compaction buffer at a time: half the team where shared memory
  // limits the occupancy (NW = 3: the d = 48 instance, 4 CTAs/SM instead of 3), else all
  __host__ __device__ static constexpr int cmp_warps() { return NW == 3 ? 2 : NW; }
  __host__ __device__ static int u1_words(int E, int NTL, int n) {
    const int lab = 3 * (n + 2) + 4 * NW * NTL;  // series scratch + La Budde partials
    const int cmp = cmp_warps() * 32 * ((3 * CS + 3) / 4);  // compaction buffer
    int w = red_words() > lab ? red_words() : lab;
    return w > cmp ? w : cmp;
  }
  __host__ __device__ static int words(int E, int NTL, int n) {
    return (E + 2) * NTL + u1_words(E, NTL, n) + 32 + 32;  // band (+2 rows: La Budde's q)
  }
};

struct TeamMem {
  double2 *hb, *u1;
  int *wv;
  double *ww;
};

template <int S, int CS, int NW>
__device__ __forceinline__ TeamMem carve(double2 *b, int E, int NTL, int n) {
  using Sh = Shape<S, CS, NW>;
  TeamMem T;
  T.hb = b; b += (E + 2) * NTL;
  T.u1 = b; b += Sh::u1_words(E, NTL, n);
  T.wv = reinterpret_cast<int *>(b); b += 32;
  T.ww = reinterpret_cast<double *>(b);
  return T;
}

struct Pattern {  // per-pattern sizes (kept opaque to loop-invariant motion)
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

// ================================================================ phased reduction
// The Hessenberg reduction in four phases of shrinking register arrays.  Live columns (index
// label > k) occupy "positions" (slot S*s + par); at the start of phases 2..4 the live
// columns of every row are compacted (through shared memory, one row per S lanes) to the
// positions 0..L-1 (ascending index order), so later phases sweep CS2 = 3CS/4, CS3 = CS/2,
// CS4 = CS/4 slots instead of CS.  kb and the published pivot rows are indexed by position.
struct PhaseSt {
  int label, buf, mypos, zl;  // zl: 1 + the label after the latest zero subdiagonal (0: none)
  double2 rs;                 // row scale (see team_term)
  uint64_t live, livec;  // indices with label > k; the live set at the last compaction
  double2 colv;
};

template <int S, int CS, int CSP, int NW, int TEAMS>
__device__ __forceinline__ void phase_steps(double2 (&A)[CSP], PhaseSt &st, int k0, int k1, int E,
                                            int NTL, double2 *hb, double2 *u1, int tid, int team) {
  using Sh = Shape<S, CS, NW>;
  constexpr int RC = Sh::RC, CC = Sh::CC;
  const int lane = tid & 31, warp = tid >> 5, rr = tid / S, par = tid % S;
  double2 *cand = u1;                                             // [2][NW][CC]
  double2 *kbuf = cand + 2 * NW * CC;                             // [2][RC]
  unsigned *keys = reinterpret_cast<unsigned *>(kbuf + 2 * RC);   // [2][NW][4]
  for (int k = k0; k < k1; ++k) {
    double2 *cb = cand + st.buf * NW * CC;  // (one row used: the pivot row)
    double2 *kb = kbuf + st.buf * RC;
    unsigned *yk = keys + st.buf * NW * 4;
    double2 *yv = reinterpret_cast<double2 *>(keys + 2 * NW * 4) + st.buf * NW * 2;
    st.buf ^= 1;
    LHAF_SP(0)
    const bool candr = st.label > k && st.label < E;
    const unsigned key = candr ? pivot_key(st.colv, st.label) : 0u;
    const unsigned wkey = __reduce_max_sync(LHAF_FULL, key);
    LHAF_SP(1)
    if (par == 0 && st.mypos >= 0) kb[st.mypos] = candr ? st.colv : c0();
    if (candr && key == wkey) {  // this warp's best row: its pivot record (and 1 / pivot)
      if constexpr (NW == 1) {   // (one warp: it is the pivot row, publish at once)
        double2 *dst = cb + par;
#pragma unroll
        for (int s = 0; s < CSP; ++s) dst[S * s] = A[s];
      }
      if (par == 0) {
        yv[2 * warp] = st.colv;
        if constexpr (NW > 1) yv[2 * warp + 1] = crecip(st.colv);
        yk[4 * warp + 1] = (unsigned)rr;
        yk[4 * warp + 2] = (unsigned)st.mypos;
      }
    }
    if (lane == 0) yk[4 * warp] = wkey;
    LHAF_SP(2)
    team_sync<NW, TEAMS>(team);
    LHAF_SP(3)

    unsigned bkey = 0u;
    int wb = 0;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      const unsigned kw = yk[4 * w];
      if (kw > bkey) { bkey = kw; wb = w; }
    }
    const int plabel = 63 - (int)(bkey & 63u);
    const int p = (int)yk[4 * wb + 1];   // pivot: physical index
    const int qp = (int)yk[4 * wb + 2];  // and its column position
    if constexpr (NW > 1) {
      // only the team's pivot row publishes (one warp's stores instead of NW speculative rows
      // contending for the shared-memory pipe), then a second barrier
      if (rr == p && (bkey >> 6) > 1u) {
        double2 *dst = cb + par;
#pragma unroll
        for (int s = 0; s < CSP; ++s) dst[S * s] = A[s];
      }
      team_sync<NW, TEAMS>(team);
    }
    const int newlabel = (rr == p) ? k + 1 : (st.label == k + 1 ? plabel : st.label);
    if (par == 0 && newlabel <= k + 1 && k + 1 - newlabel < NTL)
      hb[newlabel * NTL + k + 1 - newlabel] = (newlabel < st.zl) ? c0() : cmul(st.rs, st.colv);
    st.live &= ~(1ull << p);
    // NW > 1: one code path for A (a zero pivot runs the pass with m = 0, which leaves A
    // unchanged) -- two paths that update A differently made the compiler re-shuffle every
    // slot register at the loop back-edge (~2 CS moves per column); measured +2 % at d = 60.
    // One-warp teams keep the branch (there the single path measured 20 % slower).
    const bool elim = (bkey >> 6) > 1u;
    if (NW > 1 || elim) {
      const double2 ip = (NW > 1) ? yv[2 * wb + 1] : crecip(yv[2 * wb]);
      const double2 m = (elim && candr && rr != p) ? cmul(st.colv, ip) : c0();
      LHAF_SP(4)
      const double2 *rp = cb + par;  // the pivot row (position-indexed; stale but finite if !elim)
      const double2 *kq = kb + par;
      double xr0 = 0, xi0 = 0, yr0 = 0, yi0 = 0, xr1 = 0, xi1 = 0, yr1 = 0, yi1 = 0;
#pragma unroll
      for (int s = 0; s < CSP; ++s) {
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
      LHAF_SP(5)
#pragma unroll
      for (int x = 1; x < S; x <<= 1) sum = cadd(sum, shfl2_xor(sum, x));
      if (elim) {
        st.colv = sum;  // column p scaled by the pivot: unit subdiagonal
        if (rr == p) st.rs = ip;
      }
    }
    if (!elim) {
      st.colv = read_col<S, CSP>(A, qp, lane);  // nothing to eliminate: column p as it stands
      st.zl = k + 1;                            // H[k+1][k] = 0
    }
    LHAF_SP(6)
    st.label = newlabel;
  }
}

// Compaction of every row's live columns from CSA to CSB slots (see above), in place: the
// narrower array is the prefix A[0 .. CSB) of the same registers, and the rows pass through
// the shared-memory buffer either all at once or, where shared memory limits the occupancy,
// in two halves of the team (Shape::cmp_warps).  ipos[q] = index of the column at position q (-1: none);
// npos = the new position of each old one.
template <int S, int CS, int CSA, int CSB, int NW, int TEAMS>
__device__ __forceinline__ void compact(double2 (&A)[CSA], PhaseSt &st, int *ipos, int *npos,
                                        double2 *u1, int tid, int team) {
  using Sh = Shape<S, CS, NW>;
  constexpr int TS = Sh::TS, RC = Sh::RC;
  constexpr int NB = S * CSB;
  constexpr int HW = Sh::cmp_warps(), HROWS = HW * 32 / S;
  constexpr int NHALF = (NW + HW - 1) / HW;  // 1 or 2 passes
  const int rr = tid / S, par = tid % S, warp = tid >> 5;
  const uint64_t live = st.live;
  const int L = __popcll(live);
  for (int q = tid; q < 64; q += TS) {
    const int i = ipos[q];
    npos[q] = (i >= 0 && ((live >> i) & 1ull)) ? __popcll(live & ((1ull << i) - 1ull)) : -1;
  }
  team_sync<NW, TEAMS>(team);  // npos visible; the last column's shared-memory reads are done
  const int h = warp >= HW ? 1 : 0;
  double2 *row = u1 + (size_t)(rr - h * HROWS) * NB;
#pragma unroll
  for (int half = 0; half < NHALF; ++half) {
    if (h == half) {
#pragma unroll
      for (int s = 0; s < CSA; ++s) {
        const int np = npos[S * s + par];
        if (np >= 0) row[np] = A[s];
      }
      __syncwarp();
#pragma unroll
      for (int s = 0; s < CSB; ++s) A[s] = (S * s + par < L) ? row[S * s + par] : c0();
    }
    team_sync<NW, TEAMS>(team);
  }
  // new position table, row ownership, and zero pivot-column slots without an owner (the next
  // column's barrier orders these writes before their readers)
  for (int i = tid; i < 64; i += TS) {
    if ((live >> i) & 1ull) ipos[__popcll(live & ((1ull << i) - 1ull))] = i;
    if (i >= L) ipos[i] = -1;
  }
  st.mypos = (rr < 64 && ((live >> rr) & 1ull)) ? __popcll(live & ((1ull << rr) - 1ull)) : -1;
  st.livec = live;
  double2 *kbuf = u1 + 2 * NW * Sh::CC;
  for (int q = L + tid; q < RC; q += TS) {
    kbuf[q] = c0();
    kbuf[RC + q] = c0();
  }
}

template <int S, int CS, int NW, int TEAMS>
__device__ __forceinline__ void reduce_phased(double2 (&A)[CS], int &label, double2 &colv, int E,
                                              int NTL, double2 *hb, double2 *u1, int *ipos,
                                              int *npos, double2 *betap, int tid, int team) {
  using Sh = Shape<S, CS, NW>;
  constexpr int TS = Sh::TS;
  constexpr int CS2 = (3 * CS + 3) / 4, CS3 = (CS + 1) / 2, CS4 = (CS + 3) / 4;
  const int lane = tid & 31, rr = tid / S, par = tid % S;
  PhaseSt st;
  st.label = label;
  st.colv = colv;
  st.buf = 0;
  st.mypos = rr;
  st.zl = 0;
  st.rs = c1();
  st.live = (E >= 64 ? ~0ull : ((1ull << E) - 1ull)) & ~1ull;
  st.livec = (E >= 64 ? ~0ull : ((1ull << E) - 1ull));
  for (int q = tid; q < 64; q += TS) ipos[q] = (q < E) ? q : -1;
  team_sync<NW, TEAMS>(team);
  const int kend = E >= 2 ? E - 2 : 0;
  const int k2 = min(kend, max(0, E - 1 - S * CS2));
  const int k3 = max(k2, min(kend, max(0, E - 1 - S * CS3)));
  const int k4 = max(k3, min(kend, max(0, E - 1 - S * CS4)));
  phase_steps<S, CS, CS, NW, TEAMS>(A, st, 0, k2, E, NTL, hb, u1, tid, team);
  compact<S, CS, CS, CS2, NW, TEAMS>(A, st, ipos, npos, u1, tid, team);
  double2 (&A2)[CS2] = *reinterpret_cast<double2 (*)[CS2]>(&A);  // prefix views of A
  phase_steps<S, CS, CS2, NW, TEAMS>(A2, st, k2, k3, E, NTL, hb, u1, tid, team);
  compact<S, CS, CS2, CS3, NW, TEAMS>(A2, st, ipos, npos, u1, tid, team);
  double2 (&A3)[CS3] = *reinterpret_cast<double2 (*)[CS3]>(&A);
  phase_steps<S, CS, CS3, NW, TEAMS>(A3, st, k3, k4, E, NTL, hb, u1, tid, team);
  compact<S, CS, CS3, CS4, NW, TEAMS>(A3, st, ipos, npos, u1, tid, team);
  double2 (&A4)[CS4] = *reinterpret_cast<double2 (*)[CS4]>(&A);
  phase_steps<S, CS, CS4, NW, TEAMS>(A4, st, k4, kend, E, NTL, hb, u1, tid, team);
  // the last two columns: the carried one (label kend) and the last live one
  const int lb = st.label;
  if (E >= 1) {
    if (par == 0 && lb < E && kend + 1 - lb < NTL)
      hb[lb * NTL + kend + 1 - lb] = (lb < st.zl) ? c0() : cmul(st.rs, st.colv);
    if (E >= 2) {
      const int pl = __ffsll((long long)st.live) - 1;  // label E-1
      if (rr == pl && par == 0) *betap = st.colv;     // H[E-1][E-2], not yet scaled to 1
      const int pos = __popcll(st.livec & ((1ull << pl) - 1ull));
      const double2 cl = read_col<S, CS4>(A4, pos, lane);
      if (par == 0 && lb < E && E - lb < NTL) hb[lb * NTL + E - lb] = (lb < st.zl) ? c0() : cmul(st.rs, cl);
    }
  }
  label = st.label;
  colv = st.colv;
}

// ================================================================ one term, one team
// a4-a6 of one term: decode, build, Hessenberg reduction into the band T.hb; sign and weight
// from the decode (warp 0).  Ends without a barrier after the last band writes.
// CMP: phased reduction (compaction of the live columns).
template <int S, int CS, int NW, int TEAMS, bool CMP>
__device__ __forceinline__ void team_reduce(const PatDesc &P, const Pattern &D, const JobDev &J,
                                            uint64_t t, const TeamMem &T, int tid, int team,
                                            int &sign, double &weight) {
  using Sh = Shape<S, CS, NW>;
  constexpr int RC = Sh::RC, CC = Sh::CC;
  const int lane = tid & 31, warp = tid >> 5;
  const int H = D.H, E = D.E, o = D.o, NTL = D.NTL;
  double2 *hb = T.hb;

#ifdef LHAF_PHASE_TIMING
  long long t_last_ = clock64();
#endif
  // ---- a4: decode; ww[c] = weight of column c of B (1 for the border column)
  if (warp == 0) {
    sign = decode_term(P, J, t, lane, T.wv, weight);
    __syncwarp();
    for (int c = lane; c < CC; c += 32) {
      const int j = c - o;
      T.ww[c] = (c >= E) ? 0.0 : (j < 0) ? 1.0 : (double)T.wv[j < H ? j : j - H];
    }
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

  // ---- a6: Gauss-transform Hessenberg reduction, one barrier per column.  Each step is
  // followed by the diagonal similarity that scales the new pivot column by the pivot and the
  // pivot row by its inverse, so H has a unit subdiagonal (0 after a zero pivot) and La Budde
  // needs no subdiagonal products.  The row scaling is not applied to the registers: a pivot
  // row keeps rs = 1/pivot and multiplies its band entries by it; after a zero pivot at step
  // k, band entries of rows above k+1 in later columns are 0 (zl).
  double2 *cand = T.u1;                                       // [2][NW][CC]
  double2 *kbuf = cand + 2 * NW * CC;                         // [2][RC]
  unsigned *keys = reinterpret_cast<unsigned *>(kbuf + 2 * RC);  // [2][NW][4] (key, phys)
  int label = rr;
  double2 colv = (S == 1) ? A[0] : shfl2(A[0], lane & ~(S - 1));    // this row's B[.][k]
  int buf = 0;
  const int kend = E >= 2 ? E - 2 : 0;
  double2 *betap = reinterpret_cast<double2 *>(T.ww) + 31;  // (past npos: 64 ints)
  if constexpr (CMP) {
    reduce_phased<S, CS, NW, TEAMS>(A, label, colv, E, NTL, hb, T.u1, T.wv,
                                    reinterpret_cast<int *>(T.ww), betap, tid, team);
  } else {
  uint64_t live = (E >= 64 ? ~0ull : ((1ull << E) - 1ull)) & ~1ull;  // indices with label > k
  int zl = 0;
  double2 rs = c1();
  for (int k = 0; k < kend; ++k) {
    double2 *cb = cand + buf * NW * CC;
    double2 *kb = kbuf + buf * RC;
    unsigned *yk = keys + buf * NW * 4;
    double2 *yv = reinterpret_cast<double2 *>(keys + 2 * NW * 4) + buf * NW * 2;  // pivot, 1/pivot
    buf ^= 1;
    const bool candr = label > k && label < E;
    // pivot key: |re| + |im| as a float (monotone bits), low 6 bits = 63 - label so that ties
    // go to the smallest label; non-candidates 0; one REDUX per warp
    const unsigned key = candr ? pivot_key(colv, label) : 0u;
    const unsigned wkey = __reduce_max_sync(LHAF_FULL, key);
    if (par == 0) kb[rr] = candr ? colv : c0();
    if (candr && key == wkey) {  // this warp's best row publishes itself (and 1 / its pivot)
      double2 *dst = cb + warp * CC + par;
#pragma unroll
      for (int s = 0; s < CS; ++s) dst[S * s] = A[s];
      if (par == 0) {
        yv[2 * warp] = colv;
        if constexpr (NW > 1) yv[2 * warp + 1] = crecip(colv);  // off the post-barrier path
        yk[4 * warp + 1] = (unsigned)rr;
      }
    }
    if (lane == 0) yk[4 * warp] = wkey;
    LHAF_PHASE(6)
    team_sync<NW, TEAMS>(team);
    LHAF_PHASE(7)

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
    if (par == 0 && newlabel <= k + 1 && k + 1 - newlabel < NTL)
      hb[newlabel * NTL + k + 1 - newlabel] = (newlabel < zl) ? c0() : cmul(rs, colv);
    live &= ~(1ull << p);
    if ((bkey >> 6) > 1u) {  // nonzero pivot
      const double2 ip = (NW > 1) ? yv[2 * wb + 1] : crecip(yv[2 * wb]);
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
      colv = sum;  // column p scaled by the pivot: unit subdiagonal
      if (rr == p) rs = ip;
    } else {
      colv = read_col<S, CS>(A, p, lane);  // nothing to eliminate: column p as it stands
      zl = k + 1;                          // H[k+1][k] = 0
    }
    label = newlabel;
    LHAF_PHASE(1)
  }
  // the last two columns: the carried one (label kend) and the remaining live index
  if (E >= 1) {
    if (par == 0 && label < E && kend + 1 - label < NTL)
      hb[label * NTL + kend + 1 - label] = (label < zl) ? c0() : cmul(rs, colv);
    if (E >= 2) {
      const int pl = __ffsll((long long)live) - 1;  // label E-1
      if (rr == pl && par == 0) *betap = colv;        // H[E-1][E-2], not yet scaled to 1
      const double2 cl = read_col<S, CS>(A, pl, lane);
      if (par == 0 && label < E && E - label < NTL) hb[label * NTL + E - label] = (label < zl) ? c0() : cmul(rs, cl);
    }
  }
  }
  team_sync<NW, TEAMS>(team);
  // the last subdiagonal: scale column E-1 by it (rows above E-1; La Budde's first barrier
  // orders these writes before its reads)
  if (E >= 2 && par == 0 && label < E - 1 && E - label < NTL)
    hb[label * NTL + E - label] = cmul(hb[label * NTL + E - label], *betap);
  LHAF_PHASE(1)
}

// a7: La Budde on the band T.hb into Q = T.u1 ([E+1][NTL], Q[j][t] = coefficient of
// x^{deg q_j - t}); the whole team takes part (its first barrier orders the band writes).
template <int NW, int TEAMS>
__device__ __forceinline__ void team_labudde(const Pattern &D, const TeamMem &T, int tid, int team) {
  const int lane = tid & 31, warp = tid >> 5;
  const int n = D.n, E = D.E, NTL = D.NTL;
  const double2 *hb = T.hb;
  // q_j is stored in band row j+1, which La Budde has consumed by then (rows E, E+1 extra)
  double2 *Q = T.hb + NTL;
  double2 *part = T.u1 + 3 * (n + 2);  // [2][NW][2][NTL]
  if constexpr (NW == 1) {
    if (NTL <= 32) labudde<1>(hb, Q, E, NTL, lane);
    else labudde<2>(hb, Q, E, NTL, lane);
  } else {
    // (two rows per barrier pays at NTL <= 32; one row per barrier above, measured)
    if (NTL <= 32) labudde_team2<1, NW, TEAMS>(hb, Q, part, E, NTL, warp, lane, team);
    else labudde_team<2, NW, TEAMS>(hb, Q, part, E, NTL, warp, lane, team);
  }
}

// a8/a9 in one warp: series from c_B = q_0, c_M = q_1 (loops) or c_M = q_0; returns
// g = [lam^n] and leaves Qs, Rs, Es (degrees 0..n) in the scratch after Q.
__device__ __forceinline__ double2 warp_series(const Pattern &D, const double2 *Q, double2 *scr,
                                               int lane) {
  const int n = D.n, E = D.E, NTL = D.NTL;
  const double2 *cB = Q;
  const double2 *cM = D.loops ? Q + NTL : Q;
  (void)E;
  if (n + 2 <= 32) return series<1>(cM, cB, n, NTL, D.loops, scr, lane);
  if (n + 2 <= 64) return series<2>(cM, cB, n, NTL, D.loops, scr, lane);
  return series<5>(cM, cB, n, NTL, D.loops, scr, lane);
}

// g(t) of one term (valid in warp 0 of the team); sign and weight from the decode (warp 0).
template <int S, int CS, int NW, int TEAMS, bool CMP>
__device__ double2 team_term(const PatDesc &P, const Pattern &D, const JobDev &J, uint64_t t,
                             const TeamMem &T, int tid, int team, int &sign, double &weight) {
  team_reduce<S, CS, NW, TEAMS, CMP>(P, D, J, t, T, tid, team, sign, weight);
#ifdef LHAF_PHASE_TIMING
  long long t_last_ = clock64();
#endif
  const int lane = tid & 31, warp = tid >> 5;
  team_labudde<NW, TEAMS>(D, T, tid, team);
  LHAF_PHASE(3)
  double2 g = c0();
  if (warp == 0) g = warp_series(D, T.hb + D.NTL, T.u1, lane);
  LHAF_PHASE(4)
  team_sync<NW, TEAMS>(team);  // smem reused by the next term
  LHAF_PHASE(5)
  return g;
}

// ================================================================ kernels
template <int S, int CS, int NW, int TEAMS, int REGS, bool CMP>
__global__ void __maxnreg__(REGS)
sieve_v3(JobDev J, uint64_t ubeg, uint64_t uend, int team_words) {
  extern __shared__ double2 smem[];
  __shared__ unsigned long long s_unit;
  __shared__ double s_acc[TEAMS][6];
  constexpr int TS = 32 * NW;
  const int team = threadIdx.x / TS, tid = threadIdx.x % TS;
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
    double rh = 0, rl = 0, ih = 0, il = 0, ah = 0, al = 0;
    for (uint64_t t = tb + team; t < te; t += TEAMS) {
      int sign = 1;
      double weight = 1.0;
      const double2 g = team_term<S, CS, NW, TEAMS, CMP>(P, D, J, t, T, tid, team, sign, weight);
      if (tid == 0) {
        const double sw = sign * weight;
        dd_add(rh, rl, sw * g.x);
        dd_add(ih, il, sw * g.y);
        dd_add(ah, al, weight * hypot(g.x, g.y));
      }
    }
    if (tid == 0) {
      s_acc[team][0] = rh; s_acc[team][1] = rl; s_acc[team][2] = ih;
      s_acc[team][3] = il; s_acc[team][4] = ah; s_acc[team][5] = al;
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

// Cutoff groups (App. B.5; FLAG_CUT patterns built by lhaf_rpt_cutoff): the
// last pair is the batched mode's self-pair with weight w_b = j - eta_b.  One reduction and
// one series to degree n = n_f + eta_b per (fixed-pair term, w_b) serve every count 2m
// (+ the group's parity) with m >= |w_b|, m = w_b (mod 2): lane m of warp 0 adds
// (-1)^{k_b} C(m, k_b) [lam^{n_f + m}] f, k_b = (m - w_b) / 2, to its own accumulator; the
// unit's partial of count m goes to partials[part_base + m * units + unit - unit_begin].
template <int S, int CS, int NW, int TEAMS, int REGS, bool CMP>
__global__ void __maxnreg__(REGS)
sieve_cut_v3(JobDev J, uint64_t ubeg, uint64_t uend, int team_words) {
  extern __shared__ double2 smem[];
  __shared__ unsigned long long s_unit;
  __shared__ double s_acc[TEAMS][32][6];
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
    const int eb = P.eta_b, nf = D.n - eb;
    double rh = 0, rl = 0, ih = 0, il = 0, ah = 0, al = 0;
    for (uint64_t t = tb + team; t < te; t += TEAMS) {
      int sign = 1;
      double weight = 1.0;
      team_reduce<S, CS, NW, TEAMS, CMP>(P, D, J, t, T, tid, team, sign, weight);
      team_labudde<NW, TEAMS>(D, T, tid, team);
      if (warp == 0) {
        warp_series(D, T.hb + D.NTL, T.u1, lane);
        __syncwarp();
        const double2 *Qs = T.u1, *Es = Qs + 2 * (D.n + 2);
        // the batched pair's weight, re-derived from t (T.wv is the reduction's position table)
        const uint64_t Rb = J.upool[P.radix_off + D.H - 1];
        const int wb = (int)((t / Rb) % (uint64_t)(2 * eb + 1)) - eb, m = lane;
        if (m <= eb && m >= abs(wb) && ((m - wb) & 1) == 0) {
          const int deg = nf + m;
          double2 g;
          if (D.loops) {
            g = c0();
            for (int i = 0; i <= deg; ++i) g = cfma(Qs[i], Es[deg - i], g);
          } else {
            g = Qs[deg];
          }
          const int kb = (m - wb) / 2;
          double cb = 1.0;  // C(m, kb), exact
          for (int i = 0; i < kb; ++i) cb = cb * (double)(m - i) / (double)(i + 1);
          const double sw = (double)sign * weight * ((kb & 1) ? -cb : cb);
          dd_add(rh, rl, sw * g.x);
          dd_add(ih, il, sw * g.y);
          dd_add(ah, al, weight * cb * hypot(g.x, g.y));
        }
      }
      team_sync<NW, TEAMS>(team);  // smem reused by the next term
    }
    if (warp == 0) {
      s_acc[team][lane][0] = rh; s_acc[team][lane][1] = rl; s_acc[team][lane][2] = ih;
      s_acc[team][lane][3] = il; s_acc[team][lane][4] = ah; s_acc[team][lane][5] = al;
    }
    __syncthreads();
    if (threadIdx.x <= eb) {
      const int m = threadIdx.x;
      double a0 = 0, a1 = 0, a2 = 0, a3 = 0, a4 = 0, a5 = 0;
      for (int w = 0; w < TEAMS; ++w) {
        dd_add_dd(a0, a1, s_acc[w][m][0], s_acc[w][m][1]);
        dd_add_dd(a2, a3, s_acc[w][m][2], s_acc[w][m][3]);
        dd_add_dd(a4, a5, s_acc[w][m][4], s_acc[w][m][5]);
      }
      Partial q;
      q.re_hi = a0; q.re_lo = a1; q.im_hi = a2; q.im_lo = a3; q.abs_hi = a4; q.abs_lo = a5;
      q.pad0 = 0; q.pad1 = 0;
      J.partials[P.part_base + (uint64_t)m * P.units + (u - P.unit_begin)] = q;
    }
  }
}

// g(t) (unweighted) of pattern 0 for a list of term indices; one team per index.
template <int S, int CS, int NW, int TEAMS, int REGS, bool CMP>
__global__ void __maxnreg__(REGS)
terms_v3(JobDev J, const uint64_t *ts, int nt, double2 *g_out, int team_words) {
  extern __shared__ double2 smem[];
  constexpr int TS = 32 * NW;
  const int team = threadIdx.x / TS, tid = threadIdx.x % TS;
  double2 *tbase = smem + (size_t)team * team_words;
  for (int i = tid; i < team_words; i += TS) tbase[i] = c0();
  __syncthreads();
  const PatDesc P = J.descs[0];
  const Pattern D = pattern_of(P);
  const TeamMem T = carve<S, CS, NW>(tbase, D.E, D.NTL, D.n);
  for (int base = blockIdx.x * TEAMS; base < nt; base += gridDim.x * TEAMS) {
    const int i = base + team;
    if (i < nt) {
      int sign;
      double weight;
      const double2 g = team_term<S, CS, NW, TEAMS, CMP>(P, D, J, ts[i], T, tid, team, sign, weight);
      if (tid == 0) g_out[i] = g;
    }
  }
}

// ================================================================ host side
template <int S, int CS, int NW, int TEAMS, int REGS, bool CMP = false>
struct Inst {
  using Sh = Shape<S, CS, NW>;
  static constexpr int EMAX = Sh::EMAX;
  static constexpr int THREADS = 32 * NW * TEAMS;
  static cudaError_t sieve(const JobDev &job, int E, int NTL, int n, uint64_t ubeg, uint64_t uend,
                           int num_sms, cudaStream_t s) {
    const int tw = Sh::words(E, NTL, n);
    const size_t smem = (size_t)tw * TEAMS * sizeof(double2);
    auto *kern = sieve_v3<S, CS, NW, TEAMS, REGS, CMP>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
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
  static cudaError_t sieve_cut(const JobDev &job, int E, int NTL, int n, uint64_t ubeg,
                               uint64_t uend, int num_sms, cudaStream_t s) {
    const int tw = Sh::words(E, NTL, n);
    const size_t smem = (size_t)tw * TEAMS * sizeof(double2);
    auto *kern = sieve_cut_v3<S, CS, NW, TEAMS, REGS, CMP>;
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
    ++lhaf::g_launches;
    kern<<<(unsigned)grid, THREADS, smem, s>>>(job, ubeg, uend, tw);
    return cudaGetLastError();
  }
  static cudaError_t terms(const JobDev &job, int E, int NTL, int n, const uint64_t *t, int nt,
                           double2 *g_out, cudaStream_t s) {
    const int tw = Sh::words(E, NTL, n);
    const size_t smem = (size_t)tw * TEAMS * sizeof(double2);
    auto *kern = terms_v3<S, CS, NW, TEAMS, REGS, CMP>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int grid = (nt + TEAMS - 1) / TEAMS;
    if (grid > 1024) grid = 1024;
    ++lhaf::g_launches;
    kern<<<grid, THREADS, smem, s>>>(job, t, nt, g_out, tw);
    return cudaGetLastError();
  }
};

// <S, CS, NW, TEAMS, registers per thread>.  Each SM sub-partition has 16K registers, so a
// warp of R registers allows floor(512 / R) warps per sub-partition.
using I9 = Inst<1, 9, 1, 4, 128>;
using I17 = Inst<1, 17, 1, 4, 128>;
using I25 = Inst<1, 25, 1, 4, 168, true>;
using I32 = Inst<1, 32, 1, 4, 168, true>;
using I48 = Inst<2, 24, 3, 1, 168, true>;
using I62 = Inst<2, 31, 4, 1, 232, true>;  // 2 CTAs / SM (2 warps per 16K-register sub-partition)
using I64 = Inst<2, 32, 4, 1, 168, true>;
// (LHAF_V3_ALT=3) single-phase reduction (no compaction): a second rounding order of the same
// method, kept for the accuracy cross-checks (tests/test_gpu_variants.py)
using P25 = Inst<1, 25, 1, 4, 168>;
using P48 = Inst<2, 24, 3, 1, 168>;
using P62 = Inst<2, 31, 4, 1, 255>;
static int alt_mode() {
  static const int m = [] { const char *e = getenv("LHAF_V3_ALT"); return e ? atoi(e) : 0; }();
  return m;
}


}  // namespace v3

cudaError_t v3_ensure_tables() { return v3::ensure_inv(); }

#ifdef LHAF_STEP_PROBE
extern "C" int lhaf_debug_step_probe(long long *out) {  // [64][8][4]
  cudaDeviceSynchronize();
  return (int)cudaMemcpyFromSymbol(out, v3::g_probe, sizeof(long long) * 64 * 8 * 4);
}
#endif
#ifdef LHAF_PHASE_TIMING
extern "C" int lhaf_debug_phase_cycles(unsigned long long *out8) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out8, v3::g_phase, 8 * sizeof(unsigned long long));
  unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  return (int)cudaMemcpyToSymbol(v3::g_phase, z, sizeof z);
}
#endif

#define LHAF_V3_DISPATCH(CALL)                  \
  if (v3::alt_mode() == 3) {                    \
    if (E > 17 && E <= v3::P25::EMAX) return v3::P25::CALL; \
    if (E > 32 && E <= v3::P48::EMAX) return v3::P48::CALL; \
    if (E > 48 && E <= v3::P62::EMAX) return v3::P62::CALL; \
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

cudaError_t launch_sieve_cut_v3(const JobDev &job, int e_max, int ntl_max, int n_max, uint64_t ubeg,
                                uint64_t uend, int num_sms, cudaStream_t s) {
  if (uend <= ubeg) return cudaSuccess;
  cudaError_t e = v3::ensure_inv();
  if (e != cudaSuccess) return e;
  const int E = e_max;
#define LHAF_CUT(I) \
  if (E <= v3::I::EMAX) return v3::I::sieve_cut(job, e_max, ntl_max, n_max, ubeg, uend, num_sms, s);
  LHAF_CUT(I9) LHAF_CUT(I17) LHAF_CUT(I25) LHAF_CUT(I32) LHAF_CUT(I48) LHAF_CUT(I62) LHAF_CUT(I64)
#undef LHAF_CUT
  return cudaErrorInvalidValue;
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
