/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY.  Plain, slow, obviously-correct CPU oracle
 * for the loop hafnian of a matrix with repeated rows/columns.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load this library.  It shares no code, header, table or helper with the
 * product (paper_2108_01622_b200/); neither side includes or links the other.
 *
 * Arithmetic: x87 `long double _Complex` (64-bit mantissa) throughout; inputs arrive as
 * IEEE doubles (interleaved re, im) and are widened on entry.
 *
 * Citations: "P:nnn" = line nnn of the paper text (PAPER.md of arXiv 2108.01622).
 *
 * Functions (each follows one passage; see DESIGN.md "Oracle" for the readings):
 *   orc_expand          A_n formation: repeat row/col i n_i times, diagonal <- gamma
 *   orc_lhaf_brute      definition: sum over single-pair matchings
 *   orc_lhaf_et         eigenvalue-trace inclusion/exclusion, Eq. ET_loop / ET_poly
 *                       with explicit matrix powers; sign reading C1, odd-N phantom C7;
 *                       also returns sum_Z |f(A_Z)| (the cancellation factor kappa =
 *                       that / |lhaf| bounds the oracle's own rounding: err <~ kappa * eps_ld)
 *   orc_matched_reps    greedy pair matching, steps 1-5
 *   orc_fds_term        one repeated-pair finite-difference-sieve term g(w)
 *                       with explicit matrix powers (reading C4: X replaced by X_w)
 *   orc_lhaf_fds        full repeated-pair sieve sum, Eq. fdsieve generalised by P:505
 *                       with weights/sign of reading C5, no halving
 *
 * Parity pins: see tests/test_oracle_pins.py (closed forms, brute force, identities).
 */
#include <complex.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#include <omp.h>

typedef long double _Complex cld;

/* ------------------------------------------------------------------------- */
/* A_n formation ("repeating the ith ... rows and columns n_i times ... the diagonal
 * elements of A_n are replaced by the elements of gamma_n"; P:378 for the pure B_n).
 * Output: Ahat (N x N, interleaved re/im doubles), N = sum(reps). Index a of Ahat maps
 * to mode mu(a) where modes are listed in order 0..k-1, mode i repeated reps[i] times. */
int orc_expand(const double *A, const double *gamma, const int32_t *reps, int32_t k,
               double *Ahat_out) {
  int N = 0;
  for (int i = 0; i < k; ++i) N += reps[i];
  int *mu = (int *)malloc(sizeof(int) * (N > 0 ? N : 1));
  int a = 0;
  for (int i = 0; i < k; ++i)
    for (int c = 0; c < reps[i]; ++c) mu[a++] = i;
  for (int r = 0; r < N; ++r)
    for (int c = 0; c < N; ++c) {
      double re, im;
      if (r == c) { re = gamma[2 * mu[r]]; im = gamma[2 * mu[r] + 1]; }
      else { re = A[2 * (mu[r] * k + mu[c])]; im = A[2 * (mu[r] * k + mu[c]) + 1]; }
      Ahat_out[2 * (r * N + c)] = re;
      Ahat_out[2 * (r * N + c) + 1] = im;
    }
  free(mu);
  return N;
}

/* ------------------------------------------------------------------------- */
/* Definition: lhaf(A) = sum over single-pair matchings M of [N] of
 * prod_{(i,j) in M} A_ij, where singles (i,i) are loops weighted by A_ii.
 * Recursion: the lowest unmatched index is either a loop, or pairs with a later
 * unmatched index. */
static cld brute_rec(int N, const cld *A, unsigned char *used, int first) {
  int a = first;
  while (a < N && used[a]) ++a;
  if (a == N) return 1.0L;
  used[a] = 1;
  cld total = A[a * N + a] * brute_rec(N, A, used, a + 1);          /* a is a loop */
  for (int b = a + 1; b < N; ++b) {
    if (used[b]) continue;
    used[b] = 1;
    total += A[a * N + b] * brute_rec(N, A, used, a + 1);           /* pair (a,b) */
    used[b] = 0;
  }
  used[a] = 0;
  return total;
}

void orc_lhaf_brute(int32_t N, const double *Ahat, double *out) {
  cld *A = (cld *)malloc(sizeof(cld) * (N > 0 ? N * N : 1));
  for (int i = 0; i < N * N; ++i) A[i] = (long double)Ahat[2 * i] + I * (long double)Ahat[2 * i + 1];
  unsigned char *used = (unsigned char *)calloc(N > 0 ? N : 1, 1);
  cld r = brute_rec(N, A, used, 0);
  out[0] = (double)creall(r);
  out[1] = (double)cimagl(r);
  free(A);
  free(used);
}

/* Number of single-pair matchings visited, for the pin T(N) = telephone numbers. */
static uint64_t count_rec(int N, unsigned char *used, int first) {
  int a = first;
  while (a < N && used[a]) ++a;
  if (a == N) return 1;
  used[a] = 1;
  uint64_t total = count_rec(N, used, a + 1);
  for (int b = a + 1; b < N; ++b) {
    if (used[b]) continue;
    used[b] = 1;
    total += count_rec(N, used, a + 1);
    used[b] = 0;
  }
  used[a] = 0;
  return total;
}
uint64_t orc_count_matchings(int32_t N) {
  unsigned char used[64] = {0};
  return count_rec(N, used, 0);
}

/* ------------------------------------------------------------------------- */
/* lambda^m coefficient of sum_{j=1}^{m} (1/j!) (sum_{k=1}^{m} a_k lambda^k)^j   (Eq. ET_poly,
 * P:409-413), evaluated literally: the polynomial P = sum_k a_k lambda^k is raised to
 * successive powers, truncated at degree m. a[1..m] used. */
static cld et_poly_coeff(int m, const cld *a) {
  if (m == 0) return 0.0L;      /* the j-sum is empty for N/2 = 0; callers special-case N=0 */
  cld *P = (cld *)calloc(m + 1, sizeof(cld));
  cld *Pj = (cld *)calloc(m + 1, sizeof(cld));
  cld *tmp = (cld *)calloc(m + 1, sizeof(cld));
  for (int k = 1; k <= m; ++k) P[k] = a[k];
  memcpy(Pj, P, sizeof(cld) * (m + 1));              /* P^1 */
  cld result = 0.0L;
  long double jfact = 1.0L;
  for (int j = 1; j <= m; ++j) {
    jfact *= (long double)j;
    result += Pj[m] / jfact;
    /* Pj <- Pj * P (truncated) */
    for (int e = 0; e <= m; ++e) tmp[e] = 0.0L;
    for (int e1 = 0; e1 <= m; ++e1)
      if (Pj[e1] != 0.0L)
        for (int e2 = 1; e1 + e2 <= m; ++e2) tmp[e1 + e2] += Pj[e1] * P[e2];
    memcpy(Pj, tmp, sizeof(cld) * (m + 1));
  }
  free(P); free(Pj); free(tmp);
  return result;
}

/* a_k = Tr((C Xw)^k)/(2k) + (v Xw (C Xw)^{k-1} v^T)/2 for k=1..m, with C (dim x dim, dim = 2h),
 * Xw = [[0, diag(w)], [diag(w), 0]] (w = 1 gives the plain X of P:311).  Explicit powers. */
static void et_a_coeffs(int h, const cld *C, const cld *v, const cld *w, int m, cld *a) {
  int dim = 2 * h;
  cld *M = (cld *)malloc(sizeof(cld) * (dim * dim > 0 ? dim * dim : 1));
  cld *Pw = (cld *)malloc(sizeof(cld) * (dim * dim > 0 ? dim * dim : 1));
  cld *T = (cld *)malloc(sizeof(cld) * (dim * dim > 0 ? dim * dim : 1));
  cld *x = (cld *)malloc(sizeof(cld) * (dim > 0 ? dim : 1));
  cld *y = (cld *)malloc(sizeof(cld) * (dim > 0 ? dim : 1));
  cld *vX = (cld *)malloc(sizeof(cld) * (dim > 0 ? dim : 1));
  /* M = C Xw: column c of M = Xw-weighted column of C: (C Xw)_{r,c} = C_{r, c^} w_{c mod h},
   * where c^ is the partner index (c+h) mod dim. */
  for (int r = 0; r < dim; ++r)
    for (int c = 0; c < dim; ++c) {
      int partner = (c < h) ? c + h : c - h;
      M[r * dim + c] = C[r * dim + partner] * w[c % h];
    }
  /* row vector vX = v Xw */
  for (int c = 0; c < dim; ++c) {
    int partner = (c < h) ? c + h : c - h;
    vX[c] = v[partner] * w[c % h];
  }
  /* Pw = M^1, x = v^T (= M^0 v^T) */
  memcpy(Pw, M, sizeof(cld) * dim * dim);
  for (int r = 0; r < dim; ++r) x[r] = v[r];
  for (int k = 1; k <= m; ++k) {
    cld tr = 0.0L;
    for (int r = 0; r < dim; ++r) tr += Pw[r * dim + r];
    cld q = 0.0L;
    for (int r = 0; r < dim; ++r) q += vX[r] * x[r];
    a[k] = tr / (2.0L * k) + q / 2.0L;
    /* advance: Pw <- Pw M, x <- M x */
    for (int r = 0; r < dim; ++r)
      for (int c = 0; c < dim; ++c) {
        cld s = 0.0L;
        for (int l = 0; l < dim; ++l) s += Pw[r * dim + l] * M[l * dim + c];
        T[r * dim + c] = s;
      }
    memcpy(Pw, T, sizeof(cld) * dim * dim);
    for (int r = 0; r < dim; ++r) {
      cld s = 0.0L;
      for (int l = 0; l < dim; ++l) s += M[r * dim + l] * x[l];
      y[r] = s;
    }
    memcpy(x, y, sizeof(cld) * dim);
  }
  free(M); free(Pw); free(T); free(x); free(y); free(vX);
}

/* ------------------------------------------------------------------------- */
/* Eigenvalue-trace (Eq. ET_loop):
 *   lhaf(A) = sum_{Z in P([N/2])} s(Z) f(A_Z),
 * A_Z keeps rows/cols i and N/2+i for i in Z; f(C) = lambda^{N/2} coefficient of ET_poly
 * with v = diag(C) and X the swap matrix of C's size.  Sign: reading C1, s(Z) =
 * (-1)^{N/2-|Z|} (the printed (-1)^{|Z|} differs by the global factor (-1)^{N/2}; the
 * 2x2 pin lhaf([[a,b],[b,d]]) = b + a d fixes it).  Odd N: reading C7 -- a phantom index
 * with loop weight 1 and zero couplings is appended (lhaf unchanged).
 * Parallel over subsets with OpenMP; each subset is independent. */
void orc_lhaf_et(int32_t N0, const double *Ahat, double *out, double *out_abs) {
  int N = N0 + (N0 & 1);
  if (N == 0) { out[0] = 1.0; out[1] = 0.0; if (out_abs) *out_abs = 1.0; return; }
  cld *A = (cld *)calloc(N * N, sizeof(cld));
  for (int r = 0; r < N0; ++r)
    for (int c = 0; c < N0; ++c)
      A[r * N + c] = (long double)Ahat[2 * (r * N0 + c)] + I * (long double)Ahat[2 * (r * N0 + c) + 1];
  if (N != N0) A[(N - 1) * N + (N - 1)] = 1.0L;   /* phantom loop */
  int half = N / 2;
  uint64_t nsub = (uint64_t)1 << half;
  /* Deterministic summation: fixed blocks of subsets, each summed in order, then the block
   * sums added in block order (independent of the thread count). */
  const uint64_t BLK = 256;
  const uint64_t nblk = (nsub + BLK - 1) / BLK;
  long double *bre = (long double *)calloc(nblk, sizeof(long double));
  long double *bim = (long double *)calloc(nblk, sizeof(long double));
  long double *bab = (long double *)calloc(nblk, sizeof(long double));
#pragma omp parallel for schedule(dynamic, 1)
  for (uint64_t blk = 0; blk < nblk; ++blk)
  for (uint64_t Z = blk * BLK; Z < nsub && Z < (blk + 1) * BLK; ++Z) {
    int idx[64], h = 0;
    for (int i = 0; i < half; ++i)
      if (Z >> i & 1) idx[h++] = i;
    int dim = 2 * h;
    cld *C = (cld *)malloc(sizeof(cld) * (dim * dim > 0 ? dim * dim : 1));
    cld *v = (cld *)malloc(sizeof(cld) * (dim > 0 ? dim : 1));
    cld *w = (cld *)malloc(sizeof(cld) * (h > 0 ? h : 1));
    cld *a = (cld *)calloc(half + 1, sizeof(cld));
    /* retained index list: (i_1..i_h, N/2+i_1..N/2+i_h), so the pairs (r, r+h) of the
     * submatrix are the retained pairs (i, N/2+i) of the full matrix. */
    int keep[128];
    for (int r = 0; r < h; ++r) { keep[r] = idx[r]; keep[r + h] = idx[r] + half; }
    for (int r = 0; r < dim; ++r)
      for (int c = 0; c < dim; ++c) C[r * dim + c] = A[keep[r] * N + keep[c]];
    for (int r = 0; r < dim; ++r) v[r] = C[r * dim + r];
    for (int r = 0; r < h; ++r) w[r] = 1.0L;
    et_a_coeffs(h, C, v, w, half, a);
    cld f = et_poly_coeff(half, a);
    if ((half - h) & 1) f = -f;
    bre[blk] += creall(f);
    bim[blk] += cimagl(f);
    bab[blk] += cabsl(f);
    free(C); free(v); free(w); free(a);
  }
  long double sre = 0.0L, sim = 0.0L, sabs = 0.0L;
  for (uint64_t blk = 0; blk < nblk; ++blk) { sre += bre[blk]; sim += bim[blk]; sabs += bab[blk]; }
  free(bre); free(bim); free(bab);
  out[0] = (double)sre;
  out[1] = (double)sim;
  if (out_abs) *out_abs = (double)sabs;
  free(A);
}

/* ------------------------------------------------------------------------- */
/* Greedy pair matching, P:474-481 (reading C9):
 *   m = (0..M-1).  Repeat: (1) sort n and m descending by n (stable: ties keep the lower
 *   mode index first); (2) if n1 >= 2 n2 (n2 := 0 when only one mode remains) create
 *   (m1,m1) pairs repeated floor(n1/2) times, else (m1,m2) pairs repeated n2 times;
 *   (3) subtract; (4) drop zeros; (5) continue while sum(n) > 1.
 * A single leftover photon (sum n == 1) is returned in *leftover (else -1) -- reading C7
 * pairs it with a phantom index.
 * Output arrays p, q, eta of capacity cap; returns the number of pairs H (or -1 on overflow). */
int32_t orc_matched_reps(const int32_t *reps, int32_t k, int32_t *p, int32_t *q, int32_t *eta,
                         int32_t cap, int32_t *leftover) {
  int32_t *n = (int32_t *)malloc(sizeof(int32_t) * (k > 0 ? k : 1));
  int32_t *m = (int32_t *)malloc(sizeof(int32_t) * (k > 0 ? k : 1));
  int len = 0;
  for (int i = 0; i < k; ++i)
    if (reps[i] > 0) { n[len] = reps[i]; m[len] = i; ++len; }
  int H = 0;
  *leftover = -1;
  for (;;) {
    long total = 0;
    for (int i = 0; i < len; ++i) total += n[i];
    if (total <= 1) {
      if (total == 1) *leftover = m[0];
      break;
    }
    /* stable insertion sort, descending n, ties by ascending mode index */
    for (int i = 1; i < len; ++i) {
      int ni = n[i], mi = m[i], j = i - 1;
      while (j >= 0 && (n[j] < ni || (n[j] == ni && m[j] > mi))) {
        n[j + 1] = n[j]; m[j + 1] = m[j]; --j;
      }
      n[j + 1] = ni; m[j + 1] = mi;
    }
    int n1 = n[0], n2 = (len > 1) ? n[1] : 0;
    if (H >= cap) { free(n); free(m); return -1; }
    if (n1 >= 2 * n2) {
      p[H] = m[0]; q[H] = m[0]; eta[H] = n1 / 2; ++H;
      n[0] -= 2 * (n1 / 2);
    } else {
      p[H] = m[0]; q[H] = m[1]; eta[H] = n2; ++H;
      n[0] -= n2; n[1] -= n2;
    }
    int w = 0;
    for (int i = 0; i < len; ++i)
      if (n[i] > 0) { n[w] = n[i]; m[w] = m[i]; ++w; }
    len = w;
  }
  free(n); free(m);
  return H;
}

/* ------------------------------------------------------------------------- */
/* One repeated-pair sieve term (P:431-435 with X_z -> X_w, reading C4):
 *   g(w) = lambda^n coefficient of sum_j (1/j!) (sum_k a_k lambda^k)^j,
 *   a_k = Tr((C Xw)^k)/(2k) + v Xw (C Xw)^{k-1} v^T / 2,
 * with C (2h x 2h) the reduced matrix over the pair index list (p_1..p_h, q_1..q_h),
 * v the loop vector, w (h) the per-pair integer weights.  Explicit powers, long double. */
static cld fds_term_ld(int h, const cld *C, const cld *v, const int32_t *w, int n) {
  cld *wl = (cld *)malloc(sizeof(cld) * (h > 0 ? h : 1));
  cld *a = (cld *)calloc(n + 1, sizeof(cld));
  for (int i = 0; i < h; ++i) wl[i] = (long double)w[i];
  et_a_coeffs(h, C, v, wl, n, a);
  cld g = et_poly_coeff(n, a);
  free(wl); free(a);
  return g;
}

void orc_fds_term(int32_t h, const double *C, const double *v, const int32_t *w, int32_t n,
                  double *out) {
  int dim = 2 * h;
  cld *Cl = (cld *)malloc(sizeof(cld) * (dim * dim > 0 ? dim * dim : 1));
  cld *vl = (cld *)malloc(sizeof(cld) * (dim > 0 ? dim : 1));
  for (int i = 0; i < dim * dim; ++i) Cl[i] = (long double)C[2 * i] + I * (long double)C[2 * i + 1];
  for (int i = 0; i < dim; ++i) vl[i] = (long double)v[2 * i] + I * (long double)v[2 * i + 1];
  cld g = fds_term_ld(h, Cl, vl, w, n);
  out[0] = (double)creall(g);
  out[1] = (double)cimagl(g);
  free(Cl); free(vl);
}

/* A batch of sieve terms (the same g(w) as orc_fds_term, one per row of w: nt x h int32),
 * OpenMP over the terms.  A plain map of fds_term_ld, used by the per-term parity test (P14). */
void orc_fds_terms(int32_t h, const double *C, const double *v, const int32_t *w, int32_t nt,
                   int32_t n, double *out) {
  int dim = 2 * h;
  cld *Cl = (cld *)malloc(sizeof(cld) * (dim * dim > 0 ? dim * dim : 1));
  cld *vl = (cld *)malloc(sizeof(cld) * (dim > 0 ? dim : 1));
  for (int i = 0; i < dim * dim; ++i) Cl[i] = (long double)C[2 * i] + I * (long double)C[2 * i + 1];
  for (int i = 0; i < dim; ++i) vl[i] = (long double)v[2 * i] + I * (long double)v[2 * i + 1];
#pragma omp parallel for schedule(dynamic, 1)
  for (int32_t i = 0; i < nt; ++i) {
    cld g = fds_term_ld(h, Cl, vl, w + (size_t)i * h, n);
    out[2 * (size_t)i] = (double)creall(g);
    out[2 * (size_t)i + 1] = (double)cimagl(g);
  }
  free(Cl); free(vl);
}

/* ------------------------------------------------------------------------- */
/* Reduced matrix for a matching (reading C8): index list r = (p_1..p_H, q_1..q_H);
 * C_ab = A_{r_a r_b} including a = b (A's own diagonal = the weight of pairing two photons
 * of the same mode); v_a = gamma_{r_a}.  A phantom index (r = -1) has zero couplings and
 * loop weight 1 (reading C7). */
static void reduced(const double *A, const double *gamma, int k, int H, const int *r,
                    cld *C, cld *v) {
  int dim = 2 * H;
  for (int a = 0; a < dim; ++a) {
    if (r[a] < 0) v[a] = 1.0L;
    else v[a] = (long double)gamma[2 * r[a]] + I * (long double)gamma[2 * r[a] + 1];
    for (int b = 0; b < dim; ++b) {
      if (r[a] < 0 || r[b] < 0) { C[a * dim + b] = 0.0L; continue; }
      C[a * dim + b] = (long double)A[2 * (r[a] * k + r[b])] + I * (long double)A[2 * (r[a] * k + r[b]) + 1];
    }
  }
}

/* Full repeated-pair sieve (Eq. fdsieve, with the repeated-pair rule of P:505;
 * weights and sign per reading C5):
 *   lhaf = 2^{-n} sum_{k_1=0}^{eta_1} ... sum_{k_H=0}^{eta_H} (-1)^{sum k} prod C(eta_h, k_h) g(eta - 2k),
 * n = sum eta.  Every term is evaluated (no halving), each by explicit powers.
 * Pairs from orc_matched_reps; odd N adds the pair (leftover, phantom) x 1.
 * Mixed variant (mixed != 0): A, gamma are 2k x 2k / 2k and reps has length k; the natural
 * pairing (i, i+k) x reps_i of P:425-428 is used (reading C11).
 * Returns T (the number of terms) and writes out[2]; also writes sum|term| * 2^{-n} to
 * out_abs (the conditioning denominator kappa = out_abs / |out|). */
uint64_t orc_lhaf_fds(const double *A, const double *gamma, const int32_t *reps, int32_t k,
                      int32_t mixed, double *out, double *out_abs) {
  int32_t p[256], q[256], eta[256], leftover = -1, H = 0;
  if (!mixed) {
    H = orc_matched_reps(reps, k, p, q, eta, 255, &leftover);
    if (H < 0) return 0;
  } else {
    for (int i = 0; i < k; ++i)
      if (reps[i] > 0) { p[H] = i; q[H] = i + k; eta[H] = reps[i]; ++H; }
  }
  int kk = mixed ? 2 * k : k;
  int Hf = H + (leftover >= 0 ? 1 : 0);
  int r[512];
  for (int h = 0; h < H; ++h) { r[h] = p[h]; r[h + Hf] = q[h]; }
  if (leftover >= 0) { r[H] = leftover; r[H + Hf] = -1; eta[H] = 1; }
  int n = 0;
  for (int h = 0; h < Hf; ++h) n += eta[h];
  if (Hf == 0) { out[0] = 1.0; out[1] = 0.0; *out_abs = 1.0; return 1; }
  int dim = 2 * Hf;
  cld *C = (cld *)malloc(sizeof(cld) * dim * dim);
  cld *v = (cld *)malloc(sizeof(cld) * dim);
  reduced(A, gamma, kk, Hf, r, C, v);
  uint64_t T = 1;
  for (int h = 0; h < Hf; ++h) T *= (uint64_t)(eta[h] + 1);
  const uint64_t BLK = 64;                      /* deterministic block-ordered summation */
  const uint64_t nblk = (T + BLK - 1) / BLK;
  long double *bre = (long double *)calloc(nblk, sizeof(long double));
  long double *bim = (long double *)calloc(nblk, sizeof(long double));
  long double *bab = (long double *)calloc(nblk, sizeof(long double));
#pragma omp parallel for schedule(dynamic, 1)
  for (uint64_t blk = 0; blk < nblk; ++blk)
  for (uint64_t t = blk * BLK; t < T && t < (blk + 1) * BLK; ++t) {
    int32_t w[256];
    uint64_t rem = t;
    int ksum = 0;
    long double weight = 1.0L;
    for (int h = 0; h < Hf; ++h) {              /* mixed radix, lowest pair fastest */
      int kh = (int)(rem % (uint64_t)(eta[h] + 1));
      rem /= (uint64_t)(eta[h] + 1);
      ksum += kh;
      long double b = 1.0L;                      /* C(eta_h, k_h) */
      for (int i = 1; i <= kh; ++i) b = b * (long double)(eta[h] - kh + i) / (long double)i;
      weight *= b;
      w[h] = eta[h] - 2 * kh;
    }
    cld g = fds_term_ld(Hf, C, v, w, n);
    long double sgn = (ksum & 1) ? -1.0L : 1.0L;
    bre[blk] += sgn * weight * creall(g);
    bim[blk] += sgn * weight * cimagl(g);
    bab[blk] += weight * cabsl(g);
  }
  long double sre = 0.0L, sim = 0.0L, sabs = 0.0L;
  for (uint64_t blk = 0; blk < nblk; ++blk) { sre += bre[blk]; sim += bim[blk]; sabs += bab[blk]; }
  free(bre); free(bim); free(bab);
  long double scale = ldexpl(1.0L, -n);
  out[0] = (double)(sre * scale);
  out[1] = (double)(sim * scale);
  *out_abs = (double)(sabs * scale);
  free(C); free(v);
  return T;
}

/* ------------------------------------------------------------------------- */
/* Timing entry for the CPU baseline: sum of the sieve terms t in [t0, t1) of the same sum as
 * orc_lhaf_fds (each term by explicit powers), without the 2^{-n} prefactor.  Used only by
 * bench.py's cpu_baseline / --impl reference legs; same arithmetic as orc_lhaf_fds. */
uint64_t orc_fds_range(const double *A, const double *gamma, const int32_t *reps, int32_t k,
                       int32_t mixed, uint64_t t0, uint64_t t1, double *out) {
  int32_t p[256], q[256], eta[256], leftover = -1, H = 0;
  if (!mixed) {
    H = orc_matched_reps(reps, k, p, q, eta, 255, &leftover);
    if (H < 0) return 0;
  } else {
    for (int i = 0; i < k; ++i)
      if (reps[i] > 0) { p[H] = i; q[H] = i + k; eta[H] = reps[i]; ++H; }
  }
  int kk = mixed ? 2 * k : k;
  int Hf = H + (leftover >= 0 ? 1 : 0);
  int r[512];
  for (int h = 0; h < H; ++h) { r[h] = p[h]; r[h + Hf] = q[h]; }
  if (leftover >= 0) { r[H] = leftover; r[H + Hf] = -1; eta[H] = 1; }
  int n = 0;
  for (int h = 0; h < Hf; ++h) n += eta[h];
  if (Hf == 0) { out[0] = 1.0; out[1] = 0.0; return 0; }
  int dim = 2 * Hf;
  cld *C = (cld *)malloc(sizeof(cld) * dim * dim);
  cld *v = (cld *)malloc(sizeof(cld) * dim);
  reduced(A, gamma, kk, Hf, r, C, v);
  uint64_t T = 1;
  for (int h = 0; h < Hf; ++h) T *= (uint64_t)(eta[h] + 1);
  if (t1 > T) t1 = T;
  long double sre = 0.0L, sim = 0.0L;
#pragma omp parallel for schedule(dynamic, 1) reduction(+ : sre, sim)
  for (uint64_t t = t0; t < t1; ++t) {
    int32_t w[256];
    uint64_t rem = t;
    int ksum = 0;
    long double weight = 1.0L;
    for (int h = 0; h < Hf; ++h) {
      int kh = (int)(rem % (uint64_t)(eta[h] + 1));
      rem /= (uint64_t)(eta[h] + 1);
      ksum += kh;
      long double b = 1.0L;
      for (int i = 1; i <= kh; ++i) b = b * (long double)(eta[h] - kh + i) / (long double)i;
      weight *= b;
      w[h] = eta[h] - 2 * kh;
    }
    cld g = fds_term_ld(Hf, C, v, w, n);
    long double sgn = (ksum & 1) ? -1.0L : 1.0L;
    sre += sgn * weight * creall(g);
    sim += sgn * weight * cimagl(g);
  }
  out[0] = (double)sre;
  out[1] = (double)sim;
  free(C); free(v);
  return t1 > t0 ? t1 - t0 : 0;
}

int orc_num_threads(void) {
  int n = 1;
#pragma omp parallel
  {
#pragma omp single
    n = omp_get_num_threads();
  }
  return n;
}
