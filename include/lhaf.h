/*
 * lhaf.h -- C-ABI of the B200 loop-hafnian library for matrices with repeated rows/columns
 * (photon collisions at number-resolving detectors), after Bulmer et al., "The Boundary for
 * Quantum Advantage in Gaussian Boson Sampling", arXiv 2108.01622.
 *
 * Citations "P:nnn" are lines of the paper text; "S8(a) a4" etc. are rows of the
 * hot-path scope table in SURVEY.md.
 *
 * What is computed.  For a symmetric complex k x k matrix A, loop weights gamma (k) and a
 * photon pattern reps (k non-negative integers, N = sum reps), lhaf_rpt returns lhaf(A_n),
 * the loop hafnian (sum over single-pair matchings) of the N x N matrix A_n
 * formed by repeating row/column i of A reps[i] times and replacing the diagonal by the
 * correspondingly repeated gamma.  The method is the finite-difference sieve
 * over the repeated pairs of the greedy matching:
 *     lhaf = 2^{1-n} sum_{t < floor(T/2)} (-1)^{sum k} prod_h C(eta_h, k_h) g(eta - 2k)
 * (readings C5/C6 of DESIGN.md), one per-term evaluation g per mixed-radix index t.
 *
 * Conventions shared by every entry point.
 *  - Complex numbers are interleaved (re, im) IEEE doubles; matrices are row-major.
 *  - Host pointers unless the name ends in _dev.  The caller owns every buffer; the library
 *    copies what it needs and keeps no pointer after the call returns.  Outputs are written
 *    only when the call returns LHAF_OK.
 *  - A's diagonal is the weight of pairing two photons detected in the same mode (it is used
 *    only when some reps[i] >= 2); gamma holds the loop weights (reading C8).  A caller that
 *    holds an already-expanded matrix with the loops on its diagonal passes reps = 1 and
 *    gamma = its diagonal.
 *  - Errors are returned as lhaf_status, never thrown across the ABI; lhaf_last_error()
 *    gives a message for the calling thread's last non-OK status.
 *  - Calls are serialised internally (one device context per process); results are
 *    bit-identical for any number of ranks (fixed chunking + ordered double-double sums).
 *  - All arithmetic runs on the GPU (sm_100a kernels); there is no CPU fallback.  Without a
 *    usable CUDA device every compute call returns LHAF_E_CUDA.
 */
#ifndef LHAF_H_
#define LHAF_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  LHAF_OK = 0,
  LHAF_E_ARG = 1,           /* null pointer, k < 0 or > LHAF_MAX_MODES, negative reps, batch < 0 */
  LHAF_E_NOT_SYMMETRIC = 2, /* max|A - A^T| > 1e-12 * max(1, max|A|) */
  LHAF_E_TOO_LARGE = 3,     /* reduced dimension d > LHAF_MAX_DIM, degree n > LHAF_MAX_DEGREE,
                               or term count above the guard */
  LHAF_E_CUDA = 4,          /* CUDA runtime failure, or no device */
  LHAF_E_NCCL = 5,          /* NCCL failure (multi-rank only) */
  LHAF_E_STATE = 6,         /* library not initialised as required / inconsistent ranks */
  LHAF_E_INACCURATE = 7     /* results computed, but an error estimate exceeds the requested tolerance */
} lhaf_status;

#define LHAF_MAX_MODES 4096
#define LHAF_MAX_DIM 64       /* d = 2H (H = number of distinct pairs incl. the phantom) */
#define LHAF_MAX_DEGREE 128   /* n = sum eta (lambda degree) */
#define LHAF_MAX_PAIRS 64

/* Host-only plan of one pattern (S8(a) a2-a4).  Greedy matching of P:474-481 (reading C9:
 * stable sort by (count desc, mode asc) every round, n2 := 0 when one mode remains), the
 * phantom pair for odd N (reading C7), and the term counts.  mixed = 1 plans the mixed state
 * by the same greedy matching of the doubled pattern (reps, reps) over the 2k modes (reading
 * C11b: same value, measured far better conditioned in FP64); mixed = 2 selects the natural
 * pairing (i, i+k) x reps_i of P:425-428 (reading C11); mixed = 3 (job API, lhaf_rpt_mixed)
 * searches the matching with the least cancellation (below) -- planned here like mode 1. */
typedef struct {
  int32_t N;            /* photons = sum reps */
  int32_t H;            /* distinct pairs incl. phantom */
  int32_t d;            /* reduced dimension 2H */
  int32_t n;            /* lambda degree = sum eta */
  int32_t leftover;     /* mode of the odd leftover photon, or -1 */
  int32_t pad_;
  uint64_t T;           /* prod (eta_h + 1): full sieve term count */
  uint64_t T_eval;      /* floor(T/2): evaluated terms after halving (reading C6) */
  int32_t p[LHAF_MAX_PAIRS];   /* pair h = (p[h], q[h]); q = -1 for the phantom */
  int32_t q[LHAF_MAX_PAIRS];
  int32_t eta[LHAF_MAX_PAIRS];
} lhaf_plan_info;

/* Plan only (no GPU).  reps: k int32, k in [0, LHAF_MAX_MODES].  For mixed, reps has length
 * k and refers to a 2k-mode matrix.  Returns LHAF_E_ARG on bad input, LHAF_E_TOO_LARGE when
 * H exceeds LHAF_MAX_PAIRS. */
lhaf_status lhaf_plan(const int32_t *reps, int32_t k, int32_t mixed, lhaf_plan_info *info);

/* Mixed-radix decode of term index t for a plan (S8(a) a4, integers only, bit-exact):
 * digits k_h in [0, eta_h] with pair 0 fastest, w_h = eta_h - 2 k_h, sign = (-1)^{sum k},
 * weight = prod C(eta_h, k_h) (exact integer if < 2^64; returned as uint64).  k_out, w_out
 * have room for info->H entries. */
lhaf_status lhaf_decode(const lhaf_plan_info *info, uint64_t t, int32_t *k_out, int32_t *w_out,
                        int32_t *sign_out, uint64_t *weight_out);

/* One loop hafnian (S8(a) a1-a12).  A: k*k c128, gamma: k c128, reps: k int32.  out[2] =
 * (re, im) of lhaf(A_n).  N = 0 gives (1, 0).  Errors: E_ARG, E_NOT_SYMMETRIC, E_TOO_LARGE,
 * E_CUDA, E_NCCL.  After lhaf_init_rank(nranks > 1) the term range is sharded over the ranks
 * and every rank receives the full result (one NCCL all-reduce of chunk partials). */
lhaf_status lhaf_rpt(const double *A, const double *gamma, const int32_t *reps, int32_t k,
                     double out[2]);

/* Batch of loop hafnians sharing A (S8(a) a14; the chain-rule use of P:371-373).
 * gamma: k c128 when gamma_stride == 0 (shared), else batch rows of gamma_stride (>= k)
 * c128 each.  reps: batch*k int32 row-major.  out: batch*2 doubles.  Patterns are sharded
 * over ranks by contiguous blocks of work units. */
lhaf_status lhaf_rpt_batch(const double *A, const double *gamma, int64_t gamma_stride,
                           const int32_t *reps, int32_t k, int32_t batch, double *out);

/* Mixed-state loop hafnian (S8(a) a13): lhaf of the 2N x 2N A_n formed from the 2k x 2k
 * matrix A2 by repeating rows/cols i and i+k reps[i] times.  Evaluated with mixed mode
 * 3: every matching gives the same lhaf but not the same cancellation kappa =
 * sum|term| / |lhaf|, which sets the FP64 error; 16 greedy matchings of the
 * doubled pattern (reading C11b; ties broken by seeded relabellings of the modes, the first
 * the identity = mode 1) are each estimated on 8 work units spread over the sieve and the one
 * with the smallest sum|term| is evaluated (env LHAF_KAPPA_CANDIDATES / LHAF_KAPPA_SAMPLES).
 * Mode 1 (the identity candidate alone) and the natural pairing (i, i+k) x reps_i of
 * P:425-428 (mode 2) are selectable through the job API.  In precise mode the natural pairing
 * is used.  A2: 2k*2k c128, gamma2: 2k c128, reps: k int32. */
lhaf_status lhaf_rpt_mixed(const double *A2, const double *gamma2, const int32_t *reps,
                           int32_t k, double out[2]);

/* Cutoff-batched loop hafnians for the chain rule (App. B.5, P:517-523:
 * "all but one mode has a fixed outcome n_fixed, while one 'batched' mode takes all values
 * from 0 to the cutoff n_cut").  out[2 j], out[2 j + 1] = lhaf(A_n) for the pattern
 * reps_fixed with reps[mode] replaced by j, j = 0 .. n_cut.  A: k*k c128, gamma: k c128,
 * reps_fixed: k int32 (its entry at `mode` is ignored), 0 <= mode < k, 0 <= n_cut <= 64,
 * out: 2 (n_cut + 1) doubles.  The paper's shared evaluation: the fixed modes are matched once
 * and the batched mode becomes a self-pair (mode, mode) with eta_b = floor((n_cut - p) / 2) in
 * two groups by the parity p of its count (odd counts add one single-photon pair: with the
 * fixed part's leftover photon, or with the phantom); every term (fixed-pair term, w_b in
 * [-eta_b, eta_b]) is ONE series to degree n_f + eta_b whose coefficients serve every count
 * 2m + p with m >= |w_b|, m = w_b (mod 2), weighted by (-1)^k C(m, k), k = (m - w_b) / 2.
 * Default (series length n_f + eta_b + 1 <= 40, >= 65536 terms): the prefix-sharing tree with
 * the batched self-pair as its leaf level (every prefix of fixed pairs shared); otherwise, or
 * with LHAF_CUTOFF_PER_TERM set, one Hessenberg reduction + La Budde per term (sieve_cut_v3).
 * One sieve evaluation, one finalize.
 * n_cut = 64, or LHAF_CUTOFF_SEPARATE set in the environment, evaluates the n_cut + 1 patterns
 * as independent sieves in one batch job instead (same values up to rounding: both orders
 * carry the sieve's cancellation, ~kappa * eps per count).  Errors as lhaf_rpt_batch, plus
 * LHAF_E_ARG for a bad mode / n_cut. */
lhaf_status lhaf_rpt_cutoff(const double *A, const double *gamma, const int32_t *reps_fixed,
                            int32_t k, int32_t mode, int32_t n_cut, double *out);
/* The same, plus a per-count error estimate (the paper's accuracy mechanism: the
 * sieve's error is its cancellation times the per-term rounding): err_est[j] = kappa_j * 2^-46
 * with kappa_j = 2^{1-n} sum_t |term_t| / |lhaf_j| accumulated in the same pass (2^-46 ~ 64 eps
 * is the FP64 per-term relative error scale measured for d <= 48).  The
 * repeated-pair sieve cancels steeply with the count of one mode (tanh r = 0.6: kappa*eps ~ 2e-8,
 * 8e-5, 1e-2, 1 at counts 4, 8, 12, 16 -- profiles/r01/cutoff_kappa_t0.6.txt), so high counts
 * of a strongly squeezed mode are beyond FP64.  err_est is capped at 1 (a value at the noise
 * level of its own terms, e.g. an exact zero, has no significant digits).  tol > 0: if some
 * err_est[j] > tol, out and
 * err_est are still written and LHAF_E_INACCURATE is returned (lhaf_last_error names the first
 * such count); tol <= 0 never refuses.  err_est: n_cut + 1 doubles.  Other errors as
 * lhaf_rpt_cutoff. */
lhaf_status lhaf_rpt_cutoff_ex(const double *A, const double *gamma, const int32_t *reps_fixed,
                               int32_t k, int32_t mode, int32_t n_cut, double tol, double *out,
                               double *err_est);

/* The same pattern under many loop vectors (the threshold chain rule's
 * sub-detector batching: "this does not change the eigenvalue calculation,
 * so these calculations can be batched"): out[2 g], out[2 g + 1] = lhaf of (A, gammas row g,
 * reps), g < ngamma.  A: k*k c128, gammas: ngamma*k c128 row-major, reps: k int32, out:
 * 2 ngamma doubles.  Shared cubic step: per sieve term ONE Gauss-Hessenberg reduction of the
 * loop-free M = C X_w (the loop vectors ride along as inert rows and columns), one La Budde
 * (c_M) and one c_M^{-1/2}; per loop vector only the loop terms s_j = z'^T H^{j-1} y' by
 * Hessenberg matvecs (O(n d^2)) and the exp series (O(n^2)) -- the v5 kernel's FLAG_MG path.
 * Applies when d + ngamma <= 64, ngamma <= 16, FP64 mode and the automatic kernel choice;
 * otherwise (or with LHAF_MULTIGAMMA_SEPARATE set) the pattern is evaluated once per loop vector
 * in one batch job.  Errors as lhaf_rpt_batch. */
lhaf_status lhaf_rpt_multigamma(const double *A, const double *gammas, int32_t ngamma,
                                const int32_t *reps, int32_t k, double *out);

/* The same loop hafnian by inclusion/exclusion over the pair copies instead of the +-1 sieve
 * (the eigenvalue-trace formula ET_loop of P:403-415 with repeated pairs,
 * the comparison of Fig. 5): lhaf = sum over c_h = 0..eta_h of
 * (-1)^{n - sum c} prod C(eta_h, c_h) g(w = c), g as in the sieve.  Every term runs the same
 * device path (Hessenberg + La Budde + series at full d; excluded pairs are zero columns, not
 * deleted), there is no halving, so it evaluates prod (eta_h + 1) terms (twice the sieve's).
 * Arguments, ownership and errors as lhaf_rpt. */
lhaf_status lhaf_rpt_et(const double *A, const double *gamma, const int32_t *reps, int32_t k,
                        double out[2]);

/* Photon-number pattern probabilities of an M-mode Gaussian state (App. A,
 * P:301-320, Eq. (mixed_prob)):
 *   P(n | sigma, alpha) = exp(-alpha^dag sigma_Q^{-1} alpha / 2) / (sqrt(det sigma_Q) prod_i n_i!)
 *                         * lhaf(A_n),
 * sigma_Q = sigma + I/2, A = X (I - sigma_Q^{-1}), gamma = alpha^dag sigma_Q^{-1}; A_n and
 * gamma_n repeat indices i and i+M n_i times (lhaf_rpt_mixed, natural pairing).
 * sigma: 2M*2M c128 in the basis (a_1..a_M, a_1^dag..a_M^dag),
 *   sigma_ij = <a_i a_j^dag + a_j^dag a_i>/2 - alpha_i alpha_j^* (P:303-305);
 * alpha: 2M c128, alpha_i = <a_i> (so alpha_{i+M} = conj(alpha_i)); n: M int32 >= 0.
 * pure != 0: the caller asserts the state is pure, so A = B (+) B* and the probability is
 *   prefactor |lhaf(B_n)|^2 / prod n_i! with B = A[0:M, 0:M] and loops gamma[0:M],
 *   a loop hafnian of half the size (lhaf_rpt).
 * out[0] = P, out[1] = the imaginary residue of the evaluated expression (0 up to rounding).
 * sigma_Q is inverted on the host (LU with partial pivoting, one per call); the loop hafnian
 * runs on the device.  Errors: LHAF_E_ARG (null pointer, M < 1 or > 2048, n_i < 0, sigma_Q
 * singular or det(sigma_Q) <= 0), otherwise as lhaf_rpt / lhaf_rpt_mixed. */
lhaf_status lhaf_gbs_prob(const double *sigma, const double *alpha, int32_t M, const int32_t *n,
                          int32_t pure, double out[2]);

/* Gaussian-state constructor: the covariance sigma (2M*2M c128)
 * and mean alpha (2M c128), in lhaf_gbs_prob's basis and convention, of M single-mode squeezed
 * vacua (squeezing r_i, real, phase 0), pure loss per input mode (transmission eta_i in [0, 1];
 * eta = NULL: lossless), the interferometer a -> U a (U: M*M c128, unitary to 1e-10) and a
 * displacement beta of the output modes (M c128; NULL: none):
 *   sigma_0 per mode = [[sinh^2 r + 1/2, -cosh r sinh r], [-cosh r sinh r, sinh^2 r + 1/2]],
 *   loss sigma <- sqrt(E) sigma sqrt(E) + (I - E)/2, then S sigma S^dag, S = diag(U, U*),
 *   alpha = (beta, conj(beta)).
 * Host arithmetic; caller-owned outputs written only on LHAF_OK.  Errors: LHAF_E_ARG (null
 * pointer, M outside [1, 2048], r not finite, eta outside [0, 1], U not unitary). */
lhaf_status lhaf_gbs_state(const double *U, const double *r, const double *eta, const double *beta,
                           int32_t M, double *sigma, double *alpha);
/* P(n) of that state in one call: lhaf_gbs_state then lhaf_gbs_prob (the pure half-size form
 * when every eta_i = 1).  out[0] = P, out[1] = imaginary residue.  Errors as the two calls. */
lhaf_status lhaf_gbs_prob_state(const double *U, const double *r, const double *eta,
                                const double *beta, int32_t M, const int32_t *n, double out[2]);

/* The ingredients of lhaf_gbs_prob without a device: A (2M*2M c128), gamma (2M c128) and the
 * prefactor exp(-alpha^dag sigma_Q^{-1} alpha / 2) / sqrt(det sigma_Q) (out_pref: re, im).
 * Caller-owned outputs, written only on LHAF_OK.  Errors as lhaf_gbs_prob. */
lhaf_status lhaf_gbs_matrices(const double *sigma, const double *alpha, int32_t M, double *A,
                              double *gamma, double out_pref[2]);

/* Proposal probability of the MIS importance sampler: singles Poisson(|alpha_j|^2)
 * and photon pairs Poisson(|B_jk|^2) (j < k; 1/2 |B_jj|^2 for j = k) combined into a pattern:
 *   Q(n | B, alpha) = exp(-sum_j |alpha_j|^2 - 1/2 sum_{j,k} |B_jk|^2) / prod_i n_i! lhaf(C_n),
 * C_n = |B_n|^2 elementwise with its diagonal replaced by |alpha_n|^2 -- a loop hafnian of a
 * non-negative matrix, evaluated by the same device path (lhaf_rpt with A = |B|^2, gamma =
 * |alpha|^2).  B: M*M c128 (symmetric), alpha: M c128, n: M int32.  out[0] = Q, out[1] = the
 * imaginary residue (0).  Errors as lhaf_rpt, plus LHAF_E_ARG for M < 1 or n_i < 0. */
lhaf_status lhaf_ips_prob(const double *B, const double *alpha, int32_t M, const int32_t *n,
                          double out[2]);

/* Same three entry points with DEVICE pointers for A / gamma / out (reps stays on the host,
 * since planning is host integer work) and an explicit cudaStream_t (passed as void*; NULL =
 * the legacy default stream).  Ordering: the call first synchronises the device, so inputs
 * written on any stream (e.g. a torch side stream) are complete before they are read; A is
 * copied back for the symmetry check when 2k <= 2048.  Results land in out_dev on `stream`,
 * which is synchronised before return. */
lhaf_status lhaf_rpt_batch_dev(const double *A_dev, const double *gamma_dev, int64_t gamma_stride,
                               const int32_t *reps, int32_t k, int32_t batch, int32_t mixed,
                               double *out_dev, void *stream);

/* ---- Jobs: a planned, device-resident evaluation (for timing and multi-rank control) ----
 * lhaf_job_create plans and uploads a batch (mixed = 1: the mixed state over A2 / gamma2 by
 * the greedy matching of the doubled pattern, mixed = 2: by the natural pairing, mixed = 3:
 * by the matching search of lhaf_rpt_mixed -- host inputs, gamma_stride 0, FP64 mode; it runs
 * candidate sample evaluations on the device during the call; each reps row of length k).  lhaf_job_run evaluates work units [unit_begin, unit_end) into
 * the job's chunk-partial array (zeroed by lhaf_job_reset); lhaf_job_finalize sums the
 * partials in chunk order (double-double) and writes batch*2 doubles to out (host pointer if
 * out_is_device == 0).  One work unit = a fixed, rank-independent chunk of one pattern's
 * terms; units of a pattern are contiguous. */
typedef struct lhaf_job lhaf_job;
typedef struct {
  int32_t batch;
  int32_t d_max;
  int32_t n_max;
  int32_t kernel;        /* kernel variant id selected for this job */
  uint64_t units;        /* total work units */
  uint64_t terms;        /* total evaluated terms (sum of T_eval) */
  double flops_per_term_model; /* algorithmic FP64 flops per term of the selected kernel */
  uint64_t h2d_plan_bytes;     /* bytes of plan tables copied host->device at creation */
  int32_t precision;           /* The plan of pattern `pattern` of a job in the job's own evaluation order: the pairs and
 * multiplicities as lhaf_plan returns them, permuted for the tree variant (the pair
 * eliminated first is last), and T_eval = the terms the job evaluates (T when
 * no pair has an odd count and the tree cannot halve).  Term t of lhaf_job_terms and the
 * unit ranges of lhaf_job_run decode with this order (pair 0 fastest).  Host only.
 * Errors: E_ARG (null pointer, pattern outside [0, batch)). */
lhaf_status lhaf_job_plan(const lhaf_job *job, int32_t pattern, lhaf_plan_info *info);

/* precision mode of the job (lhaf_set_precision) */
  int32_t pad_;
} lhaf_job_info;

lhaf_status lhaf_job_create(const double *A, const double *gamma, int64_t gamma_stride,
                            const int32_t *reps, int32_t k, int32_t batch, int32_t mixed,
                            int32_t A_is_device, lhaf_job **job);
lhaf_status lhaf_job_info_get(const lhaf_job *job, lhaf_job_info *info);
lhaf_status lhaf_job_reset(lhaf_job *job, void *stream);
lhaf_status lhaf_job_run(lhaf_job *job, uint64_t unit_begin, uint64_t unit_end, void *stream);
/* All-reduce (sum) of the partial array over the ranks of lhaf_init_rank (ncclAllReduce on
 * `stream`; no-op for a single rank without a communicator).  Exact: the ranks' unit ranges are
 * disjoint and every other entry is zero (x + 0 = x), so the finalized value is bit-identical
 * for any rank count (S8(e) a12). */
lhaf_status lhaf_job_allreduce(lhaf_job *job, void *stream);
/* The same on the unit range [unit_begin, unit_end) only, plus a stream-ordered zeroing of that
 * range: a caller that evaluates a long sieve slice by slice (bench.py) zeroes the slice,
 * runs its own shard of it, and all-reduces just the slice (each unit is owned by one rank,
 * so the sum is exact and the other units are untouched).  Errors: E_ARG if the range is not
 * inside [0, units), E_STATE / E_NCCL as lhaf_job_allreduce. */
lhaf_status lhaf_job_reset_range(lhaf_job *job, uint64_t unit_begin, uint64_t unit_end, void *stream);
lhaf_status lhaf_job_allreduce_range(lhaf_job *job, uint64_t unit_begin, uint64_t unit_end,
                                     void *stream);
lhaf_status lhaf_job_finalize(lhaf_job *job, double *out, int32_t out_is_device, void *stream);
/* Optional diagnostic: per-pattern sum_t |term_t| * 2^{1-n} (the conditioning denominator:
 * kappa = abs_sum / |lhaf|).  Valid after lhaf_job_finalize.  out: batch doubles (host). */
lhaf_status lhaf_job_abs_sum(lhaf_job *job, double *out);
/* Device pointer and byte size of the partial array (for external all-reduce). */
lhaf_status lhaf_job_partials(lhaf_job *job, void **dev_ptr, size_t *bytes);
void lhaf_job_destroy(lhaf_job *job);

/* Per-term diagnostic (S8(c) pin P14): g(t) for nt sampled term indices of pattern 0 of the
 * job, computed by the same device code as the sieve.  g_out: nt*2 doubles (host). */
lhaf_status lhaf_job_terms(lhaf_job *job, const uint64_t *t, int32_t nt, double *g_out);

/* ---- Devices and ranks ---- */
/* Select the CUDA device of this process (default 0, or LHAF_DEVICE env). */
lhaf_status lhaf_set_device(int32_t device);
/* Multi-rank (one process per GPU; "each term in the sum can be computed
 * independently", S8(e)).  Rank 0 calls lhaf_get_unique_id and broadcasts the 128 bytes (e.g.
 * through torch.distributed); every rank then calls lhaf_init_rank.  NCCL is loaded at run
 * time (dlopen of libnccl.so.2).  nranks = 1 with id128 = NULL: a single rank without NCCL;
 * nranks = 1 with an id: a one-rank NCCL communicator (the all-reduce then runs through
 * ncclAllReduce exactly as with N ranks -- used to exercise that path on one GPU).
 * Errors: E_ARG (rank outside [0, nranks), null id for nranks > 1), E_NCCL (dlopen or
 * communicator creation failed; the context falls back to a single rank). */
lhaf_status lhaf_get_unique_id(void *id128);
lhaf_status lhaf_init_rank(int32_t rank, int32_t nranks, const void *id128, int32_t device);
lhaf_status lhaf_rank_info(int32_t *rank, int32_t *nranks);
/* The contiguous block of work units [*begin, *end) that rank `rank` of `nranks` evaluates
 * out of `units` (S8(e): units are rank-independent, so results are bit-identical for any
 * nranks).  Host-only integer arithmetic. */
lhaf_status lhaf_shard_units(uint64_t units, int32_t rank, int32_t nranks, uint64_t *begin,
                             uint64_t *end);

/* Precision of the per-term arithmetic ("Precise mode"; the paper's
 * accuracy discussion P:139-140).  0 (default): every stage in FP64.  1 (precise): the
 * Hessenberg reduction stays FP64, the characteristic-polynomial recursion (La Budde) and the
 * power series run in double-double -- the stages that dominate the per-term rounding error --
 * on the v5 kernel (bordered size E <= 64; larger jobs fail with E_TOO_LARGE); mixed states
 * are then planned by the natural pairing (i, i+k) (reading C11), whose sieve cancels ~100x
 * less than the greedy matching of the doubled pattern once its terms are accurate.  Cost: see
 * DESIGN.md.  Applies to jobs created afterwards.  lhaf_rpt_cutoff keeps FP64.
 * Errors: E_ARG for another mode. */
lhaf_status lhaf_set_precision(int32_t mode);
int32_t lhaf_get_precision(void);

/* Kernel override for experiments and cross-checks: 0 = automatic (the tree, variant 6, for
 * plain sieves in FP64 mode; v3 for the per-term paths), 1 = the Householder baseline
 * (lhaf_kernels.cu), 3 = v3, 5 = v5 for bordered sizes 33 <= E <= 64 (v3 below), 6 = the
 * prefix-sharing tree (lhaf_tree.cu; plain sieves -- cutoff groups, inclusion/exclusion and
 * gamma-batched jobs keep their per-term kernels) -- four independent codes of the same sum
 * (DESIGN.md sections 2-3).  Errors: E_ARG for any other id. */
lhaf_status lhaf_set_kernel(int32_t variant);

const char *lhaf_last_error(void);
const char *lhaf_version(void);
/* Number of CUDA kernel launches the library has issued in this process (all entry points,
 * all streams) -- a host counter, incremented at every launch site.  Never fails. */
uint64_t lhaf_launch_count(void);
void lhaf_shutdown(void);

#ifdef __cplusplus
}
#endif
#endif /* LHAF_H_ */
