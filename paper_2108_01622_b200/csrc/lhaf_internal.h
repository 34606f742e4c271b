// lhaf_internal.h -- structures shared by the host planner (lhaf_host.cpp) and the sm_100a
// kernels (lhaf_kernels.cu).  Product code only: the oracle (oracle/) never includes this.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include <atomic>
#include <vector>

namespace lhaf {

// kernel launches issued by the library (lhaf_launch_count; bench.py's gpu_launches)
extern std::atomic<unsigned long long> g_launches;

// One pattern of a job.  All offsets index the job's device pools.
struct PatDesc {
  int32_t d;           // reduced dimension 2H (0 when N = 0)
  int32_t H;           // pairs incl. phantom
  int32_t n;           // lambda degree = sum eta
  int32_t flags;       // bit 0: loop vector nonzero (loop terms present)
  uint64_t T_eval;     // evaluated terms floor(T/2)
  uint64_t chunk;      // terms per work unit
  uint64_t unit_begin; // first global work unit of this pattern
  uint64_t units;      // number of work units
  int32_t idx_off;     // ipool: r[d] (mode index of reduced row a; -1 = phantom)
  int32_t eta_off;     // ipool: eta[H]
  int32_t bin_off;     // dpool: for pair h, C(eta_h, k) k = 0..eta_h, concatenated
  int32_t radix_off;   // upool: R_h = prod_{h' < h} (eta_h' + 1)
  int64_t mat_off;     // cpool (double2): Ct[d*d] | uh[d] | v[d] | beta[1]
  int64_t gamma_off;   // offset (in complex entries) of this pattern's gamma row
  // FLAG_CUT (cutoff group, App. B.5): the last pair is the batched self-pair; its digit
  // j in [0, 2 eta_b] gives w = j - eta_b; outputs m = 0..eta_b (count 2m + parity) go to
  // partials[part_base + m * units + unit - unit_begin]
  int32_t eta_b;
  int32_t out_exp;     // extra power-of-two exponent of the result (input scaling, see lhaf_host.cpp)
  int64_t part_base;
};

constexpr uint32_t FLAG_LOOP = 1u;
constexpr uint32_t FLAG_CUT = 2u;
// FLAG_ET: inclusion/exclusion over pair copies (ET) instead of the +-1 sieve:
// w_h = eta_h - k_h, no halving, no 2^{-n} prefactor
constexpr uint32_t FLAG_ET = 4u;
// FLAG_MG: gamma-batched evaluation (lhaf_rpt_multigamma): eta_b holds the number G of loop
// vectors (rows of the job's gamma array, stride kdim); partials per loop vector at
// part_base + g * units + unit - unit_begin
constexpr uint32_t FLAG_MG = 8u;
constexpr int LHAF_MAX_GAMMA = 16;
// FLAG_FULL: no halving (every eta even, so no pair has an odd digit count): the whole term
// range is evaluated and the prefactor is 2^{-n} instead of 2^{1-n} (variant 6)
constexpr uint32_t FLAG_FULL = 16u;

// Chunk partial: double-double complex sum of the unit's terms + sum |term|.
struct Partial {
  double re_hi, re_lo, im_hi, im_lo;
  double abs_hi, abs_lo;
  double pad0, pad1;
};

struct JobDev {
  const PatDesc *descs;
  int32_t npat;
  const int32_t *ipool;
  const double *dpool;
  const uint64_t *upool;
  double2 *cpool;
  const double2 *A;      // k x k (or 2k x 2k) matrix
  const double2 *gamma;  // gamma rows
  int32_t kdim;          // row length of A (k, or 2k for mixed)
  Partial *partials;
  unsigned long long *counter;
};

// Launchers (lhaf_kernels.cu).  Return cudaError_t of the launch.
cudaError_t launch_prep(const JobDev &job, int d_max, cudaStream_t s);
cudaError_t launch_sieve(const JobDev &job, int variant, int d_max, int n_max,
                         uint64_t unit_begin, uint64_t unit_end, int num_sms, cudaStream_t s);
cudaError_t launch_finalize(const JobDev &job, double2 *out, double *abs_out, cudaStream_t s);
cudaError_t launch_terms(const JobDev &job, int variant, int d_max, int n_max, const uint64_t *t,
                         int nt, double2 *g_out, cudaStream_t s);
// Algorithmic FP64 flops per term of a variant at (d, n) -- DESIGN.md "Roofline".
double flops_per_term(int variant, int d, int n, bool loops);
int choose_variant(int d_max, int n_max);

// The bordered column-swapped matrix B0 of every pattern (prep of variants 3 and 5).
// e_max = max over patterns of d + (loops ? 1 : 0); ntl_max = max of min(n + (loops ? 2 : 1), E + 1).
int bordered_supported(int e_max, int n_max);
cudaError_t launch_prep_bordered(const JobDev &job, cudaStream_t s);

// Variant 3 (lhaf_v3.cu): branch-free fused per-column body, band + trailing La Budde.
// Uses the bordered column-swapped B0 of launch_prep_bordered.
cudaError_t launch_sieve_v3(const JobDev &job, int e_max, int ntl_max, int n_max, uint64_t unit_begin,
                            uint64_t unit_end, int num_sms, cudaStream_t s);
// cutoff groups (FLAG_CUT patterns): one term serves every count of the batched mode
cudaError_t launch_sieve_cut_v3(const JobDev &job, int e_max, int ntl_max, int n_max,
                                uint64_t unit_begin, uint64_t unit_end, int num_sms, cudaStream_t s);
cudaError_t launch_terms_v3(const JobDev &job, int e_max, int ntl_max, int n_max, const uint64_t *t,
                            int nt, double2 *g_out, cudaStream_t s);
double v3_flops_per_term(int d, int n, bool loops);

// Variant 5 (lhaf_v5.cu): 2-D register tile per lane, one barrier per column, 8 warps per team;
// bordered sizes 33 <= E <= 64.  Same prep (launch_prep_bordered) and flop model as v3.
int v5_supported(int e_max);
// FLAG_MG jobs (one pattern, d + G <= 64, G <= LHAF_MAX_GAMMA)
cudaError_t launch_sieve_mg_v5(const JobDev &job, int e_max, int g_max, int n_max, uint64_t unit_begin,
                               uint64_t unit_end, int num_sms, cudaStream_t s);
// prec = 1: the precise tail (double-double La Budde and series, lhaf_dd.cuh)
cudaError_t launch_sieve_v5(const JobDev &job, int e_max, int ntl_max, int n_max, uint64_t unit_begin,
                            uint64_t unit_end, int num_sms, cudaStream_t s, int prec);
cudaError_t launch_terms_v5(const JobDev &job, int e_max, int ntl_max, int n_max, const uint64_t *t,
                            int nt, double2 *g_out, cudaStream_t s, int prec);

// Variant 6 (lhaf_tree.cu): the sieve terms of a pattern as the leaves of a tree that shares
// every prefix of eliminated pairs (symmetric 2x2-block Schur complements of power series).
namespace tree {
struct TLevel {   // the nodes of one depth: K[(node * NE + e) * L + s], logc[node * L + s]
  double2 *K;
  double2 *logc;
  double *coef;   // sign * prod C(eta, k) of the node's path
  uint64_t cap;
};
}  // namespace tree
struct TreeGroup {            // patterns that share one tree shape
  int H = 0, n = 0, bord = 0, halve = 1, k_u = 0, npat = 0;
  int wmul = 2;               // digit k -> weight eta - wmul k (2: the sieve; 1: inclusion/exclusion)
  int cut_eb = -1;            // >= 0: cutoff group (FLAG_CUT, one pattern): the leaf pair is the
                              // batched self-pair, weights w_b = (eta - 2k) / 2 in [-eta_b, eta_b]
  int nf = 0;                 // cutoff group: the fixed pairs' degree (count 2m + p at nf + m)
  uint64_t part_base = 0;     // cutoff group: first partial (count m at part_base + m * units_pp)
  std::vector<int> eta;       // tree order: pair H-1 is eliminated first (depth 0)
  std::vector<int32_t> pats;  // job pattern indices, in unit order
  int32_t *d_pats = nullptr;
  uint64_t unit_base = 0;     // first job unit of the group
  uint64_t units_pp = 0;      // units per pattern = nodes at depth k_u
};
struct TreeWork {             // device buffers of the tree driver, kept across calls
  static constexpr size_t kLevelBudget = (size_t)512 << 20;  // bytes per depth
  std::vector<tree::TLevel> lv;
  std::vector<size_t> kbytes, lbytes, cbytes;
  // per depth: node-level series of the next pivot (Delta; at the last depth Delta, P, N0)
  std::vector<void *> aux;
  std::vector<size_t> abytes;
  void *scratch = nullptr, *val = nullptr, *absv = nullptr;
  size_t scratch_bytes = 0, val_bytes = 0, abs_bytes = 0;
};
void tree_plan_group(TreeGroup &g, uint64_t target_units);
double tree_cmacs_per_term(const TreeGroup &g);
// group-local units [ub, ue) of group g (their partials at g.unit_base + u)
cudaError_t tree_run(const JobDev &J, TreeGroup &g, TreeWork &w, uint64_t ub, uint64_t ue, cudaStream_t st);
void tree_work_free(TreeWork &w);

// sets lhaf_last_error() for entry points outside lhaf_host.cpp (returns its status argument)
int set_error(int status, const char *msg);

}  // namespace lhaf
