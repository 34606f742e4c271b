// lhaf_host.cpp -- C-ABI of include/lhaf.h: validation, greedy matching, term plans, work
// units, device orchestration and the multi-rank NCCL exchange.  All floating-point work of
// the method runs in the sm_100a kernels (lhaf_kernels.cu); this file does integer planning,
// memory management and launches only.  Product code: shares nothing with oracle/.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/lhaf.h"
#include "lhaf_internal.h"

using namespace lhaf;

namespace {

thread_local std::string g_err;
std::recursive_mutex g_mu;

lhaf_status fail(lhaf_status s, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}

#define CUDA_TRY(x)                                                                     \
  do {                                                                                  \
    cudaError_t e_ = (x);                                                               \
    if (e_ != cudaSuccess) return fail(LHAF_E_CUDA, "%s: %s", #x, cudaGetErrorString(e_)); \
  } while (0)

// Device memory for jobs comes from the device's default stream-ordered pool, configured in
// ensure_device() to keep freed memory (no release threshold): creating and destroying a job
// per call (lhaf_rpt*, the e2e path) then reuses pool memory instead of mapping new pages.
template <class T>
cudaError_t dmalloc(T **p, size_t bytes) {
  return cudaMallocAsync((void **)p, bytes, 0);
}
inline void dfree(void *p) {
  if (p) cudaFreeAsync(p, 0);
}

// ------------------------------------------------------------------ NCCL (dlopen)
struct Nccl {
  void *h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char *(*GetErrorString)(ncclResult_t) = nullptr;
  bool load() {
    if (h) return true;
    const char *names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char *nm : names) {
      h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
      if (h) break;
    }
    if (!h) return false;
    GetUniqueId = (decltype(GetUniqueId))dlsym(h, "ncclGetUniqueId");
    CommInitRank = (decltype(CommInitRank))dlsym(h, "ncclCommInitRank");
    AllReduce = (decltype(AllReduce))dlsym(h, "ncclAllReduce");
    CommDestroy = (decltype(CommDestroy))dlsym(h, "ncclCommDestroy");
    GetErrorString = (decltype(GetErrorString))dlsym(h, "ncclGetErrorString");
    return GetUniqueId && CommInitRank && AllReduce && CommDestroy && GetErrorString;
  }
};

struct Ctx {
  int device = -1;
  int num_sms = 0;
  int variant = 0;
  int precision = 0;  // 0: FP64 per term; 1: precise (double-double La Budde + series, v5)
  int rank = 0, nranks = 1;
  ncclComm_t comm = nullptr;
  Nccl nccl;
  uint64_t max_terms = (uint64_t)1 << 40;
};
Ctx g_ctx;

lhaf_status ensure_device() {
  if (g_ctx.device >= 0) {
    CUDA_TRY(cudaSetDevice(g_ctx.device));
    return LHAF_OK;
  }
  int dev = 0;
  if (const char *e = getenv("LHAF_DEVICE")) dev = atoi(e);
  int count = 0;
  cudaError_t ce = cudaGetDeviceCount(&count);
  if (ce != cudaSuccess || count == 0)
    return fail(LHAF_E_CUDA, "no CUDA device available (%s); the library has no CPU path",
                cudaGetErrorString(ce));
  if (dev >= count) return fail(LHAF_E_CUDA, "device %d out of range (%d devices)", dev, count);
  CUDA_TRY(cudaSetDevice(dev));
  cudaDeviceProp prop;
  CUDA_TRY(cudaGetDeviceProperties(&prop, dev));
  if (prop.major != 10)
    return fail(LHAF_E_CUDA, "device %d is sm_%d%d; this build targets sm_100a only", dev,
                prop.major, prop.minor);
  g_ctx.device = dev;
  g_ctx.num_sms = prop.multiProcessorCount;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t keep = ~(uint64_t)0;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  if (const char *e = getenv("LHAF_MAX_TERMS")) g_ctx.max_terms = strtoull(e, nullptr, 10);
  return LHAF_OK;
}

// ------------------------------------------------------------------ planning (host, integer)
// Greedy matching of P:474-481 (reading C9).  Independent implementation from oracle/.
struct Plan {
  int N = 0, H = 0, d = 0, n = 0, leftover = -1;
  uint64_t T = 1, T_eval = 0;
  std::vector<int> p, q, eta;  // q = -1 for the phantom
  int eta_b = -1;              // >= 0: cutoff group (FLAG_CUT), the last pair is batched
  bool et = false;             // inclusion/exclusion (FLAG_ET): T_eval = T
  int mg = 0;                  // > 0: gamma-batched evaluation of mg loop vectors (FLAG_MG)
};

lhaf_status make_plan(const int32_t *reps, int k, int mixed, Plan &P) {
  P = Plan();
  long N = 0;
  for (int i = 0; i < k; ++i) {
    if (reps[i] < 0) return fail(LHAF_E_ARG, "reps[%d] = %d < 0", i, reps[i]);
    N += reps[i];
  }
  if (mixed) N *= 2;
  if (N > 4 * LHAF_MAX_DEGREE) return fail(LHAF_E_TOO_LARGE, "N = %ld photons too large", N);
  P.N = (int)N;
  // precise mode plans mixed states by the natural pairing (lhaf_set_precision, reading C11)
  if ((mixed == 1 || mixed == 3) && g_ctx.precision == 1) mixed = 2;
  if (mixed == 1 || mixed == 3) {  // (3: the matching search needs A: job_create_impl)
    // mixed state, default: the greedy matching of the doubled pattern (reps, reps) over the
    // 2k modes (the same lhaf as the natural pairing; far better conditioned in FP64 -- the
    // BASELINE cfg5 sum is rounding noise with the natural pairing)
    std::vector<int32_t> r2(2 * (size_t)k);
    for (int i = 0; i < k; ++i) r2[i] = r2[i + k] = reps[i];
    lhaf_status s = make_plan(r2.data(), 2 * k, 0, P);
    P.N = (int)N;
    return s;
  }
  if (mixed) {  // mixed == 2: the natural pairing (i, i+k) x reps_i of P:425-428
    for (int i = 0; i < k; ++i)
      if (reps[i] > 0) { P.p.push_back(i); P.q.push_back(i + k); P.eta.push_back(reps[i]); }
  } else {
    struct Item { int n, m; };
    std::vector<Item> v;
    for (int i = 0; i < k; ++i)
      if (reps[i] > 0) v.push_back({reps[i], i});
    for (;;) {
      long tot = 0;
      for (auto &it : v) tot += it.n;
      if (tot <= 1) {
        if (tot == 1) P.leftover = v[0].m;
        break;
      }
      std::sort(v.begin(), v.end(), [](const Item &a, const Item &b) {
        return a.n != b.n ? a.n > b.n : a.m < b.m;  // step 1: descending n, ties: lower mode first
      });
      const int n1 = v[0].n, n2 = v.size() > 1 ? v[1].n : 0;
      if (n1 >= 2 * n2) {  // step 2: self pairs (m1, m1) x floor(n1/2)
        P.p.push_back(v[0].m); P.q.push_back(v[0].m); P.eta.push_back(n1 / 2);
        v[0].n -= 2 * (n1 / 2);
      } else {             // (m1, m2) x n2
        P.p.push_back(v[0].m); P.q.push_back(v[1].m); P.eta.push_back(n2);
        v[0].n -= n2; v[1].n -= n2;
      }
      v.erase(std::remove_if(v.begin(), v.end(), [](const Item &a) { return a.n == 0; }), v.end());
    }
    if (P.leftover >= 0) { P.p.push_back(P.leftover); P.q.push_back(-1); P.eta.push_back(1); }
  }
  P.H = (int)P.eta.size();
  if (P.H > LHAF_MAX_PAIRS) return fail(LHAF_E_TOO_LARGE, "H = %d pairs > %d", P.H, LHAF_MAX_PAIRS);
  P.d = 2 * P.H;
  long n = 0;
  for (int e : P.eta) n += e;
  P.n = (int)n;
  P.T = 1;
  for (int e : P.eta) {
    const uint64_t r = (uint64_t)e + 1;
    if (P.T > (~(uint64_t)0) / r) return fail(LHAF_E_TOO_LARGE, "term count overflows 64 bits");
    P.T *= r;
  }
  P.T_eval = P.H > 0 ? P.T / 2 : 0;
  return LHAF_OK;
}

lhaf_status check_plan_limits(const Plan &P) {
  if (P.d > LHAF_MAX_DIM) return fail(LHAF_E_TOO_LARGE, "reduced dimension d = %d > %d", P.d, LHAF_MAX_DIM);
  if (P.n > LHAF_MAX_DEGREE) return fail(LHAF_E_TOO_LARGE, "degree n = %d > %d", P.n, LHAF_MAX_DEGREE);
  if (P.T_eval > g_ctx.max_terms)
    return fail(LHAF_E_TOO_LARGE, "%llu terms > guard %llu (LHAF_MAX_TERMS)",
                (unsigned long long)P.T_eval, (unsigned long long)g_ctx.max_terms);
  return LHAF_OK;
}

// Tree order of the pairs (variant 6): the pair eliminated first (tree index H-1, depth 0) has
// an odd eta -- the smallest odd one -- so that halving (reading C6) keeps the first (eta+1)/2
// digits of the root; the others follow by descending eta, so that the pairs with the most
// digits are eliminated last, where the matrices are smallest.  Any order gives the same lhaf
// (every matching does; the sieve sum does not depend on the order of its pairs).
// Returns false (no halving) when every eta is even.
bool tree_order(Plan &P) {
  const int H = P.H;
  // cutoff groups: the batched self-pair (the plan's last pair) is eliminated last -- tree index
  // 0, the leaf level, where one series serves every count -- and never halves
  const int batched = P.eta_b >= 0 ? H - 1 : -1;
  int root = -1;
  for (int h = 0; h < H; ++h)
    if (h != batched && (P.eta[h] & 1) && (root < 0 || P.eta[h] < P.eta[root])) root = h;
  std::vector<int> rest;
  for (int h = 0; h < H; ++h)
    if (h != root && h != batched) rest.push_back(h);
  std::stable_sort(rest.begin(), rest.end(), [&](int a, int b) { return P.eta[a] > P.eta[b]; });
  if (batched >= 0) rest.insert(rest.begin(), batched);
  if (root >= 0) rest.push_back(root);
  std::vector<int> p(H), q(H), eta(H);
  for (int t = 0; t < H; ++t) { p[t] = P.p[rest[t]]; q[t] = P.q[rest[t]]; eta[t] = P.eta[rest[t]]; }
  P.p = p; P.q = q; P.eta = eta;
  return root >= 0;
}

lhaf_status check_symmetric(const double *A, int m) {
  double amax = 0.0, dmax = 0.0;
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < m; ++j) {
      const double *a = A + 2 * ((size_t)i * m + j), *b = A + 2 * ((size_t)j * m + i);
      if (!std::isfinite(a[0]) || !std::isfinite(a[1]))
        return fail(LHAF_E_ARG, "A[%d][%d] is not finite", i, j);
      amax = std::max(amax, std::hypot(a[0], a[1]));
      dmax = std::max(dmax, std::hypot(a[0] - b[0], a[1] - b[1]));
    }
  if (dmax > 1e-12 * std::max(1.0, amax))
    return fail(LHAF_E_NOT_SYMMETRIC, "max|A - A^T| = %.3e > 1e-12 * max(1, max|A|)", dmax);
  return LHAF_OK;
}

uint64_t chunk_for(uint64_t T_eval, bool small_job) {
  // Terms per work unit: T_eval split into at most 2^17 units of >= 64 terms (independent
  // of the number of ranks, so results are bit-identical for any rank count; small enough
  // units that a 1/64 slice of a 2^29-term lhaf still spreads over every SM).  LHAF_MAX_UNITS
  // overrides the unit cap (profiling runs use small units to fill the GPU with few terms).
  static const uint64_t max_units = [] {
    const char *e = getenv("LHAF_MAX_UNITS");
    const uint64_t v = e ? strtoull(e, nullptr, 10) : 0;
    return v ? v : (uint64_t)131072;
  }();
  // small jobs (< 2^16 terms in all: latency-bound) get 16-term units so that they spread
  // over every SM; others keep >= 64 terms per unit to amortise the unit fetch and partials
  const uint64_t min_chunk = small_job ? 16 : 64;
  uint64_t c = (T_eval + max_units - 1) / max_units;
  if (c < min_chunk) c = min_chunk;
  if (c > T_eval) c = T_eval;
  return c;
}

}  // namespace

int lhaf::set_error(int status, const char *msg) {
  g_err = msg;
  return status;
}

// ------------------------------------------------------------------ job
struct lhaf_job {
  int batch = 0, kdim = 0, d_max = 0, n_max = 0, variant = 1, prec = 0;
  int scale_s = 0;  // exact input scaling 2^s per photon (results multiplied back by 2^{-sN})
  int e_max = 0, ntl_max = 0;   // bordered dimension E and leading coefficients NTL
  bool any_loop = false;
  uint64_t units = 0, terms = 0, plan_bytes = 0;
  uint64_t parts = 0;  // partial records (= units, except cutoff groups: (eta_b + 1) per unit)
  std::vector<PatDesc> descs;
  // device
  PatDesc *d_descs = nullptr;
  int32_t *d_ipool = nullptr;
  double *d_dpool = nullptr;
  uint64_t *d_upool = nullptr;
  double2 *d_cpool = nullptr;
  double2 *d_A = nullptr, *d_gamma = nullptr;
  bool own_inputs = true;
  Partial *d_partials = nullptr;
  unsigned long long *d_counter = nullptr;
  double2 *d_out = nullptr;
  double *d_abs = nullptr;
  // variant 6: one tree per group of patterns of the same shape
  std::vector<TreeGroup> groups;
  TreeWork tw;
  std::vector<Plan> plans;  // per pattern, in the job's evaluation order (lhaf_job_plan)
  double tree_flops = 0.0;
  JobDev dev() const {
    JobDev J;
    J.descs = d_descs; J.npat = batch; J.ipool = d_ipool; J.dpool = d_dpool; J.upool = d_upool;
    J.cpool = d_cpool; J.A = d_A; J.gamma = d_gamma; J.kdim = kdim; J.partials = d_partials;
    J.counter = d_counter;
    return J;
  }
};

static void job_free(lhaf_job *j) {
  if (!j) return;
  cudaDeviceSynchronize();  // work on any stream may still use the buffers (as cudaFree did)
  dfree(j->d_descs); dfree(j->d_ipool); dfree(j->d_dpool); dfree(j->d_upool);
  dfree(j->d_cpool);
  if (j->own_inputs) { dfree(j->d_A); dfree(j->d_gamma); }
  dfree(j->d_partials); dfree(j->d_counter); dfree(j->d_out); dfree(j->d_abs);
  for (auto &g : j->groups) dfree(g.d_pats);
  tree_work_free(j->tw);
  delete j;
}

template <class T>
static cudaError_t upload(T **dst, const std::vector<T> &v) {
  const size_t bytes = std::max<size_t>(1, v.size()) * sizeof(T);
  cudaError_t e = dmalloc(dst, bytes);
  if (e != cudaSuccess) return e;
  if (!v.empty()) e = cudaMemcpy(*dst, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice);
  return e;
}

static lhaf_status mixed_kappa_plan(const double *A2, const double *g2, const int32_t *reps, int k,
                                    Plan &best, double *best_est);
static lhaf_status job_create_impl(const double *A, const double *gamma, int64_t gamma_stride,
                                   const int32_t *reps, int k, int batch, int mixed, bool on_device,
                                   lhaf_job **out, const std::vector<Plan> *plans_in = nullptr) {
  if (!A || !gamma || (!reps && !plans_in) || !out) return fail(LHAF_E_ARG, "null pointer argument");
  if (k < 0 || k > LHAF_MAX_MODES) return fail(LHAF_E_ARG, "k = %d out of range", k);
  if (batch < 0) return fail(LHAF_E_ARG, "batch = %d < 0", batch);
  if (mixed < 0 || mixed > 3) return fail(LHAF_E_ARG, "mixed = %d (0 pure, 1 greedy doubled, 2 natural, 3 searched)", mixed);
  if (mixed == 3 && !plans_in && g_ctx.precision == 0 && !on_device && gamma_stride == 0) {
    // kappa-aware matching per pattern (mixed_kappa_plan), then the job on those plans
    std::vector<Plan> plans(batch);
    for (int b = 0; b < batch; ++b) {
      lhaf_status s0 = check_symmetric(A, 2 * k);
      if (s0 == LHAF_OK) s0 = mixed_kappa_plan(A, gamma, reps + (size_t)b * k, k, plans[b], nullptr);
      if (s0 != LHAF_OK) return s0;
    }
    return job_create_impl(A, gamma, 0, nullptr, k, batch, 1, false, out, &plans);
  }
  const int kdim = mixed ? 2 * k : k;
  if (gamma_stride != 0 && gamma_stride < kdim)
    return fail(LHAF_E_ARG, "gamma_stride %lld < row length %d", (long long)gamma_stride, kdim);
  lhaf_status s = ensure_device();
  if (s != LHAF_OK) return s;
  if (on_device) {
    // device inputs may have been written on any stream of the caller (e.g. a torch side
    // stream): order every read below after them
    CUDA_TRY(cudaDeviceSynchronize());
    if (kdim <= 2048) {  // the same symmetry / finiteness check as for host inputs
      std::vector<double> acopy(2 * std::max<size_t>(1, (size_t)kdim * kdim));
      if (kdim > 0)
        CUDA_TRY(cudaMemcpy(acopy.data(), A, (size_t)kdim * kdim * 16, cudaMemcpyDeviceToHost));
      s = check_symmetric(acopy.data(), kdim);
      if (s != LHAF_OK) return s;
    }
  } else {
    s = check_symmetric(A, kdim);
    if (s != LHAF_OK) return s;
  }

  // host view of gamma (loop flags are planned on the host)
  int mg_rows = 0;  // FLAG_MG: the gamma array holds G rows of the job's single pattern
  if (plans_in)
    for (const Plan &Pm : *plans_in) mg_rows = std::max(mg_rows, Pm.mg);
  const size_t gamma_len = mg_rows ? (size_t)mg_rows * gamma_stride
                                   : gamma_stride ? (size_t)batch * gamma_stride : (size_t)kdim;
  std::vector<double> gcopy;
  const double *ghost = gamma;
  if (on_device) {
    gcopy.resize(2 * std::max<size_t>(1, gamma_len));
    if (gamma_len > 0 && cudaMemcpy(gcopy.data(), gamma, gamma_len * 16, cudaMemcpyDeviceToHost) != cudaSuccess)
      return fail(LHAF_E_CUDA, "reading gamma from the device failed");
    ghost = gcopy.data();
  }

  // Exact power-of-two input scaling: lhaf(4^s A, 2^s gamma) = 2^{sN} lhaf(A, gamma)
  // (each photon contributes one factor 2^s: a pair one A entry, a loop one gamma entry; the
  // phantom's loop 1 is unscaled and is always a loop).  Inputs far from unit scale are brought
  // to ~1 before upload, so that no pivot, characteristic-polynomial coefficient or series term
  // under- or overflows; the finalize multiplies by 2^{-sN}.  Host inputs only (device buffers
  // belong to the caller); |s| < 8 leaves the inputs untouched.
  int scale_s = 0;
  std::vector<double> a_scaled, g_scaled;
  if (!on_device) {
    double ma = 0.0, mg = 0.0;
    for (size_t i = 0; i < (size_t)kdim * kdim; ++i) ma = std::max(ma, std::hypot(A[2 * i], A[2 * i + 1]));
    for (size_t i = 0; i < gamma_len; ++i) mg = std::max(mg, std::hypot(ghost[2 * i], ghost[2 * i + 1]));
    const double m = std::max(std::sqrt(ma), mg);
    if (m > 0.0 && std::isfinite(m)) {
      const int s0 = -(int)std::lround(std::log2(m));
      if (std::abs(s0) >= 8 && std::abs(s0) <= 400) scale_s = s0;
    }
    if (scale_s != 0) {
      a_scaled.assign(A, A + 2 * (size_t)kdim * kdim);
      for (double &x : a_scaled) x = std::ldexp(x, 2 * scale_s);
      g_scaled.assign(ghost, ghost + 2 * gamma_len);
      for (double &x : g_scaled) x = std::ldexp(x, scale_s);
      A = a_scaled.data();
      gamma = g_scaled.data();
      ghost = g_scaled.data();
    }
  }

  // variant 6 (the prefix-sharing tree) evaluates plain sieves and inclusion/exclusion: not the
  // cutoff groups or the gamma-batched jobs (their own kernels), not precise mode.  By default a
  // job with fewer than LHAF_TREE_MIN_TERMS (65536) evaluated terms runs the per-term v3 kernel
  // instead: the tree's cost there is the latency of its many small per-level launches (BASELINE
  // cfg3, 7200 terms: 0.67 ms on the tree, 0.18 ms per term).
  bool use_tree = g_ctx.variant == 6 || (g_ctx.variant == 0 && g_ctx.precision == 0);
  if (plans_in)
    for (const Plan &Pm : *plans_in)
      if (Pm.mg > 0 || (Pm.eta_b >= 0 && (Pm.n + 1 > 40 || getenv("LHAF_CUTOFF_PER_TERM")))) use_tree = false;
  if (use_tree && g_ctx.variant == 0) {
    static const uint64_t min_terms = [] {
      const char *e = getenv("LHAF_TREE_MIN_TERMS");
      return e ? strtoull(e, nullptr, 10) : (uint64_t)65536;
    }();
    uint64_t tot = 0;
    for (int b = 0; b < batch && tot < min_terms; ++b) {
      Plan P;
      if (plans_in) P = (*plans_in)[b];
      else if (make_plan(reps + (size_t)b * k, k, mixed, P) != LHAF_OK) break;  // reported below
      tot += P.et ? P.T : P.T_eval;
    }
    if (tot < min_terms) use_tree = false;
  }

  lhaf_job *j = new lhaf_job();
  j->batch = batch;
  j->kdim = kdim;
  j->scale_s = scale_s;
  j->variant = 1;
  std::vector<int32_t> ipool;
  std::vector<double> dpool;
  std::vector<uint64_t> upool;
  int64_t cpool_words = 0;
  uint64_t unit = 0, part = 0;
  // the job's total term count decides the unit size (a function of the job only: results
  // stay independent of the rank count)
  bool small_job = true;
  {
    uint64_t tot = 0;
    for (int b = 0; b < batch && small_job; ++b) {
      Plan P;
      if (plans_in) P = (*plans_in)[b];
      else if (make_plan(reps + (size_t)b * k, k, mixed, P) != LHAF_OK) break;  // reported below
      tot += P.T_eval;
      if (tot >= 65536) small_job = false;
    }
  }
  j->descs.resize(batch);
  for (int b = 0; b < batch; ++b) {
    Plan P;
    if (plans_in) {
      P = (*plans_in)[b];
      s = LHAF_OK;
    } else {
      s = make_plan(reps + (size_t)b * k, k, mixed, P);
    }
    bool full = false;
    if (s == LHAF_OK && use_tree && P.H > 0 && !tree_order(P) && !P.et) {
      full = true;       // every eta even: no halving, the whole range [0, T)
      P.T_eval = P.T;
    }
    if (s == LHAF_OK) s = check_plan_limits(P);
    if (s != LHAF_OK) { job_free(j); return s; }
    j->plans.push_back(P);
    PatDesc &D = j->descs[b];
    memset(&D, 0, sizeof D);
    D.d = P.d; D.H = P.H; D.n = P.n; D.flags = full ? FLAG_FULL : 0;
    if (P.mg > 0) {
      // gamma-batched: M alone is reduced (no border); the loop vectors ride along (v5 MG)
      D.flags |= FLAG_MG;
      D.eta_b = P.mg;
      if (P.H > 0) {
        j->e_max = std::max(j->e_max, P.d);
        j->ntl_max = std::max(j->ntl_max, std::min(P.n + 1, P.d + 1));
      }
    } else {
      bool loops = P.leftover >= 0;  // the phantom carries loop weight 1 (reading C7)
      const double *gb = ghost + 2 * (size_t)(gamma_stride ? (size_t)b * gamma_stride : 0);
      for (int h = 0; h < P.H && !loops; ++h)
        for (int side = 0; side < 2 && !loops; ++side) {
          const int m = side ? P.q[h] : P.p[h];
          if (m >= 0 && (gb[2 * m] != 0.0 || gb[2 * m + 1] != 0.0)) loops = true;
        }
      if (loops) D.flags |= FLAG_LOOP;
      if (P.H > 0) {
        const int E = P.d + (loops ? 1 : 0);
        j->e_max = std::max(j->e_max, E);
        j->ntl_max = std::max(j->ntl_max, std::min(P.n + (loops ? 2 : 1), E + 1));
        j->any_loop |= loops;
      }
    }
    D.T_eval = P.T_eval;
    D.out_exp = -scale_s * P.N;  // the photons of this pattern (for mixed: of the 2N x 2N matrix)
    D.gamma_off = gamma_stride ? (int64_t)b * gamma_stride : 0;
    D.unit_begin = unit;
    D.part_base = (int64_t)part;
    if (P.H == 0 || P.T_eval == 0) { D.chunk = 0; D.units = 0; continue; }
    if (P.et) D.flags |= FLAG_ET;
    if (P.eta_b >= 0) {  // cutoff group: eta_b + 1 partials per unit, at most 4096 units
      D.flags |= FLAG_CUT;
      D.eta_b = P.eta_b;
      D.chunk = std::max<uint64_t>(64, (P.T_eval + 4095) / 4096);
      if (D.chunk > P.T_eval) D.chunk = P.T_eval;
    } else {
      D.chunk = use_tree ? 0 : chunk_for(P.T_eval, small_job);
    }
    D.units = use_tree ? 0 : (P.T_eval + D.chunk - 1) / D.chunk;  // tree jobs: units below
    unit += D.units;
    part += D.units * (uint64_t)(P.mg > 0 ? P.mg : P.eta_b >= 0 ? P.eta_b + 1 : 1);
    j->terms += P.T_eval;
    j->d_max = std::max(j->d_max, P.d);
    j->n_max = std::max(j->n_max, P.n);
    // index list r = (p_1..p_H, q_1..q_H)
    D.idx_off = (int32_t)ipool.size();
    for (int h = 0; h < P.H; ++h) ipool.push_back(P.p[h]);
    for (int h = 0; h < P.H; ++h) ipool.push_back(P.q[h]);
    D.eta_off = (int32_t)ipool.size();
    for (int h = 0; h < P.H; ++h) ipool.push_back(P.eta[h]);
    int acc = 0;
    for (int h = 0; h < P.H; ++h) { ipool.push_back(acc); acc += P.eta[h] + 1; }
    D.bin_off = (int32_t)dpool.size();
    for (int h = 0; h < P.H; ++h) {
      long double c = 1.0L;
      for (int kk = 0; kk <= P.eta[h]; ++kk) {
        dpool.push_back((double)c);
        c = c * (long double)(P.eta[h] - kk) / (long double)(kk + 1);
      }
    }
    D.radix_off = (int32_t)upool.size();
    uint64_t R = 1;
    for (int h = 0; h < P.H; ++h) { upool.push_back(R); R *= (uint64_t)(P.eta[h] + 1); }
    D.mat_off = cpool_words;
    cpool_words += (int64_t)(P.d + 1) * (P.d + 1) + 2 * P.d + 2;  // v1: Ct|uh|v|beta; v3/v5: E x E
  }
  if (use_tree) {
    // groups of patterns with the same tree shape; each group's units are contiguous
    std::vector<std::vector<int>> keys;
    for (int b = 0; b < batch; ++b) {
      const PatDesc &D = j->descs[b];
      if (D.H == 0 || D.T_eval == 0) continue;
      const bool et = (D.flags & FLAG_ET) != 0;
      std::vector<int> key = {D.H, D.n, (D.flags & FLAG_LOOP) ? 1 : 0, (D.flags & (FLAG_FULL | FLAG_ET)) ? 0 : 1,
                              et ? 1 : 0};
      for (int h = 0; h < D.H; ++h) key.push_back(ipool[D.eta_off + h]);
      if (D.flags & FLAG_CUT) { key.push_back(-1 - b); key.push_back(D.eta_b); }  // one pattern per cutoff group
      size_t gi = 0;
      while (gi < keys.size() && keys[gi] != key) ++gi;
      if (gi == keys.size()) {
        keys.push_back(key);
        TreeGroup g;
        g.H = D.H; g.n = D.n; g.bord = key[2]; g.halve = key[3];
        g.wmul = key[4] ? 1 : 2;  // inclusion/exclusion: w = eta - k; sieve: eta - 2k
        g.eta.assign(key.begin() + 5, key.begin() + 5 + D.H);
        if (D.flags & FLAG_CUT) { g.cut_eb = D.eta_b; g.nf = D.n - D.eta_b; }
        j->groups.push_back(g);
      }
      j->groups[gi].pats.push_back(b);
    }
    for (auto &g : j->groups) {
      g.npat = (int)g.pats.size();
      tree_plan_group(g, 65536);
      g.unit_base = unit;
      g.part_base = part;
      for (int32_t pb : g.pats) {
        PatDesc &D = j->descs[pb];
        D.unit_begin = unit;
        D.units = g.units_pp;
        D.chunk = D.T_eval / g.units_pp;  // leaves per unit
        D.part_base = (int64_t)part;
        unit += g.units_pp;
        part += g.units_pp * (uint64_t)(g.cut_eb >= 0 ? g.cut_eb + 1 : 1);
      }
      j->tree_flops = 8.0 * tree_cmacs_per_term(g);
    }
  }
  j->units = unit;
  j->parts = part;
  j->plan_bytes = j->descs.size() * sizeof(PatDesc) + ipool.size() * 4 + dpool.size() * 8 +
                  upool.size() * 8;
  cudaError_t e = cudaSuccess;
  if (e == cudaSuccess) e = upload(&j->d_descs, j->descs);
  if (e == cudaSuccess) e = upload(&j->d_ipool, ipool);
  if (e == cudaSuccess) e = upload(&j->d_dpool, dpool);
  if (e == cudaSuccess) e = upload(&j->d_upool, upool);
  if (e == cudaSuccess) e = dmalloc(&j->d_cpool, std::max<int64_t>(1, cpool_words) * sizeof(double2));
  if (e == cudaSuccess) e = dmalloc(&j->d_partials, std::max<uint64_t>(1, j->parts) * sizeof(Partial));
  if (e == cudaSuccess) e = cudaMemset(j->d_partials, 0, std::max<uint64_t>(1, j->parts) * sizeof(Partial));
  if (e == cudaSuccess) e = dmalloc(&j->d_counter, sizeof(unsigned long long));
  for (auto &g : j->groups)
    if (e == cudaSuccess) e = upload(&g.d_pats, g.pats);
  if (e == cudaSuccess) e = dmalloc(&j->d_out, std::max(1, batch) * sizeof(double2));
  if (e == cudaSuccess) e = dmalloc(&j->d_abs, std::max(1, batch) * sizeof(double));
  if (on_device) {
    j->own_inputs = false;
    j->d_A = (double2 *)A;
    j->d_gamma = (double2 *)gamma;
  } else {
    if (e == cudaSuccess) e = dmalloc(&j->d_A, std::max<size_t>(1, (size_t)kdim * kdim) * sizeof(double2));
    if (e == cudaSuccess) e = dmalloc(&j->d_gamma, std::max<size_t>(1, gamma_len) * sizeof(double2));
    if (e == cudaSuccess && kdim > 0)
      e = cudaMemcpy(j->d_A, A, (size_t)kdim * kdim * sizeof(double2), cudaMemcpyHostToDevice);
    if (e == cudaSuccess && gamma_len > 0)
      e = cudaMemcpy(j->d_gamma, gamma, gamma_len * sizeof(double2), cudaMemcpyHostToDevice);
  }
  j->variant = use_tree ? 6 : g_ctx.variant ? g_ctx.variant : choose_variant(j->e_max, j->n_max);
  j->prec = g_ctx.precision;
  if (j->prec && !use_tree) j->variant = 5;  // the precise tail lives in the v5 kernel (every E <= 64)
  // inclusion/exclusion: excluded pairs are deleted -- on the tree (default: a deleted
  // pair's children copy the parent's leading block) or per term on v5 (lhaf_set_kernel(5))
  if (j->variant == 0 || (j->variant == 5 && !v5_supported(j->e_max))) j->variant = 3;
  if (j->prec && j->variant != 5 && j->variant != 6) {
    job_free(j);
    return fail(LHAF_E_TOO_LARGE, "precise mode needs d <= 63 (bordered size <= 64)");
  }
  if (j->variant >= 3 && j->variant != 6 && !bordered_supported(j->e_max, j->n_max)) j->variant = 1;
  // tree jobs build their roots per run; the bordered B0 serves lhaf_job_terms (v3 per term)
  if (e == cudaSuccess && !(j->variant == 6 && !bordered_supported(j->e_max, j->n_max)))
    e = (j->variant >= 3) ? launch_prep_bordered(j->dev(), 0) : launch_prep(j->dev(), j->d_max, 0);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    job_free(j);
    return fail(LHAF_E_CUDA, "job setup: %s", cudaGetErrorString(e));
  }
  *out = j;
  return LHAF_OK;
}

static cudaError_t run_sieve(lhaf_job *j, uint64_t b, uint64_t e, cudaStream_t st) {
  if (j->variant == 6) {
    for (auto &g : j->groups) {
      const uint64_t gb = g.unit_base, ge = gb + (uint64_t)g.npat * g.units_pp;
      const uint64_t lo = std::max(b, gb), hi = std::min(e, ge);
      if (lo < hi) {
        cudaError_t r = tree_run(j->dev(), g, j->tw, lo - gb, hi - gb, st);
        if (r != cudaSuccess) return r;
      }
    }
    return cudaSuccess;
  }
  if (j->variant == 5)
    return launch_sieve_v5(j->dev(), j->e_max, j->ntl_max, j->n_max, b, e, g_ctx.num_sms, st, j->prec);
  if (j->variant == 3)
    return launch_sieve_v3(j->dev(), j->e_max, j->ntl_max, j->n_max, b, e, g_ctx.num_sms, st);
  return launch_sieve(j->dev(), j->variant, j->d_max, j->n_max, b, e, g_ctx.num_sms, st);
}

static void shard(uint64_t units, uint64_t r, uint64_t R, uint64_t &b, uint64_t &e) {
  // units * r / R without 64-bit overflow (units < 2^40 guard, R <= 2^16)
  b = (uint64_t)(((unsigned __int128)units * r) / R);
  e = (uint64_t)(((unsigned __int128)units * (r + 1)) / R);
}

static void rank_units(uint64_t units, uint64_t &b, uint64_t &e) {
  shard(units, (uint64_t)g_ctx.rank, (uint64_t)g_ctx.nranks, b, e);
}

static lhaf_status job_allreduce_impl(lhaf_job *j, cudaStream_t st) {
  // no communicator: a single rank without NCCL (nothing to exchange); a 1-rank communicator
  // (lhaf_init_rank(0, 1, id, dev) with an id) runs the same ncclAllReduce as N ranks do
  if (!g_ctx.comm && g_ctx.nranks <= 1) return LHAF_OK;
  if (j->units == 0) return LHAF_OK;
  if (!g_ctx.comm) return fail(LHAF_E_STATE, "multi-rank all-reduce without a communicator");
  const size_t count = (size_t)j->units * (sizeof(Partial) / sizeof(double));
  ncclResult_t r = g_ctx.nccl.AllReduce(j->d_partials, j->d_partials, count, ncclDouble, ncclSum,
                                        g_ctx.comm, st);
  if (r != ncclSuccess) return fail(LHAF_E_NCCL, "ncclAllReduce: %s", g_ctx.nccl.GetErrorString(r));
  return LHAF_OK;
}

static lhaf_status evaluate(lhaf_job *j, double *out_host, double *out_dev, cudaStream_t st) {
  uint64_t b, e;
  rank_units(j->units, b, e);
  CUDA_TRY(cudaMemsetAsync(j->d_partials, 0, std::max<uint64_t>(1, j->units) * sizeof(Partial), st));
  CUDA_TRY(run_sieve(j, b, e, st));
  lhaf_status s = job_allreduce_impl(j, st);
  if (s != LHAF_OK) return s;
  double2 *dst = out_dev ? (double2 *)out_dev : j->d_out;
  CUDA_TRY(launch_finalize(j->dev(), dst, j->d_abs, st));
  if (out_host)
    CUDA_TRY(cudaMemcpyAsync(out_host, dst, (size_t)j->batch * sizeof(double2), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return LHAF_OK;
}

// ------------------------------------------------------------------ kappa-aware matching
// Every matching of the repeated rows gives the same loop hafnian, but not the same
// cancellation: kappa = sum|term| / |lhaf| sets the FP64 error of the sum, and for
// the BASELINE mixed state it varies ~40x between matchings that differ only in how the greedy
// rule breaks ties.  Mixed mode 3: C candidate matchings -- the greedy matching
// of the doubled pattern with the 2k modes relabelled by seeded permutations (candidate 0 =
// the identity, i.e. mode 1) -- each estimated by evaluating S work units spread over its sieve
// (sum|term| of the sample x units / S), and the one with the smallest estimate is kept.
static uint64_t splitmix64(uint64_t &x) {
  uint64_t z = (x += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
static int env_int(const char *name, int dflt) {
  const char *e = getenv(name);
  return e ? atoi(e) : dflt;
}
static lhaf_status mixed_kappa_plan(const double *A2, const double *g2, const int32_t *reps, int k,
                                    Plan &best, double *best_est) {
  const int C = std::max(1, env_int("LHAF_KAPPA_CANDIDATES", 16));
  const int S = std::max(1, env_int("LHAF_KAPPA_SAMPLES", 8));
  const int k2 = 2 * k;
  std::vector<int32_t> r2(k2);
  for (int i = 0; i < k; ++i) r2[i] = r2[i + k] = reps[i];
  double best_abs = INFINITY;
  bool have = false;
  for (int c = 0; c < C; ++c) {
    std::vector<int> lab(k2);  // mode i gets label lab[i]
    for (int i = 0; i < k2; ++i) lab[i] = i;
    uint64_t seed = 0x5EEDull + (uint64_t)c;
    for (int i = k2 - 1; c > 0 && i > 0; --i) std::swap(lab[i], lab[splitmix64(seed) % (uint64_t)(i + 1)]);
    std::vector<int32_t> rl(k2);
    std::vector<int> inv(k2);
    for (int i = 0; i < k2; ++i) { rl[lab[i]] = r2[i]; inv[lab[i]] = i; }
    Plan P;
    lhaf_status s = make_plan(rl.data(), k2, 0, P);
    if (s != LHAF_OK) return s;
    for (int h = 0; h < P.H; ++h) {
      P.p[h] = P.p[h] >= 0 ? inv[P.p[h]] : -1;
      P.q[h] = P.q[h] >= 0 ? inv[P.q[h]] : -1;
    }
    if (P.leftover >= 0) P.leftover = inv[P.leftover];
    std::vector<Plan> plans{P};
    lhaf_job *j = nullptr;
    s = job_create_impl(A2, g2, 0, nullptr, k, 1, 1, false, &j, &plans);
    if (s != LHAF_OK) return s;
    double est = 0.0;
    if (j->units > 0) {
      const uint64_t U = j->units, n = std::min<uint64_t>(U, (uint64_t)S);
      cudaError_t e = cudaMemsetAsync(j->d_partials, 0, U * sizeof(Partial), 0);
      for (uint64_t t = 0; t < n && e == cudaSuccess; ++t) {
        const uint64_t u = (uint64_t)(((double)t + 0.5) * (double)U / (double)n);
        e = run_sieve(j, u, u + 1, 0);
      }
      if (e == cudaSuccess) e = launch_finalize(j->dev(), j->d_out, j->d_abs, 0);
      double a = 0.0;
      if (e == cudaSuccess) e = cudaMemcpy(&a, j->d_abs, sizeof(double), cudaMemcpyDeviceToHost);
      if (e != cudaSuccess) {
        job_free(j);
        return fail(LHAF_E_CUDA, "matching search: %s", cudaGetErrorString(e));
      }
      est = a * (double)U / (double)n;
    }
    job_free(j);
    if (!have || est < best_abs) { best_abs = est; best = P; have = true; }
  }
  if (best_est) *best_est = best_abs;
  return LHAF_OK;
}

// ------------------------------------------------------------------ C-ABI
extern "C" {

const char *lhaf_last_error(void) { return g_err.c_str(); }
const char *lhaf_version(void) { return "lhaf-b200 0.2 (sm_100a)"; }
uint64_t lhaf_launch_count(void) { return lhaf::g_launches.load(); }

lhaf_status lhaf_plan(const int32_t *reps, int32_t k, int32_t mixed, lhaf_plan_info *info) {
  if (!info || (k > 0 && !reps)) return fail(LHAF_E_ARG, "null pointer argument");
  if (k < 0 || k > LHAF_MAX_MODES) return fail(LHAF_E_ARG, "k = %d out of range", k);
  Plan P;
  lhaf_status s = make_plan(reps, k, mixed, P);
  if (s != LHAF_OK) return s;
  memset(info, 0, sizeof *info);
  info->N = P.N; info->H = P.H; info->d = P.d; info->n = P.n; info->leftover = P.leftover;
  info->T = P.T; info->T_eval = P.T_eval;
  for (int h = 0; h < P.H; ++h) { info->p[h] = P.p[h]; info->q[h] = P.q[h]; info->eta[h] = P.eta[h]; }
  return LHAF_OK;
}

lhaf_status lhaf_decode(const lhaf_plan_info *info, uint64_t t, int32_t *k_out, int32_t *w_out,
                        int32_t *sign_out, uint64_t *weight_out) {
  if (!info || !k_out || !w_out || !sign_out || !weight_out) return fail(LHAF_E_ARG, "null pointer");
  if (t >= info->T) return fail(LHAF_E_ARG, "t = %llu >= T", (unsigned long long)t);
  uint64_t rem = t, weight = 1;
  int ks = 0;
  for (int h = 0; h < info->H; ++h) {
    const uint64_t r = (uint64_t)info->eta[h] + 1;
    const int kd = (int)(rem % r);
    rem /= r;
    k_out[h] = kd;
    w_out[h] = info->eta[h] - 2 * kd;
    ks += kd;
    uint64_t c = 1;  // C(eta, kd), exact while it fits
    for (int i = 1; i <= kd; ++i) c = c * (uint64_t)(info->eta[h] - kd + i) / (uint64_t)i;
    weight *= c;
  }
  *sign_out = (ks & 1) ? -1 : 1;
  *weight_out = weight;
  return LHAF_OK;
}

lhaf_status lhaf_set_device(int32_t device) {
  std::lock_guard<std::recursive_mutex> lk(g_mu);
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || device < 0 || device >= count)
    return fail(LHAF_E_CUDA, "cannot select device %d", device);
  g_ctx.device = -1;
  setenv("LHAF_DEVICE", std::to_string(device).c_str(), 1);
  return ensure_device();
}

lhaf_status lhaf_set_precision(int32_t mode) {
  if (mode != 0 && mode != 1) return fail(LHAF_E_ARG, "unknown precision mode %d (0 = FP64, 1 = precise)", mode);
  g_ctx.precision = mode;
  return LHAF_OK;
}

int32_t lhaf_get_precision(void) { return g_ctx.precision; }

lhaf_status lhaf_set_kernel(int32_t variant) {
  if (variant != 0 && variant != 1 && variant != 3 && variant != 5 && variant != 6)
    return fail(LHAF_E_ARG, "unknown kernel variant %d (0 = default, 1 = Householder, 3 = v3, 5 = v5, 6 = tree)", variant);
  g_ctx.variant = variant;
  return LHAF_OK;
}

lhaf_status lhaf_job_create(const double *A, const double *gamma, int64_t gamma_stride,
                            const int32_t *reps, int32_t k, int32_t batch, int32_t mixed,
                            int32_t A_is_device, lhaf_job **job) {
  std::lock_guard<std::recursive_mutex> lk(g_mu);
  return job_create_impl(A, gamma, gamma_stride, reps, k, batch, mixed, A_is_device != 0, job);
}

lhaf_status lhaf_job_info_get(const lhaf_job *j, lhaf_job_info *info) {
  if (!j || !info) return fail(LHAF_E_ARG, "null pointer");
  info->batch = j->batch; info->d_max = j->d_max; info->n_max = j->n_max; info->kernel = j->variant;
  info->precision = j->prec;
  info->units = j->units; info->terms = j->terms; info->h2d_plan_bytes = j->plan_bytes;
  // model flops of the first non-empty pattern (batches here are uniform in d)
  info->flops_per_term_model = 0.0;
  for (const auto &D : j->descs)
    if (D.d > 0) {
      const bool lp = (D.flags & FLAG_LOOP) != 0;
      info->flops_per_term_model = (j->variant == 6)  ? j->tree_flops
                                   : (j->variant >= 3) ? v3_flops_per_term(D.d, D.n, lp)
                                                       : flops_per_term(j->variant, D.d, D.n, true);
      break;
    }
  return LHAF_OK;
}

lhaf_status lhaf_job_plan(const lhaf_job *j, int32_t pattern, lhaf_plan_info *info) {
  if (!j || !info) return fail(LHAF_E_ARG, "null pointer");
  if (pattern < 0 || pattern >= (int32_t)j->plans.size())
    return fail(LHAF_E_ARG, "pattern %d outside the job's %d", pattern, (int)j->plans.size());
  const Plan &P = j->plans[pattern];
  memset(info, 0, sizeof *info);
  info->N = P.N; info->H = P.H; info->d = P.d; info->n = P.n; info->leftover = P.leftover;
  info->T = P.T;
  info->T_eval = P.T_eval;
  for (int h = 0; h < P.H && h < LHAF_MAX_PAIRS; ++h) {
    info->p[h] = P.p[h]; info->q[h] = P.q[h]; info->eta[h] = P.eta[h];
  }
  return LHAF_OK;
}

lhaf_status lhaf_job_reset(lhaf_job *j, void *stream) {
  if (!j) return fail(LHAF_E_ARG, "null job");
  CUDA_TRY(cudaMemsetAsync(j->d_partials, 0, std::max<uint64_t>(1, j->units) * sizeof(Partial),
                           (cudaStream_t)stream));
  return LHAF_OK;
}

lhaf_status lhaf_job_reset_range(lhaf_job *j, uint64_t ub, uint64_t ue, void *stream) {
  if (!j) return fail(LHAF_E_ARG, "null job");
  if (ue > j->units || ub > ue) return fail(LHAF_E_ARG, "unit range outside the job");
  if (ue > ub)
    CUDA_TRY(cudaMemsetAsync(j->d_partials + ub, 0, (ue - ub) * sizeof(Partial), (cudaStream_t)stream));
  return LHAF_OK;
}

lhaf_status lhaf_job_allreduce_range(lhaf_job *j, uint64_t ub, uint64_t ue, void *stream) {
  std::lock_guard<std::recursive_mutex> lk(g_mu);
  if (!j) return fail(LHAF_E_ARG, "null job");
  if (ue > j->units || ub > ue) return fail(LHAF_E_ARG, "unit range outside the job");
  if (!g_ctx.comm && g_ctx.nranks <= 1) return LHAF_OK;
  if (ue == ub) return LHAF_OK;
  if (!g_ctx.comm) return fail(LHAF_E_STATE, "multi-rank all-reduce without a communicator");
  const size_t count = (size_t)(ue - ub) * (sizeof(Partial) / sizeof(double));
  ncclResult_t r = g_ctx.nccl.AllReduce(j->d_partials + ub, j->d_partials + ub, count, ncclDouble,
                                        ncclSum, g_ctx.comm, (cudaStream_t)stream);
  if (r != ncclSuccess) return fail(LHAF_E_NCCL, "ncclAllReduce: %s", g_ctx.nccl.GetErrorString(r));
  return LHAF_OK;
}

lhaf_status lhaf_job_run(lhaf_job *j, uint64_t ub, uint64_t ue, void *stream) {
  std::lock_guard<std::recursive_mutex> lk(g_mu);
  if (!j) return fail(LHAF_E_ARG, "null job");
  if (ue > j->units || ub > ue) return fail(LHAF_E_ARG, "unit range [%llu, %llu) outside [0, %llu)",
                                            (unsigned long long)ub, (unsigned long long)ue,
                                            (unsigned long long)j->units);
  lhaf_status s = ensure_device();
  if (s != LHAF_OK) return s;
  CUDA_TRY(run_sieve(j, ub, ue, (cudaStream_t)stream));
  return LHAF_OK;
}

lhaf_status lhaf_job_allreduce(lhaf_job *j, void *stream) {
  std::lock_guard<std::recursive_mutex> lk(g_mu);
  if (!j) return fail(LHAF_E_ARG, "null job");
  return job_allreduce_impl(j, (cudaStream_t)stream);
}

lhaf_status lhaf_job_finalize(lhaf_job *j, double *out, int32_t out_is_device, void *stream) {
  std::lock_guard<std::recursive_mutex> lk(g_mu);
  if (!j || !out) return fail(LHAF_E_ARG, "null pointer");
  cudaStream_t st = (cudaStream_t)stream;
  double2 *dst = out_is_device ? (double2 *)out : j->d_out;
  CUDA_TRY(launch_finalize(j->dev(), dst, j->d_abs, st));
  if (!out_is_device) {
    CUDA_TRY(cudaMemcpyAsync(out, dst, (size_t)j->batch * sizeof(double2), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
  }
  return LHAF_OK;
}

lhaf_status lhaf_job_abs_sum(lhaf_job *j, double *out) {
  if (!j || !out) return fail(LHAF_E_ARG, "null pointer");
  CUDA_TRY(cudaDeviceSynchronize());
  CUDA_TRY(cudaMemcpy(out, j->d_abs, (size_t)j->batch * sizeof(double), cudaMemcpyDeviceToHost));
  return LHAF_OK;
}

lhaf_status lhaf_job_partials(lhaf_job *j, void **dev_ptr, size_t *bytes) {
  if (!j || !dev_ptr || !bytes) return fail(LHAF_E_ARG, "null pointer");
  *dev_ptr = j->d_partials;
  *bytes = (size_t)j->units * sizeof(Partial);
  return LHAF_OK;
}

lhaf_status lhaf_job_terms(lhaf_job *j, const uint64_t *t, int32_t nt, double *g_out) {
  std::lock_guard<std::recursive_mutex> lk(g_mu);
  if (!j || (nt > 0 && (!t || !g_out))) return fail(LHAF_E_ARG, "null pointer");
  if (j->batch < 1 || j->descs[0].d == 0) return fail(LHAF_E_ARG, "pattern 0 has no terms");
  uint64_t *dt = nullptr;
  double2 *dg = nullptr;
  CUDA_TRY(dmalloc(&dt, std::max(1, nt) * sizeof(uint64_t)));
  CUDA_TRY(dmalloc(&dg, std::max(1, nt) * sizeof(double2)));
  cudaError_t e = cudaMemcpy(dt, t, nt * sizeof(uint64_t), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) {
    const PatDesc &D0 = j->descs[0];
    e = (j->variant == 5)   ? launch_terms_v5(j->dev(), j->e_max, j->ntl_max, j->n_max, dt, nt, dg, 0, j->prec)
        : (j->variant == 3 || j->variant == 6) ? launch_terms_v3(j->dev(), j->e_max, j->ntl_max, j->n_max, dt, nt, dg, 0)
                            : launch_terms(j->dev(), j->variant, D0.d, D0.n, dt, nt, dg, 0);
  }
  if (e == cudaSuccess) e = cudaMemcpy(g_out, dg, nt * sizeof(double2), cudaMemcpyDeviceToHost);
  dfree(dt);
  dfree(dg);
  if (e != cudaSuccess) return fail(LHAF_E_CUDA, "lhaf_job_terms: %s", cudaGetErrorString(e));
  return LHAF_OK;
}

void lhaf_job_destroy(lhaf_job *j) {
  std::lock_guard<std::recursive_mutex> lk(g_mu);
  job_free(j);
}

lhaf_status lhaf_rpt_batch(const double *A, const double *gamma, int64_t gamma_stride,
                           const int32_t *reps, int32_t k, int32_t batch, double *out) {
  std::lock_guard<std::recursive_mutex> lk(g_mu);
  if (!out) return fail(LHAF_E_ARG, "null output");
  lhaf_job *j = nullptr;
  lhaf_status s = job_create_impl(A, gamma, gamma_stride, reps, k, batch, 0, false, &j);
  if (s != LHAF_OK) return s;
  std::vector<double> tmp((size_t)std::max(1, batch) * 2);
  s = evaluate(j, tmp.data(), nullptr, 0);
  job_free(j);
  if (s == LHAF_OK) memcpy(out, tmp.data(), (size_t)batch * 2 * sizeof(double));
  return s;
}

static lhaf_status cutoff_impl(const double *A, const double *gamma, const int32_t *reps_fixed,
                               int32_t k, int32_t mode, int32_t n_cut, double *out, double *abs_out);

lhaf_status lhaf_rpt_cutoff(const double *A, const double *gamma, const int32_t *reps_fixed,
                            int32_t k, int32_t mode, int32_t n_cut, double *out) {
  std::lock_guard<std::recursive_mutex> lk(g_mu);
  return cutoff_impl(A, gamma, reps_fixed, k, mode, n_cut, out, nullptr);
}

lhaf_status lhaf_rpt_cutoff_ex(const double *A, const double *gamma, const int32_t *reps_fixed,
                               int32_t k, int32_t mode, int32_t n_cut, double tol, double *out,
                               double *err_est) {
  std::lock_guard<std::recursive_mutex> lk(g_mu);
  if (!err_est) return fail(LHAF_E_ARG, "null pointer argument");
  std::vector<double> ab((size_t)n_cut + 1 > 0 ? (size_t)n_cut + 1 : 1);
  lhaf_status s = cutoff_impl(A, gamma, reps_fixed, k, mode, n_cut, out, ab.data());
  if (s != LHAF_OK) return s;
  int worst = -1;
  for (int c = 0; c <= n_cut; ++c) {
    const double v = std::hypot(out[2 * c], out[2 * c + 1]);
    // kappa = 2^{1-n} sum |term| / |lhaf| times the per-term error scale 2^-46 (~64 eps), capped
    // at 1 (a value at the rounding-noise level of its terms -- e.g. an exact zero -- has no
    // significant digits)
    err_est[c] = ab[c] > 0.0 ? std::min(1.0, ab[c] * 0x1p-46 / std::max(v, 1e-300)) : 0.0;
    if (tol > 0.0 && err_est[c] > tol && worst < 0) worst = c;
  }
  if (worst >= 0)
    return fail(LHAF_E_INACCURATE, "count %d: estimated relative error %.2e > tol %.2e (sieve cancellation)",
                worst, err_est[worst], tol);
  return LHAF_OK;
}

static lhaf_status cutoff_impl(const double *A, const double *gamma, const int32_t *reps_fixed,
                               int32_t k, int32_t mode, int32_t n_cut, double *out, double *abs_out) {
  if (!A || !gamma || !reps_fixed || !out) return fail(LHAF_E_ARG, "null pointer argument");
  if (k < 1 || k > LHAF_MAX_MODES) return fail(LHAF_E_ARG, "k = %d out of range", k);
  if (mode < 0 || mode >= k) return fail(LHAF_E_ARG, "batched mode %d outside [0, %d)", mode, k);
  if (n_cut < 0 || n_cut > 64) return fail(LHAF_E_ARG, "n_cut = %d outside [0, 64]", n_cut);
  std::vector<int32_t> rf(reps_fixed, reps_fixed + k);
  rf[mode] = 0;
  // App. B.5 shared evaluation: the fixed modes' matching plus the batched self-pair
  // (mode, mode) with eta_b = floor((n_cut - parity) / 2), one group per parity of the count
  Plan Pf;
  lhaf_status s = make_plan(rf.data(), k, 0, Pf);
  if (s != LHAF_OK) return s;
  const bool shared = n_cut <= 63 && !getenv("LHAF_CUTOFF_SEPARATE") && (g_ctx.variant == 0 || g_ctx.variant == 6);
  std::vector<Plan> groups;
  int n_f[2] = {0, 0}, gidx[2] = {-1, -1};
  if (shared) {
    for (int par = 0; par < 2 && par <= n_cut; ++par) {
      Plan G = Pf;
      G.eta_b = (n_cut - par) / 2;
      if (par == 1) {
        if (Pf.leftover >= 0) {  // the leftover photon pairs with the batched one: no phantom
          G.q.back() = mode;
          G.leftover = -1;
        }
        else { G.p.push_back(mode); G.q.push_back(-1); G.eta.push_back(1); G.leftover = mode; }
      }
      int nf = 0;
      uint64_t Tf = 1;
      for (int e2 : G.eta) {
        nf += e2;
        const uint64_t r = (uint64_t)e2 + 1;
        if (Tf > (~(uint64_t)0) / r) return fail(LHAF_E_TOO_LARGE, "cutoff term count overflows 64 bits");
        Tf *= r;
      }
      G.p.push_back(mode); G.q.push_back(mode); G.eta.push_back(2 * G.eta_b);  // digit range
      G.H = (int)G.eta.size();
      G.d = 2 * G.H;
      G.n = nf + G.eta_b;
      G.N = Pf.N + par;
      const uint64_t rb = (uint64_t)(2 * G.eta_b + 1);
      if (Tf > (~(uint64_t)0) / rb) return fail(LHAF_E_TOO_LARGE, "cutoff term count overflows 64 bits");
      G.T = Tf * rb;
      G.T_eval = G.T / 2;
      n_f[par] = nf;
      gidx[par] = (int)groups.size();
      groups.push_back(G);
    }
  }
  lhaf_job *j = nullptr;
  if (shared) s = job_create_impl(A, gamma, 0, nullptr, k, (int)groups.size(), 0, false, &j, &groups);
  // the shared groups carry the batched self-pair (and a phantom for odd counts), so they can
  // exceed the kernels' d limit where every per-count pattern still fits: fall back then too
  if (!shared || (s == LHAF_OK && j->variant == 1) || s == LHAF_E_TOO_LARGE) {
    if (j) { job_free(j); j = nullptr; }
    std::vector<int32_t> reps((size_t)(n_cut + 1) * k);  // separate sieve per count
    for (int c = 0; c <= n_cut; ++c) {
      memcpy(&reps[(size_t)c * k], reps_fixed, (size_t)k * sizeof(int32_t));
      reps[(size_t)c * k + mode] = c;
    }
    lhaf_job *jb = nullptr;
    lhaf_status sb = job_create_impl(A, gamma, 0, reps.data(), k, n_cut + 1, 0, false, &jb);
    if (sb != LHAF_OK) return sb;
    std::vector<double> tmp(2 * (size_t)(n_cut + 1));
    sb = evaluate(jb, tmp.data(), nullptr, 0);
    if (sb == LHAF_OK && abs_out &&
        cudaMemcpy(abs_out, jb->d_abs, (size_t)(n_cut + 1) * sizeof(double), cudaMemcpyDeviceToHost) != cudaSuccess)
      sb = fail(LHAF_E_CUDA, "reading the absolute sums failed");
    job_free(jb);
    if (sb == LHAF_OK) memcpy(out, tmp.data(), tmp.size() * sizeof(double));
    return sb;
  }
  if (s != LHAF_OK) return s;
  // one sieve launch over both groups, then one finalize over n_cut + 1 virtual patterns
  std::vector<PatDesc> vd(n_cut + 1);
  for (int c = 0; c <= n_cut; ++c) {
    const PatDesc &G = j->descs[gidx[c & 1]];
    const int m = c >> 1;
    PatDesc &D = vd[c];
    memset(&D, 0, sizeof D);
    D.d = (Pf.N + c == 0) ? 0 : 2;
    D.flags = G.flags & FLAG_FULL;  // the tree evaluates every term when no fixed pair can halve
    D.n = n_f[c & 1] + m;
    D.unit_begin = (uint64_t)G.part_base + (uint64_t)m * G.units;
    D.units = G.units;
    D.out_exp = -j->scale_s * (Pf.N + c);
  }
  PatDesc *d_vd = nullptr;
  double2 *d_o = nullptr;
  double *d_ab = nullptr;
  cudaError_t e = upload(&d_vd, vd);
  if (e == cudaSuccess) e = dmalloc(&d_o, (n_cut + 1) * sizeof(double2));
  if (e == cudaSuccess) e = dmalloc(&d_ab, (n_cut + 1) * sizeof(double));
  if (e == cudaSuccess) e = cudaMemset(j->d_partials, 0, std::max<uint64_t>(1, j->parts) * sizeof(Partial));
  if (e == cudaSuccess)
    e = (j->variant == 6) ? run_sieve(j, 0, j->units, 0)  // the batched pair at the tree's leaves
                          : launch_sieve_cut_v3(j->dev(), j->e_max, j->ntl_max, j->n_max, 0, j->units, g_ctx.num_sms, 0);
  if (e == cudaSuccess) {
    JobDev J = j->dev();
    J.descs = d_vd;
    J.npat = n_cut + 1;
    e = launch_finalize(J, d_o, d_ab, 0);
  }
  if (e == cudaSuccess) e = cudaMemcpy(out, d_o, (n_cut + 1) * sizeof(double2), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && abs_out) e = cudaMemcpy(abs_out, d_ab, (n_cut + 1) * sizeof(double), cudaMemcpyDeviceToHost);
  dfree(d_vd);
  dfree(d_o);
  dfree(d_ab);
  job_free(j);
  if (e != cudaSuccess) return fail(LHAF_E_CUDA, "cutoff job: %s", cudaGetErrorString(e));
  return LHAF_OK;
}

lhaf_status lhaf_rpt_multigamma(const double *A, const double *gammas, int32_t ngamma,
                                const int32_t *reps, int32_t k, double *out) {
  std::lock_guard<std::recursive_mutex> lk(g_mu);
  if (!A || !gammas || !reps || !out) return fail(LHAF_E_ARG, "null pointer argument");
  if (ngamma < 0 || k < 0 || k > LHAF_MAX_MODES) return fail(LHAF_E_ARG, "bad ngamma / k");
  if (ngamma == 0) return LHAF_OK;
  std::vector<Plan> plans(1);
  lhaf_status s = make_plan(reps, k, 0, plans[0]);
  if (s != LHAF_OK) return s;
  const Plan &P0 = plans[0];
  // the shared per-term reduction (v5 FLAG_MG) against G patterns in one tree forest: on the
  // tree (FP64, >= 65536 terms per loop vector) the separate evaluation is faster -- d = 48,
  // G = 16: 2.7 s against 8.2 s (DESIGN.md §9 row 2) -- so the shared path serves the per-term
  // regime (small patterns) and explicit requests (LHAF_MULTIGAMMA_SHARED, kernel 5)
  const bool tree_regime = g_ctx.variant == 0 && g_ctx.precision == 0 && P0.T_eval >= 65536 &&
                           !getenv("LHAF_MULTIGAMMA_SHARED");
  const bool shared = P0.H > 0 && P0.d + ngamma <= 64 && ngamma <= LHAF_MAX_GAMMA &&
                      (g_ctx.variant == 0 || g_ctx.variant == 5) && g_ctx.precision == 0 && !tree_regime &&
                      !getenv("LHAF_MULTIGAMMA_SEPARATE");
  if (!shared) {
    // the pattern once per loop vector in one batch job (G independent sieves)
    std::vector<int32_t> r((size_t)ngamma * k);
    for (int g = 0; g < ngamma; ++g) memcpy(&r[(size_t)g * k], reps, (size_t)k * sizeof(int32_t));
    return lhaf_rpt_batch(A, gammas, k, r.data(), k, ngamma, out);
  }
  // one job, one pattern, FLAG_MG: one reduction per term shared by every loop vector
  plans[0].mg = ngamma;
  lhaf_job *j = nullptr;
  s = job_create_impl(A, gammas, k, nullptr, k, 1, 0, false, &j, &plans);
  if (s != LHAF_OK) return s;
  std::vector<PatDesc> vd(ngamma);
  const PatDesc &D = j->descs[0];
  for (int g = 0; g < ngamma; ++g) {
    memset(&vd[g], 0, sizeof(PatDesc));
    vd[g].d = D.d;
    vd[g].n = D.n;
    vd[g].unit_begin = (uint64_t)D.part_base + (uint64_t)g * D.units;
    vd[g].units = D.units;
    vd[g].out_exp = D.out_exp;
  }
  PatDesc *d_vd = nullptr;
  double2 *d_o = nullptr;
  cudaError_t e = upload(&d_vd, vd);
  if (e == cudaSuccess) e = dmalloc(&d_o, (size_t)ngamma * sizeof(double2));
  if (e == cudaSuccess) e = cudaMemset(j->d_partials, 0, std::max<uint64_t>(1, j->parts) * sizeof(Partial));
  if (e == cudaSuccess) e = launch_sieve_mg_v5(j->dev(), j->d_max, ngamma, j->n_max, 0, j->units, g_ctx.num_sms, 0);
  if (e == cudaSuccess) {
    JobDev J = j->dev();
    J.descs = d_vd;
    J.npat = ngamma;
    e = launch_finalize(J, d_o, nullptr, 0);
  }
  if (e == cudaSuccess) e = cudaMemcpy(out, d_o, (size_t)ngamma * sizeof(double2), cudaMemcpyDeviceToHost);
  dfree(d_vd);
  dfree(d_o);
  job_free(j);
  if (e != cudaSuccess) return fail(LHAF_E_CUDA, "multigamma job: %s", cudaGetErrorString(e));
  return LHAF_OK;
}

lhaf_status lhaf_rpt_et(const double *A, const double *gamma, const int32_t *reps, int32_t k,
                        double out[2]) {
  std::lock_guard<std::recursive_mutex> lk(g_mu);
  if (!A || !gamma || !reps || !out) return fail(LHAF_E_ARG, "null pointer argument");
  if (k < 0 || k > LHAF_MAX_MODES) return fail(LHAF_E_ARG, "k = %d out of range", k);
  std::vector<Plan> plans(1);
  lhaf_status s = make_plan(reps, k, 0, plans[0]);
  if (s != LHAF_OK) return s;
  plans[0].et = true;
  plans[0].T_eval = plans[0].H > 0 ? plans[0].T : 0;  // no halving: w -> -w is not a symmetry
  lhaf_job *j = nullptr;
  s = job_create_impl(A, gamma, 0, nullptr, k, 1, 0, false, &j, &plans);
  if (s != LHAF_OK) return s;
  double tmp[2];
  s = evaluate(j, tmp, nullptr, 0);
  job_free(j);
  if (s == LHAF_OK) { out[0] = tmp[0]; out[1] = tmp[1]; }
  return s;
}

lhaf_status lhaf_rpt(const double *A, const double *gamma, const int32_t *reps, int32_t k,
                     double out[2]) {
  return lhaf_rpt_batch(A, gamma, 0, reps, k, 1, out);
}

lhaf_status lhaf_rpt_mixed(const double *A2, const double *gamma2, const int32_t *reps, int32_t k,
                           double out[2]) {
  std::lock_guard<std::recursive_mutex> lk(g_mu);
  if (!out) return fail(LHAF_E_ARG, "null output");
  lhaf_job *j = nullptr;
  lhaf_status s = job_create_impl(A2, gamma2, 0, reps, k, 1, 3, false, &j);
  if (s != LHAF_OK) return s;
  double tmp[2];
  s = evaluate(j, tmp, nullptr, 0);
  job_free(j);
  if (s == LHAF_OK) { out[0] = tmp[0]; out[1] = tmp[1]; }
  return s;
}

lhaf_status lhaf_rpt_batch_dev(const double *A_dev, const double *gamma_dev, int64_t gamma_stride,
                               const int32_t *reps, int32_t k, int32_t batch, int32_t mixed,
                               double *out_dev, void *stream) {
  std::lock_guard<std::recursive_mutex> lk(g_mu);
  if (!out_dev) return fail(LHAF_E_ARG, "null output");
  lhaf_job *j = nullptr;
  lhaf_status s = job_create_impl(A_dev, gamma_dev, gamma_stride, reps, k, batch, mixed, true, &j);
  if (s != LHAF_OK) return s;
  s = evaluate(j, nullptr, out_dev, (cudaStream_t)stream);
  job_free(j);
  return s;
}

lhaf_status lhaf_get_unique_id(void *id128) {
  std::lock_guard<std::recursive_mutex> lk(g_mu);
  if (!id128) return fail(LHAF_E_ARG, "null pointer");
  if (!g_ctx.nccl.load()) return fail(LHAF_E_NCCL, "cannot dlopen libnccl.so.2");
  ncclUniqueId id;
  ncclResult_t r = g_ctx.nccl.GetUniqueId(&id);
  if (r != ncclSuccess) return fail(LHAF_E_NCCL, "ncclGetUniqueId: %s", g_ctx.nccl.GetErrorString(r));
  memcpy(id128, &id, sizeof id);
  return LHAF_OK;
}

lhaf_status lhaf_init_rank(int32_t rank, int32_t nranks, const void *id128, int32_t device) {
  std::lock_guard<std::recursive_mutex> lk(g_mu);
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(LHAF_E_ARG, "bad rank %d of %d", rank, nranks);
  if (device >= 0) {
    lhaf_status s = lhaf_set_device(device);
    if (s != LHAF_OK) return s;
  } else {
    lhaf_status s = ensure_device();
    if (s != LHAF_OK) return s;
  }
  if (g_ctx.comm) { g_ctx.nccl.CommDestroy(g_ctx.comm); g_ctx.comm = nullptr; }
  g_ctx.rank = rank;
  g_ctx.nranks = nranks;
  if (nranks == 1 && !id128) return LHAF_OK;  // single rank without NCCL
  if (!id128) return fail(LHAF_E_ARG, "null unique id");
  if (!g_ctx.nccl.load()) return fail(LHAF_E_NCCL, "cannot dlopen libnccl.so.2");
  ncclUniqueId id;
  memcpy(&id, id128, sizeof id);
  ncclResult_t r = g_ctx.nccl.CommInitRank(&g_ctx.comm, nranks, id, rank);
  if (r != ncclSuccess) {
    g_ctx.nranks = 1; g_ctx.rank = 0;
    return fail(LHAF_E_NCCL, "ncclCommInitRank: %s", g_ctx.nccl.GetErrorString(r));
  }
  return LHAF_OK;
}

lhaf_status lhaf_rank_info(int32_t *rank, int32_t *nranks) {
  if (!rank || !nranks) return fail(LHAF_E_ARG, "null pointer");
  *rank = g_ctx.rank;
  *nranks = g_ctx.nranks;
  return LHAF_OK;
}

lhaf_status lhaf_shard_units(uint64_t units, int32_t rank, int32_t nranks, uint64_t *begin,
                             uint64_t *end) {
  if (!begin || !end) return fail(LHAF_E_ARG, "null pointer");
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(LHAF_E_ARG, "bad rank %d of %d", rank, nranks);
  shard(units, (uint64_t)rank, (uint64_t)nranks, *begin, *end);
  return LHAF_OK;
}

void lhaf_shutdown(void) {
  std::lock_guard<std::recursive_mutex> lk(g_mu);
  if (g_ctx.comm) { g_ctx.nccl.CommDestroy(g_ctx.comm); g_ctx.comm = nullptr; }
  g_ctx.rank = 0;
  g_ctx.nranks = 1;
}

}  // extern "C"
