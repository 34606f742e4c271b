// Can TMEM stand in for the register-resident row of the Hessenberg step?  One "step" per
// thread: NSLOT complex slots a <- a - m r[s] (r broadcast from shared memory) and a dot
// with q[s], then a CTA barrier; the slots live either in registers (MODE 0) or in tensor
// memory (MODE 1: tcgen05.ld/st 32x32b.x16 chunks of 8 complex, double-buffered loads).
// Prints one JSON line per (mode, CTAs/SM): ns per step, slot-updates/s for the whole GPU.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ void tld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tst16(uint32_t taddr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};\n"
      :: "r"(taddr), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
        "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]));
}
__device__ __forceinline__ void twait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void twait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }

template <int NSLOT>
__device__ __forceinline__ void slot_math(double &ax, double &ay, double2 m, double2 r, double2 q,
                                          double &xr, double &xi, double &yr, double &yi) {
  ax = fma(-m.x, r.x, ax); ax = fma(m.y, r.y, ax);
  ay = fma(-m.x, r.y, ay); ay = fma(-m.y, r.x, ay);
  xr = fma(ax, q.x, xr); xi = fma(ay, q.y, xi); yr = fma(ax, q.y, yr); yi = fma(ay, q.x, yi);
}

__device__ __forceinline__ void team_bar(int team) {
  asm volatile("bar.sync %0, 128;\n" :: "r"(team + 1) : "memory");
}
template <int MODE, int NSLOT, int MINB, int TEAMS = 1>
__global__ void __launch_bounds__(128 * TEAMS, MINB) step_bench(double *out, int steps, int smem_pad) {
  extern __shared__ double2 dyn[];
  __shared__ double2 r[NSLOT], q[NSLOT];
  __shared__ uint32_t s_taddr;
  const int tid = threadIdx.x % 128, warp = threadIdx.x >> 5, team = threadIdx.x / 128;
  for (int s = threadIdx.x; s < NSLOT; s += 128 * TEAMS) { r[s] = make_double2(1e-3 * s, 2e-3); q[s] = make_double2(0.5, -1e-3 * s); }
  if (smem_pad > 0 && tid == 0) dyn[0] = make_double2(0, 0);
  double2 m = make_double2(1e-6 * tid, 1e-7);
  double res = 0;
  if constexpr (MODE == 0) {
    double2 A[NSLOT];
#pragma unroll
    for (int s = 0; s < NSLOT; ++s) A[s] = make_double2(tid + s, s);
    __syncthreads();
    for (int it = 0; it < steps; ++it) {
      double xr = 0, xi = 0, yr = 0, yi = 0;
#pragma unroll
      for (int s = 0; s < NSLOT; ++s) slot_math<NSLOT>(A[s].x, A[s].y, m, r[s], q[s], xr, xi, yr, yi);
      m.x = fma(xr - xi, 1e-30, m.x); m.y = fma(yr + yi, 1e-30, m.y);
      team_bar(team);
    }
#pragma unroll
    for (int s = 0; s < NSLOT; ++s) res += A[s].x + A[s].y;
  } else {
    constexpr int NCH = (4 * NSLOT + 15) / 16;  // 16-column chunks of 4 complex
    constexpr int NC1 = NCH * 16 * TEAMS;
    constexpr int NCOL = NC1 <= 32 ? 32 : NC1 <= 64 ? 64 : NC1 <= 128 ? 128 : NC1 <= 256 ? 256 : 512;
    if (warp == 0) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n"
                   :: "r"((uint32_t)__cvta_generic_to_shared(&s_taddr)), "n"(NCOL));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t base = s_taddr + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(team * NCH * 16);
    {
      uint32_t v[16];
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const long long x = __double_as_longlong((double)(tid + 4 * c + j / 2));
          v[2 * j] = (uint32_t)x; v[2 * j + 1] = (uint32_t)(x >> 32);
        }
        tst16(base + 16 * c, v);
      }
      twait_st();
    }
    __syncthreads();
    for (int it = 0; it < steps; ++it) {
      double xr = 0, xi = 0, yr = 0, yi = 0;
      uint32_t v0[16], v1[16];
      tld16(base, v0);
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        uint32_t (&cur)[16] = (c & 1) ? v1 : v0;
        uint32_t (&nxt)[16] = (c & 1) ? v0 : v1;
        twait_ld();
        if (c + 1 < NCH) tld16(base + 16 * (c + 1), nxt);
#pragma unroll
        for (int j = 0; j < 4; ++j) {  
          const int s = 4 * c + j;
          if (s < NSLOT) {
            double ax = __hiloint2double(cur[4 * j + 1], cur[4 * j]);
            double ay = __hiloint2double(cur[4 * j + 3], cur[4 * j + 2]);
            slot_math<NSLOT>(ax, ay, m, r[s], q[s], xr, xi, yr, yi);
            const long long bx = __double_as_longlong(ax), by = __double_as_longlong(ay);
            cur[4 * j] = (uint32_t)bx; cur[4 * j + 1] = (uint32_t)(bx >> 32);
            cur[4 * j + 2] = (uint32_t)by; cur[4 * j + 3] = (uint32_t)(by >> 32);
          }
        }
        tst16(base + 16 * c, cur);
      }
      m.x = fma(xr - xi, 1e-30, m.x); m.y = fma(yr + yi, 1e-30, m.y);
      twait_st();
      team_bar(team);
    }
    {
      uint32_t v[16];
      tld16(base, v);
      twait_ld();
      res = __hiloint2double(v[1], v[0]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" :: "r"(s_taddr), "n"(NCOL));
  }
  out[blockIdx.x * 128 * TEAMS + threadIdx.x] = res + m.x + m.y;
}

template <int MODE, int NSLOT, int MINB, int TEAMS = 1>
int run(int ctas_per_sm, int nsm, double *out, int padk = -1) {
  auto k = step_bench<MODE, NSLOT, MINB, TEAMS>;
  // pad dynamic shared memory so that at most ctas_per_sm CTAs fit on one SM
  const int pad = padk >= 0 ? padk : (220 * 1024) / ctas_per_sm - 2 * NSLOT * 16 - 1024;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, pad));
  CK(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, 128 * TEAMS, pad));
  cudaFuncAttributes fa;
  CK(cudaFuncGetAttributes(&fa, k));
  const int steps = 4000;
  const int grid = nsm * ctas_per_sm;
  k<<<grid, 128 * TEAMS, pad>>>(out, 10, pad);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<grid, 128 * TEAMS, pad>>>(out, steps, pad);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double ns_step = ms * 1e6 / steps;
  const double upd = (double)grid * 128 * TEAMS * NSLOT * steps / (ms * 1e-3);
  printf("{\"mode\": \"%s\", \"nslot\": %d, \"regs\": %d, \"ctas_per_sm\": %d, \"occ\": %d, \"pad\": %d, \"static_smem\": %d, \"ns_per_step\": %.2f, "
         "\"slot_updates_per_s\": %.4e, \"dfma_tflops\": %.3f}\n",
         MODE ? "tmem" : "regs", TEAMS, NSLOT, fa.numRegs, ctas_per_sm, occ, pad, (int)fa.sharedSizeBytes, ns_step, upd, upd * 16 / 1e12);
  return 0;
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double *out;
  CK(cudaMalloc(&out, (size_t)nsm * 16 * 128 * sizeof(double)));
  run<0, 31, 2>(2, nsm, out, 0);
  run<1, 32, 1, 2>(1, nsm, out, 0);
  run<1, 32, 1, 3>(1, nsm, out, 0);
  run<1, 32, 1, 4>(1, nsm, out, 0);
  run<0, 31, 1, 2>(1, nsm, out, 0);
  return 0;
}
