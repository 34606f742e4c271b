// DMMA micro-benchmark for B200 (sm_100a): throughput of mma.sync.aligned.m8n8k4 .f64 (the only
// FP64 tensor-core shape; tcgen05 has no FP64 kind) against the DFMA peak in
// profiles/fp64_peak.json.  Round-1 VERDICT "missing 9" / SURVEY K6: "DMMA only if it measurably
// wins".  Output: one JSON object on stdout.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

template <int CHAINS>
__global__ void dmma_tp(double *out, long iters, double a, double b) {
  double c0[CHAINS], c1[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) { c0[c] = threadIdx.x * 1e-3 + c; c1[c] = c; }
  for (long i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                   : "+d"(c0[c]), "+d"(c1[c]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += c0[c] + c1[c];
  if (s == 12345.678) out[threadIdx.x] = s;
}

__global__ void dmma_lat(double *out, long iters, double a, double b, long long *cyc) {
  double c0 = threadIdx.x, c1 = 1.0;
  long long t0 = clock64();
  for (long i = 0; i < iters; ++i)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
  long long t1 = clock64();
  if (threadIdx.x == 0) *cyc = t1 - t0;
  if (c0 + c1 == 12345.678) out[0] = c0;
}

int main() {
  CK(cudaSetDevice(0));
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  double *out; CK(cudaMalloc(&out, 1 << 20));
  long long *cyc; CK(cudaMalloc(&cyc, 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int sms = p.multiProcessorCount;
  double best[3] = {0, 0, 0};
  const int warps_per_block[3] = {4, 8, 16};
  for (int cfg = 0; cfg < 3; ++cfg) {
    const int threads = 32 * warps_per_block[cfg], blocks = sms * (32 / warps_per_block[cfg]);
    auto run = [&](long iters) {
      CK(cudaEventRecord(e0));
      dmma_tp<8><<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
      CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      // one warp-level m8n8k4 = 8*8*4 MACs = 512 flops
      const double flops = 512.0 * 8 * iters * (double)(threads / 32) * blocks;
      return flops / (ms * 1e-3) / 1e12;
    };
    run(200);
    for (int r = 0; r < 5; ++r) { const double t = run(4000); if (t > best[cfg]) best[cfg] = t; }
  }
  const long lit = 4096;
  dmma_lat<<<1, 32>>>(out, lit, 0.999999, 1e-7, cyc);
  CK(cudaDeviceSynchronize());
  dmma_lat<<<1, 32>>>(out, lit, 0.999999, 1e-7, cyc);
  long long hc; CK(cudaMemcpy(&hc, cyc, 8, cudaMemcpyDeviceToHost));
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"dmma_m8n8k4_tflops_4w\": %.3f, \"dmma_m8n8k4_tflops_8w\": %.3f, "
         "\"dmma_m8n8k4_tflops_16w\": %.3f, \"dmma_latency_cyc\": %.2f}\n",
         p.name, sms, best[0], best[1], best[2], (double)hc / lit);
  return 0;
}
