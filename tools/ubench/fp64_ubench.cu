// FP64 roofline micro-benchmarks for B200 (sm_100a): DFMA throughput (burst and
// sustained), DFMA latency, 32-bit SHFL throughput, LDS.128 throughput.
// Output: one JSON object on stdout. Used to derive the "% FP64 peak" denominator.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <chrono>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

template <int CHAINS>
__global__ void dfma_tp(double *out, long iters, double a, double b) {
  double x[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x * 1e-3 + c;
  for (long i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = fma(x[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += x[c];
  if (s == 12345.678) out[threadIdx.x] = s;
}

__global__ void dfma_lat(double *out, long iters, double a, double b, long long *cyc) {
  double x = threadIdx.x;
  long long t0 = clock64();
  for (long i = 0; i < iters; ++i) x = fma(x, a, b);
  long long t1 = clock64();
  if (threadIdx.x == 0) *cyc = t1 - t0;
  if (x == 12345.678) out[0] = x;
}

__global__ void shfl_tp(double *out, long iters) {
  unsigned v0 = threadIdx.x, v1 = threadIdx.x * 3, v2 = threadIdx.x * 5, v3 = threadIdx.x * 7;
  for (long i = 0; i < iters; ++i) {
    v0 = __shfl_xor_sync(0xffffffffu, v0, 1);
    v1 = __shfl_xor_sync(0xffffffffu, v1, 2);
    v2 = __shfl_xor_sync(0xffffffffu, v2, 4);
    v3 = __shfl_xor_sync(0xffffffffu, v3, 8);
  }
  if ((v0 ^ v1 ^ v2 ^ v3) == 0xdeadbeef) out[0] = v0;
}

__global__ void lds_tp(double *out, long iters) {
  __shared__ double2 buf[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) buf[i] = make_double2(i, i);
  __syncthreads();
  double2 acc = make_double2(0, 0);
  int idx = threadIdx.x & 1023;
  for (long i = 0; i < iters; ++i) {
    double2 v = buf[(idx + i) & 1023];
    acc.x += v.x; acc.y += v.y;
  }
  if (acc.x == 1.2345) out[0] = acc.y;
}

int main(int argc, char **argv) {
  int dev = 0; CK(cudaSetDevice(dev));
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  double *out; CK(cudaMalloc(&out, 1 << 20));
  long long *cyc; CK(cudaMalloc(&cyc, 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int sms = p.multiProcessorCount;
  // DFMA throughput: 8 chains/thread, 256 threads/block, 8 blocks/SM.
  const int threads = 256, blocks = sms * 8;
  auto run_dfma = [&](long iters) {
    CK(cudaEventRecord(e0));
    dfma_tp<8><<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * iters * (double)threads * blocks;
    return flops / (ms * 1e-3) / 1e12;
  };
  run_dfma(1000);
  double burst = 0;
  for (int r = 0; r < 5; ++r) { double t = run_dfma(20000); if (t > burst) burst = t; }
  // sustained: back-to-back for >= 4 s, report the mean rate
  auto t0 = std::chrono::steady_clock::now();
  double sum_flops = 0; float total_ms = 0; int nl = 0;
  while (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() < 5.0) {
    long iters = 200000;
    CK(cudaEventRecord(e0));
    dfma_tp<8><<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    total_ms += ms; sum_flops += 2.0 * 8 * iters * (double)threads * blocks; ++nl;
  }
  double sustained = sum_flops / (total_ms * 1e-3) / 1e12;
  // DFMA latency (one warp, dependent chain)
  dfma_lat<<<1, 32>>>(out, 100000, 0.999999, 1e-7, cyc);
  long long hc; CK(cudaMemcpy(&hc, cyc, 8, cudaMemcpyDeviceToHost));
  double lat = hc / 100000.0;
  // SHFL throughput: 4 shuffles per iteration per thread
  long siters = 100000;
  shfl_tp<<<sms * 8, 256>>>(out, 1000);
  CK(cudaEventRecord(e0));
  shfl_tp<<<sms * 8, 256>>>(out, siters);
  CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
  float sms_ms; cudaEventElapsedTime(&sms_ms, e0, e1);
  // lanes per clock per SM, using the SM clock inferred from DFMA burst assuming 64 DFMA/clk/SM
  double shfl_lanes_per_s = 4.0 * siters * 256.0 * sms * 8 / (sms_ms * 1e-3);
  // LDS.128 throughput
  long liters = 100000;
  lds_tp<<<sms * 8, 256>>>(out, 1000);
  CK(cudaEventRecord(e0));
  lds_tp<<<sms * 8, 256>>>(out, liters);
  CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
  float lds_ms; cudaEventElapsedTime(&lds_ms, e0, e1);
  double lds_bytes_per_s = 16.0 * liters * 256.0 * sms * 8 / (lds_ms * 1e-3);
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"cc\": \"%d.%d\", \"clock_attr_mhz\": %.0f, "
         "\"regs_per_sm\": %d, \"smem_per_sm\": %zu, \"smem_optin_per_block\": %zu, "
         "\"fp64_tflops_burst\": %.3f, \"fp64_tflops_sustained\": %.3f, \"sustained_launches\": %d, "
         "\"dfma_latency_cyc\": %.2f, \"shfl32_lanes_per_s_chip\": %.4e, \"lds128_bytes_per_s_chip\": %.4e}\n",
         p.name, sms, p.major, p.minor, clk_khz / 1e3, p.regsPerMultiprocessor,
         p.sharedMemPerMultiprocessor, p.sharedMemPerBlockOptin, burst, sustained, nl, lat,
         shfl_lanes_per_s, lds_bytes_per_s);
  return 0;
}
