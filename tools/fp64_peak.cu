// FP64-pipe peak of this GPU, measured: a DFMA-chain microbenchmark.
//
// Every thread runs 8 independent FMA chains (x = x * a + b), so the pipe,
// not the 4-cycle-ish DFMA latency, is the limit; the grid is a whole number
// of resident CTAs per SM.  Reported:
//   tinstr_s  FP64 thread-instructions per second (the unit ncu's
//             smsp__sass_thread_inst_executed_op_dfma_pred_on counts), best of
//             `reps` timed launches (CUDA events);
//   sm_mhz    the SM clock during the best launch, from clock64() over
//             %globaltimer in one thread of CTA 0;
//   per_clk_per_sm  tinstr_s / (SMs x sm_mhz): the FP64 lanes per SM the
//             pipe actually delivers.
// bench.py runs this once (build/fp64_peak) and quotes the chi2 pass's FP64
// fraction against tinstr_s, measured on the same box in the same run.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e_ = (x);                                                          \
    if (e_ != cudaSuccess) {                                                       \
      std::fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));                \
      std::exit(1);                                                                \
    }                                                                              \
  } while (0)

constexpr int kChains = 8;

__global__ void __launch_bounds__(256) dfma_chains(double* out, long long* clk, int iters,
                                                   double a, double b) {
  double x[kChains];
#pragma unroll
  for (int k = 0; k < kChains; ++k) x[k] = 1.0 + 1e-3 * (threadIdx.x + k);
  long long c0 = 0, t0 = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    c0 = clock64();
  }
  for (int i = 0; i < iters; ++i) {
#pragma unroll 16
    for (int u = 0; u < 16; ++u)
#pragma unroll
      for (int k = 0; k < kChains; ++k) x[k] = __fma_rn(x[k], a, b);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const long long c1 = clock64();
    long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    clk[0] = c1 - c0;
    clk[1] = t1 - t0;
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < kChains; ++k) s += x[k];
  if (s == 12345.678) out[blockIdx.x * blockDim.x + threadIdx.x] = s;  // keeps the chains live
}

int main(int argc, char** argv) {
  const int dev = argc > 1 ? std::atoi(argv[1]) : 0;
  const int reps = argc > 2 ? std::atoi(argv[2]) : 5;
  const int iters = argc > 3 ? std::atoi(argv[3]) : 16384;
  CK(cudaSetDevice(dev));
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, dev));
  int per_sm = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, dfma_chains, 256, 0));
  const int blocks = prop.multiProcessorCount * per_sm;
  double* out;
  long long* clk;
  CK(cudaMalloc(&out, sizeof(double) * blocks * 256));
  CK(cudaMalloc(&clk, sizeof(long long) * 2));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  const double a = 0.99999999, b = 1e-9;
  dfma_chains<<<blocks, 256>>>(out, clk, iters / 4, a, b);  // warm-up (clocks ramp)
  CK(cudaDeviceSynchronize());
  double best_s = 1e30, best_mhz = 0.0;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(e0));
    dfma_chains<<<blocks, 256>>>(out, clk, iters, a, b);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    long long h[2];
    CK(cudaMemcpy(h, clk, sizeof(h), cudaMemcpyDeviceToHost));
    if (ms * 1e-3 < best_s) {
      best_s = ms * 1e-3;
      best_mhz = h[1] > 0 ? (double)h[0] / (double)h[1] * 1e3 : 0.0;
    }
  }
  const double instr = (double)blocks * 256.0 * iters * 16.0 * kChains;
  const double rate = instr / best_s;
  std::printf("{\"tinstr_s\": %.6e, \"sm_mhz\": %.1f, \"sms\": %d, \"ctas_per_sm\": %d, "
              "\"per_clk_per_sm\": %.2f, \"seconds\": %.6f, \"instr\": %.6e, "
              "\"how\": \"DFMA chains (8 independent per thread), best of %d launches, CUDA events; "
              "clock from clock64/globaltimer\"}\n",
              rate / 1e12, best_mhz, prop.multiProcessorCount, per_sm,
              best_mhz > 0 ? rate / (prop.multiProcessorCount * best_mhz * 1e6) : 0.0, best_s, instr,
              reps);
  return 0;
}
