// FP64 DFMA peak microbenchmark (roofline denominator for the path tracker).
// Each thread runs 8 independent DFMA chains; grid = SMs x 8 blocks x 256 threads.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_chain(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x * 1e-9, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  double x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (s == 12345.678) out[0] = s;
}
int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"clock_khz\": %d, \"cc\": \"%d.%d\", \"regs_per_sm\": %d, \"smem_per_sm\": %zu}\n",
         p.name, p.multiProcessorCount, clk, p.major, p.minor, p.regsPerMultiprocessor, p.sharedMemPerMultiprocessor);
  double* d; cudaMalloc(&d, 8);
  int blocks = p.multiProcessorCount * 8, threads = 256, iters = 4000;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) dfma_chain<<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(e0); dfma_chain<<<blocks, threads>>>(d, iters, 0.999999, 1e-7); cudaEventRecord(e1);
    cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  double flops = 2.0 * 8 * 16 * (double)iters * blocks * threads;
  printf("{\"fp64_tflops_burst\": %.3f, \"ms\": %.3f}\n", flops / best / 1e9, best);
  // sustained: back-to-back for ~3 s
  cudaEventRecord(e0); int n = 0; float tot = 0;
  while (tot < 3000.f) { dfma_chain<<<blocks, threads>>>(d, iters, 0.999999, 1e-7); ++n;
    if (n % 20 == 0) { cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&tot, e0, e1);} }
  cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&tot, e0, e1);
  printf("{\"fp64_tflops_sustained\": %.3f, \"launches\": %d}\n", flops * n / tot / 1e9, n);
  return 0;
}
