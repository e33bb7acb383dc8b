// Latency of dependent DFMA / DMUL chains, FP64 division, hypot and an LDS round trip on one warp.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, double a, double b, int iters) {
  __shared__ double sm[1024];
  double x = threadIdx.x * 1e-3 + 1.0;
  sm[threadIdx.x] = x;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = fma(x, a, b);
  long long t1 = clock64();
  for (int i = 0; i < iters; ++i) x = x * a;
  long long t2 = clock64();
  for (int i = 0; i < iters; ++i) x = b / x;
  long long t3 = clock64();
  for (int i = 0; i < iters; ++i) x = hypot(x, a);
  long long t4 = clock64();
  int idx = threadIdx.x;
  for (int i = 0; i < iters; ++i) { double v = sm[idx]; idx = ((int)v + i) & 31; x += v; }
  long long t5 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; }
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 1024 * 8); cudaMallocManaged(&c, 5 * 8);
  int it = 4096;
  k<<<1, 32>>>(o, c, 0.9999999, 1e-9, it); cudaDeviceSynchronize();
  k<<<1, 32>>>(o, c, 0.9999999, 1e-9, it); cudaDeviceSynchronize();
  printf("{\"dfma_lat\": %.1f, \"dmul_lat\": %.1f, \"ddiv_lat\": %.1f, \"hypot_lat\": %.1f, \"lds_dep_lat\": %.1f}\n",
         c[0] / (double)it, c[1] / (double)it, c[2] / (double)it, c[3] / (double)it, c[4] / (double)it);
  return 0;
}
