// Non-templated helpers: batched singular values (condition_and_rank,
// linalg.py:13-32), the all-pairs points_match test behind _dedup
// (filtering.py:73-78,140-150), and the rectangular Jacobian rank used by
// _restricted_regular (filtering.py:130-137).
#pragma once
#include "homotopy.cuh"
#include "linalg.cuh"

// one thread per matrix; A[P][m][n] row-major, sv[P][n] descending
__global__ void svd_kernel(int m, int n, long long P, const cd* A, cd* scratch, double* sv) {
  long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  cd* a = scratch + p * (size_t)m * n;
  for (int i = 0; i < m * n; ++i) a[i] = A[p * m * n + i];
  double s[NID_MAX_VARS];
  bool fin = true;
  for (int i = 0; i < m * n; ++i) fin = fin && cfinite(a[i]);
  if (!fin) {
    for (int j = 0; j < n; ++j) sv[p * n + j] = NAN;
    return;
  }
  jacobi_svd(a, m, n, n, nullptr, n, s);
  sort_desc(s, n);
  for (int j = 0; j < n; ++j) sv[p * n + j] = s[j];
}

// points_match(a = X[j], b = X[i]) for all i < j:  max|a-b| <= max(1e-8, 1e-6 max(1, |b|_inf))
__global__ void match_pairs_kernel(int n, int ncmp, long long P, const cd* X, const double* tolb, int* pairs,
                                   long long maxp, unsigned long long* count) {
  long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= P) return;
  for (long long i = 0; i < j; ++i) {
    const double tol = tolb[i];
    double d = 0.0;
    bool hit = true;
    for (int v = 0; v < ncmp; ++v) {
      cd a = X[j * n + v], b = X[i * n + v];
      double e = hypot(a.re - b.re, a.im - b.im);
      d = nanmax(d, e);
      if (!(d <= tol)) {
        hit = false;
        break;
      }
    }
    if (hit) {
      unsigned long long k = atomicAdd(count, 1ull);
      if ((long long)k < maxp) {
        pairs[2 * k] = (int)i;
        pairs[2 * k + 1] = (int)j;
      }
    }
  }
}

__global__ void match_tol_kernel(int n, int ncmp, long long P, const cd* X, double* tolb) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P) return;
  double s = 1.0;
  for (int v = 0; v < ncmp; ++v) s = nanmax(s, cabsd(X[i * n + v]));
  tolb[i] = fmax(1e-8, 1e-6 * s);
}

// K7 pre-pass: order-preserving compaction of the succeeded endpoints
// (status converged / singular_endpoint) of one shard -- what a rank sends to
// the classification rank.  256 paths per block: pass 1
// counts per block, the host scans the block counts, pass 2 writes each
// block's endpoints at its offset (ballot ranks inside the warp, warp totals
// through shared memory), with the path's global index
// first_index + i * index_stride.
__global__ void __launch_bounds__(256) finite_count_kernel(long long P, const int8_t* status, int* block_counts) {
  const long long i = (long long)blockIdx.x * 256 + threadIdx.x;
  const int st = i < P ? status[i] : NID_FAILED;
  const int cnt = __syncthreads_count(st == NID_CONVERGED || st == NID_SINGULAR_ENDPOINT);
  if (threadIdx.x == 0) block_counts[blockIdx.x] = cnt;
}

__global__ void __launch_bounds__(256) finite_compact_kernel(long long P, int n, const cd* x, const int8_t* status,
                                                             const long long* block_off, long long first_index,
                                                             long long index_stride, cd* out, long long* index_out) {
  __shared__ int wtot[8];
  const long long i = (long long)blockIdx.x * 256 + threadIdx.x;
  const int st = i < P ? status[i] : NID_FAILED;
  const bool keep = st == NID_CONVERGED || st == NID_SINGULAR_ENDPOINT;
  const unsigned m = __ballot_sync(0xffffffffu, keep);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) wtot[w] = __popc(m);
  __syncthreads();
  int base = 0;
  for (int k = 0; k < w; ++k) base += wtot[k];
  if (keep) {
    const long long dst = block_off[blockIdx.x] + base + __popc(m & ((1u << lane) - 1u));
    for (int v = 0; v < n; ++v) out[dst * n + v] = x[i * n + v];
    if (index_out) index_out[dst] = first_index + i * index_stride;
  }
}
