// Common device arithmetic: complex128, NaN-propagating reductions and the
// thread-group ("one group of n lanes per path") collectives.
#pragma once
#ifdef __CUDACC_RTC__
// NVRTC (csrc JIT, paper_1804_03807_b200/jit.py): no host headers
typedef signed char int8_t;
typedef unsigned char uint8_t;
typedef int int32_t;
typedef unsigned int uint32_t;
typedef long long int64_t;
typedef unsigned long long uint64_t;
#define INFINITY __longlong_as_double(0x7ff0000000000000ULL)
#define NAN __longlong_as_double(0x7ff8000000000000ULL)
#define NID_NO_STD_HEADERS 1
#else
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#endif

#include "nid.h"

#define NID_HD __host__ __device__ __forceinline__
#define NID_D __device__ __forceinline__

// 16-byte aligned so a complex loads/stores as one 128-bit access
struct __align__(16) cd {
  double re, im;
};

NID_HD cd mkc(double r, double i) { return cd{r, i}; }
NID_HD cd operator+(cd a, cd b) { return cd{a.re + b.re, a.im + b.im}; }
NID_HD cd operator-(cd a, cd b) { return cd{a.re - b.re, a.im - b.im}; }
NID_HD cd operator-(cd a) { return cd{-a.re, -a.im}; }
NID_HD cd operator*(cd a, cd b) {
  return cd{fma(a.re, b.re, -a.im * b.im), fma(a.re, b.im, a.im * b.re)};
}
NID_HD cd operator*(double s, cd a) { return cd{s * a.re, s * a.im}; }
NID_HD cd cfma(cd a, cd b, cd c) {  // a*b + c
  return cd{fma(a.re, b.re, fma(-a.im, b.im, c.re)), fma(a.re, b.im, fma(a.im, b.re, c.im))};
}
NID_HD cd cfms(cd c, cd a, cd b) {  // c - a*b
  return cd{fma(-a.re, b.re, fma(a.im, b.im, c.re)), fma(-a.re, b.im, fma(-a.im, b.re, c.im))};
}
// complex product and difference with every step rounded separately (no
// FMA contraction), the arithmetic of LAPACK's reference-style updates
NID_HD cd cmul_nf(cd a, cd b) {
#ifdef __CUDA_ARCH__
  return cd{__dsub_rn(__dmul_rn(a.re, b.re), __dmul_rn(a.im, b.im)),
            __dadd_rn(__dmul_rn(a.re, b.im), __dmul_rn(a.im, b.re))};
#else
  return cd{a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
#endif
}
NID_HD cd csub_nf(cd a, cd b) {
#ifdef __CUDA_ARCH__
  return cd{__dsub_rn(a.re, b.re), __dsub_rn(a.im, b.im)};
#else
  return cd{a.re - b.re, a.im - b.im};
#endif
}
NID_HD double cabs1(cd a) { return fabs(a.re) + fabs(a.im); }
NID_HD double cabsd(cd a) { return hypot(a.re, a.im); }
NID_HD bool cfinite(cd a) { return isfinite(a.re) && isfinite(a.im); }
// Smith's complex division (robust against overflow).
NID_HD cd cdiv(cd a, cd b) {
  if (fabs(b.re) >= fabs(b.im)) {
    double r = b.im / b.re, den = b.re + b.im * r;
    return cd{(a.re + a.im * r) / den, (a.im - a.re * r) / den};
  }
  double r = b.re / b.im, den = b.im + b.re * r;
  return cd{(a.re * r + a.im) / den, (a.im * r - a.re) / den};
}
NID_HD cd crecip(cd b) { return cdiv(cd{1.0, 0.0}, b); }
// 1/b with a single real division: b is scaled by an exact power of two so
// |b|^2 can neither overflow nor underflow (rounding-level equal to crecip)
// 1/d for a normal d with |d| in [1e-300, 1e300]: the MUFU seed refined by
// two Newton steps (quadratic: ~2^-23 -> 2^-46 -> full precision), no
// division slow path
NID_D double rcp_nr(double d) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
  double e = fma(-d, y, 1.0);
  y = fma(y, e, y);
  e = fma(-d, y, 1.0);
  return fma(y, e, y);
}
NID_D cd crecip_fast(cd b) {
  const double m = fmax(fabs(b.re), fabs(b.im));
  if (m > 1e-150 && m < 1e150) {  // |b|^2 safely representable: one reciprocal
    const double d = rcp_nr(fma(b.re, b.re, b.im * b.im));
    return cd{b.re * d, -b.im * d};
  }
  if (!(m > 0.0) || !isfinite(m)) return crecip(b);
  const double s = ldexp(1.0, -ilogb(m));
  const double re = b.re * s, im = b.im * s;
  const double d = s / fma(re, re, im * im);
  return cd{re * d, -im * d};
}
// |a| by one square root when |a|^2 is safely representable (hypot otherwise);
// within an ulp of hypot
NID_HD double cabs_fast(cd a) {
  const double m = fmax(fabs(a.re), fabs(a.im));
  if (m > 1e-150 && m < 1e150) return sqrt(fma(a.re, a.re, a.im * a.im));
  return hypot(a.re, a.im);
}
// |a|^2 (for max-norm comparisons: one sqrt at the end instead of a hypot per entry)
NID_HD double cabs2(cd a) { return fma(a.re, a.re, a.im * a.im); }

// max that propagates NaN like numpy's np.max
NID_HD double nanmax(double a, double b) {
  if (isnan(a) || isnan(b)) return a + b;
  return a > b ? a : b;
}

static constexpr double NOISE_ULPS = 50.0 * 2.220446049250313e-16;  // tracker.py:31
static constexpr double CONVERGED_RESIDUAL = 1e-8;                   // tracker.py:46
static constexpr double SINGULARITY_TOL = 1e-8;                      // linalg.py:10

// ---------------------------------------------------------------------------
// A path group: N consecutive lanes of a warp (lane lg = 0..N-1 owns row lg).
// floor(32/N) groups per warp; leftover lanes form an inert group.
// All collectives read only lanes of the caller's own group, so they are
// safe in group-divergent code.
template <int N>
struct Grp {
  int lane, lg, gbase, gid;  // gid: group index in warp
  unsigned mask;  // sync mask of the *_sync intrinsics: the group's lanes (safe in
                  // group-divergent code) or the full warp (converged compute rounds)
  unsigned bits;  // the group's own lanes
  bool real;      // false for the leftover lanes
  NID_D static Grp make() {
    Grp g;
    g.lane = threadIdx.x & 31;
    constexpr int P = 32 / N;
    g.gid = g.lane / N;
    g.real = g.gid < P;
    g.gbase = g.gid * N;
    g.lg = g.lane - g.gbase;
    int cnt = g.real ? N : (32 - P * N);
    unsigned m = (cnt >= 32) ? 0xffffffffu : ((1u << cnt) - 1u);
    g.mask = m << g.gbase;
    g.bits = g.mask;
    return g;
  }
  // the same group, for code every lane of the warp executes together
  NID_D Grp warpwide() const {
    Grp w = *this;
    w.mask = 0xffffffffu;
    return w;
  }
  NID_D int src(int j) const { int s = gbase + j; return s < 32 ? s : lane; }
};

NID_D double shfl_d(unsigned mask, double v, int src) { return __shfl_sync(mask, v, src); }
NID_D cd shfl_c(unsigned mask, cd v, int src) {
  return cd{__shfl_sync(mask, v.re, src), __shfl_sync(mask, v.im, src)};
}

// tree reduction inside the group (lanes lg + s < N only), result broadcast
template <int N, class Op>
NID_D double group_reduce(const Grp<N>& g, double v, Op op) {
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) {
    if (s < N) {
      bool ok = (g.lg + s < N) && (g.lane + s < 32);
      double o = __shfl_sync(g.mask, v, ok ? g.lane + s : g.lane);
      if (ok) v = op(v, o);
    }
  }
  return __shfl_sync(g.mask, v, g.gbase);
}

struct OpNanMax {
  NID_D double operator()(double a, double b) const { return nanmax(a, b); }
};
struct OpMax {
  NID_D double operator()(double a, double b) const { return fmax(a, b); }
};
struct OpSum {
  NID_D double operator()(double a, double b) const { return a + b; }
};

template <int N>
NID_D double group_nanmax(const Grp<N>& g, double v) { return group_reduce<N>(g, v, OpNanMax()); }
template <int N>
NID_D double group_sum(const Grp<N>& g, double v) { return group_reduce<N>(g, v, OpSum()); }
template <int N>
NID_D bool group_all(const Grp<N>& g, bool b) {
  unsigned bal = __ballot_sync(g.mask, !b) & g.bits;
  return bal == 0;
}

// all-gather of one complex per lane: out[v] = value held by lane v of the group
template <int N>
NID_D void group_gather(const Grp<N>& g, cd own, cd (&out)[N]) {
#pragma unroll
  for (int v = 0; v < N; ++v) out[v] = shfl_c(g.mask, own, g.src(v));
}

// select element lg of a register array without dynamic indexing
template <int N>
NID_D cd pick(const cd (&a)[N], int i) {
  cd r = a[0];
#pragma unroll
  for (int v = 1; v < N; ++v)
    if (v == i) r = a[v];
  return r;
}
