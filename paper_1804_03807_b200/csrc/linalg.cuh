// K2: per-path complex LU with partial pivoting (zgesv semantics) and the
// one-sided Jacobi SVD used for condition numbers, ranks and the min-norm
// least-squares fallback.
//
// Replaces newton_step (linalg.py:35-51: np.linalg.solve = LAPACK zgesv,
// falling back to lstsq rcond=1e-14 = zgelsd when zgesv reports an exactly
// zero pivot or returns non-finite values) and condition_and_rank
// (linalg.py:13-32: zgesdd singular values).
#pragma once
#include "nid_common.cuh"

// Group LU solve of A x = b, in place: lane lg holds row lg of A and b[lg];
// on return every lane holds the full solution in A[0..N-1] and mine =
// x[lg].  Rows are never moved: the pivot row of step k is broadcast from
// its lane, and each lane remembers the step it pivoted (mystep); the
// back substitution finds step k's lane by ballot.  Pivot choice is
// LAPACK's izamax rule (largest |Re|+|Im| in column k among unused rows,
// ties to the row first in LAPACK's swapped order, `pos`).  Elimination
// arithmetic is unfused, as LAPACK's zgetf2/zgetrs update loops round it,
// so exactly rank-deficient Jacobians produce the same exact zero pivot
// (and the same lstsq fallback) as zgesv.  The k loops run at runtime
// (uniform across the warp) to keep the kernel inside the instruction
// cache.  Returns false on an exactly zero pivot or a non-finite solution.
template <int N>
NID_D bool group_lu_solve(const Grp<N>& g, cd (&A)[N], cd b, cd& mine) {
  bool used = false;
  int pos = g.lg, mystep = N;
  bool bad = false;
#pragma unroll 1
  for (int k = 0; k < N; ++k) {
    const cd ak = pick<N>(A, k);
    double key = used ? -1.0 : cabs1(ak);
    if (isnan(key)) key = -0.5;
    double bk = key;
    int bp = pos, bl = g.lg;
#pragma unroll
    for (int s = 16; s >= 1; s >>= 1) {
      if (s < N) {
        const bool ok = (g.lg + s < N) && (g.lane + s < 32);
        const int src = ok ? g.lane + s : g.lane;
        const double ok_k = __shfl_sync(g.mask, bk, src);
        const int ok_p = __shfl_sync(g.mask, bp, src);
        const int ok_l = __shfl_sync(g.mask, bl, src);
        if (ok && (ok_k > bk || (ok_k == bk && ok_p < bp))) {
          bk = ok_k;
          bp = ok_p;
          bl = ok_l;
        }
      }
    }
    bk = __shfl_sync(g.mask, bk, g.gbase);
    bp = __shfl_sync(g.mask, bp, g.gbase);
    bl = __shfl_sync(g.mask, bl, g.gbase);
    if (!(bk > 0.0)) bad = true;
    const bool me = (g.lg == bl);
    if (!me && pos == k) pos = bp;
    if (me) {
      pos = k;
      used = true;
      mystep = k;
    }
    const int src = g.src(bl);
    const cd inv = crecip(shfl_c(g.mask, ak, src));
    const cd l = cmul_nf(ak, inv);
#pragma unroll
    for (int j = 1; j < N; ++j) {
      if (j > k) {  // warp-uniform test
        const cd pj = shfl_c(g.mask, A[j], src);
        if (!used) A[j] = csub_nf(A[j], cmul_nf(l, pj));
      }
    }
    const cd pb = shfl_c(g.mask, b, src);
    if (!used) b = csub_nf(b, cmul_nf(l, pb));
  }
  bool fin = true;
  mine = cd{0.0, 0.0};
#pragma unroll 1
  for (int k = N - 1; k >= 0; --k) {
    const cd ak = pick<N>(A, k);
    const unsigned who = __ballot_sync(g.mask, mystep == k) & g.bits;
    const int src = who ? (__ffs(who) - 1) : g.lane;
    cd xk = cdiv(b, ak);
    xk = shfl_c(g.mask, xk, src);
    fin = fin && cfinite(xk);
    if (k == g.lg) mine = xk;
    if (mystep < k) b = csub_nf(b, cmul_nf(ak, xk));
#pragma unroll
    for (int j = 0; j < N; ++j)
      if (j == k) A[j] = xk;
  }
  return !bad && fin;
}

// ---------------------------------------------------------------------------
// One-sided (Hestenes) Jacobi SVD of an m x n complex matrix (m >= n) stored
// row-major in A (leading dimension lda), run by one thread.  Columns are
// rotated until pairwise orthogonal; the singular values are the column
// norms.  V (n x n, ldv) accumulates the right rotations when non-null.
static __device__ __noinline__ void jacobi_svd(cd* A, int m, int n, int lda, cd* V, int ldv, double* sv) {
  if (V) {
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) V[i * ldv + j] = cd{i == j ? 1.0 : 0.0, 0.0};
  }
  const double eps = 2.220446049250313e-16;
  for (int sweep = 0; sweep < 60; ++sweep) {
    bool rotated = false;
    for (int p = 0; p < n - 1; ++p) {
      for (int q = p + 1; q < n; ++q) {
        double al = 0.0, be = 0.0;
        cd ga = cd{0.0, 0.0};
        for (int i = 0; i < m; ++i) {
          cd ap = A[i * lda + p], aq = A[i * lda + q];
          al += ap.re * ap.re + ap.im * ap.im;
          be += aq.re * aq.re + aq.im * aq.im;
          ga.re += ap.re * aq.re + ap.im * aq.im;  // conj(ap) * aq
          ga.im += ap.re * aq.im - ap.im * aq.re;
        }
        double gabs = hypot(ga.re, ga.im);
        if (!(gabs > eps * sqrt(al * be)) || gabs == 0.0) continue;
        rotated = true;
        cd ph = cd{ga.re / gabs, -ga.im / gabs};  // e^{-i phi}
        double zeta = (be - al) / (2.0 * gabs);
        double tt = (zeta >= 0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        double c = 1.0 / sqrt(1.0 + tt * tt), s = c * tt;
        for (int i = 0; i < m; ++i) {
          cd ap = A[i * lda + p], aq = A[i * lda + q] * ph;
          A[i * lda + p] = cd{c * ap.re - s * aq.re, c * ap.im - s * aq.im};
          A[i * lda + q] = cd{s * ap.re + c * aq.re, s * ap.im + c * aq.im};
        }
        if (V) {
          for (int i = 0; i < n; ++i) {
            cd vp = V[i * ldv + p], vq = V[i * ldv + q] * ph;
            V[i * ldv + p] = cd{c * vp.re - s * vq.re, c * vp.im - s * vq.im};
            V[i * ldv + q] = cd{s * vp.re + c * vq.re, s * vp.im + c * vq.im};
          }
        }
      }
    }
    if (!rotated) break;
  }
  for (int j = 0; j < n; ++j) {
    double s2 = 0.0;
    for (int i = 0; i < m; ++i) {
      cd a = A[i * lda + j];
      s2 += a.re * a.re + a.im * a.im;
    }
    sv[j] = sqrt(s2);
  }
}

// descending insertion sort of singular values
NID_D void sort_desc(double* s, int n) {
  for (int i = 1; i < n; ++i) {
    double v = s[i];
    int j = i - 1;
    while (j >= 0 && s[j] < v) {
      s[j + 1] = s[j];
      --j;
    }
    s[j + 1] = v;
  }
}

// condition_and_rank on singular values (linalg.py:13-32)
NID_D void cond_rank_from_sv(const double* s_desc, int k, double tol, double& cond, int& rank) {
  double smax = s_desc[0];
  if (!(smax > 0.0) || !isfinite(smax)) {
    cond = INFINITY;
    rank = 0;
    return;
  }
  rank = 0;
  for (int i = 0; i < k; ++i) rank += (s_desc[i] > tol * smax);
  double smin = s_desc[k - 1];
  cond = (smin == 0.0) ? INFINITY : smax / smin;
}

// Min-norm least squares x = argmin |A x - b| with rcond 1e-14 (zgelsd
// semantics), square or tall A (m x n, row-major lda).  A is destroyed;
// V (n x n) and sv (n) are scratch.
static __device__ __noinline__ void lstsq_minnorm(cd* A, int m, int n, int lda, const cd* b, cd* V, double* sv, cd* x) {
  jacobi_svd(A, m, n, lda, V, n, sv);
  double smax = 0.0;
  for (int j = 0; j < n; ++j) smax = fmax(smax, sv[j]);
  for (int i = 0; i < n; ++i) x[i] = cd{0.0, 0.0};
  for (int j = 0; j < n; ++j) {
    if (!(sv[j] > 1e-14 * smax)) continue;
    cd d = cd{0.0, 0.0};  // a_j^H b
    for (int i = 0; i < m; ++i) {
      cd a = A[i * lda + j];
      d.re += a.re * b[i].re + a.im * b[i].im;
      d.im += a.re * b[i].im - a.im * b[i].re;
    }
    double s2 = sv[j] * sv[j];
    cd cj = cd{d.re / s2, d.im / s2};
    for (int i = 0; i < n; ++i) x[i] = cfma(V[i * n + j], cj, x[i]);
  }
}
