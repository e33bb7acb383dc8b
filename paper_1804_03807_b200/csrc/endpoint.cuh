// K4/K5/K6: endpoint solutions, double-double polish, refine + classify.
//
//   endpoint_kernel  _endpoint_solution + the cond > 1e4 double-double polish
//                    of _finish (tracker.py:255-259, 319-331)
//   dd_polish        _dd_polish (tracker.py:262-302) with solve_dd
//                    (linalg.py:54-76) in complex double-double
//   refine_kernel    newton_refine (tracker.py:410-428) + condition_and_rank
//                    (linalg.py:13-32) + classify (tracker.py:438-455)
//   ddrefine_kernel  refine_dd (tracker.py:431-435)
//
// All run one path group per point; the O(n^3) serial parts (Jacobi SVD,
// double-double elimination) run on the group's lane 0 over a per-group
// global scratch slab while the other lanes evaluate rows.
#pragma once
#include "dd.cuh"
#include "homotopy.cuh"
#include "linalg.cuh"

// CDD evaluation of target row `row` (t = 1) and its Jacobian row, term by
// term with repeated products in variable order (polynomials.py:293-314).
template <int N>
NID_D void cdd_row(const HomDev& H, int row, const cdd (&x)[N], const cd* prm, cdd& rv, cdd* Jrow) {
  // One prefix and one suffix pass over each term's variables give the value
  // and every partial derivative (the reference multiplies each derivative
  // term out on its own, polynomials.py:293-314: the same products, other
  // association, a double-double rounding apart).
  rv = cdd_zero();
  if (row >= H.n) return;
  const int k0 = H.row_off[row], k1 = H.row_off[row + 1];
  cdd Jr[N];
#pragma unroll
  for (int j = 0; j < N; ++j) Jr[j] = cdd_zero();
  const cdd one = cdd_from(cd{1.0, 0.0});
#pragma unroll 1
  for (int k = k0; k < k1; ++k) {
    cd c = H.ct[k];
    if (H.pslot != nullptr && H.pslot[k] >= 0) c = prm[H.pslot[k]];
    if (c.re == 0.0 && c.im == 0.0) continue;
    const uint4 ew = H.expo[k];
    const unsigned w[4] = {ew.x, ew.y, ew.z, ew.w};
    cdd F[N], D[N], P[N];
    int var[N];
    int K = 0;
#pragma unroll 1
    for (int u = 0; u < N; ++u) {
      const int a = expo_at(w, u);
      if (a == 0) continue;
      cdd pw = one;
      for (int e = 1; e < a; ++e) pw = cdd_mul(pw, x[u]);
      F[K] = a == 1 ? x[u] : cdd_mul(pw, x[u]);
      const dd aa = dd{(double)a, 0.0};
      D[K] = a == 1 ? pw : cdd{dd_mul(pw.re, aa), dd_mul(pw.im, aa)};
      var[K] = u | (a == 1 ? 16 : 0);  // bit 4: D[K] is one
      ++K;
    }
    cdd p = cdd_from(c);
#pragma unroll 1
    for (int q = 0; q < K; ++q) {
      P[q] = p;
      p = cdd_mul(p, F[q]);
    }
    rv = cdd_add(rv, p);
    // products with the constant one are skipped (they are exact in
    // double-double, so the results are the same bit for bit): the derivative
    // factor of an exponent-1 variable, the empty suffix of the last position
    // and the suffix update after the first
    cdd sfx = one;
#pragma unroll 1
    for (int q = K - 1; q >= 0; --q) {
      cdd d = (var[q] & 16) ? P[q] : cdd_mul(P[q], D[q]);
      if (q < K - 1) d = cdd_mul(d, sfx);
      const int u = var[q] & 15;
#pragma unroll
      for (int j = 0; j < N; ++j)
        if (j == u) Jr[j] = cdd_add(Jr[j], d);
      if (q > 0) sfx = q == K - 1 ? F[q] : cdd_mul(sfx, F[q]);
    }
  }
#pragma unroll
  for (int j = 0; j < N; ++j) Jrow[j] = Jr[j];
}

// per-group double-double scratch layout (cdd units)
template <int N>
struct DDSlab {
  static constexpr int J = 0;                  // N*N
  static constexpr int R = N * N;              // N
  static constexpr int A = N * N + N;          // N*(N+1) augmented
  static constexpr int PT = 2 * N * N + 2 * N; // N
  static constexpr int DX = 2 * N * N + 3 * N; // N
  static constexpr int SIZE = 2 * N * N + 4 * N;
};

// _dd_polish at t = 1 starting from the group's point x (full copy in every
// lane).  On success writes the polished point to out (full copy) and
// returns true; returns false where the reference returns None.
template <int N>
NID_D bool dd_polish(const Grp<N>& g, const HomDev& H, const cd* prm, const cd (&x)[N], int steps, cdd* sl,
                     cd (&out)[N]) {
  using L = DDSlab<N>;
  cdd* Js = sl + L::J;
  cdd* Rs = sl + L::R;
  cdd* As = sl + L::A;
  cdd* Ps = sl + L::PT;
  cdd* Ds = sl + L::DX;
  if (g.lg == 0)
    for (int v = 0; v < N; ++v) Ps[v] = cdd_from(x[v]);
  __syncwarp(g.mask);
  int fail = 0;
  for (int it = 0; it < steps; ++it) {
    cdd pt[N];
#pragma unroll
    for (int v = 0; v < N; ++v) pt[v] = Ps[v];
    cdd rv;
    cdd_row<N>(H, g.lg, pt, prm, rv, Js + g.lg * N);
    Rs[g.lg] = rv;
    __syncwarp(g.mask);
    // normal equations row p = lg: A_pq = sum_k conj(J_kp) J_kq, b_p = -sum_k conj(J_kp) r_k
    {
      const int p = g.lg;
      for (int q = 0; q < N; ++q) {
        cdd acc = cdd_zero();
        for (int k = 0; k < N; ++k) acc = cdd_add(acc, cdd_mul(cdd_conj(Js[k * N + p]), Js[k * N + q]));
        As[p * (N + 1) + q] = acc;
      }
      cdd acc = cdd_zero();
      for (int k = 0; k < N; ++k) acc = cdd_add(acc, cdd_mul(cdd_conj(Js[k * N + p]), Rs[k]));
      As[p * (N + 1) + N] = cdd_neg(acc);
    }
    __syncwarp(g.mask);
    int stop = 0;
    double scale = 0.0;
    if (g.lg == 0) {
      for (int i = 0; i < N; ++i) scale = fmax(scale, cdd_abs(As[i * (N + 1) + i]));
      if (scale == 0.0) scale = 1.0;
      const double lam = 1e-26 * scale;
      for (int i = 0; i < N; ++i) As[i * (N + 1) + i] = cdd_add_real(As[i * (N + 1) + i], lam);
    }
    __syncwarp(g.mask);
    // solve_dd: Gaussian elimination, partial pivoting on |.| (linalg.py:54-76),
    // lane i eliminating row i (the same operations per entry as the serial
    // loop); the pivot is the first largest |A_ik|, i >= k
    for (int k = 0; k < N && !fail; ++k) {
      double a = g.lg >= k ? cdd_abs(As[g.lg * (N + 1) + k]) : -1.0;
      if (!(a == a)) a = -1.0;
      const double best = group_reduce<N>(g, a, OpMax());
      const unsigned eq = (__ballot_sync(g.mask, g.lg >= k && a == best) & g.bits) >> g.gbase;
      const int piv = eq ? __ffs(eq) - 1 : k;
      if (!(best > 0.0)) {
        fail = 1;
        break;
      }
      if (piv != k) {
        for (int j = g.lg; j <= N; j += N) {
          const cdd tmp = As[k * (N + 1) + j];
          As[k * (N + 1) + j] = As[piv * (N + 1) + j];
          As[piv * (N + 1) + j] = tmp;
        }
      }
      __syncwarp(g.mask);
      if (g.lg > k) {
        const int i = g.lg;
        const cdd f = cdd_div(As[i * (N + 1) + k], As[k * (N + 1) + k]);
        if (!(f.re.hi == 0.0 && f.im.hi == 0.0))
          for (int j = k; j <= N; ++j)
            As[i * (N + 1) + j] = cdd_sub(As[i * (N + 1) + j], cdd_mul(f, As[k * (N + 1) + j]));
      }
      __syncwarp(g.mask);
    }
    if (g.lg == 0 && !fail) {
      for (int k = N - 1; k >= 0; --k) {
        cdd s = As[k * (N + 1) + N];
        for (int j = k + 1; j < N; ++j) s = cdd_sub(s, cdd_mul(As[k * (N + 1) + j], Ds[j]));
        Ds[k] = cdd_div(s, As[k * (N + 1) + k]);
      }
      double mx = 0.0;
      for (int v = 0; v < N; ++v) {
        Ps[v] = cdd_add(Ps[v], Ds[v]);
        mx = fmax(mx, cdd_abs(Ds[v]));
      }
      if (mx < 1e-14 * scale) stop = 1;
    }
    fail = __shfl_sync(g.mask, fail, g.gbase);
    stop = __shfl_sync(g.mask, stop, g.gbase);
    __syncwarp(g.mask);
    if (fail) return false;
    if (stop) break;
  }
  bool fin = true;
#pragma unroll
  for (int v = 0; v < N; ++v) {
    out[v] = cdd_to(Ps[v]);
    fin = fin && cfinite(out[v]);
  }
  __syncwarp(g.mask);
  return fin;
}

// condition_and_rank (linalg.py:13-32) of the group's Jacobian, one row per
// lane, by a one-sided (Hestenes) Jacobi SVD run by the whole group: the rows
// are orthogonalised pairwise (the singular values of J are those of its
// transpose), N/2 disjoint pairs per round in round-robin order, each lane
// fetching its partner's row by shuffles and both lanes of a pair forming the
// same rotation from the same operands; the singular values are the row norms.
// (The parity hook svd_kernel keeps the serial jacobi_svd of linalg.cuh, which
// until round 2 also served here on the group's lane 0 over a global scratch
// slab: 1.2 s of endpoint_kernel<14> for C4's 400,000 endpoints.)  `cs` is unused.
template <int N>
NID_D void group_cond_rank(const Grp<N>& g, const cd (&Jrow)[N], cd* cs, double& cond, int& rank) {
  (void)cs;
  cd u[N];
  bool fin = true;
#pragma unroll
  for (int v = 0; v < N; ++v) {
    u[v] = Jrow[v];
    fin = fin && cfinite(u[v]);
  }
  if (!group_all<N>(g, fin)) {
    cond = INFINITY;
    rank = 0;
    return;
  }
  constexpr int M = (N + 1) & ~1;  // players of the round-robin (a dummy for odd N)
  const double eps = 2.220446049250313e-16;
  if (N > 1) {
#pragma unroll 1
    for (int sweep = 0; sweep < 60; ++sweep) {
      bool rotated = false;
#pragma unroll 1
      for (int r = 0; r < M - 1; ++r) {
        // circle method: player M-1 stays, the others rotate
        int partner;
        if (g.lg == M - 1) {
          partner = (r * (M / 2)) % (M - 1);
        } else {
          partner = (r - g.lg) % (M - 1);
          if (partner < 0) partner += M - 1;
          if (partner == g.lg) partner = M - 1;
        }
        const bool idle = partner >= N;
        const int src = g.gbase + (idle ? g.lg : partner);
        cd w[N];
#pragma unroll
        for (int i = 0; i < N; ++i) w[i] = shfl_c(g.mask, u[i], src);
        if (!idle) {
          const bool low = g.lg < partner;  // the pair's first vector is the lower lane's row
          double al = 0.0, be = 0.0;
          cd ga = cd{0.0, 0.0};
#pragma unroll
          for (int i = 0; i < N; ++i) {
            const cd ap = low ? u[i] : w[i], aq = low ? w[i] : u[i];
            al += ap.re * ap.re + ap.im * ap.im;
            be += aq.re * aq.re + aq.im * aq.im;
            ga.re += ap.re * aq.re + ap.im * aq.im;  // conj(ap) * aq
            ga.im += ap.re * aq.im - ap.im * aq.re;
          }
          const double gabs = hypot(ga.re, ga.im);
          if (gabs > eps * sqrt(al * be) && gabs != 0.0) {
            rotated = true;
            const cd ph = cd{ga.re / gabs, -ga.im / gabs};  // e^{-i phi}
            const double zeta = (be - al) / (2.0 * gabs);
            const double tt = (zeta >= 0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
            const double c = 1.0 / sqrt(1.0 + tt * tt), sn = c * tt;
#pragma unroll
            for (int i = 0; i < N; ++i) {
              const cd ap = low ? u[i] : w[i];
              const cd aq = (low ? w[i] : u[i]) * ph;
              u[i] = low ? cd{c * ap.re - sn * aq.re, c * ap.im - sn * aq.im}
                         : cd{sn * ap.re + c * aq.re, sn * ap.im + c * aq.im};
            }
          }
        }
      }
      if (!(__ballot_sync(g.mask, rotated) & g.bits)) break;
    }
  }
  double s2 = 0.0;
#pragma unroll
  for (int i = 0; i < N; ++i) s2 += u[i].re * u[i].re + u[i].im * u[i].im;
  const double sv = sqrt(s2);
  const double smax = group_reduce<N>(g, sv, OpMax());
  const double smin = -group_reduce<N>(g, -sv, OpMax());
  if (!(smax > 0.0) || !isfinite(smax)) {
    cond = INFINITY;
    rank = 0;
    return;
  }
  rank = __popc(__ballot_sync(g.mask, sv > SINGULARITY_TOL * smax) & g.bits);
  cond = (smin == 0.0) ? INFINITY : smax / smin;
}

struct EndpointArgs {
  HomDev H;
  long long P;
  int dd_steps;  // 0 disables the polish
  // double-double tracking (_track_dd, tracker.py:486-497): no cond > 1e4 polish
  // inside _finish (the _DDView has no eval_generic); instead every endpoint is
  // polished with dd_steps steps and taken when its double residual is finite
  // and <= 4 x the endpoint residual
  int dd_mode;
  const cd* params;
  int param_div;
  cd* x_end;
  const int8_t* status;
  double* resid;
  double* cond;
  int8_t* regular;
  cdd* ddscratch;  // per group DDSlab<N>::SIZE
  cd* cscratch;    // per group 2*N*N
  unsigned long long* counters;  // [4] dd polished count
};

template <int N>
__global__ void __launch_bounds__(128) endpoint_kernel(EndpointArgs E) {
  const Grp<N> g = Grp<N>::make();
  if (!g.real) return;
  const long long gslot = (long long)(blockIdx.x * blockDim.x + threadIdx.x) / 32 * (32 / N) + g.gid;
  const long long ngroups = (long long)gridDim.x * blockDim.x / 32 * (32 / N);
  cdd* dsl = E.ddscratch + gslot * DDSlab<N>::SIZE;
  cd* csl = E.cscratch + gslot * (2 * N * N);
  unsigned long long polished = 0;
  for (long long p = gslot; p < E.P; p += ngroups) {
    const int st = E.status[p];
    if (st != NID_CONVERGED && st != NID_SINGULAR_ENDPOINT) {
      if (g.lg == 0) {
        E.cond[p] = NAN;
        E.regular[p] = -1;
      }
      continue;
    }
    const cd* prm = E.params ? E.params + (p / E.param_div) * E.H.nparam : nullptr;
    cd x[N];
#pragma unroll
    for (int v = 0; v < N; ++v) x[v] = E.x_end[p * N + v];
    double res = E.resid[p];
    cd hv, J[N];
    double sS, sT, cond;
    int rank;
    eval_row<N>(E.H, g.lg, x, 1.0, prm, hv, J, sS, sT, false);
    group_cond_rank<N>(g, J, csl, cond, rank);
    if (E.dd_mode ? E.dd_steps > 0 : (st == NID_CONVERGED && cond > 1e4 && E.dd_steps > 0)) {
      cd better[N];
      if (dd_polish<N>(g, E.H, prm, x, E.dd_steps, dsl, better)) {
        cd hb = eval_row_value<N>(E.H, g.lg, better, 1.0, prm);
        double res2 = group_nanmax<N>(g, cabsd(hb));
        if (isfinite(res2) && res2 <= (E.dd_mode ? res * 4.0 : fmax(res * 4.0, 1e-14))) {
#pragma unroll
          for (int v = 0; v < N; ++v) x[v] = better[v];
          res = res2;
          eval_row<N>(E.H, g.lg, x, 1.0, prm, hv, J, sS, sT, false);
          group_cond_rank<N>(g, J, csl, cond, rank);
          polished += 1;
        }
      }
    }
    E.x_end[p * N + g.lg] = pick<N>(x, g.lg);
    if (g.lg == 0) {
      E.resid[p] = res;
      E.cond[p] = cond;
      E.regular[p] = cond < 1.0 / SINGULARITY_TOL ? 1 : 0;
    }
  }
  if (g.lg == 0 && polished) atomicAdd(E.counters, polished);
}

// ---------------------------------------------------------------------------
// newton_refine + classify (and the t=1 damped Newton it shares with _finish)

struct RefineArgs {
  HomDev H;
  long long P;
  double tol;
  int iters;
  int n_original;
  double inf_thr;
  cd* x;
  double* resid;
  double* cond;
  int8_t* regular;
  int* rank;
  int8_t* slack;
  cd* cscratch;  // per group 3*N*N + 2*N
};

// LU with the lstsq fallback for a group-divergent context (refine)
template <int N>
NID_D void group_newton_step(const Grp<N>& g, const HomDev& H, const cd (&x)[N], const cd* prm, cd (&J)[N],
                             cd hv, cd* sc, cd (&dx)[N]) {
  cd mine;
#pragma unroll
  for (int v = 0; v < N; ++v) dx[v] = J[v];
  bool ok = group_lu_solve<N>(g, dx, -hv, mine);
  if (!ok) {
#pragma unroll
    for (int v = 0; v < N; ++v) sc[g.lg * N + v] = J[v];
    sc[N * N + g.lg] = -hv;
    __syncwarp(g.mask);
    if (g.lg == 0) {
      double sv[N];
      lstsq_minnorm(sc, N, N, N, sc + N * N, sc + N * N + N, sv, sc + 2 * N * N + N);
    }
    __syncwarp(g.mask);
#pragma unroll
    for (int v = 0; v < N; ++v) dx[v] = sc[2 * N * N + N + v];
    __syncwarp(g.mask);
  }
}

// _damped_newton (tracker.py:210-238) at t=1; x in/out (full copy), returns residual
template <int N>
NID_D double group_damped_newton(const Grp<N>& g, const HomDev& H, cd (&x)[N], const cd* prm, double tol, int iters,
                                 cd* sc) {
  cd hv, J[N];
  double sS, sT;
  eval_row<N>(H, g.lg, x, 1.0, prm, hv, J, sS, sT, false);
  double res = group_nanmax<N>(g, cabsd(hv));
  for (int it = 0; it < iters; ++it) {
    if (!isfinite(res) || res <= tol) break;
    cd dx[N];
    group_newton_step<N>(g, H, x, prm, J, hv, sc, dx);
    double lam = 1.0;
    bool improved = false;
    for (int tr = 0; tr < 8; ++tr) {
      cd xt[N];
#pragma unroll
      for (int v = 0; v < N; ++v) xt[v] = x[v] + cd{lam, 0.0} * dx[v];
      cd ht, Jt[N];
      eval_row<N>(H, g.lg, xt, 1.0, prm, ht, Jt, sS, sT, false);
      double rt = group_nanmax<N>(g, cabsd(ht));
      if (isfinite(rt) && rt < res) {
#pragma unroll
        for (int v = 0; v < N; ++v) {
          x[v] = xt[v];
          J[v] = Jt[v];
        }
        hv = ht;
        res = rt;
        improved = true;
        break;
      }
      lam *= 0.5;
    }
    if (!improved) break;
  }
  return res;
}

template <int N>
__global__ void __launch_bounds__(128) refine_kernel(RefineArgs R) {
  const Grp<N> g = Grp<N>::make();
  if (!g.real) return;
  const long long gslot = (long long)(blockIdx.x * blockDim.x + threadIdx.x) / 32 * (32 / N) + g.gid;
  const long long ngroups = (long long)gridDim.x * blockDim.x / 32 * (32 / N);
  cd* sc = R.cscratch + gslot * (3 * N * N + 2 * N);
  for (long long p = gslot; p < R.P; p += ngroups) {
    cd x[N];
#pragma unroll
    for (int v = 0; v < N; ++v) x[v] = R.x[p * N + v];
    double res = group_damped_newton<N>(g, R.H, x, nullptr, R.tol, R.iters, sc);
    cd hv, J[N];
    double sS, sT, cond;
    int rank;
    eval_row<N>(R.H, g.lg, x, 1.0, nullptr, hv, J, sS, sT, false);
    group_cond_rank<N>(g, J, sc, cond, rank);
    // classify (tracker.py:438-455)
    bool fin = true;
    double mx = 0.0, ms = 0.0;
#pragma unroll
    for (int v = 0; v < N; ++v) {
      fin = fin && cfinite(x[v]);
      double a = cabsd(x[v]);
      mx = nanmax(mx, a);
      if (v >= R.n_original) ms = nanmax(ms, a);
    }
    int cls;
    if (!fin || mx > R.inf_thr) cls = NID_CLS_AT_INFINITY;
    else if (R.n_original >= N || ms < 1e-8) cls = NID_CLS_ZERO_SLACK;
    else cls = NID_CLS_NONZERO_SLACK;
    R.x[p * N + g.lg] = pick<N>(x, g.lg);
    if (g.lg == 0) {
      R.resid[p] = res;
      R.cond[p] = cond;
      R.regular[p] = cond < 1.0 / SINGULARITY_TOL ? 1 : 0;
      R.rank[p] = rank;
      R.slack[p] = (int8_t)cls;
    }
  }
}

struct DDRefineArgs {
  HomDev H;
  long long P;
  int steps;
  cd* x;
  int8_t* ok;
  cdd* ddscratch;
};

template <int N>
__global__ void __launch_bounds__(128) ddrefine_kernel(DDRefineArgs D) {
  const Grp<N> g = Grp<N>::make();
  if (!g.real) return;
  const long long gslot = (long long)(blockIdx.x * blockDim.x + threadIdx.x) / 32 * (32 / N) + g.gid;
  const long long ngroups = (long long)gridDim.x * blockDim.x / 32 * (32 / N);
  cdd* dsl = D.ddscratch + gslot * DDSlab<N>::SIZE;
  for (long long p = gslot; p < D.P; p += ngroups) {
    cd x[N], out[N];
#pragma unroll
    for (int v = 0; v < N; ++v) x[v] = D.x[p * N + v];
    bool ok = dd_polish<N>(g, D.H, nullptr, x, D.steps, dsl, out);
    if (ok) D.x[p * N + g.lg] = pick<N>(out, g.lg);
    if (g.lg == 0) D.ok[p] = ok ? 1 : 0;
  }
}

// ---------------------------------------------------------------------------
// parity hooks: batched H/J/scale and Newton steps

struct EvalArgs {
  HomDev H;
  long long P;
  const cd* x;
  const double* t;
  const cd* params;
  int param_div;
  cd* Hout;
  cd* Jout;
  double* scale;
};

template <int N>
__global__ void __launch_bounds__(128) eval_kernel(EvalArgs E) {
  const Grp<N> g = Grp<N>::make();
  if (!g.real) return;
  const long long gslot = (long long)(blockIdx.x * blockDim.x + threadIdx.x) / 32 * (32 / N) + g.gid;
  const long long ngroups = (long long)gridDim.x * blockDim.x / 32 * (32 / N);
  for (long long p = gslot; p < E.P; p += ngroups) {
    cd x[N];
#pragma unroll
    for (int v = 0; v < N; ++v) x[v] = E.x[p * N + v];
    const cd* prm = E.params ? E.params + (p / E.param_div) * E.H.nparam : nullptr;
    cd hv, J[N];
    double sS, sT;
    const double t = E.t[p];
    eval_row<N>(E.H, g.lg, x, t, prm, hv, J, sS, sT, true);
    double mS = group_reduce<N>(g, sS, OpMax());
    double mT = group_reduce<N>(g, sT, OpMax());
    E.Hout[p * N + g.lg] = hv;
#pragma unroll
    for (int v = 0; v < N; ++v) E.Jout[(p * N + g.lg) * N + v] = J[v];
    if (g.lg == 0) E.scale[p] = E.H.tw ? mT : (1.0 - t) * mS + t * mT;
  }
}

struct NewtonArgs {
  long long P;
  const cd* J;
  const cd* r;
  cd* dx;
  cd* cscratch;
};

template <int N>
__global__ void __launch_bounds__(128) newton_kernel(NewtonArgs A) {
  const Grp<N> g = Grp<N>::make();
  if (!g.real) return;
  const long long gslot = (long long)(blockIdx.x * blockDim.x + threadIdx.x) / 32 * (32 / N) + g.gid;
  const long long ngroups = (long long)gridDim.x * blockDim.x / 32 * (32 / N);
  cd* sc = A.cscratch + gslot * (3 * N * N + 2 * N);
  for (long long p = gslot; p < A.P; p += ngroups) {
    cd dx[N], mine;
#pragma unroll
    for (int v = 0; v < N; ++v) dx[v] = A.J[(p * N + g.lg) * N + v];
    cd rr = A.r[p * N + g.lg];
    bool ok = group_lu_solve<N>(g, dx, -rr, mine);
    if (!ok) {
#pragma unroll
      for (int v = 0; v < N; ++v) sc[g.lg * N + v] = A.J[(p * N + g.lg) * N + v];
      sc[N * N + g.lg] = -rr;
      __syncwarp(g.mask);
      if (g.lg == 0) {
        double sv[N];
        lstsq_minnorm(sc, N, N, N, sc + N * N, sc + N * N + N, sv, sc + 2 * N * N + N);
      }
      __syncwarp(g.mask);
      mine = sc[2 * N * N + N + g.lg];
      __syncwarp(g.mask);
    }
    A.dx[p * N + g.lg] = mine;
  }
}
