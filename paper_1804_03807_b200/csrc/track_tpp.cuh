// K3 + K4, thread-per-path: the persistent path tracker.
//
// Each thread tracks one path at a time and refills from a global atomic
// claim counter -- the GPU form of the reference's claim-guarded work crew
// (parallel.py:37-109).  Because every thread of a warp walks the SAME term
// table, the evaluation loops are warp-uniform: coefficients and exponents
// are broadcast loads, a variable absent from a term is skipped by a
// uniform branch (sparse cost), and the point x stays in registers.  The
// Jacobian and the Newton right-hand side live in shared memory, laid out
// [element][thread] so that every access of a warp is one conflict-free
// 512-byte line set whatever row permutation each thread has.
//
// Per warp loop iteration: control (per thread), one evaluation round (the
// threads that need H/J), one LU round (the threads that need a Newton
// step).  The control state machine replays, branch for branch,
//   track           tracker.py:341-407  (secant predictor, step control,
//                                        endgame, snap, infinity test)
//   _correct        tracker.py:184-207  (residual-judged Newton, noise floor)
//   _finish         tracker.py:305-338  (t=1 polish + endpoint verdict)
//   _damped_newton  tracker.py:210-238  (8 halvings, never accept increase)
// newton_step (linalg.py:35-51) is an LU with LAPACK's partial pivoting
// (izamax on |Re|+|Im|, unfused updates) and the zgelsd min-norm fallback.
#pragma once
#include "homotopy.cuh"
#include "linalg.cuh"
#include "track.cuh"

namespace tpp {

// shared-memory element (i, j) of this thread's augmented matrix
struct Mat {
  cd* base;  // smem + threadIdx.x
  int stride;  // blockDim.x
  NID_D cd& at(int i, int j, int ncol) const { return base[(i * ncol + j) * stride]; }
};

// x^a for a >= 1 by repeated products (the reference's power table)
NID_D cd upow(cd x, int a) {
  cd r = x;
#pragma unroll 1
  for (int e = 1; e < a; ++e) r = r * x;
  return r;
}

// One target/merged term: accumulate c x^a into hv and its partials into Jr.
template <int N>
NID_D void term_tpp(const HomDev& H, int k, const cd (&x)[N], double t, cd alpha, const cd* prm, bool ml, cd& hv,
                    cd (&Jr)[N]) {
  const uint4 ew = __ldg(H.expo + k);
  const unsigned w[4] = {ew.x, ew.y, ew.z, ew.w};
  cd ct = ldg_c(H.ct + k);
  if (H.pslot != nullptr) {
    const int s = __ldg(H.pslot + k);
    if (s >= 0) ct = prm[s];
  }
  const cd c = H.td ? t * ct : alpha * ldg_c(H.cs + k) + t * ct;
  cd P[N];
  cd p = cd{1.0, 0.0};
  if (ml) {
#pragma unroll
    for (int v = 0; v < N; ++v) {
      if (expo_at(w, v)) {  // warp-uniform: every thread walks the same term
        P[v] = p;
        p = p * x[v];
      }
    }
    hv = cfma(c, p, hv);
    cd s = c;
#pragma unroll
    for (int v = N - 1; v >= 0; --v) {
      if (expo_at(w, v)) {
        Jr[v] = cfma(P[v], s, Jr[v]);
        s = s * x[v];
      }
    }
  } else {
#pragma unroll
    for (int v = 0; v < N; ++v) {
      const int a = expo_at(w, v);
      if (a) {
        P[v] = p;
        p = p * (a == 1 ? x[v] : upow(x[v], a));
      }
    }
    hv = cfma(c, p, hv);
    cd s = c;
#pragma unroll
    for (int v = N - 1; v >= 0; --v) {
      const int a = expo_at(w, v);
      if (a == 1) {
        Jr[v] = cfma(P[v], s, Jr[v]);
        s = s * x[v];
      } else if (a > 1) {
        const cd q = upow(x[v], a - 1);
        Jr[v] = cfma(P[v] * ((double)a * q), s, Jr[v]);
        s = s * (q * x[v]);
      }
    }
  }
}

// Evaluate H(x,t) and J into shared memory (row i: J[i][0..n-1], -H_i in
// column n).  Returns max_i |H_i| (NaN-propagating) and, when want_scale,
// the noise scale (1-t) max_i S_i + t max_i T_i (tracker.py:91-92).
// Terms are taken two at a time with separate accumulators so that their
// product chains overlap (the loop is latency-bound otherwise).
template <int N>
NID_D double eval_tpp(const HomDev& H, const cd (&x)[N], double t, const cd* prm, const Mat& M, bool want_scale,
                      double& scale) {
  const cd alpha = (1.0 - t) * H.gamma;
  double r2 = 0.0, mS = 0.0, mT = 0.0;
  const bool ml = H.multilinear != 0;
#pragma unroll 1
  for (int i = 0; i < N; ++i) {
    cd hv = cd{0.0, 0.0}, hv2 = cd{0.0, 0.0};
    cd Jr[N], Jr2[N];
#pragma unroll
    for (int v = 0; v < N; ++v) {
      Jr[v] = cd{0.0, 0.0};
      Jr2[v] = cd{0.0, 0.0};
    }
    const int k0 = __ldg(H.row_off + i), k1 = __ldg(H.row_off + i + 1);
    int k = k0;
#pragma unroll 1
    for (; k + 1 < k1; k += 2) {
      term_tpp<N>(H, k, x, t, alpha, prm, ml, hv, Jr);
      term_tpp<N>(H, k + 1, x, t, alpha, prm, ml, hv2, Jr2);
    }
    if (k < k1) term_tpp<N>(H, k, x, t, alpha, prm, ml, hv, Jr);
    hv = hv + hv2;
#pragma unroll
    for (int v = 0; v < N; ++v) Jr[v] = Jr[v] + Jr2[v];
    double sS = 0.0, sT = 0.0;
    if (want_scale) {  // abs sums in a separate pass
      double ax[N];
#pragma unroll
      for (int v = 0; v < N; ++v) ax[v] = cabsd(x[v]);
#pragma unroll 1
      for (int kk = k0; kk < k1; ++kk) {
        const uint4 ew = __ldg(H.expo + kk);
        const unsigned w[4] = {ew.x, ew.y, ew.z, ew.w};
        double m = 1.0;
#pragma unroll
        for (int v = 0; v < N; ++v) {
          const int a = expo_at(w, v);
          if (a) {
            double pv = 1.0;
#pragma unroll 1
            for (int e = 0; e < a; ++e) pv = __dmul_rn(pv, ax[v]);
            m = __dmul_rn(m, pv);
          }
        }
        if (!H.td) sS = __dadd_rn(sS, __dmul_rn(__ldg(H.acs + kk), m));
        sT = __dadd_rn(sT, __dmul_rn(__ldg(H.act + kk), m));
      }
    }
    if (H.td) {  // G_i = x_i^{d_i} - 1 in closed form
      const int d = H.tddeg[i];
      const cd xi = pick<N>(x, i);
      cd q = cd{1.0, 0.0};
#pragma unroll 1
      for (int e = 1; e < d; ++e) q = q * xi;
      hv = cfma(alpha, q * xi - cd{1.0, 0.0}, hv);
      const cd dj = alpha * ((double)d * q);
#pragma unroll
      for (int v = 0; v < N; ++v)
        if (v == i) Jr[v] = Jr[v] + dj;
      if (want_scale) {
        const double axi = cabsd(xi);
        double m = 1.0;
#pragma unroll 1
        for (int e = 0; e < d; ++e) m = __dmul_rn(m, axi);
        sS = __dadd_rn(1.0, m);
      }
    }
#pragma unroll
    for (int v = 0; v < N; ++v) M.at(i, v, N + 1) = Jr[v];
    M.at(i, N, N + 1) = -hv;
    r2 = nanmax(r2, cabs2(hv));
    mS = fmax(mS, sS);
    mT = fmax(mT, sT);
  }
  scale = (1.0 - t) * mS + t * mT;
  if (r2 < 1e290) return sqrt(r2);  // NaN falls through to the exact path too
  double resid = 0.0;               // huge or non-finite: the exact max of hypot
#pragma unroll 1
  for (int i = 0; i < N; ++i) resid = nanmax(resid, cabsd(-M.at(i, N, N + 1)));
  return resid;
}

// LU with partial pivoting of the augmented matrix in smem (rows permuted
// implicitly: perm nibbles), then back substitution into dx[] (registers).
// LAPACK zgesv semantics: izamax pivot (first max of |Re|+|Im| in the
// permuted order), multipliers a_ik * (1/a_kk), unfused updates.  Returns
// false on an exactly zero pivot or a non-finite solution.
template <int N>
NID_D bool lu_tpp(const Mat& M, cd (&dx)[N]) {
  unsigned long long perm = 0;
#pragma unroll
  for (int i = 0; i < N; ++i) perm |= (unsigned long long)i << (4 * i);
  bool bad = false;
#pragma unroll 1
  for (int k = 0; k < N; ++k) {
    // pivot search over logical rows k..N-1 (loads issued together)
    int pk = k;
    double best = -1.0;
#pragma unroll
    for (int i = 0; i < N; ++i) {
      if (i >= k) {  // warp-uniform
        const int r = (perm >> (4 * i)) & 15;
        const double key = cabs1(M.at(r, k, N + 1));
        if (key > best) {
          best = key;
          pk = i;
        }
      }
    }
    if (!(best > 0.0)) bad = true;
    // swap logical rows k and pk
    const unsigned long long rk = (perm >> (4 * k)) & 15, rp = (perm >> (4 * pk)) & 15;
    perm &= ~((15ull << (4 * k)) | (15ull << (4 * pk)));
    perm |= (rp << (4 * k)) | (rk << (4 * pk));
    const int r0 = (int)rp;
    // pivot row (columns k+1..N) into registers; j is compile-time, k uniform
    cd prow[N + 1];
#pragma unroll
    for (int j = 1; j <= N; ++j)
      if (j > k) prow[j] = M.at(r0, j, N + 1);
    // the reciprocal of the pivot replaces it (the back substitution multiplies)
    const cd inv = crecip_fast(M.at(r0, k, N + 1));
    M.at(r0, k, N + 1) = inv;
#pragma unroll 2
    for (int i = k + 1; i < N; ++i) {
      const int r = (perm >> (4 * i)) & 15;
      const cd l = cmul_nf(M.at(r, k, N + 1), inv);
#pragma unroll
      for (int j = 1; j <= N; ++j) {
        if (j > k) {
          cd& a = M.at(r, j, N + 1);
          a = csub_nf(a, cmul_nf(l, prow[j]));
        }
      }
    }
  }
  bool fin = true;
#pragma unroll
  for (int k = N - 1; k >= 0; --k) {
    const int r = (perm >> (4 * k)) & 15;
    cd s = M.at(r, N, N + 1);
#pragma unroll
    for (int j = k + 1; j < N; ++j) s = csub_nf(s, cmul_nf(M.at(r, j, N + 1), dx[j]));
    dx[k] = cmul_nf(s, M.at(r, k, N + 1));
    fin = fin && cfinite(dx[k]);
  }
  return !bad && fin;
}

template <int N>
NID_D double norm_inf(const cd (&v)[N]) {
  double m = 0.0;
#pragma unroll
  for (int i = 0; i < N; ++i) m = nanmax(m, cabsd(v[i]));
  return m;
}

template <int N>
NID_D bool all_finite(const cd (&v)[N]) {
  bool f = true;
#pragma unroll
  for (int i = 0; i < N; ++i) f = f && cfinite(v[i]);
  return f;
}

// per-thread shared-memory footprint (complex entries): augmented matrix,
// accepted point x, x_prev (tracking) / x_base (finish), dx of the damped Newton
template <int N>
constexpr int smem_per_thread() {
  return N * (N + 1) + 3 * N;
}

}  // namespace tpp


// consume a Newton step dx (tracker.py:200-205 / 223-233) -- shared by the
// LU round and the lstsq fallback so that dx never outlives its round
#define NID_APPLY_STEP(dxv)                                    \
  do {                                                         \
    if (mode == M_CORR) {                                      \
      bool fin_ = true;                                        \
      _Pragma("unroll") for (int v = 0; v < N; ++v) {          \
        xe[v] = xe[v] + (dxv)[v];                              \
        fin_ = fin_ && cfinite(xe[v]);                         \
      }                                                        \
      if (!fin_) {                                             \
        c_ok = false;                                          \
        c_its = c_it + 1;                                      \
        act = A_CORR_DONE;                                     \
      } else {                                                 \
        c_it += 1;                                             \
        c_phase = (c_it >= c_iters) ? 2 : 1;                   \
        need_scale = (c_phase == 2);                           \
        act = A_EVAL;                                          \
      }                                                        \
    } else {                                                   \
      dn_lam = 1.0;                                            \
      dn_trial = 0;                                            \
      _Pragma("unroll") for (int v = 0; v < N; ++v) {          \
        ds[v * T] = (dxv)[v];                                  \
        xe[v] = xs[v * T] + (dxv)[v];                          \
      }                                                        \
      act = A_EVAL;                                            \
    }                                                          \
  } while (0)

template <int N>
__global__ void __launch_bounds__(128) track_tpp_kernel(TrackArgs A) {
  using namespace tpp;
  extern __shared__ cd smem_tpp[];
  const int T = blockDim.x;
  const Mat M{smem_tpp + threadIdx.x, T};
  cd* const xos = smem_tpp + N * (N + 1) * T + threadIdx.x;  // accepted point x
  cd* const xs = xos + N * T;                                  // x_prev (tracking) / x_base (finish)
  cd* const ds = xs + N * T;                                   // dx of the damped Newton
  const NidTrackParams& q = A.prm;

  cd xe[N];
#pragma unroll
  for (int v = 0; v < N; ++v) xe[v] = cd{0.0, 0.0};
  long long path = -1;
  const cd* prm = nullptr;
  double te = 0.0, c_tol = 0.0, c_tol_eff = 0.0, dn_lam = 1.0, dn_res = 0.0, t = 0.0, step = 0.0, prev_step = 0.0,
         hstep = 0.0, t_try = 0.0, entry_norm = 0.0, norm_now = 0.0, move_cap = 0.0, t_from = 0.0, out_t = 0.0,
         out_res = 0.0, resid = 0.0, scale = 0.0;
  int mode = M_CORR, c_ctx = CTX_PRE, c_iters = 0, c_it = 0, c_phase = 0, c_its = 0, dn_it = 0, dn_trial = 0,
      used = 0, out_status = 0;
  bool c_ok = false, have_prev = false, endgame = false, need_scale = false, out_hasx = false, fallback = false;
  unsigned long long n_eval = 0, n_jac = 0, n_scale = 0, n_fb = 0;
  int act = A_CLAIM;

  while (true) {
    // ------------------------------------------------------------ control (per thread)
    while (act > A_SOLVE) {
      switch (act) {
        case A_CLAIM: {
          const unsigned long long idx = atomicAdd(A.next, 1ull);
          if ((long long)idx >= A.P) {
            act = A_IDLE;
            break;
          }
          path = (long long)idx;
          if (A.starts) {
#pragma unroll
            for (int v = 0; v < N; ++v) xe[v] = A.starts[path * N + v];
          } else {
            long long rem = A.first_index + path;
#pragma unroll
            for (int v = N - 1; v >= 0; --v) {
              const int d = A.deg[v];
              const long long k = rem % d;
              rem /= d;
              xe[v] = A.roots[A.root_off[v] + (int)k];
            }
          }
          prm = A.params ? A.params + (path / A.param_div) * A.H.nparam : nullptr;
          te = 0.0;
          used = 0;
          fallback = false;
          mode = M_CORR;  // precondition _correct(h, x0, 0, tol*10, 3) (tracker.py:356)
          c_ctx = CTX_PRE;
          c_tol = q.corrector_tol * 10.0;
          c_iters = 3;
          c_it = 0;
          c_phase = 0;
          need_scale = true;
          act = A_EVAL;
          break;
        }
        case A_ON_EVAL: {
          if (mode == M_CORR) {  // _correct loop body (tracker.py:191-207)
            if (c_phase == 0) c_tol_eff = fmax(c_tol, NOISE_ULPS * scale);
            if (c_phase == 2 || (c_phase == 0 && c_iters == 0)) {
              c_ok = resid <= fmax(c_tol, NOISE_ULPS * scale);
              c_its = c_iters;
              act = A_CORR_DONE;
            } else if (!isfinite(resid)) {
              c_ok = false;
              c_its = c_it;
              act = A_CORR_DONE;
            } else if (resid <= c_tol_eff) {
              c_ok = true;
              c_its = c_it;
              act = A_CORR_DONE;
            } else {
              act = A_SOLVE;
            }
          } else {  // _damped_newton (tracker.py:216-238)
            if (dn_trial < 0) {
              dn_res = resid;
              act = A_DN_CONT;
            } else if (isfinite(resid) && resid < dn_res) {
#pragma unroll
              for (int v = 0; v < N; ++v) xs[v * T] = xe[v];  // accepted trial is the new base
              dn_res = resid;
              dn_it += 1;
              dn_trial = -1;
              act = A_DN_CONT;
            } else {
              dn_lam *= 0.5;
              dn_trial += 1;
              if (dn_trial < 8) {
#pragma unroll
                for (int v = 0; v < N; ++v) xe[v] = xs[v * T] + cd{dn_lam, 0.0} * ds[v * T];
                act = A_EVAL;
              } else {
                dn_it += 1;  // not improved: break
                act = A_DECIDE;
              }
            }
          }
          break;
        }
        case A_CORR_DONE: {
          if (c_ctx == CTX_PRE) {
            if (!c_ok) {
              out_status = NID_FAILED;
              out_hasx = false;
              out_t = 0.0;
              out_res = NAN;
              act = A_WRITE;
              break;
            }
#pragma unroll
            for (int v = 0; v < N; ++v) xos[v * T] = xe[v];
            t = 0.0;
            step = q.initial_step;
            have_prev = false;
            prev_step = 0.0;
            used = 0;
            entry_norm = norm_inf<N>(xe);
            endgame = false;
            act = A_LOOP_TOP;
            break;
          }
          if (c_ok) {
            if (norm_inf<N>(xe) > q.infinity_threshold) {
              out_status = NID_AT_INFINITY;
              out_hasx = false;
              out_t = t_try;
              out_res = NAN;
              act = A_WRITE;
              break;
            }
#pragma unroll
            for (int v = 0; v < N; ++v) {
              xs[v * T] = xos[v * T];
              xos[v * T] = xe[v];
            }
            prev_step = hstep;
            have_prev = true;
            t = t_try;
            if (t >= 1.0) {
              act = A_FINISH;
              break;
            }
            if (c_its <= 2) step = fmin(step * 2.0, q.max_step);
            act = A_LOOP_TOP;
          } else {
            step = hstep * 0.5;
            if (step < q.min_step) {
              if (endgame) {
                act = A_FINISH;
              } else {
                out_status = NID_FAILED;
                out_hasx = false;
                out_t = t;
                out_res = NAN;
                act = A_WRITE;
              }
              break;
            }
            act = A_LOOP_TOP;
          }
          break;
        }
        case A_LOOP_TOP: {  // tracker.py:367-387
          if (used >= q.max_steps) {
            if (endgame) {
              act = A_FINISH;
            } else {
              out_status = NID_FAILED;
              out_hasx = false;
              out_t = t;
              out_res = NAN;
              act = A_WRITE;
            }
            break;
          }
          const double rem = 1.0 - t;
          cd xo[N];
#pragma unroll
          for (int v = 0; v < N; ++v) xo[v] = xos[v * T];
          if (!endgame && t >= q.endgame_start) {
            endgame = true;
            entry_norm = norm_inf<N>(xo);
          }
          if (rem <= q.snap_remaining) {
            act = A_FINISH;
            break;
          }
          used += 1;
          double hs = fmin(fmin(step, q.max_step), rem);
          if (endgame) hs = fmin(hs, q.endgame_contraction * rem);
          double tt = t + hs;
          if (1.0 - tt < 1e-14) tt = 1.0;
          hstep = hs;
          t_try = tt;
          if (have_prev && prev_step > 0.0) {
            const cd ratio = cd{hs / prev_step, 0.0};
#pragma unroll
            for (int v = 0; v < N; ++v) xe[v] = xo[v] + (xo[v] - xs[v * T]) * ratio;
          } else {
#pragma unroll
            for (int v = 0; v < N; ++v) xe[v] = xo[v];
          }
          te = tt;
          mode = M_CORR;
          c_ctx = CTX_STEP;
          c_tol = q.corrector_tol;
          c_iters = q.max_corrector_iters;
          c_it = 0;
          c_phase = 0;
          need_scale = true;
          act = A_EVAL;
          break;
        }
        case A_FINISH: {  // tracker.py:315-317
          cd xo[N];
#pragma unroll
          for (int v = 0; v < N; ++v) xo[v] = xos[v * T];
          norm_now = all_finite<N>(xo) ? norm_inf<N>(xo) : INFINITY;
          move_cap = 0.05 * (1.0 + norm_now);
          t_from = t;
          mode = M_DN;
          dn_it = 0;
          dn_trial = -1;
#pragma unroll
          for (int v = 0; v < N; ++v) {
            xs[v * T] = xo[v];
            xe[v] = xo[v];
          }
          te = 1.0;
          need_scale = false;
          act = A_EVAL;
          break;
        }
        case A_DN_CONT:  // loop head of _damped_newton
          if (dn_it >= q.final_newton_iters || !isfinite(dn_res) || dn_res <= q.corrector_tol) act = A_DECIDE;
          else act = A_SOLVE;
          break;
        case A_DECIDE: {  // tracker.py:318-338
          cd xb[N];
#pragma unroll
          for (int v = 0; v < N; ++v) xb[v] = xs[v * T];
          const double res = dn_res;
          double moved = INFINITY;
          if (all_finite<N>(xb)) {
            moved = 0.0;
#pragma unroll
            for (int v = 0; v < N; ++v) moved = nanmax(moved, cabsd(xb[v] - xos[v * T]));
          }
          out_hasx = false;
          out_res = NAN;
          if (isfinite(res) && res <= CONVERGED_RESIDUAL && moved <= move_cap) {
            out_status = NID_CONVERGED;
            out_hasx = true;
            out_t = 1.0;
            out_res = res;
          } else if (norm_now > q.soft_infinity || (norm_now + 1e-6) / (entry_norm + 1e-6) >= 8.0) {
            out_status = NID_AT_INFINITY;
            out_t = t_from;
          } else if (isfinite(res) && res <= 1e-4 && moved <= move_cap) {
            out_status = NID_SINGULAR_ENDPOINT;
            out_hasx = true;
            out_t = t_from;
            out_res = res;
          } else {
            out_status = NID_FAILED;
            out_t = t_from;
          }
          act = A_WRITE;
          break;
        }
        case A_WRITE: {
          A.status[path] = (int8_t)out_status;
          A.steps[path] = used;
          A.t_reached[path] = out_t;
          A.resid[path] = out_res;
#pragma unroll
          for (int v = 0; v < N; ++v) A.x_end[path * N + v] = out_hasx ? xs[v * T] : cd{NAN, NAN};
          act = A_CLAIM;
          break;
        }
        default:
          act = A_IDLE;
          break;
      }
    }

    // ------------------------------------------------------------ evaluation round
    const bool want_eval = act == A_EVAL;
    if (!__any_sync(0xffffffffu, act != A_IDLE)) break;
    if (want_eval) {
      double sc = 0.0;
      const double r = eval_tpp<N>(A.H, xe, te, prm, M, need_scale || fallback, sc);
      if (fallback) {
        // zgesv failed on this point: min-norm least squares (zgelsd) on the
        // re-evaluated Jacobian, copied out of the [element][thread] layout
        fallback = false;
        cd* sc2 = A.scratch + (size_t)(blockIdx.x * blockDim.x + threadIdx.x) * (3 * N * N + 2 * N);
        for (int i = 0; i < N; ++i) {
          for (int j = 0; j < N; ++j) sc2[i * N + j] = M.at(i, j, N + 1);
          sc2[N * N + i] = M.at(i, N, N + 1);
        }
        double sv[N];
        lstsq_minnorm(sc2, N, N, N, sc2 + N * N, sc2 + N * N + N, sv, sc2 + 2 * N * N + N);
        cd dx[N];
#pragma unroll
        for (int v = 0; v < N; ++v) dx[v] = sc2[2 * N * N + N + v];
        NID_APPLY_STEP(dx);
      } else {
        n_eval += 1;
        n_scale += need_scale ? 1 : 0;
        resid = r;
        scale = sc;
        act = A_ON_EVAL;
      }
    }
    // consume evaluations now so that the LU round below serves them
    if (act == A_ON_EVAL) {
      // (the same transitions as the control switch, for the common case)
      if (mode == M_CORR) {
        if (c_phase == 0) c_tol_eff = fmax(c_tol, NOISE_ULPS * scale);
        if (!(c_phase == 2 || (c_phase == 0 && c_iters == 0)) && isfinite(resid) && !(resid <= c_tol_eff))
          act = A_SOLVE;
      } else if (dn_trial < 0 && dn_it < q.final_newton_iters && isfinite(resid) && resid > q.corrector_tol) {
        dn_res = resid;
        act = A_SOLVE;
      }
    }
    // ------------------------------------------------------------ LU round
    if (__any_sync(0xffffffffu, act == A_SOLVE)) {
      if (act == A_SOLVE) {
        n_jac += 1;
        cd dx[N];
        if (lu_tpp<N>(M, dx)) {
          NID_APPLY_STEP(dx);
        } else {
          n_fb += 1;
          fallback = true;
          act = A_EVAL;
        }
      }
    }
  }
  atomicAdd(A.counters + 0, n_eval);
  atomicAdd(A.counters + 1, n_jac);
  atomicAdd(A.counters + 2, n_scale);
  atomicAdd(A.counters + 3, n_fb);
}
