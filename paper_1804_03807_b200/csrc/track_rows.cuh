// K3 + K4: the persistent path tracker, row-split thread-per-path layout.
//
// A block serves 32 paths (lane l of every warp belongs to path slot l) with
// G warps: warp g evaluates and eliminates the rows i == g (mod G) of all 32
// paths.  Every warp therefore walks ONE row's term table for 32 different
// paths -- the evaluation loops are warp-uniform (coefficients and
// exponents are broadcast loads, absent variables are skipped by uniform
// branches, the point stays in registers) -- and each thread's serial chain
// is 1/G of a path's work.  Each path's augmented Jacobian [J | -H] lives in
// shared memory laid out [element][slot], so a warp's access is one
// conflict-free 512-byte transaction whatever each path's row permutation.
//
// Paths are claimed from a global atomic counter and slots refilled as
// paths retire -- the GPU form of the reference's claim-guarded work crew
// (parallel.py:37-109).  Per block loop iteration: claim, control (each of
// a path's G threads runs the same deterministic state machine on the same
// data), one evaluation phase, one LU phase; phases are separated by block
// barriers.  The state machine replays, branch for branch,
//   track           tracker.py:341-407  (secant predictor, step control,
//                                        endgame, snap, infinity test)
//   _correct        tracker.py:184-207  (residual-judged Newton, noise floor)
//   _finish         tracker.py:305-338  (t=1 polish + endpoint verdict)
//   _damped_newton  tracker.py:210-238  (8 halvings, never accept increase)
// newton_step (linalg.py:35-51) is an LU with LAPACK's partial pivoting
// (izamax on |Re|+|Im| in row-swap order, unfused updates) with the zgelsd
// min-norm fallback.
#pragma once
#include "homotopy.cuh"
#include "linalg.cuh"
#include "track.cuh"

namespace rows {

constexpr int SLOTS = 32;  // paths per block

template <int N>
constexpr int groups() {  // G: warps per block = threads per path
  return N <= 3 ? 1 : (N <= 6 ? 2 : (N <= 10 ? 4 : 8));
}

// shared-memory layout (complex units unless noted), each [item][slot]
template <int N>
struct Layout {
  static constexpr int G = groups<N>();
  static constexpr int AUG = N * (N + 1);     // augmented matrix
  static constexpr int XO = AUG;              // accepted point
  static constexpr int XS = XO + N;           // x_prev / damped-Newton base
  static constexpr int DS = XS + N;           // damped-Newton direction
  static constexpr int DXS = DS + N;          // Newton step exchange (fallback)
  static constexpr int CPLX = DXS + N;
  // doubles after the complex area: per-group partial maxima
  static constexpr int R2 = 0;                // G entries: max |H_i|^2
  static constexpr int SS = G;                // G entries: max start abs sums
  static constexpr int ST = 2 * G;            // G entries: max target abs sums
  static constexpr int PK = 3 * G;            // G entries: pivot key
  static constexpr int PP = 4 * G;            // G entries: pivot logical position (as double)
  static constexpr int DBL = 5 * G;
  static constexpr size_t bytes() { return (size_t)SLOTS * (CPLX * sizeof(cd) + DBL * sizeof(double) + 8); }
};

template <int N>
NID_D cd& A(cd* base, int i, int j) {  // augmented matrix element of this slot
  return base[(i * (N + 1) + j) * SLOTS];
}

NID_D cd upow(cd x, int a) {
  cd r = x;
#pragma unroll 1
  for (int e = 1; e < a; ++e) r = r * x;
  return r;
}

// one term c x^a of the merged table: value into hv, partials into Jr
template <int N>
NID_D void term(const HomDev& H, int k, const cd (&x)[N], double t, cd alpha, const cd* prm, bool ml, cd& hv,
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
      if (expo_at(w, v)) {  // warp-uniform
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

// rows g, g+G, ... of H and J at (x, t) into the slot's augmented matrix;
// partial max |H_i|^2 and abs-sum maxima into the slot's double area
template <int N>
NID_D void eval_rows(const HomDev& H, int g, const cd (&x)[N], double t, const cd* prm, cd* aug, double* dbl,
                     bool want_scale) {
  using L = Layout<N>;
  const cd alpha = (1.0 - t) * H.gamma;
  const bool ml = H.multilinear != 0;
  double r2 = 0.0, mS = 0.0, mT = 0.0;
#pragma unroll 1
  for (int i = g; i < N; i += L::G) {
    cd hv = cd{0.0, 0.0};
    cd Jr[N];
#pragma unroll
    for (int v = 0; v < N; ++v) Jr[v] = cd{0.0, 0.0};
    const int k0 = __ldg(H.row_off + i), k1 = __ldg(H.row_off + i + 1);
#pragma unroll 1
    for (int k = k0; k < k1; ++k) term<N>(H, k, x, t, alpha, prm, ml, hv, Jr);
    double sS = 0.0, sT = 0.0;
    if (want_scale) {
      double ax[N];
#pragma unroll
      for (int v = 0; v < N; ++v) ax[v] = cabsd(x[v]);
#pragma unroll 1
      for (int k = k0; k < k1; ++k) {
        const uint4 ew = __ldg(H.expo + k);
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
        if (!H.td) sS = __dadd_rn(sS, __dmul_rn(__ldg(H.acs + k), m));
        sT = __dadd_rn(sT, __dmul_rn(__ldg(H.act + k), m));
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
    for (int v = 0; v < N; ++v) A<N>(aug, i, v) = Jr[v];
    A<N>(aug, i, N) = -hv;
    r2 = nanmax(r2, cabs2(hv));
    mS = fmax(mS, sS);
    mT = fmax(mT, sT);
  }
  dbl[(L::R2 + g) * SLOTS] = r2;
  dbl[(L::SS + g) * SLOTS] = mS;
  dbl[(L::ST + g) * SLOTS] = mT;
}

// combine the G partial maxima (after a barrier): residual max|H_i| and scale
template <int N>
NID_D double combine_resid(const cd* aug, const double* dbl, double t, double& scale) {
  using L = Layout<N>;
  double r2 = 0.0, mS = 0.0, mT = 0.0;
#pragma unroll
  for (int g = 0; g < L::G; ++g) {
    r2 = nanmax(r2, dbl[(L::R2 + g) * SLOTS]);
    mS = fmax(mS, dbl[(L::SS + g) * SLOTS]);
    mT = fmax(mT, dbl[(L::ST + g) * SLOTS]);
  }
  scale = (1.0 - t) * mS + t * mT;
  if (r2 < 1e290) return sqrt(r2);  // NaN takes the exact path as well
  double resid = 0.0;
#pragma unroll 1
  for (int i = 0; i < N; ++i) resid = nanmax(resid, cabsd(A<N>(const_cast<cd*>(aug), i, N)));
  return resid;
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

}  // namespace rows

// consume a Newton step dx (tracker.py:200-205 / 223-233)
#define NID_ROWS_APPLY(dxv)                                    \
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
        if (g == 0) ds[v * S] = (dxv)[v];                      \
        xe[v] = xs[v * S] + (dxv)[v];                          \
      }                                                        \
      act = A_EVAL;                                            \
    }                                                          \
  } while (0)

template <int N>
__global__ void __launch_bounds__(rows::groups<N>() * 32, 2) track_rows_kernel(TrackArgs Ar) {
  using namespace rows;
  using L = Layout<N>;
  constexpr int G = L::G;
  constexpr int S = SLOTS;
  extern __shared__ __align__(16) unsigned char smem_rows[];
  const int lane = threadIdx.x & 31;
  const int g = threadIdx.x >> 5;  // row group
  cd* const cbase = reinterpret_cast<cd*>(smem_rows);
  double* const dbase = reinterpret_cast<double*>(cbase + (size_t)L::CPLX * S);
  long long* const claim_slot = reinterpret_cast<long long*>(dbase + (size_t)L::DBL * S);
  cd* const aug = cbase + lane;        // this slot's augmented matrix
  cd* const xos = cbase + L::XO * S + lane;
  cd* const xs = cbase + L::XS * S + lane;
  cd* const ds = cbase + L::DS * S + lane;
  cd* const dxs = cbase + L::DXS * S + lane;
  double* const dbl = dbase + lane;
  const NidTrackParams& q = Ar.prm;

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
    // ------------------------------------------------------------ claim phase
    if (g == 0 && act == A_CLAIM) claim_slot[lane] = (long long)atomicAdd(Ar.next, 1ull);
    __syncthreads();
    if (act == A_CLAIM) {
      const long long idx = claim_slot[lane];
      if (idx >= Ar.P) {
        act = A_IDLE;
      } else {
        path = idx;
        if (Ar.starts) {
#pragma unroll
          for (int v = 0; v < N; ++v) xe[v] = Ar.starts[path * N + v];
        } else {
          long long rem = Ar.first_index + path;
#pragma unroll
          for (int v = N - 1; v >= 0; --v) {
            const int d = Ar.deg[v];
            const long long k = rem % d;
            rem /= d;
            xe[v] = Ar.roots[Ar.root_off[v] + (int)k];
          }
        }
        prm = Ar.params ? Ar.params + (path / Ar.param_div) * Ar.H.nparam : nullptr;
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
      }
    }
    __syncthreads();  // claim slots are reused next iteration

    // ------------------------------------------------------------ control
    // The slot's vectors x (xos) and x_prev / damped-Newton base (xs) live in
    // shared memory; within a control phase they are read as committed at
    // its start and new values are staged in registers (pend_*), committed
    // by the slot's thread 0 after the phase barrier.
    cd pend_xo[N], pend_xs[N];
    bool has_xo = false, has_xs = false;
    while (act > A_SOLVE && act != A_CLAIM) {
      switch (act) {
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
              for (int v = 0; v < N; ++v) pend_xs[v] = xe[v];  // accepted trial is the new base
              has_xs = true;
              dn_res = resid;
              dn_it += 1;
              dn_trial = -1;
              act = A_DN_CONT;
            } else {
              dn_lam *= 0.5;
              dn_trial += 1;
              if (dn_trial < 8) {
#pragma unroll
                for (int v = 0; v < N; ++v) xe[v] = xs[v * S] + cd{dn_lam, 0.0} * ds[v * S];
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
            for (int v = 0; v < N; ++v) pend_xo[v] = xe[v];
            has_xo = true;
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
              pend_xs[v] = xos[v * S];  // x_prev <- x
              pend_xo[v] = xe[v];       // x <- x_new
            }
            has_xs = has_xo = true;
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
          if (!endgame && t >= q.endgame_start) {
            endgame = true;
            double m = 0.0;
#pragma unroll
            for (int v = 0; v < N; ++v) m = nanmax(m, cabsd(has_xo ? pend_xo[v] : xos[v * S]));
            entry_norm = m;
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
            for (int v = 0; v < N; ++v) {
              const cd xo = has_xo ? pend_xo[v] : xos[v * S];
              const cd xp = has_xs ? pend_xs[v] : xs[v * S];
              xe[v] = xo + (xo - xp) * ratio;
            }
          } else {
#pragma unroll
            for (int v = 0; v < N; ++v) xe[v] = has_xo ? pend_xo[v] : xos[v * S];
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
          bool fin = true;
          double m = 0.0;
#pragma unroll
          for (int v = 0; v < N; ++v) {
            const cd xo = has_xo ? pend_xo[v] : xos[v * S];
            fin = fin && cfinite(xo);
            m = nanmax(m, cabsd(xo));
            pend_xs[v] = xo;  // damped-Newton base x1 <- x
            xe[v] = xo;
          }
          has_xs = true;
          norm_now = fin ? m : INFINITY;
          move_cap = 0.05 * (1.0 + norm_now);
          t_from = t;
          mode = M_DN;
          dn_it = 0;
          dn_trial = -1;
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
          const double res = dn_res;
          bool finb = true;
          double moved = 0.0;
#pragma unroll
          for (int v = 0; v < N; ++v) {
            const cd xb = has_xs ? pend_xs[v] : xs[v * S];
            finb = finb && cfinite(xb);
            moved = nanmax(moved, cabsd(xb - xos[v * S]));
          }
          if (!finb) moved = INFINITY;
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
          if (g == 0) {
            Ar.status[path] = (int8_t)out_status;
            Ar.steps[path] = used;
            Ar.t_reached[path] = out_t;
            Ar.resid[path] = out_res;
#pragma unroll
            for (int v = 0; v < N; ++v)
              Ar.x_end[path * N + v] = out_hasx ? (has_xs ? pend_xs[v] : xs[v * S]) : cd{NAN, NAN};
          }
          act = A_CLAIM;
          break;
        }
        default:
          act = A_IDLE;
          break;
      }
    }

    // exit when every slot of the block is idle
    if (!__syncthreads_or(act != A_IDLE)) break;
    if (g == 0) {  // commit the staged vectors (everyone has read the old ones)
      if (has_xo) {
#pragma unroll
        for (int v = 0; v < N; ++v) xos[v * S] = pend_xo[v];
      }
      if (has_xs) {
#pragma unroll
        for (int v = 0; v < N; ++v) xs[v * S] = pend_xs[v];
      }
    }

    // ------------------------------------------------------------ evaluation phase
    const bool want_eval = act == A_EVAL;
    if (want_eval) eval_rows<N>(Ar.H, g, xe, te, prm, aug, dbl, need_scale || fallback);
    __syncthreads();
    if (want_eval) {
      double sc = 0.0;
      const double r = combine_resid<N>(aug, dbl, te, sc);
      if (fallback) {
        act = A_ON_SOLVE;  // resolved below by thread 0 of the slot
      } else {
        n_eval += (g == 0);
        n_scale += (g == 0 && need_scale);
        resid = r;
        scale = sc;
        act = A_ON_EVAL;
        // the common case of the state machine: the corrector wants a step
        if (mode == M_CORR) {
          if (c_phase == 0) c_tol_eff = fmax(c_tol, NOISE_ULPS * scale);
          if (!(c_phase == 2 || (c_phase == 0 && c_iters == 0)) && isfinite(resid) && !(resid <= c_tol_eff))
            act = A_SOLVE;
        } else if (dn_trial < 0 && dn_it < q.final_newton_iters && isfinite(resid) && resid > q.corrector_tol) {
          dn_res = resid;
          act = A_SOLVE;
        }
      }
    }
    // zgesv failed earlier for this slot: min-norm least squares (zgelsd) on
    // the re-evaluated augmented matrix, solved by the slot's thread 0
    if (__syncthreads_or(act == A_ON_SOLVE && fallback)) {
      if (act == A_ON_SOLVE && fallback && g == 0) {
        cd* sc2 = Ar.scratch + (size_t)(blockIdx.x * S + lane) * (3 * N * N + 2 * N);
        for (int i = 0; i < N; ++i) {
          for (int j = 0; j < N; ++j) sc2[i * N + j] = A<N>(aug, i, j);
          sc2[N * N + i] = A<N>(aug, i, N);
        }
        double sv[N];
        lstsq_minnorm(sc2, N, N, N, sc2 + N * N, sc2 + N * N + N, sv, sc2 + 2 * N * N + N);
        for (int v = 0; v < N; ++v) dxs[v * S] = sc2[2 * N * N + N + v];
      }
      __syncthreads();
      if (act == A_ON_SOLVE && fallback) {
        fallback = false;
        cd dx[N];
#pragma unroll
        for (int v = 0; v < N; ++v) dx[v] = dxs[v * S];
        NID_ROWS_APPLY(dx);
      }
      __syncthreads();
    }

    // ------------------------------------------------------------ LU phase
    if (__syncthreads_or(act == A_SOLVE)) {
      const bool solving = act == A_SOLVE;
      // implicit row permutation (identical in the slot's G threads)
      unsigned long long perm = 0, pinv = 0;
#pragma unroll
      for (int i = 0; i < N; ++i) {
        perm |= (unsigned long long)i << (4 * i);
        pinv |= (unsigned long long)i << (4 * i);
      }
      bool bad = false;
#pragma unroll 1
      for (int k = 0; k < N; ++k) {
        // local pivot candidates: my physical rows r (r % G == g) at logical positions >= k
        if (solving) {
          double best = -1.0;
          int bpos = N;
#pragma unroll
          for (int r = g; r < N; r += G) {
            const int pos = (pinv >> (4 * r)) & 15;
            if (pos >= k) {
              const double key = cabs1(A<N>(aug, r, k));
              if (key > best || (key == best && pos < bpos)) {
                best = key;
                bpos = pos;
              }
            }
          }
          dbl[(L::PK + g) * S] = best;
          dbl[(L::PP + g) * S] = (double)bpos;
        }
        __syncthreads();
        if (solving) {
          double best = -1.0;
          int pk = k;
#pragma unroll
          for (int gg = 0; gg < G; ++gg) {
            const double key = dbl[(L::PK + gg) * S];
            const int pos = (int)dbl[(L::PP + gg) * S];
            if (pos < N && (key > best || (key == best && pos < pk))) {
              best = key;
              pk = pos;
            }
          }
          if (!(best > 0.0)) bad = true;
          // swap logical rows k and pk
          const unsigned long long rk = (perm >> (4 * k)) & 15, rp = (perm >> (4 * pk)) & 15;
          perm &= ~((15ull << (4 * k)) | (15ull << (4 * pk)));
          perm |= (rp << (4 * k)) | (rk << (4 * pk));
          pinv &= ~((15ull << (4 * rk)) | (15ull << (4 * rp)));
          pinv |= ((unsigned long long)k << (4 * rp)) | ((unsigned long long)pk << (4 * rk));
          const int r0 = (int)rp;
          cd prow[N + 1];
#pragma unroll
          for (int j = 1; j <= N; ++j)
            if (j > k) prow[j] = A<N>(aug, r0, j);
          const cd inv = crecip_fast(A<N>(aug, r0, k));
#pragma unroll 1
          for (int r = g; r < N; r += G) {
            const int pos = (pinv >> (4 * r)) & 15;
            if (pos > k) {
              const cd l = cmul_nf(A<N>(aug, r, k), inv);
#pragma unroll
              for (int j = 1; j <= N; ++j) {
                if (j > k) {
                  cd& a = A<N>(aug, r, j);
                  a = csub_nf(a, cmul_nf(l, prow[j]));
                }
              }
            }
          }
        }
        __syncthreads();
        // the pivot's reciprocal replaces it (written after every thread read it)
        if (solving && g == ((perm >> (4 * k)) & 15) % G) {
          const int r0 = (perm >> (4 * k)) & 15;
          A<N>(aug, r0, k) = crecip_fast(A<N>(aug, r0, k));
        }
      }
      __syncthreads();
      if (solving) {
        n_jac += (g == 0);
        cd dx[N];
        bool fin = true;
#pragma unroll
        for (int k = N - 1; k >= 0; --k) {
          const int r = (perm >> (4 * k)) & 15;
          cd s = A<N>(aug, r, N);
#pragma unroll
          for (int j = k + 1; j < N; ++j) s = csub_nf(s, cmul_nf(A<N>(aug, r, j), dx[j]));
          dx[k] = cmul_nf(s, A<N>(aug, r, k));
          fin = fin && cfinite(dx[k]);
        }
        if (!bad && fin) {
          NID_ROWS_APPLY(dx);
        } else {
          n_fb += (g == 0);
          fallback = true;
          act = A_EVAL;
        }
      }
      __syncthreads();  // the augmented matrices are rewritten by the next evaluation
    }
  }
  if (g == 0) {
    atomicAdd(Ar.counters + 0, n_eval);
    atomicAdd(Ar.counters + 1, n_jac);
    atomicAdd(Ar.counters + 2, n_scale);
    atomicAdd(Ar.counters + 3, n_fb);
  }
}
