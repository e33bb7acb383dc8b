// K3 + K4: the persistent path tracker.
//
// One group of n lanes tracks one path at a time (lane i owns row i of H and
// J and coordinate i of x).  Groups claim path indices from a global atomic
// counter -- the GPU form of the reference's claim-guarded work crew
// (parallel.py:37-109) -- and refill their slot the moment a path retires.
//
// Every loop iteration is one homotopy evaluation (H, J and, on request, the
// noise scale) at each group's current point, followed by one group LU solve
// if any group in the warp needs a Newton step.  What the evaluation is for
// is decided by a per-group state machine that replays, branch for branch,
//   track           tracker.py:341-407  (secant predictor, step control,
//                                        endgame, snap, infinity test)
//   _correct        tracker.py:184-207  (residual-judged Newton, noise floor)
//   _finish         tracker.py:305-338  (t=1 polish + endpoint verdict)
//   _damped_newton  tracker.py:210-238  (8 halvings, never accept increase)
// The endpoint Solution (condition number, regularity, double-double polish,
// tracker.py:255-302,319-331) is computed afterwards by the endpoint kernel
// for the paths that need one.
#pragma once
#include "homotopy.cuh"
#include "linalg.cuh"

struct TrackArgs {
  HomDev H;
  NidTrackParams prm;
  long long P;            // paths in this launch
  long long first_index;  // total-degree start index of path 0
  const cd* starts;       // [P][n] or null for total-degree starts
  int deg[NID_MAX_VARS];  // total-degree start degrees
  const cd* params;       // per-path target coefficients
  int param_div;
  unsigned long long* next;  // claim counter
  cd* x_end;
  int8_t* status;
  int* steps;
  double* t_reached;
  double* resid;
  unsigned long long* counters;  // evals, jacs, scales, lstsq fallbacks
  cd* scratch;                   // per-group lstsq scratch, 3*n*n + 2*n complex each
};

enum { M_IDLE = 0, M_CORR = 1, M_DN = 2 };
enum { CTX_PRE = 0, CTX_STEP = 1 };

template <int N>
struct PathState {
  long long path;
  int mode;
  // corrector
  int c_ctx, c_iters, c_it, c_phase;
  double c_tol, c_tol_eff;
  // damped newton
  int dn_it, dn_trial, dn_iters;
  double dn_lam, dn_res, dn_tol;
  // tracking
  double t, step, prev_step, hstep, t_try, entry_norm, norm_now, move_cap, t_from;
  int used;
  bool have_prev, endgame;
  // own coordinates
  cd xo, xpo, xbo, dxo;
  // evaluation point
  double te;
  bool need_scale;
  const cd* prm;
};

template <int N>
struct Tracker {
  const TrackArgs& A;
  const Grp<N>& g;
  PathState<N>& s;
  cd (&xe)[N];
  unsigned long long& n_eval;

  NID_D void write_result(int status, bool has_x, double t_reached, double res) {
    long long p = s.path;
    if (g.lg == 0) {
      A.status[p] = (int8_t)status;
      A.steps[p] = s.used;
      A.t_reached[p] = t_reached;
      A.resid[p] = res;
    }
    A.x_end[p * N + g.lg] = has_x ? s.xbo : cd{NAN, NAN};
  }

  NID_D void claim() {
    unsigned long long idx = 0;
    if (g.lg == 0) idx = atomicAdd(A.next, 1ull);
    idx = __shfl_sync(g.mask, idx, g.gbase);
    if ((long long)idx >= A.P) {
      s.mode = M_IDLE;
      s.path = -1;
      return;
    }
    s.path = (long long)idx;
    if (A.starts) {
#pragma unroll
      for (int v = 0; v < N; ++v) xe[v] = A.starts[s.path * N + v];
    } else {
      long long rem = A.first_index + s.path;
#pragma unroll
      for (int v = N - 1; v >= 0; --v) {
        int d = A.deg[v];
        long long k = rem % d;
        rem /= d;
        double ang = 3.141592653589793 * (2.0 * (double)k / (double)d);
        double sn, cs;
        sincos(ang, &sn, &cs);
        xe[v] = cd{cs, sn};
      }
    }
    s.xo = pick<N>(xe, g.lg);
    s.prm = A.params ? A.params + (s.path / A.param_div) * A.H.nparam : nullptr;
    s.te = 0.0;
    start_corrector(CTX_PRE, A.prm.corrector_tol * 10.0, 3);
  }

  NID_D void start_corrector(int ctx, double tol, int iters) {
    s.mode = M_CORR;
    s.c_ctx = ctx;
    s.c_tol = tol;
    s.c_iters = iters;
    s.c_it = 0;
    s.c_phase = 0;
    s.need_scale = true;
  }

  NID_D double group_max_abs_own(cd v) { return group_nanmax<N>(g, cabsd(v)); }

  // top of the `while steps_used < max_steps` loop (tracker.py:367-387)
  NID_D void loop_top() {
    const NidTrackParams& q = A.prm;
    if (s.used >= q.max_steps) {
      if (s.endgame) start_finish();
      else finish_path(NID_FAILED, false, s.t, NAN);
      return;
    }
    double rem = 1.0 - s.t;
    if (!s.endgame && s.t >= q.endgame_start) {
      s.endgame = true;
      s.entry_norm = group_max_abs_own(s.xo);
    }
    if (rem <= q.snap_remaining) {
      start_finish();
      return;
    }
    s.used += 1;
    double hs = fmin(fmin(s.step, q.max_step), rem);
    if (s.endgame) hs = fmin(hs, q.endgame_contraction * rem);
    double tt = s.t + hs;
    if (1.0 - tt < 1e-14) tt = 1.0;
    s.hstep = hs;
    s.t_try = tt;
    cd xp = s.xo;
    if (s.have_prev && s.prev_step > 0.0) xp = s.xo + (s.xo - s.xpo) * cd{hs / s.prev_step, 0.0};
    group_gather<N>(g, xp, xe);
    s.te = tt;
    start_corrector(CTX_STEP, q.corrector_tol, q.max_corrector_iters);
  }

  NID_D void corrector_done(bool ok, int its) {
    const NidTrackParams& q = A.prm;
    if (s.c_ctx == CTX_PRE) {
      if (!ok) {
        s.used = 0;
        finish_path(NID_FAILED, false, 0.0, NAN);
        return;
      }
      s.xo = pick<N>(xe, g.lg);
      s.t = 0.0;
      s.step = q.initial_step;
      s.have_prev = false;
      s.prev_step = 0.0;
      s.used = 0;
      s.entry_norm = group_max_abs_own(s.xo);
      s.endgame = false;
      loop_top();
      return;
    }
    if (ok) {
      cd xn = pick<N>(xe, g.lg);
      if (group_max_abs_own(xn) > q.infinity_threshold) {
        finish_path(NID_AT_INFINITY, false, s.t_try, NAN);
        return;
      }
      s.xpo = s.xo;
      s.prev_step = s.hstep;
      s.have_prev = true;
      s.xo = xn;
      s.t = s.t_try;
      if (s.t >= 1.0) {
        start_finish();
        return;
      }
      if (its <= 2) s.step = fmin(s.step * 2.0, q.max_step);
    } else {
      s.step = s.hstep * 0.5;
      if (s.step < q.min_step) {
        if (s.endgame) start_finish();
        else finish_path(NID_FAILED, false, s.t, NAN);
        return;
      }
    }
    loop_top();
  }

  // _finish, first half (tracker.py:315-317)
  NID_D void start_finish() {
    bool fin = group_all<N>(g, cfinite(s.xo));
    s.norm_now = fin ? group_max_abs_own(s.xo) : INFINITY;
    s.move_cap = 0.05 * (1.0 + s.norm_now);
    s.t_from = s.t;
    s.mode = M_DN;
    s.dn_it = 0;
    s.dn_trial = -1;
    s.dn_iters = A.prm.final_newton_iters;
    s.dn_tol = A.prm.corrector_tol;
    s.xbo = s.xo;
    group_gather<N>(g, s.xo, xe);
    s.te = 1.0;
    s.need_scale = false;
  }

  // _finish, verdict (tracker.py:318-338)
  NID_D void finish_decide() {
    const NidTrackParams& q = A.prm;
    double res = s.dn_res;
    bool fin = group_all<N>(g, cfinite(s.xbo));
    double moved = fin ? group_max_abs_own(s.xbo - s.xo) : INFINITY;
    if (isfinite(res) && res <= CONVERGED_RESIDUAL && moved <= s.move_cap) {
      finish_path(NID_CONVERGED, true, 1.0, res);
      return;
    }
    double growth = (s.norm_now + 1e-6) / (s.entry_norm + 1e-6);
    if (s.norm_now > q.soft_infinity || growth >= 8.0) {
      finish_path(NID_AT_INFINITY, false, s.t_from, NAN);
      return;
    }
    if (isfinite(res) && res <= 1e-4 && moved <= s.move_cap) {
      finish_path(NID_SINGULAR_ENDPOINT, true, s.t_from, res);
      return;
    }
    finish_path(NID_FAILED, false, s.t_from, NAN);
  }

  NID_D void finish_path(int status, bool has_x, double t_reached, double res) {
    write_result(status, has_x, t_reached, res);
    claim();
  }

  // damped Newton: loop head (tracker.py:219-223)
  NID_D bool dn_continue() {
    if (s.dn_it >= s.dn_iters || !isfinite(s.dn_res) || s.dn_res <= s.dn_tol) {
      finish_decide();
      return false;
    }
    return true;  // solve with the Jacobian at xbo (just evaluated)
  }

  NID_D void dn_trial_point() {
    cd xt = s.xbo + cd{s.dn_lam, 0.0} * s.dxo;
    group_gather<N>(g, xt, xe);
    s.te = 1.0;
  }

  // Consume an evaluation; returns true when a Newton solve is wanted.
  NID_D bool on_eval(double resid, double scale) {
    if (s.mode == M_CORR) {
      if (s.c_phase == 0) s.c_tol_eff = fmax(s.c_tol, NOISE_ULPS * scale);
      if (s.c_phase == 2 || (s.c_phase == 0 && s.c_iters == 0)) {
        double te2 = fmax(s.c_tol, NOISE_ULPS * scale);
        corrector_done(resid <= te2, s.c_iters);
        return false;
      }
      if (!isfinite(resid)) {
        corrector_done(false, s.c_it);
        return false;
      }
      if (resid <= s.c_tol_eff) {
        corrector_done(true, s.c_it);
        return false;
      }
      return true;
    }
    if (s.mode == M_DN) {
      if (s.dn_trial < 0) {
        s.dn_res = resid;
        return dn_continue();
      }
      if (isfinite(resid) && resid < s.dn_res) {  // accepted trial: new base
        s.xbo = s.xbo + cd{s.dn_lam, 0.0} * s.dxo;
        s.dn_res = resid;
        s.dn_it += 1;
        s.dn_trial = -1;
        return dn_continue();
      }
      s.dn_lam *= 0.5;
      s.dn_trial += 1;
      if (s.dn_trial < 8) {
        dn_trial_point();
        return false;
      }
      s.dn_it += 1;  // not improved: break (tracker.py:235-237)
      finish_decide();
      return false;
    }
    return false;
  }

  // Consume the Newton step dx (full vector in every lane, mine = dx[lg]).
  NID_D void on_solve(const cd (&dx)[N], cd mine) {
    if (s.mode == M_CORR) {
      bool fin = true;
#pragma unroll
      for (int v = 0; v < N; ++v) {
        xe[v] = xe[v] + dx[v];
        fin = fin && cfinite(xe[v]);
      }
      if (!fin) {
        corrector_done(false, s.c_it + 1);
        return;
      }
      s.c_it += 1;
      s.c_phase = (s.c_it >= s.c_iters) ? 2 : 1;
      s.need_scale = (s.c_phase == 2);
      return;
    }
    if (s.mode == M_DN) {
      s.dxo = mine;
      s.dn_lam = 1.0;
      s.dn_trial = 0;
      dn_trial_point();
    }
  }
};

template <int N>
__global__ void __launch_bounds__(128) track_kernel(TrackArgs A) {
  const Grp<N> g = Grp<N>::make();
  PathState<N> s;
  cd xe[N];
  unsigned long long n_eval = 0, n_jac = 0, n_scale = 0, n_fb = 0;
#pragma unroll
  for (int v = 0; v < N; ++v) xe[v] = cd{0.0, 0.0};
  s.mode = M_IDLE;
  s.path = -1;
  s.need_scale = false;
  s.te = 0.0;
  s.prm = nullptr;
  Tracker<N> tr{A, g, s, xe, n_eval};
  if (g.real) tr.claim();
  const int gslot = (blockIdx.x * blockDim.x + threadIdx.x) / 32 * (32 / N) + g.gid;

  while (true) {
    const bool act = s.mode != M_IDLE;
    if (!__any_sync(0xffffffffu, act)) break;
    const bool ws = __any_sync(0xffffffffu, act && s.need_scale);
    cd hv;
    cd J[N];
    double sS, sT;
    eval_row<N>(A.H, act ? g.lg : N, xe, s.te, s.prm, hv, J, sS, sT, ws);
    const double resid = group_nanmax<N>(g, cabsd(hv));
    double scale = 0.0;
    if (ws) {
      double mS = group_reduce<N>(g, sS, OpMax());
      double mT = group_reduce<N>(g, sT, OpMax());
      scale = (1.0 - s.te) * mS + s.te * mT;
    }
    bool want = false;
    if (act) {
      n_eval += 1;
      n_scale += s.need_scale ? 1 : 0;
      want = tr.on_eval(resid, scale);
    }
    if (__any_sync(0xffffffffu, want)) {
      cd dx[N];
      cd mine;
      cd rhs = -hv;
      bool ok = group_lu_solve<N>(g, J, rhs, dx, mine);
      if (want) {
        n_jac += 1;
        if (!ok) {
          // zgesv failed: min-norm least squares on the re-evaluated Jacobian
          n_fb += 1;
          cd* sc = A.scratch + (size_t)gslot * (3 * N * N + 2 * N);
          cd hv2;
          eval_row<N>(A.H, g.lg, xe, s.te, s.prm, hv2, J, sS, sT, false);
#pragma unroll
          for (int v = 0; v < N; ++v) sc[g.lg * N + v] = J[v];
          sc[N * N + g.lg] = -hv2;
          __syncwarp(g.mask);
          if (g.lg == 0) {
            double sv[N];
            lstsq_minnorm(sc, N, N, N, sc + N * N, sc + N * N + N, sv, sc + 2 * N * N + N);
          }
          __syncwarp(g.mask);
#pragma unroll
          for (int v = 0; v < N; ++v) dx[v] = sc[2 * N * N + N + v];
          mine = pick<N>(dx, g.lg);
          __syncwarp(g.mask);
        }
        tr.on_solve(dx, mine);
      }
    }
  }
  if (g.real && g.lg == 0) {
    atomicAdd(A.counters + 0, n_eval);
    atomicAdd(A.counters + 1, n_jac);
    atomicAdd(A.counters + 2, n_scale);
    atomicAdd(A.counters + 3, n_fb);
  }
}
