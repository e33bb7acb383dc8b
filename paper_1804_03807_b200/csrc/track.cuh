// K3 + K4: the persistent path tracker.
//
// One group of n lanes tracks one path at a time (lane i owns row i of H and
// J and coordinate i of x).  Groups claim path indices from a global atomic
// counter -- the GPU form of the reference's claim-guarded work crew
// (parallel.py:37-109) -- and refill their slot the moment a path retires.
//
// The warp loop alternates two uniform compute rounds -- one homotopy
// evaluation (H, J and, on request, the noise scale) or one group LU solve
// -- with a single copy of a control state machine.  LU rounds take
// priority, so a group's Jacobian is never overwritten while it waits for
// its solve.  The state machine replays, branch for branch,
//   track           tracker.py:341-407  (secant predictor, step control,
//                                        endgame, snap, infinity test)
//   _correct        tracker.py:184-207  (residual-judged Newton, noise floor)
//   _finish         tracker.py:305-338  (t=1 polish + endpoint verdict)
//   _damped_newton  tracker.py:210-238  (8 halvings, never accept increase)
// Every transition exists once in the code (the kernel must fit the
// instruction cache); group-uniform control scalars live in shared memory,
// only per-lane coordinates and the row/Jacobian data stay in registers.
// The endpoint Solution (condition number, regularity, double-double
// polish, tracker.py:255-302,319-331) is computed afterwards by the endpoint
// kernel for the paths that need one.
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
  int root_off[NID_MAX_VARS];  // offsets of each variable's roots of unity in `roots`
  const cd* roots;             // exp(2 pi i k / d_v), k < d_v
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

// control actions
enum : int {
  A_IDLE = 0,
  A_EVAL,        // wait for an evaluation round at (xe, te)
  A_SOLVE,       // wait for an LU round on the last evaluation's J
  A_ON_EVAL,     // consume an evaluation
  A_ON_SOLVE,    // consume a Newton step
  A_CLAIM,       // take the next path
  A_GATHER,      // all-gather own_next into xe, then evaluate
  A_LOOP_TOP,    // top of track()'s while loop
  A_CORR_DONE,   // _correct returned (c_ok, c_its)
  A_FINISH,      // _finish: start the t=1 damped Newton
  A_DN_CONT,     // _damped_newton loop head
  A_DECIDE,      // _finish verdict
  A_WRITE        // write the path's record, then claim
};
enum : int { M_CORR = 1, M_DN = 2 };
enum : int { CTX_PRE = 0, CTX_STEP = 1 };

// group-uniform control state (one copy per group, in shared memory)
struct GroupState {
  long long path;
  const cd* prm;
  double te, c_tol, c_tol_eff, dn_lam, dn_res, t, step, prev_step, hstep, t_try, entry_norm, norm_now,
      move_cap, t_from, out_t, out_res, resid, scale;
  int mode, c_ctx, c_iters, c_it, c_phase, c_its, dn_it, dn_trial, dn_iters, used, out_status;
  bool c_ok, have_prev, endgame, need_scale, out_hasx, fallback;
};

template <int N>
__global__ void __launch_bounds__(128) track_kernel(TrackArgs A) {
  constexpr int GPW = 32 / N;  // groups per warp
  __shared__ GroupState gs_all[4 * GPW];
  const Grp<N> g = Grp<N>::make();
  const Grp<N> gw = g.warpwide();
  const int warp = threadIdx.x >> 5;
  GroupState& S = gs_all[warp * GPW + (g.real ? g.gid : 0)];
  const int gslot = (blockIdx.x * blockDim.x + threadIdx.x) / 32 * GPW + g.gid;
  const NidTrackParams& q = A.prm;

  // per-lane data
  cd xe[N];                   // the point being evaluated (full copy in every lane)
  cd J[N];                    // Jacobian row lg of the last evaluation
  cd hv = cd{0.0, 0.0};       // H_lg of the last evaluation
  cd mine = cd{0.0, 0.0};     // dx[lg]
  cd xo = cd{0.0, 0.0}, xpo = cd{0.0, 0.0}, xbo = cd{0.0, 0.0}, dxo = cd{0.0, 0.0}, own_next = cd{0.0, 0.0};
#pragma unroll
  for (int v = 0; v < N; ++v) {
    xe[v] = cd{0.0, 0.0};
    J[v] = cd{0.0, 0.0};
  }
  unsigned long long n_eval = 0, n_jac = 0, n_scale = 0, n_fb = 0;
  int act = g.real ? A_CLAIM : A_IDLE;

  while (true) {
    // ------------------------------------------------------------ control
    while (act > A_SOLVE) {
      switch (act) {
        case A_CLAIM: {
          unsigned long long idx = 0;
          if (g.lg == 0) idx = atomicAdd(A.next, 1ull);
          idx = __shfl_sync(g.mask, idx, g.gbase);
          if ((long long)idx >= A.P) {
            act = A_IDLE;
            break;
          }
          const long long p = (long long)idx;
          S.path = p;
          if (A.starts) {
#pragma unroll
            for (int v = 0; v < N; ++v) xe[v] = A.starts[p * N + v];
          } else {
            long long rem = A.first_index + p;
#pragma unroll
            for (int v = N - 1; v >= 0; --v) {
              const int d = A.deg[v];
              const long long k = rem % d;
              rem /= d;
              xe[v] = A.roots[A.root_off[v] + (int)k];
            }
          }
          xo = pick<N>(xe, g.lg);
          S.prm = A.params ? A.params + (p / A.param_div) * A.H.nparam : nullptr;
          S.te = 0.0;
          S.used = 0;
          S.fallback = false;
          // _correct(h, x0, 0, tol*10, 3) precondition (tracker.py:356)
          S.mode = M_CORR;
          S.c_ctx = CTX_PRE;
          S.c_tol = q.corrector_tol * 10.0;
          S.c_iters = 3;
          S.c_it = 0;
          S.c_phase = 0;
          S.need_scale = true;
          act = A_EVAL;
          break;
        }
        case A_GATHER:
          group_gather<N>(g, own_next, xe);
          act = A_EVAL;
          break;
        case A_ON_EVAL: {
          const double resid = S.resid;
          if (S.mode == M_CORR) {  // _correct loop body (tracker.py:191-207)
            if (S.c_phase == 0) S.c_tol_eff = fmax(S.c_tol, NOISE_ULPS * S.scale);
            if (S.c_phase == 2 || (S.c_phase == 0 && S.c_iters == 0)) {
              S.c_ok = resid <= fmax(S.c_tol, NOISE_ULPS * S.scale);
              S.c_its = S.c_iters;
              act = A_CORR_DONE;
            } else if (!isfinite(resid)) {
              S.c_ok = false;
              S.c_its = S.c_it;
              act = A_CORR_DONE;
            } else if (resid <= S.c_tol_eff) {
              S.c_ok = true;
              S.c_its = S.c_it;
              act = A_CORR_DONE;
            } else {
              act = A_SOLVE;
            }
          } else {  // _damped_newton (tracker.py:216-238)
            if (S.dn_trial < 0) {
              S.dn_res = resid;
              act = A_DN_CONT;
            } else if (isfinite(resid) && resid < S.dn_res) {
              xbo = xbo + cd{S.dn_lam, 0.0} * dxo;
              S.dn_res = resid;
              S.dn_it += 1;
              S.dn_trial = -1;
              act = A_DN_CONT;
            } else {
              S.dn_lam *= 0.5;
              S.dn_trial += 1;
              if (S.dn_trial < 8) {
                own_next = xbo + cd{S.dn_lam, 0.0} * dxo;
                act = A_GATHER;
              } else {
                S.dn_it += 1;  // not improved: break
                act = A_DECIDE;
              }
            }
          }
          break;
        }
        case A_ON_SOLVE: {
          if (S.mode == M_CORR) {
            bool fin = true;
#pragma unroll
            for (int v = 0; v < N; ++v) {
              xe[v] = xe[v] + J[v];  // J holds dx after an LU round
              fin = fin && cfinite(xe[v]);
            }
            if (!fin) {
              S.c_ok = false;
              S.c_its = S.c_it + 1;
              act = A_CORR_DONE;
            } else {
              S.c_it += 1;
              S.c_phase = (S.c_it >= S.c_iters) ? 2 : 1;
              S.need_scale = (S.c_phase == 2);
              act = A_EVAL;
            }
          } else {
            dxo = mine;
            S.dn_lam = 1.0;
            S.dn_trial = 0;
            own_next = xbo + dxo;
            act = A_GATHER;
          }
          break;
        }
        case A_CORR_DONE: {
          if (S.c_ctx == CTX_PRE) {
            if (!S.c_ok) {
              S.out_status = NID_FAILED;
              S.out_hasx = false;
              S.out_t = 0.0;
              S.out_res = NAN;
              act = A_WRITE;
              break;
            }
            xo = pick<N>(xe, g.lg);
            S.t = 0.0;
            S.step = q.initial_step;
            S.have_prev = false;
            S.prev_step = 0.0;
            S.used = 0;
            S.entry_norm = group_nanmax<N>(g, cabsd(xo));
            S.endgame = false;
            act = A_LOOP_TOP;
            break;
          }
          if (S.c_ok) {
            const cd xn = pick<N>(xe, g.lg);
            if (group_nanmax<N>(g, cabsd(xn)) > q.infinity_threshold) {
              S.out_status = NID_AT_INFINITY;
              S.out_hasx = false;
              S.out_t = S.t_try;
              S.out_res = NAN;
              act = A_WRITE;
              break;
            }
            xpo = xo;
            S.prev_step = S.hstep;
            S.have_prev = true;
            xo = xn;
            S.t = S.t_try;
            if (S.t >= 1.0) {
              act = A_FINISH;
              break;
            }
            if (S.c_its <= 2) S.step = fmin(S.step * 2.0, q.max_step);
            act = A_LOOP_TOP;
          } else {
            S.step = S.hstep * 0.5;
            if (S.step < q.min_step) {
              if (S.endgame) {
                act = A_FINISH;
              } else {
                S.out_status = NID_FAILED;
                S.out_hasx = false;
                S.out_t = S.t;
                S.out_res = NAN;
                act = A_WRITE;
              }
              break;
            }
            act = A_LOOP_TOP;
          }
          break;
        }
        case A_LOOP_TOP: {  // tracker.py:367-387
          if (S.used >= q.max_steps) {
            if (S.endgame) {
              act = A_FINISH;
            } else {
              S.out_status = NID_FAILED;
              S.out_hasx = false;
              S.out_t = S.t;
              S.out_res = NAN;
              act = A_WRITE;
            }
            break;
          }
          const double rem = 1.0 - S.t;
          if (!S.endgame && S.t >= q.endgame_start) {
            S.endgame = true;
            S.entry_norm = group_nanmax<N>(g, cabsd(xo));
          }
          if (rem <= q.snap_remaining) {
            act = A_FINISH;
            break;
          }
          S.used += 1;
          double hs = fmin(fmin(S.step, q.max_step), rem);
          if (S.endgame) hs = fmin(hs, q.endgame_contraction * rem);
          double tt = S.t + hs;
          if (1.0 - tt < 1e-14) tt = 1.0;
          S.hstep = hs;
          S.t_try = tt;
          own_next = (S.have_prev && S.prev_step > 0.0) ? xo + (xo - xpo) * cd{hs / S.prev_step, 0.0} : xo;
          S.te = tt;
          S.mode = M_CORR;
          S.c_ctx = CTX_STEP;
          S.c_tol = q.corrector_tol;
          S.c_iters = q.max_corrector_iters;
          S.c_it = 0;
          S.c_phase = 0;
          S.need_scale = true;
          act = A_GATHER;
          break;
        }
        case A_FINISH: {  // tracker.py:315-317
          const bool fin = group_all<N>(g, cfinite(xo));
          S.norm_now = fin ? group_nanmax<N>(g, cabsd(xo)) : INFINITY;
          S.move_cap = 0.05 * (1.0 + S.norm_now);
          S.t_from = S.t;
          S.mode = M_DN;
          S.dn_it = 0;
          S.dn_trial = -1;
          S.dn_iters = q.final_newton_iters;
          xbo = xo;
          own_next = xo;
          S.te = 1.0;
          S.need_scale = false;
          act = A_GATHER;
          break;
        }
        case A_DN_CONT:  // loop head of _damped_newton
          if (S.dn_it >= S.dn_iters || !isfinite(S.dn_res) || S.dn_res <= q.corrector_tol) act = A_DECIDE;
          else act = A_SOLVE;
          break;
        case A_DECIDE: {  // tracker.py:318-338
          const double res = S.dn_res;
          const bool fin = group_all<N>(g, cfinite(xbo));
          const double moved = fin ? group_nanmax<N>(g, cabsd(xbo - xo)) : INFINITY;
          S.out_hasx = false;
          S.out_res = NAN;
          if (isfinite(res) && res <= CONVERGED_RESIDUAL && moved <= S.move_cap) {
            S.out_status = NID_CONVERGED;
            S.out_hasx = true;
            S.out_t = 1.0;
            S.out_res = res;
          } else if (S.norm_now > q.soft_infinity ||
                     (S.norm_now + 1e-6) / (S.entry_norm + 1e-6) >= 8.0) {
            S.out_status = NID_AT_INFINITY;
            S.out_t = S.t_from;
          } else if (isfinite(res) && res <= 1e-4 && moved <= S.move_cap) {
            S.out_status = NID_SINGULAR_ENDPOINT;
            S.out_hasx = true;
            S.out_t = S.t_from;
            S.out_res = res;
          } else {
            S.out_status = NID_FAILED;
            S.out_t = S.t_from;
          }
          act = A_WRITE;
          break;
        }
        case A_WRITE: {
          const long long p = S.path;
          if (g.lg == 0) {
            A.status[p] = (int8_t)S.out_status;
            A.steps[p] = S.used;
            A.t_reached[p] = S.out_t;
            A.resid[p] = S.out_res;
          }
          A.x_end[p * N + g.lg] = S.out_hasx ? xbo : cd{NAN, NAN};
          act = A_CLAIM;
          break;
        }
        default:
          act = A_IDLE;
          break;
      }
    }

    // ------------------------------------------------------------ compute rounds
    // reconverge the warp: every group's lanes run the rounds together, with
    // warp-wide masks on the collectives
    __syncwarp();
    if (__any_sync(0xffffffffu, act == A_SOLVE)) {
      // LU round, in place: J becomes the Newton step dx (full copy per lane)
      const bool ok = group_lu_solve<N>(gw, J, -hv, mine);
      if (act == A_SOLVE) {
        n_jac += 1;
        if (!ok) {
          // zgesv failed: evaluate J again at the same point (the LU consumed
          // it) and take the min-norm least-squares step (zgelsd) instead
          n_fb += 1;
          S.fallback = true;
          act = A_EVAL;
          continue;
        }
        act = A_ON_SOLVE;
      }
      continue;
    }
    const bool want_eval = act == A_EVAL;
    if (!__any_sync(0xffffffffu, want_eval)) break;
    const bool ws = __any_sync(0xffffffffu, want_eval && S.need_scale);
    double sS, sT;
    const double te = want_eval ? S.te : 0.0;
    eval_row<N>(A.H, want_eval ? g.lg : N, xe, te, want_eval ? S.prm : nullptr, hv, J, sS, sT, ws);
    const double resid = group_nanmax<N>(gw, cabsd(hv));
    double scale = 0.0;
    if (ws) {
      const double mS = group_reduce<N>(gw, sS, OpMax());
      const double mT = group_reduce<N>(gw, sT, OpMax());
      scale = (1.0 - te) * mS + te * mT;
    }
    if (want_eval && S.fallback) {
      S.fallback = false;
      cd* sc = A.scratch + (size_t)gslot * (3 * N * N + 2 * N);
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
      for (int v = 0; v < N; ++v) J[v] = sc[2 * N * N + N + v];
      mine = pick<N>(J, g.lg);
      __syncwarp(g.mask);
      act = A_ON_SOLVE;
    } else if (want_eval) {
      n_eval += 1;
      n_scale += S.need_scale ? 1 : 0;
      S.resid = resid;
      S.scale = scale;
      act = A_ON_EVAL;
    }
  }
  if (g.real && g.lg == 0) {
    atomicAdd(A.counters + 0, n_eval);
    atomicAdd(A.counters + 1, n_jac);
    atomicAdd(A.counters + 2, n_scale);
    atomicAdd(A.counters + 3, n_fb);
  }
}
