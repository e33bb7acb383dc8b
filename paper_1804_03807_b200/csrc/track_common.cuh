// Shared definitions of the persistent path tracker (csrc/track_ctl.cuh):
// launch arguments and the control actions of its state machine.
#pragma once
#include "homotopy.cuh"
#include "linalg.cuh"

constexpr int NID_MAX_RUNS = 256;

struct TrackArgs {
  HomDev H;
  NidTrackParams prm;
  long long P;            // paths in this launch
  long long first_index;  // total-degree start index of path 0
  long long index_stride; // start index of path i: first_index + i * index_stride
  const cd* starts;       // [P][n] or null for total-degree starts
  int deg[NID_MAX_VARS];  // total-degree start degrees
  int root_off[NID_MAX_VARS];  // offsets of each variable's roots of unity in `roots`
  const cd* roots;             // exp(2 pi i k / d_v), k < d_v
  const cd* params;       // per-path target coefficients
  int param_div;
  const double* ptw;      // per-path polyhedral t-exponent rows [P][nterms] (cells batched) or null
  unsigned long long* next;  // claim counter
  cd* x_end;
  int8_t* status;
  int* steps;
  double* t_reached;
  double* resid;
  unsigned long long* counters;  // evals, jacs, scales, lstsq fallbacks
  cd* scratch;                   // per-group lstsq scratch, 3*n*n + 2*n complex each
  cd* gstate;                    // per-slot accepted/previous point, DN direction [block][3n][32]
  int lat_slots;                 // per-slot evaluation when at most this many of a block's slots evaluate (track_rec.cuh)
  // per-step trace of accepted steps (auxiliary kernel only, track_aux.cuh):
  // (t, step, corrector iterations) rows [P][trace_cap][3], counts [P]; null: off
  double* trace;
  int* trace_n;
  int trace_cap;
  int static_claim;  // P <= blocks x 32: slot s of block b tracks path s * blocks + b (set by the launcher)
  // the streamed-record evaluator's run descriptors (HomDev::runs) in the launch's
  // parameter bank: loop bounds, factor counts and patterns are then uniform
  // constant-bank loads (a table with more runs is not streamed)
  uint4 runs_c[NID_MAX_RUNS];
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

