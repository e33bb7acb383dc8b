/*
 * nid.h -- C-ABI of the B200 batched homotopy path tracker (libnid.so).
 *
 * Plain C types only: caller-owned host buffers or device pointers, sizes,
 * int status returns (0 = ok, nonzero = error; message in nid_last_error()).
 * No exceptions cross the ABI.  Complex numbers are interleaved (re, im)
 * float64 pairs.  One process per GPU; handles are per device and
 * thread-compatible, not thread-safe.
 *
 * Each entry point replaces one reference interface of the pure-Python
 * package `nidpipe` (/root/reference/pkg/src/nidpipe):
 *
 *   nid_homotopy_create   LinearHomotopy(start, target, gamma)       tracker.py:57-106
 *                         PolyhedralHomotopy(g, cell, supports)      polyhedral.py:730-791
 *   nid_eval_batch        LinearHomotopy.eval / .jac / .eval_scale    tracker.py:81-92
 *                         (+ _StackedEvaluator, polynomials.py:202-256,282-287)
 *   nid_newton_step_batch newton_step (zgesv, lstsq fallback)          linalg.py:35-51
 *   nid_svd_batch         condition_and_rank (singular values)         linalg.py:13-32
 *   nid_track_batch       work_crew(jobs, p, lambda x0: track(h, x0))  parallel.py:69-109,
 *                         track / _correct / _finish / _damped_newton  tracker.py:184-407
 *                         _endpoint_solution / _dd_polish              tracker.py:255-302
 *   nid_track_batch_strided  the same over a rank's strided share of the
 *                         start-path indices (one process per GPU)     parallel.py:69-109
 *   nid_track_trace       track(h, x0, params, trace=list)              tracker.py:341-407
 *   nid_track_cells       solve_start_system's per-cell solve_cell loop cascade.py:134-141,
 *                         (cells batched, one t-exponent row per path) polyhedral.py:794-811
 *   nid_refine_batch      newton_refine + classify                     tracker.py:410-455
 *   nid_dd_refine_batch   refine_dd                                    tracker.py:431-435
 *   nid_match_pairs       points_match over all pairs (for _dedup)     filtering.py:73-78,140-150
 *   nid_init_devices / nid_use_device / nid_compact_finite / nid_gather_endpoints
 *                         the work crew across GPUs: results re-united    parallel.py:91-106,131-134
 */
#ifndef NID_H
#define NID_H

#ifndef NID_NO_STD_HEADERS
#include <stddef.h>
#include <stdint.h>
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define NID_MAX_VARS 16

/* Path statuses (tracker.py:36-39) */
#define NID_CONVERGED 0
#define NID_AT_INFINITY 1
#define NID_SINGULAR_ENDPOINT 2
#define NID_FAILED 3

/* Slack classes (tracker.py:41-43, classify :438-455) */
#define NID_CLS_AT_INFINITY 1
#define NID_CLS_ZERO_SLACK 4
#define NID_CLS_NONZERO_SLACK 5

/* The TrackParams fields (tracker.py:113-127); precision: 0 double,
 * 1 double_double (every H / J evaluation in complex double-double rounded
 * to double, no evaluation-noise floor, every endpoint polished:
 * _DDView / _track_dd, tracker.py:458-497). */
typedef struct NidTrackParams {
  double initial_step, min_step, max_step, corrector_tol;
  int32_t max_corrector_iters, max_steps;
  double infinity_threshold, endgame_start, endgame_contraction, snap_remaining;
  int32_t final_newton_iters;
  int32_t dd_refine_singular;
  double soft_infinity;
  int32_t precision;
  int32_t _pad;
} NidTrackParams;

/*
 * A lowered LinearHomotopy H = (1-t) gamma G + t F.  Rows of G and F are
 * merged: each term carries its exponent vector (NID_MAX_VARS bytes,
 * variable v at byte v) and its start/target coefficients (0 where the
 * monomial is absent on that side).  Terms of row i are
 * [row_off[i], row_off[i+1]).  param_slot[k] >= 0 marks a target
 * coefficient supplied per path (membership targets): the value is
 * params[(path / param_div) * nparam + param_slot[k]].
 */
typedef struct NidHomotopyDesc {
  int32_t n;            /* variables == rows, 1..NID_MAX_VARS */
  int32_t nterms;
  const int32_t* row_off;   /* [n+1] */
  const uint8_t* expo;      /* [nterms * NID_MAX_VARS] */
  const double* coef_start; /* [nterms * 2] */
  const double* coef_target;/* [nterms * 2] */
  const int8_t* param_slot; /* [nterms] or NULL */
  int32_t nparam;
  double gamma_re, gamma_im;
  /* start_kind 1: the start system is total degree, G_i = x_i^{d_i} - 1 with
   * d_i = start_degrees[i]; it is evaluated in closed form and the term
   * table then carries only the target system (coef_start all zero). */
  int32_t start_kind;
  const int32_t* start_degrees;
  /* start_kind 2: a per-cell polyhedral homotopy (PolyhedralHomotopy,
   * polyhedral.py:730-791).  H(x, t) = sum_k c_k t^{term_texp[k]} x^{a_k}
   * with c_k = coef_target[k] (coef_start all zero, gamma unused); the
   * Jacobian terms carry the weight of the term they differentiate and the
   * noise scale is max_i sum_k |c_k| t^{w_k} |x|^{a_k}.  term_texp holds the
   * rescaled exponents (0 on the cell's pairs).  Tracked only through the
   * parameter-bank kernel (at most 256 terms); larger tables are refused. */
  const double* term_texp;  /* [nterms], start_kind 2 only */
} NidHomotopyDesc;

typedef struct NidHomotopy NidHomotopy;

/* Per-path results of nid_track_batch (all arrays length P, x_end P*n*2). */
typedef struct NidPathOut {
  double* x_end;        /* endpoint (polished) coordinates, NaN when none */
  int8_t* status;
  int32_t* steps;
  double* t_reached;
  double* residual;
  double* condition;
  int8_t* regular;      /* 1 regular, 0 singular, -1 no endpoint */
} NidPathOut;

/* Aggregate work counters of the last nid_track_batch call (the executed
 * counts of the reference's h.eval / h.jac / h.eval_scale calls). */
typedef struct NidCounters {
  long long evals, jacs, scales, paths, dd_polished, lstsq_fallbacks;
  double kernel_ms_track, kernel_ms_endpoint;
} NidCounters;

const char* nid_last_error(void);
int nid_device_count(int* count);
int nid_init(int device);
int nid_shutdown(void);

/* Several GPUs in one process (the one-process-per-GPU
 * launch uses nid_init and torch.distributed instead).  nid_init_devices
 * creates a context on every listed CUDA device and enables peer access
 * between them; nid_use_device(i) makes devs[i] the calling thread's current
 * device for the handles it creates next.  A handle remembers its device and
 * every call on it runs there, so a host thread per device can track its
 * shard (nid_track_batch_strided with first_index = i, index_stride = ndev)
 * concurrently. */
int nid_init_devices(int ndev, const int* devs);
int nid_use_device(int i);

int nid_homotopy_create(const NidHomotopyDesc* desc, NidHomotopy** out);
int nid_homotopy_destroy(NidHomotopy* h);

/* Host-only test hook (no device needed): lowers a term table into the
 * column-owner stream that nid_homotopy_create builds for tables streamed from
 * L2 (csrc/col_lower.h: the merged-monomial form of the reference's stacked
 * evaluator, polynomials.py:202-256) for `groups` warps.  Copies up to
 * cap_pieces 16-byte pieces (4 words each) and cap_runs run descriptors (4
 * words each) and returns the full counts; cgrun / cgbase [17]: each warp's
 * first run and first piece.  *eligible = 0 when the table does not take the
 * stream (then nothing else is written).  tests/test_col_lower.py decodes the
 * stream and checks it against the term table. */
int nid_col_lower(const NidHomotopyDesc* desc, int groups, unsigned* pieces, long long cap_pieces,
                  long long* n_pieces, unsigned* runs, long long cap_runs, long long* n_runs, int* cgrun,
                  int* cgbase, int* eligible);

/* Evaluate H, J and the noise scale at P points (host buffers):
 * x[P*n*2], t[P], params[P? per param_div] -> H[P*n*2], J[P*n*n*2] (row-major), scale[P]. */
int nid_eval_batch(NidHomotopy* h, int P, const double* x, const double* t, const double* params,
                   int param_div, double* H, double* J, double* scale);

/* Solve J dx = -r for P square systems of size n (host buffers). */
int nid_newton_step_batch(int n, int P, const double* J, const double* r, double* dx);

/* Singular values (descending) of P m x n matrices, m <= 32, n <= 16 (host buffers). */
int nid_svd_batch(int m, int n, int P, const double* A, double* sv);

/*
 * Track P paths.  starts: host x0[P*n*2], or NULL for the total-degree start
 * system of the homotopy, with start path indices [first_index, first_index+P)
 * (mixed radix over `degrees`, last variable fastest).  Results go to host
 * buffers in `out`.  `device_io` != 0 means every pointer (starts, params,
 * out arrays) is a device pointer and nothing is copied; the complex arrays
 * (starts, params, x_end) must then be 16-byte aligned.
 */
int nid_track_batch(NidHomotopy* h, const NidTrackParams* prm, int P, const double* starts,
                    long long first_index, const int32_t* degrees, const double* params,
                    int param_div, NidPathOut* out, int device_io, void* stream);

/* nid_track_batch with total-degree start path indices first_index + i * index_stride
 * (i < P): a rank's strided share of the path index space (multi-GPU sharding,
 * work_crew's job list split across processes, parallel.py:69-109).
 * nid_track_batch is the index_stride == 1 case. */
int nid_track_batch_strided(NidHomotopy* h, const NidTrackParams* prm, int P, const double* starts,
                            long long first_index, long long index_stride, const int32_t* degrees,
                            const double* params, int param_div, NidPathOut* out, int device_io,
                            void* stream);

/* track(h, x0, params, trace=list) (tracker.py:341-407): nid_track_batch on
 * host buffers that also records, per path, the (t, step, corrector
 * iterations) triple of every accepted step (tracker.py:393-394):
 * trace[(p * trace_cap + k) * 3 .. +3) for k < min(trace_n[p], trace_cap);
 * trace_n[p] is the path's accepted-step count (it may exceed trace_cap:
 * max_steps is always enough). */
int nid_track_trace(NidHomotopy* h, const NidTrackParams* prm, int P, const double* starts, const double* params,
                    int param_div, NidPathOut* out, int trace_cap, double* trace, int32_t* trace_n);

int nid_last_counters(NidCounters* c);

/* Many mixed cells of one polyhedral homotopy (start_kind 2) in one launch:
 * path p starts at starts[p] and uses the t-exponent row
 * path_texp[p * nterms .. (p+1) * nterms) instead of the handle's term_texp.
 * Replaces the per-cell loop of solve_start_system (cascade.py:134-141) over
 * solve_cell (polyhedral.py:794-811).  Outputs as nid_track_batch. */
int nid_track_cells(NidHomotopy* h, const NidTrackParams* prm, int P, const double* starts,
                    const double* path_texp, NidPathOut* out, int device_io, void* stream);

/* newton_refine(f, x, tol, iters) on P points, then classify (n_original,
 * infinity_threshold): x in/out [P*n*2], residual, condition, regular,
 * rank, slack class.  The homotopy is evaluated at t = 1 (target rows). */
int nid_refine_batch(NidHomotopy* h, int P, double* x, double tol, int iters, int n_original,
                     double infinity_threshold, double* residual, double* condition, int8_t* regular,
                     int32_t* rank, int8_t* slack_class);

/* refine_dd(f, x, steps): double-double polish at t = 1; x in/out.  ok[P] = 1 if
 * the polish produced a point (else x is left unchanged). */
int nid_dd_refine_batch(NidHomotopy* h, int P, double* x, int steps, int8_t* ok);

/* For points X[P*n*2] (any order): for every pair i<j, set bit (i,j) when
 * points_match(X[j][:ncmp], X[i][:ncmp]) (scale from X[i]).  Returns the
 * matching pairs as (i, j) int32 pairs in `pairs` (capacity max_pairs);
 * *npairs gets the total count (may exceed capacity). */
int nid_match_pairs(int n, int ncmp, int P, const double* X, int32_t* pairs, long long max_pairs,
                    long long* npairs);

/* The endpoint exchange of a stage (the reference has no
 * counterpart: its work crew returns results through one process's memory,
 * parallel.py:91-106).  nid_compact_finite: on the current device, the
 * succeeded (converged / singular_endpoint) endpoints of x_end[P*n*2] in path
 * order into x_out, with their global path indices first_index + i *
 * index_stride in index_out (or NULL); device pointers.
 * nid_gather_endpoints: the same for nparts shards living on the devices
 * part_device[p] (indices into nid_init_devices' list), each compacted on its
 * own GPU and copied peer to peer (NVLink) into x_out / index_out on the root
 * device, part after part; *total = endpoints gathered.  The shards' tracking
 * calls must have completed (both run their kernels on the default stream of
 * the part's device and synchronize before returning). */
int nid_compact_finite(int n, long long P, const double* x_end, const int8_t* status, long long first_index,
                       long long index_stride, double* x_out, long long* index_out, long long capacity,
                       long long* count, void* stream);
int nid_gather_endpoints(int nparts, const int* part_device, const double* const* x_end, const int8_t* const* status,
                         const long long* counts, const long long* first_index, const long long* index_stride, int n,
                         int root_device, double* x_out, long long* index_out, long long capacity, long long* total);

#ifdef __cplusplus
}
#endif
#endif
