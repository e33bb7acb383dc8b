"""Path tracking on the GPU behind the reference's tracker API.

Mirrors `nidpipe.tracker` (pkg/src/nidpipe/tracker.py): the status and
slack constants (:33-46), `Solution` (:137-154), `PathResult` (:157-166),
`track` (:341-407), `newton_refine` (:410-428), `refine_dd` (:431-435),
`classify` (:438-455), plus `newton_step` / `condition_and_rank`
(linalg.py:13-51).  Every numeric call goes through libnid.so; there is no
CPU path.  `track_batch` is the batched entry point the drivers use: it is
the GPU replacement of `work_crew(jobs, p, lambda x0: track(h, x0, params))`
(cascade.py:230,312, filtering.py:115).
"""

from __future__ import annotations

import ctypes as C
import weakref
from dataclasses import dataclass

import numpy as np

from . import _lib
from .homotopy import DeviceHomotopy, LinearHomotopy, TrackParams, lower, params_c, system_homotopy  # noqa: F401
from .polys import PolySystem

REGULAR = "regular"
SINGULAR = "singular"
CONVERGED = "converged"
AT_INFINITY = "at_infinity"
SINGULAR_ENDPOINT = "singular_endpoint"
FAILED = "failed"
ZERO_SLACK = "zero_slack"
NONZERO_SLACK = "nonzero_slack"
NOT_APPLICABLE = "not_applicable"
ZERO_SLACK_TOL = 1e-8
CONVERGED_RESIDUAL = 1e-8
SINGULARITY_TOL = 1e-8

STATUS_NAMES = (CONVERGED, AT_INFINITY, SINGULAR_ENDPOINT, FAILED)
STATUS_CODES = {s: i for i, s in enumerate(STATUS_NAMES)}
SLACK_NAMES = {_lib.CLS_AT_INFINITY: AT_INFINITY, _lib.CLS_ZERO: ZERO_SLACK, _lib.CLS_NONZERO: NONZERO_SLACK}


@dataclass(frozen=True)
class Solution:
    coordinates: np.ndarray
    residual: float
    condition: float
    regularity: str = REGULAR
    slack_class: str = NOT_APPLICABLE

    def __post_init__(self):
        object.__setattr__(self, "coordinates", np.asarray(self.coordinates, dtype=np.complex128))

    @property
    def is_regular(self) -> bool:
        return self.regularity == REGULAR


@dataclass(frozen=True)
class PathResult:
    status: str
    endpoint: Solution | None
    steps_used: int
    t_reached: float

    @property
    def succeeded(self) -> bool:
        return self.status in (CONVERGED, SINGULAR_ENDPOINT)


@dataclass
class TrackResults:
    """Struct-of-arrays results of one batched launch, in job order."""

    x: np.ndarray  # [P, n] endpoint coordinates (NaN where none)
    status: np.ndarray  # int8 codes (STATUS_NAMES)
    steps: np.ndarray
    t_reached: np.ndarray
    residual: np.ndarray
    condition: np.ndarray
    regular: np.ndarray  # 1 regular, 0 singular, -1 none
    counters: dict
    traces: list | None = None  # per path [(t, step, corrector iterations), ...] when requested

    def __len__(self):
        return int(self.status.size)

    @property
    def succeeded(self) -> np.ndarray:
        return (self.status == 0) | (self.status == 2)

    def counts(self) -> dict:
        return {name: int(np.sum(self.status == i)) for i, name in enumerate(STATUS_NAMES)}

    def result(self, i: int) -> PathResult:
        st = STATUS_NAMES[int(self.status[i])]
        ep = None
        if st in (CONVERGED, SINGULAR_ENDPOINT):
            ep = Solution(self.x[i].copy(), float(self.residual[i]), float(self.condition[i]),
                          REGULAR if self.regular[i] == 1 else SINGULAR)
        return PathResult(st, ep, int(self.steps[i]), float(self.t_reached[i]))

    def path_results(self) -> list[PathResult]:
        return [self.result(i) for i in range(len(self))]


def _device_of(h) -> DeviceHomotopy:
    if isinstance(h, DeviceHomotopy):
        return h
    if isinstance(h, LinearHomotopy) or (hasattr(h, "lowered") and hasattr(h, "device")):  # + PolyhedralHomotopy
        return h.device()
    if all(hasattr(h, a) for a in ("start", "target", "gamma")):
        # a reference nidpipe.tracker.LinearHomotopy (duck-typed: only
        # .start/.target/.gamma and .polys[i].terms are read)
        # cached per object without keeping it alive: the entry (and with it
        # the uploaded device table) goes when the reference object does
        key = id(h)
        cache = _FOREIGN.get(key)
        if cache is None or cache[0]() is not h:
            cache = (weakref.ref(h), LinearHomotopy(h.start, h.target, complex(h.gamma)))
            _FOREIGN[key] = cache
            weakref.finalize(h, _FOREIGN.pop, key, None)
        return cache[1].device()
    raise TypeError("expected a LinearHomotopy or PolyhedralHomotopy (the GPU path tracks lowered homotopies)")


_FOREIGN: dict = {}


_TRACK_FIELDS = ("t_reached", "residual", "condition", "status", "steps", "regular")
_SUM_COUNTERS = ("evals", "jacs", "scales", "paths", "dd_polished", "lstsq_fallbacks")


def track_batch(h, starts=None, params: TrackParams = TrackParams(), *, degrees=None, first_index: int = 0,
                count: int | None = None, index_stride: int = 1, target_params=None, param_div: int = 1,
                out: TrackResults | None = None, trace: bool = False) -> TrackResults:
    """`_track_local` on one rank.  Under an active multi-rank context
    (`parallel.activate`) every rank tracks its strided share of the job
    groups (a group = param_div consecutive paths, e.g. one membership
    candidate's paths) and one all_gather returns the whole batch's records,
    in job order, on every rank: the GPU form of the reference's fan-outs
    cascade.py:229-230, :311-312 and filtering.py:114-115 across processes."""
    from . import parallel

    ctx = parallel.active()
    if ctx is None or out is not None or trace:
        return _track_local(h, starts, params, degrees=degrees, first_index=first_index, count=count,
                            index_stride=index_stride, target_params=target_params, param_div=param_div, out=out,
                            trace=trace)
    n = _dim_of(h)
    d = max(1, int(param_div))
    if starts is not None:
        st = np.ascontiguousarray(starts, dtype=np.complex128).reshape(-1, n)
        P = st.shape[0]
    else:
        if degrees is None or count is None:
            raise ValueError("give start points, or degrees and count for total-degree starts")
        if d != 1:
            raise ValueError("device-generated starts shard path by path (param_div must be 1)")
        st, P = None, int(count)
    if P % d:
        raise ValueError("path count must be a multiple of param_div")
    G = P // d
    mine = parallel.group_shard(G, ctx.rank, ctx.world)
    kw = dict(param_div=d)
    if st is not None:
        kw["starts"] = st.reshape(G, d, n)[mine].reshape(-1, n)
    else:
        kw.update(starts=None, degrees=degrees, count=len(mine), first_index=first_index + ctx.rank * index_stride,
                  index_stride=index_stride * ctx.world)
    if target_params is not None:
        tp = np.ascontiguousarray(target_params, dtype=np.complex128)
        kw["target_params"] = tp.reshape(G, -1)[mine]
    if len(mine):
        loc = _track_local(h, kw.pop("starts"), params, **kw)
    else:
        loc = TrackResults(np.empty((0, n), np.complex128), np.empty(0, np.int8), np.empty(0, np.int32), np.empty(0),
                           np.empty(0), np.empty(0), np.empty(0, np.int8), dict.fromkeys(_SUM_COUNTERS, 0))
    # one row per group: [x (2 n d) | the six scalar fields (d each)]
    rows = np.concatenate([loc.x.view(np.float64).reshape(len(mine), -1)] +
                          [np.asarray(getattr(loc, f), np.float64).reshape(len(mine), d) for f in _TRACK_FIELDS], axis=1)
    full = parallel.allgather_rows(ctx, rows, G)
    x = np.ascontiguousarray(full[:, : 2 * n * d]).view(np.complex128).reshape(P, n)
    cols = [full[:, 2 * n * d + i * d: 2 * n * d + (i + 1) * d].reshape(P) for i in range(len(_TRACK_FIELDS))]
    res = TrackResults(x, cols[3].astype(np.int8), cols[4].astype(np.int32), cols[0].copy(), cols[1].copy(),
                       cols[2].copy(), cols[5].astype(np.int8), {})
    sums = parallel.allreduce_sum(ctx, [loc.counters.get(k, 0) for k in _SUM_COUNTERS])
    res.counters = dict(zip(_SUM_COUNTERS, sums))
    res.counters["kernel_ms_track"] = ctx.max_over_ranks(loc.counters.get("kernel_ms_track", 0.0))
    res.counters["kernel_ms_endpoint"] = ctx.max_over_ranks(loc.counters.get("kernel_ms_endpoint", 0.0))
    res.counters["ranks"] = ctx.world
    return res


def _dim_of(h) -> int:
    if hasattr(h, "n"):
        return int(h.n)
    if hasattr(h, "dim"):
        return int(h.dim)
    return int(h.target.nvars)


def _track_local(h, starts=None, params: TrackParams = TrackParams(), *, degrees=None, first_index: int = 0,
                 count: int | None = None, index_stride: int = 1, target_params=None, param_div: int = 1,
                 out: TrackResults | None = None, trace: bool = False) -> TrackResults:
    """Track many paths of h in one launch.

    starts: [P, n] start points, or None with `degrees` for total-degree
    starts generated on the device for path indices first_index + i * index_stride,
    i < count.
    target_params: per-path target coefficients ([P/param_div, nparam]) for
    homotopies lowered with parameter slots (membership tests).
    trace: also record every path's accepted steps (explicit starts only;
    small batches); `out.traces[i]` is then the list of (t, step, corrector
    iterations) tuples the reference's trace hook receives (tracker.py:393-394).
    params.precision == "double_double" tracks with every evaluation in
    complex double-double (tracker.py:458-497)."""
    L = _lib.lib()
    dev = _device_of(h)
    n = dev.n
    if starts is not None:
        st = np.ascontiguousarray(starts, dtype=np.complex128).reshape(-1, n)
        P = st.shape[0]
        deg = None
    else:
        if degrees is None or count is None:
            raise ValueError("give start points, or degrees and count for total-degree starts")
        st = None
        P = int(count)
        deg = np.ascontiguousarray(degrees, dtype=np.int32)
    prm = None if target_params is None else np.ascontiguousarray(target_params, dtype=np.complex128)
    if out is None:  # (callers may pass preallocated, e.g. pinned, host arrays)
        out = TrackResults(np.empty((P, n), np.complex128), np.empty(P, np.int8), np.empty(P, np.int32),
                           np.empty(P, np.float64), np.empty(P, np.float64), np.empty(P, np.float64),
                           np.empty(P, np.int8), {})
    o = _lib.PathOutC(_lib.ptr(out.x), _lib.ptr(out.status), _lib.ptr(out.steps), _lib.ptr(out.t_reached),
                      _lib.ptr(out.residual), _lib.ptr(out.condition), _lib.ptr(out.regular))
    pc = params_c(params)
    if trace:
        if st is None:
            raise ValueError("step traces need explicit start points")
        cap = max(1, int(pc.max_steps))
        tr = np.zeros((P, cap, 3), np.float64)
        tn = np.zeros(P, np.int32)
        _lib.check(L.nid_track_trace(dev.handle, C.byref(pc), P, _lib.ptr(st), _lib.ptr(prm), int(param_div),
                                     C.byref(o), cap, _lib.ptr(tr), _lib.ptr(tn)), L)
        out.traces = [[(float(t), float(hs), int(it)) for t, hs, it in tr[i, :min(int(tn[i]), cap)]]
                      for i in range(P)]
    else:
        _lib.check(L.nid_track_batch_strided(dev.handle, C.byref(pc), P, _lib.ptr(st), int(first_index),
                                             int(index_stride), _lib.ptr(deg), _lib.ptr(prm), int(param_div),
                                             C.byref(o), 0, None), L)
    out.counters = _lib.last_counters()
    return out


def track(h, x0, params: TrackParams = TrackParams(), trace: list | None = None) -> PathResult:
    """Track one path (tracker.py:341-407) -- a batch of one on the GPU.  A
    trace list receives (t, step, corrector_iterations) per accepted step."""
    res = track_batch(h, np.asarray(x0, dtype=np.complex128)[None], params, trace=trace is not None)
    if trace is not None:
        trace.extend(res.traces[0])
    return res.result(0)


def newton_step(J, r):
    """Solve J dx = -r (zgesv; min-norm lstsq fallback) on the GPU (linalg.py:35-51)."""
    J = np.ascontiguousarray(J, dtype=np.complex128)
    r = np.ascontiguousarray(r, dtype=np.complex128)
    single = J.ndim == 2
    if single:
        J, r = J[None], r[None]
    P, n, m = J.shape
    if n != m:
        raise ValueError("newton_step on the GPU needs square Jacobians")
    dx = np.empty((P, n), np.complex128)
    L = _lib.lib()
    _lib.check(L.nid_newton_step_batch(n, P, _lib.ptr(J), _lib.ptr(r), _lib.ptr(dx)), L)
    return dx[0] if single else dx


def singular_values(A) -> np.ndarray:
    A = np.ascontiguousarray(A, dtype=np.complex128)
    single = A.ndim == 2
    if single:
        A = A[None]
    P, m, n = A.shape
    if m < n:
        A = np.ascontiguousarray(np.conj(np.swapaxes(A, 1, 2)))
        P, m, n = A.shape
    sv = np.empty((P, n), np.float64)
    L = _lib.lib()
    _lib.check(L.nid_svd_batch(m, n, P, _lib.ptr(A), _lib.ptr(sv)), L)
    return sv[0] if single else sv


def condition_and_rank(J, tol: float = SINGULARITY_TOL):
    """linalg.py:13-32, singular values from the GPU Jacobi SVD."""
    J = np.asarray(J, dtype=np.complex128)
    if J.size == 0:
        raise ValueError("empty matrix")
    if not np.all(np.isfinite(J.view(np.float64))):
        return float("inf"), 0
    s = singular_values(J)
    smax = float(s[0])
    if smax == 0.0:
        return float("inf"), 0
    rank = int(np.sum(s > tol * smax))
    smin = float(s[min(J.shape) - 1])
    return (float("inf") if smin == 0.0 else smax / smin), rank


@dataclass
class RefineResults:
    x: np.ndarray
    residual: np.ndarray
    condition: np.ndarray
    regular: np.ndarray
    rank: np.ndarray
    slack: np.ndarray  # slack class codes

    def solution(self, i, with_slack=False) -> Solution:
        return Solution(self.x[i].copy(), float(self.residual[i]), float(self.condition[i]),
                        REGULAR if self.regular[i] else SINGULAR,
                        SLACK_NAMES[int(self.slack[i])] if with_slack else NOT_APPLICABLE)


def refine_batch(f: PolySystem, X, tol: float = 1e-12, max_iters: int = 10, n_original: int | None = None,
                 infinity_threshold: float = 1e8, h: LinearHomotopy | None = None) -> RefineResults:
    """`_refine_local`; under an active multi-rank context the points are
    sharded like the paths of track_batch and gathered back in order."""
    from . import parallel

    ctx = parallel.active()
    if ctx is None:
        return _refine_local(f, X, tol, max_iters, n_original, infinity_threshold, h)
    n = f.nvars
    X = np.array(X, dtype=np.complex128).reshape(-1, n)
    P = X.shape[0]
    mine = parallel.group_shard(P, ctx.rank, ctx.world)
    loc = _refine_local(f, X[mine], tol, max_iters, n_original, infinity_threshold, h)
    rows = np.concatenate([loc.x.view(np.float64).reshape(len(mine), 2 * n)] +
                          [np.asarray(a, np.float64).reshape(len(mine), 1)
                           for a in (loc.residual, loc.condition, loc.regular, loc.rank, loc.slack)], axis=1)
    full = parallel.allgather_rows(ctx, rows, P)
    c = full[:, 2 * n:]
    return RefineResults(np.ascontiguousarray(full[:, : 2 * n]).view(np.complex128).reshape(P, n), c[:, 0].copy(),
                         c[:, 1].copy(), c[:, 2].astype(np.int8), c[:, 3].astype(np.int32), c[:, 4].astype(np.int8))


def _refine_local(f: PolySystem, X, tol: float = 1e-12, max_iters: int = 10, n_original: int | None = None,
                  infinity_threshold: float = 1e8, h: LinearHomotopy | None = None) -> RefineResults:
    """newton_refine + classify for many points in one launch."""
    h = h or system_homotopy(f)
    dev = h.device()
    n = dev.n
    X = np.array(X, dtype=np.complex128).reshape(-1, n)
    P = X.shape[0]
    res = RefineResults(X, np.empty(P), np.empty(P), np.empty(P, np.int8), np.empty(P, np.int32),
                        np.empty(P, np.int8))
    if P == 0:
        return res
    L = _lib.lib()
    _lib.check(L.nid_refine_batch(dev.handle, P, _lib.ptr(X), float(tol), int(max_iters),
                                  int(n if n_original is None else n_original), float(infinity_threshold),
                                  _lib.ptr(res.residual), _lib.ptr(res.condition), _lib.ptr(res.regular),
                                  _lib.ptr(res.rank), _lib.ptr(res.slack)), L)
    return res


def newton_refine(f: PolySystem, x, tol: float = 1e-12, max_iters: int = 10) -> Solution:
    """tracker.py:410-428"""
    return refine_batch(f, np.asarray(x, dtype=np.complex128)[None], tol, max_iters).solution(0)


def refine_dd_batch(f: PolySystem, X, steps: int = 3, h: LinearHomotopy | None = None):
    """refine_dd for many points; sharded under an active multi-rank context."""
    from . import parallel

    ctx = parallel.active()
    if ctx is None:
        return _refine_dd_local(f, X, steps, h)
    n = f.nvars
    X = np.array(X, dtype=np.complex128).reshape(-1, n)
    mine = parallel.group_shard(len(X), ctx.rank, ctx.world)
    lx, lok = _refine_dd_local(f, X[mine], steps, h)
    rows = np.concatenate([lx.view(np.float64).reshape(len(mine), 2 * n), lok.astype(np.float64).reshape(-1, 1)], axis=1)
    full = parallel.allgather_rows(ctx, rows, len(X))
    return (np.ascontiguousarray(full[:, : 2 * n]).view(np.complex128).reshape(len(X), n), full[:, 2 * n].astype(np.int8))


def _refine_dd_local(f: PolySystem, X, steps: int = 3, h: LinearHomotopy | None = None):
    h = h or system_homotopy(f)
    dev = h.device()
    X = np.array(X, dtype=np.complex128).reshape(-1, dev.n)
    ok = np.empty(X.shape[0], np.int8)
    if X.shape[0]:
        L = _lib.lib()
        _lib.check(L.nid_dd_refine_batch(dev.handle, X.shape[0], _lib.ptr(X), int(steps), _lib.ptr(ok)), L)
    return X, ok


def refine_dd(f: PolySystem, x, steps: int = 3) -> np.ndarray:
    """tracker.py:431-435"""
    return refine_dd_batch(f, np.asarray(x, dtype=np.complex128)[None], steps)[0][0]


def classify(coords, n_original: int, infinity_threshold: float = 1e8, zero_tol: float = ZERO_SLACK_TOL) -> str:
    """Three-way slack classification (tracker.py:438-455); pure bookkeeping."""
    c = np.asarray(coords, dtype=np.complex128)
    if not np.all(np.isfinite(c.view(np.float64))) or float(np.max(np.abs(c))) > infinity_threshold:
        return AT_INFINITY
    s = c[n_original:]
    if s.size == 0 or float(np.max(np.abs(s))) < zero_tol:
        return ZERO_SLACK
    return NONZERO_SLACK


def track_batch_device(h, params: TrackParams, P: int, out: dict, *, degrees=None, first_index: int = 0,
                       index_stride: int = 1, starts_ptr: int = 0, params_ptr: int = 0, param_div: int = 1,
                       stream: int = 0) -> dict:
    """Device-resident variant of `track_batch`: every buffer is a device
    pointer (e.g. torch CUDA tensors' data_ptr()), nothing is copied, and the
    kernels run on `stream`.  `out` maps x_end/status/steps/t_reached/
    residual/condition/regular to device pointers.  Total-degree starts are
    the path indices first_index + i * index_stride (a rank's strided shard)."""
    L = _lib.lib()
    dev = _device_of(h)
    deg = None if degrees is None else np.ascontiguousarray(degrees, dtype=np.int32)
    o = _lib.PathOutC(out["x_end"], out["status"], out["steps"], out["t_reached"], out["residual"],
                      out["condition"], out["regular"])
    pc = params_c(params)
    _lib.check(L.nid_track_batch_strided(dev.handle, C.byref(pc), int(P), C.c_void_p(starts_ptr or None),
                                         int(first_index), int(index_stride), _lib.ptr(deg),
                                         C.c_void_p(params_ptr or None), int(param_div), C.byref(o), 1,
                                         C.c_void_p(stream or None)), L)
    return _lib.last_counters()
