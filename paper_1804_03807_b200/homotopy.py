"""LinearHomotopy and TrackParams (the reference's plugin surface) and their
lowering to the C-ABI descriptor.

`LinearHomotopy(start, target, gamma)` mirrors tracker.py:57-106 and
`TrackParams` mirrors tracker.py:109-134 (same fields, defaults and
ValueError validation).  Lowering merges start and target rows into one
sorted term table with a start and a target coefficient per monomial
(SURVEY.md §8(b)); the table is uploaded once per homotopy and cached.
"""

from __future__ import annotations

import ctypes as C
import weakref
from dataclasses import dataclass, field, fields

import numpy as np

from . import _lib
from .polys import PolySystem


@dataclass(frozen=True)
class TrackParams:
    initial_step: float = 0.1
    min_step: float = 1e-8
    max_step: float = 0.2
    corrector_tol: float = 1e-10
    max_corrector_iters: int = 4
    max_steps: int = 2000
    infinity_threshold: float = 1e8
    endgame_start: float = 0.9
    endgame_contraction: float = 0.5
    snap_remaining: float = 2e-8
    final_newton_iters: int = 40
    soft_infinity: float = 1e4
    precision: str = "double"
    dd_refine_singular: int = 3

    def __post_init__(self):
        if not (self.min_step < self.initial_step <= self.max_step):
            raise ValueError("need min_step < initial_step <= max_step")
        for name in ("corrector_tol", "min_step", "infinity_threshold"):
            if getattr(self, name) <= 0:
                raise ValueError(f"{name} must be positive")
        if self.precision not in ("double", "double_double"):
            raise ValueError(f"unknown precision {self.precision!r}")

    def to_c(self) -> _lib.TrackParamsC:
        return _lib.TrackParamsC(
            self.initial_step, self.min_step, self.max_step, self.corrector_tol,
            int(self.max_corrector_iters), int(self.max_steps), self.infinity_threshold,
            self.endgame_start, self.endgame_contraction, self.snap_remaining,
            int(self.final_newton_iters), int(self.dd_refine_singular), self.soft_infinity,
            1 if self.precision == "double_double" else 0, 0)


def params_c(params) -> _lib.TrackParamsC:
    """The C-ABI struct of any TrackParams-shaped object: this package's
    TrackParams, or the reference's own `nidpipe.tracker.TrackParams`
    (tracker.py:109-134, same field names), re-validated here."""
    if not isinstance(params, TrackParams):
        params = TrackParams(**{f.name: getattr(params, f.name) for f in fields(TrackParams) if hasattr(params, f.name)})
    return params.to_c()


@dataclass(frozen=True)
class Lowered:
    n: int
    row_off: np.ndarray  # int32 [n+1]
    expo: np.ndarray  # uint8 [T, 16]
    cs: np.ndarray  # complex128 [T]
    ct: np.ndarray  # complex128 [T]
    pslot: np.ndarray | None  # int8 [T]
    nparam: int
    gamma: complex
    start_degrees: np.ndarray | None = None  # int32 [n] when the start is total degree
    texp: np.ndarray | None = None  # float64 [T]: per-cell polyhedral t-exponents (start_kind 2)

    @property
    def nterms(self) -> int:
        return int(self.cs.size)


def lower(start, target, gamma: complex = 1.0 + 0j, param_terms: dict | None = None) -> Lowered:
    """Merge rows of start and target into one term table.

    param_terms maps (row, exponent tuple) -> slot for target coefficients
    supplied per path (the term is added to the table if absent)."""
    n = start.nvars
    if target.nvars != n or len(start.polys) != len(target.polys):
        raise ValueError("start and target systems must have the same shape")
    if len(start.polys) != n:
        raise ValueError("the GPU tracker needs a square homotopy (rows == variables)")
    if n > _lib.MAX_VARS:
        raise ValueError(f"at most {_lib.MAX_VARS} variables are supported")
    param_terms = param_terms or {}
    tdeg = total_degree_degrees(start)
    offs = [0]
    ex, cs, ct, sl = [], [], [], []
    prow = {r for (r, _e) in param_terms}
    for i in range(n):
        sp, tp = start.polys[i], target.polys[i]
        if tdeg is None and sp is tp and i not in prow:
            # a row shared by both systems (every row of a system homotopy, all but
            # the last of a cascade homotopy): its terms are already merged and
            # sorted (make_poly), and both coefficients are the row's own
            for e, c in tp.terms:
                ex.append(e)
                cs.append(c)
                ct.append(c)
                sl.append(-1)
            offs.append(len(cs))
            continue
        acc: dict[tuple, list] = {}
        if tdeg is None:  # a total-degree start is evaluated in closed form instead
            for e, c in sp.terms:
                acc.setdefault(e if type(e) is tuple else tuple(int(v) for v in e), [0j, 0j])[0] += complex(c)
        for e, c in tp.terms:
            acc.setdefault(e if type(e) is tuple else tuple(int(v) for v in e), [0j, 0j])[1] += complex(c)
        for (r, e), _ in param_terms.items():
            if r == i:
                acc.setdefault(tuple(e), [0j, 0j])
        for e in sorted(acc):
            a, b = acc[e]
            ex.append(e)
            cs.append(a)
            ct.append(b)
            sl.append(param_terms.get((i, e), -1))
        offs.append(len(cs))
    T = len(cs)
    expo = np.zeros((T, _lib.MAX_VARS), dtype=np.uint8)
    if T:
        arr = np.array(ex, dtype=np.int64).reshape(T, n)
        if arr.max(initial=0) > 255:
            raise ValueError("exponents above 255 are not supported")
        expo[:, :n] = arr
    pslot = np.array(sl, dtype=np.int8) if param_terms else None
    nparam = (max(param_terms.values()) + 1) if param_terms else 0
    return Lowered(n, np.array(offs, dtype=np.int32), expo, np.array(cs, dtype=np.complex128),
                   np.array(ct, dtype=np.complex128), pslot, nparam, complex(gamma),
                   None if tdeg is None else np.array(tdeg, dtype=np.int32))


def total_degree_degrees(start) -> list[int] | None:
    """d_i when row i of `start` is exactly x_i^{d_i} - 1 for every i, else None."""
    n = start.nvars
    if len(start.polys) != n:
        return None
    degs = []
    for i, p in enumerate(start.polys):
        terms = dict((tuple(int(v) for v in e), complex(c)) for e, c in p.terms)
        if len(terms) != 2 or terms.get((0,) * n) != -1.0 + 0j:
            return None
        (e, c), = [(e, c) for e, c in terms.items() if any(e)]
        if c != 1.0 + 0j or sum(1 for v in e if v) != 1 or e[i] < 1:
            return None
        degs.append(int(e[i]))
    return degs


class DeviceHomotopy:
    """An uploaded term table (one NidHomotopy handle)."""

    def __init__(self, low: Lowered):
        L = _lib.lib()
        self.low = low
        self._keep = (low.row_off, low.expo, low.cs, low.ct, low.pslot, low.start_degrees, low.texp)
        kind = 2 if low.texp is not None else (0 if low.start_degrees is None else 1)
        d = _lib.HomotopyDescC(
            low.n, low.nterms, _lib.ptr(low.row_off), _lib.ptr(low.expo), _lib.ptr(low.cs), _lib.ptr(low.ct),
            _lib.ptr(low.pslot), low.nparam, low.gamma.real, low.gamma.imag,
            kind, _lib.ptr(low.start_degrees), _lib.ptr(low.texp))
        h = C.c_void_p()
        _lib.check(L.nid_homotopy_create(C.byref(d), C.byref(h)), L)
        self.handle = h
        self._fin = weakref.finalize(self, L.nid_homotopy_destroy, h)

    @property
    def n(self) -> int:
        return self.low.n



@dataclass(frozen=True)
class LinearHomotopy:
    """h(x, t) = (1 - t) * gamma * start(x) + t * target(x) (tracker.py:57-106)."""

    start: PolySystem
    target: PolySystem
    gamma: complex = 1.0 + 0j
    _cache: dict = field(default_factory=dict, repr=False, compare=False)

    def __post_init__(self):
        if self.start.nvars != self.target.nvars or len(self.start.polys) != len(self.target.polys):
            raise ValueError("start and target systems must have the same shape")

    @property
    def dim(self) -> int:
        return self.start.nvars

    def lowered(self) -> Lowered:
        low = self._cache.get("low")
        if low is None:
            low = lower(self.start, self.target, self.gamma)
            self._cache["low"] = low
        return low

    def device(self) -> DeviceHomotopy:
        dev = self._cache.get("dev")
        if dev is None:
            dev = DeviceHomotopy(self.lowered())
            self._cache["dev"] = dev
        return dev

    # Batched GPU evaluation (the reference evaluates one point at a time)
    def evaluate(self, X, T, params=None, param_div=1):
        """H, J and eval_scale at points X[P, n] and times T[P] on the GPU."""
        return eval_batch(self.device(), X, T, params, param_div)

    def eval(self, x, t):
        return self.evaluate(np.asarray(x)[None], np.array([t]))[0][0]

    def jac(self, x, t):
        return self.evaluate(np.asarray(x)[None], np.array([t]))[1][0]

    def eval_scale(self, x, t):
        return float(self.evaluate(np.asarray(x)[None], np.array([t]))[2][0])


def system_homotopy(f: PolySystem) -> LinearHomotopy:
    """A plain system as a homotopy evaluated at t = 1 (tracker.py:241-252,433)."""
    return LinearHomotopy(f, f, 1.0 + 0j)


def eval_batch(dev: DeviceHomotopy, X, T, params=None, param_div=1):
    L = _lib.lib()
    n = dev.n
    X = np.ascontiguousarray(X, dtype=np.complex128).reshape(-1, n)
    P = X.shape[0]
    T = np.ascontiguousarray(np.broadcast_to(np.asarray(T, dtype=np.float64), (P,)))
    H = np.empty((P, n), np.complex128)
    J = np.empty((P, n, n), np.complex128)
    S = np.empty(P, np.float64)
    prm = None if params is None else np.ascontiguousarray(params, dtype=np.complex128)
    _lib.check(L.nid_eval_batch(dev.handle, P, _lib.ptr(X), _lib.ptr(T), _lib.ptr(prm), int(param_div),
                                _lib.ptr(H), _lib.ptr(J), _lib.ptr(S)), L)
    return H, J, S
