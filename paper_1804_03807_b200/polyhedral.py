"""Per-cell polyhedral tracking on the GPU.

Mirrors the reference's polyhedral start-system surface
(`nidpipe/polyhedral.py`):

  * `PolyhedralHomotopy(g, cell, supports)`  polyhedral.py:730-791 -- lowered
    to a term table whose coefficient k is c_k t^{w_k} (start_kind 2 of the
    C-ABI, `include/nid.h`), with w the cell's lifted slacks rescaled so the
    smallest positive one is 1 (exponents <= SLACK_MARGIN become 0)
  * `binomial_solutions(V, beta)`            polyhedral.py:696-727
  * `solve_cell(cell, g, supports, params)`  polyhedral.py:794-811, one launch
  * `solve_cells(cells, g, supports, params)` every cell of a mixed
    subdivision in ONE launch (`nid_track_cells`: each path carries its
    cell's t-exponent row), results in cell order (what
    `solve_start_system`'s consume loop collects, cascade.py:134-141)

Mixed-cell enumeration (the CPU LP, polyhedral.py:597-621) stays on the host
and is not part of this package: cells are the reference's `MixedCell`
objects (duck-typed: `.pairs`, `.texps`, `.volume`) or `Cell` below.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .homotopy import DeviceHomotopy, Lowered, TrackParams, eval_batch, params_c

SLACK_MARGIN = 1e-9  # polyhedral.py:30


@dataclass(frozen=True)
class Cell:
    """A fine mixed cell (polyhedral.py:75-87): one edge (a, b) per support
    and the t-exponent of every support point (0 on the chosen pairs)."""

    pairs: tuple
    texps: tuple
    volume: int = 0
    normal: tuple = ()


def supports_of(f) -> tuple:
    """Sorted, deduplicated exponent sets per polynomial (polyhedral.py:45-52)."""
    out = []
    for i, p in enumerate(f.polys):
        if not p.terms:
            raise ValueError(f"polynomial {i} is zero; it has no Newton polytope")
        out.append(tuple(sorted({tuple(int(v) for v in e) for e, _ in p.terms})))
    return tuple(out)


def rescaled_texps(cell) -> np.ndarray:
    """The cell's t-exponents, row after row, divided by the smallest one
    above SLACK_MARGIN; the others become 0 (polyhedral.py:784-789)."""
    raw = np.concatenate([np.asarray(t, dtype=np.float64) for t in cell.texps]) if cell.texps else np.zeros(0)
    pos = raw[raw > SLACK_MARGIN]
    scale = 1.0 / pos.min() if pos.size else 1.0
    return np.where(raw > SLACK_MARGIN, raw * scale, 0.0)


def lower_polyhedral(g, cell, supports) -> Lowered:
    """Term table of the cell's homotopy: row i = g's row i in support order
    (the reference pairs supports[i] with g.polys[i].terms positionally)."""
    n = g.nvars
    if len(g.polys) != n:
        raise ValueError("the GPU tracker needs a square system (rows == variables)")
    if n > _lib.MAX_VARS:
        raise ValueError(f"at most {_lib.MAX_VARS} variables are supported")
    offs, ex, ct = [0], [], []
    for i, p in enumerate(g.polys):
        pts = supports[i]
        if len(p.terms) != len(pts):
            raise ValueError("start system terms must align with the support")
        if len(cell.texps[i]) != len(pts):
            raise ValueError("the cell needs one t-exponent per support point")
        for e, (_, c) in zip(pts, p.terms):
            ex.append(tuple(int(v) for v in e))
            ct.append(complex(c))
        offs.append(len(ct))
    T = len(ct)
    expo = np.zeros((T, _lib.MAX_VARS), dtype=np.uint8)
    if T:
        arr = np.array(ex, dtype=np.int64).reshape(T, n)
        if arr.min(initial=0) < 0 or arr.max(initial=0) > 255:
            raise ValueError("exponents must lie in 0..255")
        expo[:, :n] = arr
    return Lowered(n, np.array(offs, dtype=np.int32), expo, np.zeros(T, np.complex128),
                   np.array(ct, dtype=np.complex128), None, 0, 1.0 + 0j, None,
                   np.ascontiguousarray(rescaled_texps(cell)))


@dataclass(frozen=True)
class PolyhedralHomotopy:
    """Per-cell continuation (polyhedral.py:730-791): at t = 0 only the
    cell's binomial system survives, at t = 1 the homotopy is g itself."""

    g: object
    cell: object
    supports: tuple
    _cache: dict = field(default_factory=dict, repr=False, compare=False)

    @property
    def dim(self) -> int:
        return self.g.nvars

    def lowered(self) -> Lowered:
        low = self._cache.get("low")
        if low is None:
            low = lower_polyhedral(self.g, self.cell, self.supports)
            self._cache["low"] = low
        return low

    def device(self) -> DeviceHomotopy:
        dev = self._cache.get("dev")
        if dev is None:
            dev = DeviceHomotopy(self.lowered())
            self._cache["dev"] = dev
        return dev

    def evaluate(self, X, T):
        return eval_batch(self.device(), X, T)

    def eval(self, x, t):
        return self.evaluate(np.asarray(x)[None], np.array([t]))[0][0]

    def jac(self, x, t):
        return self.evaluate(np.asarray(x)[None], np.array([t]))[1][0]

    def eval_scale(self, x, t):
        return float(self.evaluate(np.asarray(x)[None], np.array([t]))[2][0])


def _hermite_lower(V):
    """(L, U): U unimodular, L = V U lower triangular with a positive
    diagonal.  Column Euclid row by row; exact integer arithmetic on plain
    Python ints (columns stored as lists)."""
    n = len(V)
    Mc = [[int(V[r][c]) for r in range(n)] for c in range(n)]  # Mc[c] = column c of M
    Uc = [[int(r == c) for r in range(n)] for c in range(n)]
    for k in range(n):
        while True:
            cols = [j for j in range(k, n) if Mc[j][k] != 0]
            if not cols:
                raise ValueError("the cell's edge matrix is singular")
            p = min(cols, key=lambda j: abs(Mc[j][k]))
            if p != k:
                Mc[k], Mc[p] = Mc[p], Mc[k]
                Uc[k], Uc[p] = Uc[p], Uc[k]
            rest = [j for j in range(k + 1, n) if Mc[j][k] != 0]
            if not rest:
                break
            mk, uk, piv = Mc[k], Uc[k], Mc[k][k]
            for j in rest:
                q = Mc[j][k] // piv
                Mc[j] = [a - q * b for a, b in zip(Mc[j], mk)]
                Uc[j] = [a - q * b for a, b in zip(Uc[j], uk)]
        if Mc[k][k] < 0:
            Mc[k] = [-a for a in Mc[k]]
            Uc[k] = [-a for a in Uc[k]]
    L = np.array(Mc, dtype=np.int64).T
    U = np.array(Uc, dtype=np.int64).T
    return L, U


def binomial_solutions(V, beta) -> np.ndarray:
    """All solutions of y^(rows of V) = beta in the complex torus
    (polyhedral.py:696-727): with L = V U lower triangular, solve w^L = beta
    level by level (L[k][k] roots per level, every branch at once), then
    y_l = prod_j w_j^{U[l][j]}.  Returns [|det V|, n] complex128."""
    n = len(V)
    L, U = _hermite_lower(V)
    beta = np.asarray(beta, dtype=np.complex128)
    W = np.ones((1, 0), dtype=np.complex128)
    for k in range(n):
        rhs = np.full(W.shape[0], beta[k])
        for j in range(k):
            rhs = rhs / W[:, j] ** int(L[k, j])
        m = int(L[k, k])
        r = np.abs(rhs) ** (1.0 / m)
        th = np.angle(rhs)
        ls = np.arange(m)
        wk = r[:, None] * np.exp(1j * (th[:, None] + 2.0 * np.pi * ls[None, :]) / m)
        W = np.concatenate([np.repeat(W, m, axis=0), wk.reshape(-1, 1)], axis=1)
    Y = np.ones((W.shape[0], n), dtype=np.complex128)
    for l in range(n):
        for j in range(n):
            e = int(U[l, j])
            if e:
                Y[:, l] *= W[:, j] ** e
    return Y


def _coeff_maps(g):
    cached = getattr(g, "_cache", None)
    if isinstance(cached, dict) and "coeff_of" in cached:
        return cached["coeff_of"]
    maps = [dict((tuple(int(v) for v in e), complex(c)) for e, c in p.terms) for p in g.polys]
    if isinstance(cached, dict):
        cached["coeff_of"] = maps
    return maps


def cell_starts(cell, g) -> np.ndarray:
    """The cell's binomial start system and its roots (polyhedral.py:800-808)."""
    n = g.nvars
    coeff_of = _coeff_maps(g)
    V, beta = [], []
    for i, (a, b) in enumerate(cell.pairs):
        a, b = tuple(int(v) for v in a), tuple(int(v) for v in b)
        V.append([b[j] - a[j] for j in range(n)])
        beta.append(-coeff_of[i][a] / coeff_of[i][b])
    return binomial_solutions(V, beta)


def solve_cell(cell, g, supports, params: TrackParams = TrackParams(), mode: str = "gpu"):
    """Track the cell's volume-many paths from its binomial system to g at
    t = 1 (polyhedral.py:794-811) in one launch; list[PathResult]."""
    if mode != "gpu":
        raise ValueError(f"unknown mode {mode!r}: this package tracks on the GPU")
    from .tracker import track_batch

    starts = cell_starts(cell, g)
    h = PolyhedralHomotopy(g, cell, tuple(supports))
    return track_batch(h, starts, _cell_params(params)).path_results()


def _cell_params(params):
    """Cells are tracked in double precision whatever params.precision says:
    the reference's PolyhedralHomotopy evaluates generically (double-double)
    only at t = 1 (polyhedral.py:783-791), so its double-double mode cannot
    track a cell; the start roots are polished by the continuation that
    follows."""
    if getattr(params, "precision", "double") == "double":
        return params
    from dataclasses import fields as _fields

    kw = {f.name: getattr(params, f.name) for f in _fields(TrackParams) if hasattr(params, f.name)}
    kw["precision"] = "double"
    return TrackParams(**kw)


def track_cells(cells, g, supports, params: TrackParams = TrackParams()):
    """Every cell's paths in ONE launch (`nid_track_cells`): the starts of all
    cells concatenated in cell order, each path carrying its cell's rescaled
    t-exponent row.  Returns (TrackResults, per-cell path counts)."""
    import ctypes as C

    from .tracker import TrackResults

    cells = list(cells)
    if not cells:
        raise ValueError("no cells")
    supports = tuple(supports)
    h = PolyhedralHomotopy(g, cells[0], supports)
    dev = h.device()
    n, T = g.nvars, h.lowered().nterms
    starts, rows, counts = [], [], []
    for cell in cells:
        st = cell_starts(cell, g)
        w = rescaled_texps(cell)
        if w.size != T:
            raise ValueError("the cell needs one t-exponent per support point")
        starts.append(st)
        rows.append(np.broadcast_to(w, (len(st), T)))
        counts.append(len(st))
    st = np.ascontiguousarray(np.concatenate(starts), dtype=np.complex128)
    tw = np.ascontiguousarray(np.concatenate(rows), dtype=np.float64)
    P = st.shape[0]
    out = TrackResults(np.empty((P, n), np.complex128), np.empty(P, np.int8), np.empty(P, np.int32),
                       np.empty(P, np.float64), np.empty(P, np.float64), np.empty(P, np.float64),
                       np.empty(P, np.int8), {})
    o = _lib.PathOutC(_lib.ptr(out.x), _lib.ptr(out.status), _lib.ptr(out.steps), _lib.ptr(out.t_reached),
                      _lib.ptr(out.residual), _lib.ptr(out.condition), _lib.ptr(out.regular))
    L = _lib.lib()
    pc = params_c(_cell_params(params))
    _lib.check(L.nid_track_cells(dev.handle, C.byref(pc), P, _lib.ptr(st), _lib.ptr(tw), C.byref(o), 0, None), L)
    out.counters = _lib.last_counters()
    return out, counts


def solve_cells(cells, g, supports, params: TrackParams = TrackParams(), mode: str = "gpu"):
    """Every cell in order, results concatenated as solve_start_system's
    consume loop collects them (cascade.py:134-141); one launch for all."""
    if mode != "gpu":
        raise ValueError(f"unknown mode {mode!r}: this package tracks on the GPU")
    res, _ = track_cells(cells, g, supports, params)
    return res.path_results()


def random_coefficient_system(supports, nvars: int, seed: int):
    """Unit-modulus random coefficients on exactly the given supports, drawn
    from the reference's START_COEFFS stream (polyhedral.py:645-652), so the
    same seed gives the same start system g on both sides."""
    from . import rng as rngmod
    from .polys import PolySystem, make_poly

    gen = rngmod.stream(seed, rngmod.START_COEFFS)
    polys = []
    for pts in supports:
        coeffs = rngmod.unit_complex(gen, len(pts))
        polys.append(make_poly(nvars, list(zip(pts, coeffs))))
    return PolySystem(nvars, tuple(polys))


# ---------------------------------------------------------------- pipeline


@dataclass
class PipelineStats:
    """parallel.py:156-164, plus the GPU consumer's batch count."""

    produced: int = 0
    consumed: int = 0
    batches: int = 0
    makespan: float = 0.0
    producer_blocked: float = 0.0
    consumer_idle: float = 0.0
    first_consume_before_last_produce: bool = False
    producer_error: str | None = None


def pipeline_cells(producer, g, supports, params: TrackParams = TrackParams(), queue_capacity: int = 64,
                   max_batch_cells: int = 4096, track=None):
    """Cell producer -> GPU consumer pipeline (the paper's pipelining of
    cell enumeration with path tracking; the reference's `_pipelined_cells`
    cascade.py:163-211 over `pipeline_run` parallel.py:166-231).

    The producer (any iterable of cells -- e.g. the reference's CPU LP
    enumeration feeding a queue) runs in its own thread behind a bounded
    queue.  ONE consumer thread owns the GPU: it blocks for the first
    available cell, drains whatever else is queued (up to max_batch_cells)
    and tracks that batch in one launch (`track_cells`); the C call releases
    the GIL, so enumeration continues while the GPU tracks.  A producer error
    closes the queue; what was produced is still tracked and the error is
    reported in the stats, as in the reference.

    Returns (list of PathResult in cell order, per-cell path counts,
    PipelineStats).  `track(cells, g, supports, params) -> (TrackResults,
    counts)` replaces the GPU call in host-logic tests."""
    import queue
    import threading
    import time
    import traceback

    if queue_capacity < 1:
        raise ValueError("queue capacity must be positive")
    track = track or track_cells
    stats = PipelineStats()
    buf: queue.Queue = queue.Queue(maxsize=queue_capacity)
    done = object()
    per_cell: dict = {}
    produce_done_at = [None]
    first_consume_at = [None]
    consumer_error: list = []

    def produce():
        idx = 0
        try:
            for cell in producer:
                t0 = time.perf_counter()
                buf.put((idx, cell))
                stats.producer_blocked += time.perf_counter() - t0
                idx += 1
        except Exception:  # noqa: BLE001 -- reported, as parallel.py:199-200
            stats.producer_error = traceback.format_exc(limit=4)
        finally:
            stats.produced = idx
            produce_done_at[0] = time.perf_counter()
            buf.put(done)

    def consume():
        finished = False
        while not finished:
            t0 = time.perf_counter()
            got = buf.get()
            stats.consumer_idle += time.perf_counter() - t0
            if got is done:
                return
            batch = [got]
            while len(batch) < max_batch_cells:
                try:
                    nxt = buf.get_nowait()
                except queue.Empty:
                    break
                if nxt is done:
                    finished = True
                    break
                batch.append(nxt)
            if first_consume_at[0] is None:
                first_consume_at[0] = time.perf_counter()
            try:
                res, counts = track([c for _, c in batch], g, supports, params)
            except Exception:  # noqa: BLE001 -- re-raised on the calling thread
                consumer_error.append(traceback.format_exc(limit=6))
                while not finished and buf.get() is not done:  # unblock the producer
                    pass
                return
            rows = res.path_results()
            pos = 0
            for (i, _), k in zip(batch, counts):
                per_cell[i] = (rows[pos:pos + k], k)
                pos += k
            stats.batches += 1

    t_start = time.perf_counter()
    pt = threading.Thread(target=produce, name="nid-cell-producer")
    ct = threading.Thread(target=consume, name="nid-gpu-consumer")
    pt.start()
    ct.start()
    pt.join()
    ct.join()
    stats.makespan = time.perf_counter() - t_start
    if consumer_error:
        raise RuntimeError(f"GPU consumer failed:\n{consumer_error[0]}")
    stats.consumed = len(per_cell)
    if first_consume_at[0] is not None and produce_done_at[0] is not None:
        stats.first_consume_before_last_produce = first_consume_at[0] < produce_done_at[0]
    results, counts = [], []
    for i in sorted(per_cell):
        rows, k = per_cell[i]
        results.extend(rows)
        counts.append(k)
    return results, counts, stats
