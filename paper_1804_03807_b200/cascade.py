"""Top-dimensional continuation and the cascade of embedded homotopies on the
GPU (mode="gpu"), with the reference's signatures and records
(pkg/src/nidpipe/cascade.py:47-337).

Every stage batches all of its paths into one `track_batch` launch (the
reference fans them out through `work_crew`), and refines + classifies all
endpoints of a level in one `refine_batch` launch.

Difference from the reference, by scope: `solve_top`
starts from the total-degree system G_i = x_i^{d_i} - 1 instead of the
polyhedral random-coefficient system; gamma is the reference's own draw
`stream(seed, GAMMA)` (cascade.py:226).
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

from . import rng as rngmod
from .homotopy import LinearHomotopy, TrackParams
from .polys import PolySystem, make_poly, variable_poly
from .systems import EmbeddedSystem, total_degree_start
from .tracker import (
    AT_INFINITY,
    NONZERO_SLACK,
    ZERO_SLACK,
    PathResult,
    Solution,
    TrackResults,
    refine_batch,
    track_batch,
)

from . import refbridge

GPU_MODES = ("gpu",)


def _check_mode(mode: str) -> bool:
    """True: track here on the GPU.  False: a CPU work-crew mode of the
    reference ("thread" / "process"), which the caller delegates to nidpipe
    (refbridge).  Anything else raises ValueError (parallel.py:109)."""
    return refbridge.check_mode(mode)


@dataclass
class TopStats:
    """cascade.py:47-59"""

    cells: int = 0
    mixed_volume: int = 0
    start_paths: int = 0
    start_failures: int = 0
    continuation_paths: int = 0
    at_infinity: int = 0
    finite: int = 0
    failures: int = 0
    lifting_attempt: int = 0
    time_start_system: float = 0.0
    time_continuation: float = 0.0


@dataclass
class CascadeLevel:
    """cascade.py:62-88"""

    dimension: int
    embedding: EmbeddedSystem
    starts: int
    at_infinity: int
    zero_slack: list = field(default_factory=list)
    nonzero_slack: list = field(default_factory=list)
    failures: int = 0

    @property
    def counts(self) -> dict:
        return {"dimension": self.dimension, "starts": self.starts, "at_infinity": self.at_infinity,
                "zero_slack": len(self.zero_slack), "nonzero_slack": len(self.nonzero_slack),
                "failures": self.failures}


@dataclass
class WitnessSuperset:
    """cascade.py:91-107"""

    levels: list
    embedding: EmbeddedSystem
    seed: int

    def candidates(self, dimension: int) -> list:
        for lv in self.levels:
            if lv.dimension == dimension:
                return lv.zero_slack
        return []

    @property
    def stage_counts(self) -> list:
        return [lv.counts for lv in self.levels]


def top_homotopy(emb: EmbeddedSystem, seed: int | None = None) -> tuple[LinearHomotopy, tuple]:
    seed = emb.seed if seed is None else seed
    system = emb.system if emb.k > 0 else emb.base
    g = total_degree_start(system)
    gamma = rngmod.gamma_for(seed)
    return LinearHomotopy(g, system, gamma), tuple(system.degrees())


def solve_top(emb: EmbeddedSystem, p: int = 1, seed: int | None = None, params: TrackParams = TrackParams(),
              mode: str = "gpu", cell_log: list | None = None, return_arrays: bool = False, cells=None):
    """Continuation onto the embedded system (cascade.py:214-246).  Returns
    (results, TopStats).

    Start system: the total-degree system by default.  With `cells` (the
    fine mixed cells of the system's lifted supports, e.g. the reference's
    `enumerate_cells(lift_supports(supports_of(system), seed, attempt))`,
    which stays a host-side CPU LP) it is the reference's default polyhedral
    start instead (solve_start_system, cascade.py:110-160): the random-
    coefficient system g on the same supports, all cells tracked to g in one
    launch (`polyhedral.track_cells`), then g -> system from g's roots."""
    if not _check_mode(mode):
        return refbridge.solve_top(emb, p, seed, params, mode, cell_log)
    if cells is not None:
        return _solve_top_polyhedral(emb, seed, params, cells, cell_log, return_arrays, p)
    h, degrees = top_homotopy(emb, seed)
    total = int(np.prod(degrees, dtype=np.int64))
    stats = TopStats(start_paths=total)
    t0 = time.perf_counter()
    res = track_batch(h, None, params, degrees=degrees, count=total)
    stats.time_continuation = time.perf_counter() - t0
    return _top_stats(res, stats, total, return_arrays)


def _top_stats(res, stats, total, return_arrays):
    c = res.counts()
    stats.continuation_paths = total
    stats.at_infinity = c["at_infinity"]
    stats.finite = c["converged"] + c["singular_endpoint"]
    stats.failures = c["failed"]
    if stats.continuation_paths and stats.finite == 0:
        raise RuntimeError("all continuation paths failed")
    return (res if return_arrays else res.path_results()), stats


def _solve_top_polyhedral(emb, seed, params, cells, cell_log, return_arrays, p=1):
    """p >= 2: cells stream through the producer -> GPU consumer pipeline
    (polyhedral.pipeline_cells; the reference's _pipelined_cells,
    cascade.py:163-211), so a lazy cell enumeration overlaps the tracking."""
    from . import polyhedral as ph

    seed = emb.seed if seed is None else seed
    system = emb.system if emb.k > 0 else emb.base
    supports = ph.supports_of(system)
    g = ph.random_coefficient_system(supports, system.nvars, seed)
    stats = TopStats()
    seen: list = []

    def tee():
        for c in cells:
            seen.append(c)
            yield c

    t0 = time.perf_counter()
    if p >= 2:
        rows, _, pst = ph.pipeline_cells(tee(), g, supports, params)
        if pst.producer_error:
            raise RuntimeError(f"cell producer failed:\n{pst.producer_error}")
        x0 = np.array([r.endpoint.coordinates for r in rows if r.succeeded and r.endpoint is not None],
                      np.complex128).reshape(-1, system.nvars)
        stats.start_paths = len(rows)
    else:
        start, _ = ph.track_cells(list(tee()), g, supports, params)
        x0 = start.x[start.succeeded]
        stats.start_paths = len(start)
    stats.time_start_system = time.perf_counter() - t0
    stats.cells = len(seen)
    stats.mixed_volume = int(sum(int(c.volume) for c in seen))
    if cell_log is not None:
        cell_log.extend(seen)
    stats.start_failures = int(stats.start_paths - len(x0))
    h = LinearHomotopy(g, system, rngmod.gamma_for(seed))
    t0 = time.perf_counter()
    res = track_batch(h, x0, params)
    stats.time_continuation = time.perf_counter() - t0
    return _top_stats(res, stats, len(x0), return_arrays)


def _classify_arrays(x: np.ndarray, status_ok: np.ndarray, n_at_inf: int, n_fail: int, emb_level: EmbeddedSystem,
                     dimension: int, params: TrackParams, starts: int) -> CascadeLevel:
    lv = CascadeLevel(dimension, emb_level, starts=starts, at_infinity=n_at_inf, failures=n_fail)
    system = emb_level.system if emb_level.k else emb_level.base
    pts = x[status_ok]
    if len(pts):
        rr = refine_batch(system, pts, tol=1e-13, max_iters=6, n_original=emb_level.n_original,
                          infinity_threshold=params.infinity_threshold)
        for i in range(len(pts)):
            sol = rr.solution(i, with_slack=True)
            if sol.slack_class == AT_INFINITY:
                lv.at_infinity += 1
            elif sol.slack_class == ZERO_SLACK:
                lv.zero_slack.append(sol)
            else:
                lv.nonzero_slack.append(sol)
    return lv


def _classify_level(results, emb_level: EmbeddedSystem, dimension: int, params: TrackParams) -> CascadeLevel:
    """Refine + three-way classification of tracked paths (cascade.py:249-277)."""
    if isinstance(results, TrackResults):
        ok = results.succeeded
        c = results.counts()
        return _classify_arrays(results.x, ok, c["at_infinity"], c["failed"], emb_level, dimension, params,
                                len(results))
    n = emb_level.nvars
    at_inf = sum(1 for r in results if r.status == AT_INFINITY)
    ok = np.array([r.status != AT_INFINITY and r.succeeded and r.endpoint is not None for r in results], bool)
    fails = len(results) - at_inf - int(ok.sum())
    x = np.zeros((len(results), n), np.complex128)
    for i, r in enumerate(results):
        if ok[i]:
            x[i] = r.endpoint.coordinates
    return _classify_arrays(x, ok, at_inf, fails, emb_level, dimension, params, len(results))


def _slack_removal_homotopy(emb: EmbeddedSystem, gamma: complex) -> LinearHomotopy:
    """Last hyperplane row x gamma deforms into z_d = 0 (cascade.py:280-293)."""
    system = emb.system
    nv = system.nvars
    rows_s = list(system.polys)
    rows_t = list(system.polys)
    rows_s[-1] = make_poly(nv, [(e, gamma * c) for e, c in rows_s[-1].terms])
    rows_t[-1] = variable_poly(nv, nv - 1)
    return LinearHomotopy(PolySystem(nv, tuple(rows_s), system.names), PolySystem(nv, tuple(rows_t), system.names))


def cascade_step(level: CascadeLevel, p: int = 1, params: TrackParams = TrackParams(), mode: str = "gpu") -> CascadeLevel:
    """Track the level's nonzero-slack solutions one dimension down (cascade.py:296-322)."""
    if not _check_mode(mode):
        return refbridge.cascade_step(level, p, params, mode)
    if level.dimension < 1:
        raise ValueError("cannot cascade below dimension 0")
    emb = level.embedding
    nxt = emb.level(emb.k - 1)
    if not level.nonzero_slack:
        return CascadeLevel(level.dimension - 1, nxt, starts=0, at_infinity=0)
    gamma = rngmod.gamma_for(emb.seed, level.dimension)
    h = _slack_removal_homotopy(emb, gamma)
    starts = np.array([s.coordinates for s in level.nonzero_slack])
    res = track_batch(h, starts, params)
    c = res.counts()
    return _classify_arrays(res.x[:, :-1], res.succeeded, c["at_infinity"], c["failed"], nxt,
                            level.dimension - 1, params, len(res))


def run_cascade(top_results, emb: EmbeddedSystem, p: int = 1, params: TrackParams = TrackParams(),
                mode: str = "gpu") -> WitnessSuperset:
    """cascade.py:325-337"""
    if not _check_mode(mode):
        return refbridge.run_cascade(top_results, emb, p, params, mode)
    levels = [_classify_level(top_results, emb, emb.k, params)]
    while levels[-1].dimension > 0:
        levels.append(cascade_step(levels[-1], p, params, mode))
    return WitnessSuperset(levels, emb, emb.seed)
