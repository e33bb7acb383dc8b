"""`decompose(mode="gpu")`: the reference's fixed-recipe solver
(`nidpipe/blackbox.py:36-110`) with every tracking stage on the GPU.

embed -> solve_top from the polyhedral start (all mixed cells in one launch,
then the continuation) -> run_cascade -> filter_junk -> classify_isolated,
returning the fields of the reference's `DecompositionReport`
(report.py:51-70).  Two host-side pieces are not re-implemented here:

  * mixed-cell enumeration (the CPU LP, polyhedral.py:597-621): pass `cells`
    (e.g. a cell log of the reference), or have `nidpipe` importable and the
    reference's `lift_supports` / `enumerate_cells` are called with the same
    tie-retry loop as solve_start_system (cascade.py:124-149);
  * `square_up` of non-square inputs (systems.py): the input must be square.
"""

from __future__ import annotations

import time
from . import polyhedral as ph
from .cascade import TopStats, run_cascade, solve_top
from .filtering import classify_isolated, filter_junk
from . import refbridge
from .homotopy import TrackParams
from .report import DecompositionReport, Timings
from .systems import embed


# the record decompose returns: the reference's DecompositionReport fields
# (report.py:51-70) plus the cascade's WitnessSuperset
Decomposition = DecompositionReport


def enumerate_cells_host(system, seed: int) -> list:
    """The fine mixed cells of the system's lifted supports, from the
    reference's CPU LP with the tie-retry loop of solve_start_system
    (cascade.py:124-149).  Needs `nidpipe` importable."""
    try:
        import nidpipe.polyhedral as rph
    except ImportError as e:  # pragma: no cover - depends on the host
        raise RuntimeError("mixed-cell enumeration needs the reference package (nidpipe) on the host; "
                           "pass cells= instead") from e
    supports = ph.supports_of(system)
    for attempt in range(6):
        cells: list = []
        try:
            rph.enumerate_cells(rph.lift_supports(supports, seed, attempt), lambda c: cells.append(c) or True)
            return cells
        except rph.TieDetected:
            continue
    raise RuntimeError("could not find a generic lifting for the start system")


def decompose(f, top_dimension: int | None = None, seed: int = 0, tasks: int = 1, precision: str = "double",
              mode: str = "gpu", cell_log: list | None = None, cells=None,
              input_path: str | None = None) -> DecompositionReport:
    """Numerical irreducible decomposition with every path on the GPU
    (blackbox.py:36-110).  mode "thread" / "process" is the reference's CPU
    work crew: delegated to nidpipe.blackbox.decompose when it is importable."""
    if not refbridge.check_mode(mode):
        return refbridge.decompose(f, top_dimension, seed, tasks, precision, mode, cell_log)
    if len(f.polys) != f.nvars:
        raise ValueError("give a square system (square_up stays with the reference)")
    warnings: list = []
    n = f.nvars
    if top_dimension is None:
        top_dimension = n - 1
        warnings.append(f"no top dimension given; defaulting to {top_dimension} "
                        "(an overestimate causes significant extra work)")
    if not 0 <= top_dimension < n:
        raise ValueError(f"top dimension must be in 0..{n - 1}, got {top_dimension}")
    if precision not in ("double", "dd"):
        raise ValueError(f"unknown precision {precision!r}")
    params = TrackParams(precision="double_double" if precision == "dd" else "double")
    timings = Timings()
    emb = embed(f, top_dimension, seed)
    system = emb.system if emb.k > 0 else emb.base
    t0 = time.perf_counter()
    if cells is None:
        cells = enumerate_cells_host(system, seed)
    timings.cells = time.perf_counter() - t0
    top_results, top_stats = solve_top(emb, tasks, seed, params, mode, cell_log, cells=cells)
    timings.start_system = top_stats.time_start_system + timings.cells
    timings.continuation = top_stats.time_continuation
    t0 = time.perf_counter()
    superset = run_cascade(top_results, emb, tasks, params, mode)
    timings.cascade = time.perf_counter() - t0
    t0 = time.perf_counter()
    witness_sets, stages = filter_junk(superset, tasks, params, mode)
    isolated, suspects, iso_stages = classify_isolated(superset.candidates(0), witness_sets, f, tasks, params, mode)
    timings.filtering = time.perf_counter() - t0
    return DecompositionReport(seed, top_dimension, tasks, precision, n, tuple(getattr(f, "names", ()) or ()),
                               witness_sets, isolated, suspects, [lv.counts for lv in superset.levels],
                               stages + iso_stages, top_stats, timings, input_path, warnings, superset)
