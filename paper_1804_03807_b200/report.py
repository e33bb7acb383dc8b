"""Decomposition report of `decompose(mode="gpu")`: the deterministic JSON
payload and the text summary of the reference (`nidpipe/report.py:22-170`).

The payload layout, key order, point canonicalisation (coordinates of the
original variables, points sorted by their (re, im) pairs rounded to 9
decimals), float formatting (shortest repr through `json`), `sort_keys`,
two-space indent and trailing newline are the reference's
(`report_to_jsonable` :81-124, `report_to_json` :127-128), so a report built
from the same records serialises to the same bytes (same seed +
same configuration + p = 1 gives a byte-identical report).  Records are read
by attribute, so the reference's own `DecompositionReport` / `WitnessSet` /
`FilterStage` / `TopStats` objects serialise through this module too.
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field

import numpy as np

_TIMING_ROWS = (("start system", "start_system"), ("continuation", "continuation"), ("top total", "top_total"),
                ("cascade", "cascade"), ("filter", "filtering"), ("grand total", "grand_total"))


@dataclass
class Timings:
    """report.py:22-48; seconds per stage.  `cells` is this package's extra:
    the host-side mixed-cell LP, which the reference books under the start
    system (it is included in `start_system` here as well)."""

    start_system: float = 0.0
    continuation: float = 0.0
    cascade: float = 0.0
    filtering: float = 0.0
    cells: float = 0.0

    @property
    def top_total(self) -> float:
        return self.start_system + self.continuation

    @property
    def grand_total(self) -> float:
        return self.top_total + self.cascade + self.filtering

    def table(self) -> str:
        w = max(len(label) for label, _ in _TIMING_ROWS)
        return "\n".join(f"{label:<{w}}  {getattr(self, attr):10.3f} s" for label, attr in _TIMING_ROWS)

    # dict-style access for callers of the earlier timings dict
    def __getitem__(self, key: str) -> float:
        return getattr(self, key)


@dataclass
class DecompositionReport:
    """report.py:51-70"""

    seed: int
    top_dimension: int
    tasks: int
    precision: str
    nvars: int
    names: tuple
    witness_sets: list
    isolated: list
    suspects: list
    cascade_counts: list
    filter_stages: list
    top_stats: object
    timings: Timings = field(default_factory=Timings)
    input_path: str | None = None
    warnings: list = field(default_factory=list)
    superset: object = None  # the cascade's WitnessSuperset (not serialised)

    @property
    def degrees(self) -> dict:
        return {w.dimension: w.degree for w in self.witness_sets}


def _canonical_points(solutions, n: int) -> list:
    """The points' first n coordinates as [[re, im], ...], in the report's
    canonical order (report.py:73-78)."""
    pts = np.array([np.asarray(s.coordinates)[:n] for s in solutions], np.complex128).reshape(-1, n)
    if len(pts) == 0:
        return []
    # the sort key of the reference: per coordinate (round(re, 9), round(im, 9)),
    # with Python's correctly rounded round() (numpy's scaled rint can differ in
    # the last place); stable, so equal keys keep their input order as there
    rows = [[[float(z.real), float(z.imag)] for z in p] for p in pts]
    return sorted(rows, key=lambda r: [round(c, 9) for ri in r for c in ri])


_STAGE_FIELDS = ("candidate_dimension", "against_dimension", "candidates", "degree", "paths_tracked", "removed")


def report_to_jsonable(rep) -> dict:
    """report.py:81-124"""
    n = rep.nvars
    ts = rep.top_stats
    wsets = {}
    for w in sorted(rep.witness_sets, key=lambda w: -w.dimension):
        wsets[str(w.dimension)] = {"degree": w.degree, "points": _canonical_points(w.points, n)}
    return {
        "seed": rep.seed,
        "input": getattr(rep, "input_path", None),
        "nvars": rep.nvars,
        "variables": list(rep.names),
        "top_dimension": rep.top_dimension,
        "tasks": rep.tasks,
        "precision": rep.precision,
        "witness_sets": wsets,
        "isolated": _canonical_points(rep.isolated, n),
        "suspects": _canonical_points(rep.suspects, n),
        "counts": {
            "mixed_volume": ts.mixed_volume,
            "cells": ts.cells,
            "start_paths": ts.start_paths,
            "continuation_paths": ts.continuation_paths,
            "top_at_infinity": ts.at_infinity,
            "top_finite": ts.finite,
            "cascade_levels": rep.cascade_counts,
            "filter_stages": [{k: getattr(s, k) for k in _STAGE_FIELDS} for s in rep.filter_stages],
        },
        "warnings": list(rep.warnings),
    }


def report_to_json(rep) -> str:
    """report.py:127-128"""
    return json.dumps(report_to_jsonable(rep), sort_keys=True, indent=2) + "\n"


def summary_text(rep) -> str:
    """report.py:131-170"""
    ts = rep.top_stats
    out = [f"seed {rep.seed}, top dimension {rep.top_dimension}, {rep.tasks} task(s), {rep.precision} precision",
           f"mixed volume {ts.mixed_volume} over {ts.cells} cells; {ts.continuation_paths} paths to the top system "
           f"({ts.finite} finite, {ts.at_infinity} at infinity, {ts.failures} failed)",
           "",
           "cascade levels (starts / at infinity / zero slack / nonzero slack):"]
    out += [f"  dim {c['dimension']}: {c['starts']:>4} / {c['at_infinity']:>3} / {c['zero_slack']:>3} / "
            f"{c['nonzero_slack']:>3}" for c in rep.cascade_counts]
    if rep.filter_stages:
        out += ["", "membership filters (candidates at dim -> tested against dim: paths, removed):"]
        out += [f"  {s.candidates} at dim {s.candidate_dimension} -> dim {s.against_dimension} (degree {s.degree}): "
                f"{s.paths_tracked} paths, removed {s.removed}" for s in rep.filter_stages]
    out.append("")
    if rep.witness_sets:
        out.append("witness sets: " + ", ".join(f"dimension {w.dimension} degree {w.degree}" for w in rep.witness_sets))
    else:
        out.append("witness sets: none")
    out.append(f"isolated solutions: {len(rep.isolated)}")
    out.append(f"WARNING: {len(rep.suspects)} isolated-singular suspect(s) remain (deflation not available)"
               if rep.suspects else "no isolated singular suspects")
    out += [f"WARNING: {w}" for w in rep.warnings]
    out += ["", "timings:", rep.timings.table()]
    return "\n".join(out) + "\n"


def report_from_jsonable(d: dict) -> DecompositionReport:
    """Rebuild the records of a serialised report (counts and points; residuals
    and conditions are not part of the payload and come back as NaN)."""
    from .cascade import TopStats
    from .filtering import FilterStage, WitnessSet
    from .tracker import Solution

    def sols(points):
        return [Solution(np.array([complex(re, im) for re, im in p]), float("nan"), float("nan")) for p in points]

    c = d["counts"]
    ts = TopStats(cells=c["cells"], mixed_volume=c["mixed_volume"], start_paths=c["start_paths"],
                  continuation_paths=c["continuation_paths"], at_infinity=c["top_at_infinity"], finite=c["top_finite"])
    wsets = [WitnessSet(int(k), None, sols(v["points"])) for k, v in d["witness_sets"].items()]
    wsets.sort(key=lambda w: -w.dimension)
    stages = [FilterStage(**{k: s[k] for k in _STAGE_FIELDS}) for s in c["filter_stages"]]
    return DecompositionReport(d["seed"], d["top_dimension"], d["tasks"], d["precision"], d["nvars"],
                               tuple(d["variables"]), wsets, sols(d["isolated"]), sols(d["suspects"]),
                               c["cascade_levels"], stages, ts, Timings(), d.get("input"), list(d["warnings"]))
