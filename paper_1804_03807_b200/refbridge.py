"""Delegation of the CPU modes to the reference.

The drivers of this package keep the reference's signatures, including the
`mode` string (`cascade.py:219,300,330`, `filtering.py:97,157,210`,
`blackbox.py:42`).  `mode="gpu"` runs here; `mode="thread"` / `"process"`
are the reference's CPU work crew and are handed to `nidpipe` itself when it
is importable -- this package has no CPU tracker.  Inputs built with this
package's value types are converted term by term to the reference's; records
the reference returns are passed through unchanged (they carry the same
fields as this package's).  Unknown modes raise ValueError as in
`parallel.py:109`.
"""

from __future__ import annotations

from dataclasses import fields

CPU_MODES = ("thread", "process")


def reference():
    """The reference package, or an ImportError that says what is missing."""
    try:
        import nidpipe  # noqa: F401
        import nidpipe.blackbox
        import nidpipe.cascade
        import nidpipe.filtering
        import nidpipe.tracker
    except ImportError as e:
        raise ImportError("mode='thread'/'process' is the reference's CPU work crew: the nidpipe package must be "
                          "importable (this package tracks on the GPU only, mode='gpu')") from e
    return nidpipe


def check_mode(mode: str) -> bool:
    """True for the GPU mode, False for a CPU mode (delegate); raises for
    anything else."""
    if mode == "gpu":
        return True
    if mode in CPU_MODES:
        return False
    raise ValueError(f"unknown work crew mode {mode!r}")


def _is_ref(obj) -> bool:
    return type(obj).__module__.startswith("nidpipe.")


def to_ref_system(s):
    if s is None or _is_ref(s):
        return s
    rp = reference().polynomials
    return rp.PolySystem(s.nvars, tuple(rp.make_poly(s.nvars, p.terms) for p in s.polys), tuple(s.names))


def to_ref_embedding(e):
    if e is None or _is_ref(e):
        return e
    return reference().systems.EmbeddedSystem(to_ref_system(e.base), e.k, e.gammas, e.hyper_coeffs, e.seed)


def to_ref_params(p):
    if _is_ref(p):
        return p
    rt = reference().tracker
    return rt.TrackParams(**{f.name: getattr(p, f.name) for f in fields(rt.TrackParams)})


def to_ref_solution(s):
    if s is None or _is_ref(s):
        return s
    return reference().tracker.Solution(s.coordinates, s.residual, s.condition, s.regularity, s.slack_class)


def to_ref_path_result(r):
    if _is_ref(r):
        return r
    return reference().tracker.PathResult(r.status, to_ref_solution(r.endpoint), r.steps_used, r.t_reached)


def to_ref_level(lv):
    if _is_ref(lv):
        return lv
    return reference().cascade.CascadeLevel(lv.dimension, to_ref_embedding(lv.embedding), lv.starts, lv.at_infinity,
                                            [to_ref_solution(s) for s in lv.zero_slack],
                                            [to_ref_solution(s) for s in lv.nonzero_slack], lv.failures)


def to_ref_superset(ss):
    if _is_ref(ss):
        return ss
    return reference().cascade.WitnessSuperset([to_ref_level(lv) for lv in ss.levels], to_ref_embedding(ss.embedding),
                                               ss.seed)


def to_ref_witness_set(w):
    if _is_ref(w):
        return w
    return reference().filtering.WitnessSet(w.dimension, to_ref_embedding(w.embedding),
                                            [to_ref_solution(s) for s in w.points], w.label)


# ---- the delegated drivers (same argument order as the reference's)

def solve_top(emb, p, seed, params, mode, cell_log):
    return reference().cascade.solve_top(to_ref_embedding(emb), p, seed, to_ref_params(params), mode, cell_log)


def cascade_step(level, p, params, mode):
    return reference().cascade.cascade_step(to_ref_level(level), p, to_ref_params(params), mode)


def run_cascade(top_results, emb, p, params, mode):
    if hasattr(top_results, "path_results"):
        top_results = top_results.path_results()
    return reference().cascade.run_cascade([to_ref_path_result(r) for r in top_results], to_ref_embedding(emb), p,
                                           to_ref_params(params), mode)


def membership_test(w, q, p, params, mode):
    return reference().filtering.membership_test(to_ref_witness_set(w), q, p, to_ref_params(params), mode)


def filter_junk(superset, p, params, mode):
    return reference().filtering.filter_junk(to_ref_superset(superset), p, to_ref_params(params), mode)


def classify_isolated(candidates, witness_sets, original, p, params, mode):
    return reference().filtering.classify_isolated([to_ref_solution(s) for s in candidates],
                                                   [to_ref_witness_set(w) for w in witness_sets],
                                                   to_ref_system(original), p, to_ref_params(params), mode)


def decompose(f, top_dimension, seed, tasks, precision, mode, cell_log):
    return reference().blackbox.decompose(to_ref_system(f), top_dimension, seed, tasks, precision, mode, cell_log)


def track(h, x0, params, trace):
    """The reference's CPU `track` on this package's LinearHomotopy (used by
    `tracker.track(..., mode=...)` callers that ask for a CPU mode)."""
    rt = reference().tracker
    if not _is_ref(h):
        h = rt.LinearHomotopy(to_ref_system(h.start), to_ref_system(h.target), complex(h.gamma))
    return rt.track(h, x0, to_ref_params(params), trace)
