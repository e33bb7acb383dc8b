"""Generate golden fixtures by running the REFERENCE (nidpipe) itself.

Runs only in the build container, where the reference is importable:

    PYTHONPATH=/root/reference/pkg/src:. python tests/golden/make_golden.py [--only NAME ...]

Inputs are built with this framework's seeded config builders
(`paper_1804_03807_b200/configs.py`) and converted to reference objects term
by term (`nidpipe.polynomials.make_poly`), so the fixtures pin the reference's
outputs on exactly the systems the tests and the GPU path use.  Nothing here
is needed at run time on the GPU box: the .npz files are committed.
"""

from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import nidpipe.cascade as rc  # noqa: E402
import nidpipe.filtering as rf  # noqa: E402
import nidpipe.linalg as rl  # noqa: E402
import nidpipe.polynomials as rp  # noqa: E402
import nidpipe.systems as rs  # noqa: E402
import nidpipe.tracker as rt  # noqa: E402
from nidpipe.parallel import JobFailure, work_crew  # noqa: E402

from paper_1804_03807_b200 import configs, systems  # noqa: E402

PROCS = int(os.environ.get("GOLDEN_PROCS", "8"))
STATUS = {"converged": 0, "at_infinity": 1, "singular_endpoint": 2, "failed": 3}


def ref_sys(s):
    return rp.PolySystem(s.nvars, tuple(rp.make_poly(s.nvars, p.terms) for p in s.polys))


def ref_emb(e):
    return rs.EmbeddedSystem(ref_sys(e.base), e.k, e.gammas, e.hyper_coeffs, e.seed)


def save(name, **arrays):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")


def pack_results(results, n):
    P = len(results)
    st = np.zeros(P, np.int8)
    steps = np.zeros(P, np.int32)
    treach = np.zeros(P)
    x = np.full((P, n), np.nan + 0j)
    res = np.full(P, np.nan)
    cond = np.full(P, np.nan)
    reg = np.full(P, -1, np.int8)
    for i, r in enumerate(results):
        if isinstance(r, JobFailure):
            r = rt.PathResult("failed", None, 0, 0.0)
        st[i] = STATUS[r.status]
        steps[i] = r.steps_used
        treach[i] = r.t_reached
        if r.endpoint is not None:
            x[i] = r.endpoint.coordinates
            res[i] = r.endpoint.residual
            cond[i] = r.endpoint.condition
            reg[i] = 1 if r.endpoint.regularity == "regular" else 0
    return dict(status=st, steps=steps, t_reached=treach, x=x, residual=res, condition=cond, regular=reg)


def track_problem(prob, index):
    h = rt.LinearHomotopy(ref_sys(prob.start), ref_sys(prob.target), prob.gamma)
    starts = np.concatenate([systems.total_degree_starts(prob.degrees, int(i), 1) for i in index])
    t0 = time.time()
    res = work_crew(list(starts), PROCS, lambda x0: rt.track(h, x0), mode="process")
    print(f"{prob.name}: {len(index)} paths in {time.time() - t0:.1f}s")
    return dict(index=np.asarray(index, np.int64), starts=starts, **pack_results(res, prob.n))


def gen_eval():
    """H, J and scale of several homotopies at seeded points."""
    gen = np.random.default_rng(1234)
    out = {}
    probs = [configs.c1(), configs.c2(), configs.c5(), configs.c3_top(configs.c3_mini()),
             configs.c3_top(configs.c3())]
    for p in probs:
        h = rt.LinearHomotopy(ref_sys(p.start), ref_sys(p.target), p.gamma)
        n = p.n
        X = gen.normal(size=(6, n)) + 1j * gen.normal(size=(6, n))
        X[0] *= 1e-3
        X[1] *= 30.0
        T = np.array([0.0, 0.3, 0.5, 0.9, 0.999, 1.0])
        out[p.name + "_x"] = X
        out[p.name + "_t"] = T
        out[p.name + "_H"] = np.array([h.eval(x, t) for x, t in zip(X, T)])
        out[p.name + "_J"] = np.array([h.jac(x, t) for x, t in zip(X, T)])
        out[p.name + "_scale"] = np.array([h.eval_scale(x, t) for x, t in zip(X, T)])
    save("eval_golden", **out)


def gen_linalg():
    gen = np.random.default_rng(99)
    out = {}
    for n in (2, 4, 7, 10, 14):
        J = gen.normal(size=(8, n, n)) + 1j * gen.normal(size=(8, n, n))
        r = gen.normal(size=(8, n)) + 1j * gen.normal(size=(8, n))
        J[1, :, 0] = 0.0  # exactly singular: zgesv fails, lstsq path
        J[2, 1] = J[2, 0]  # rank deficient but no exact zero pivot
        J[3] = np.diag(np.logspace(0, -12, n)) @ J[3]  # ill-conditioned
        J[4, n - 1] = 0.0
        J[5] = np.eye(n)
        out[f"n{n}_J"] = J
        out[f"n{n}_r"] = r
        out[f"n{n}_dx"] = np.array([rl.newton_step(J[i], r[i]) for i in range(8)])
        cr = [rl.condition_and_rank(J[i]) for i in range(8)]
        out[f"n{n}_cond"] = np.array([c for c, _ in cr])
        out[f"n{n}_rank"] = np.array([k for _, k in cr])
        out[f"n{n}_sv"] = np.array([np.linalg.svd(J[i], compute_uv=False) for i in range(8)])
    # rectangular (restricted-Jacobian shape) rank tests
    A = gen.normal(size=(4, 14, 8)) + 1j * gen.normal(size=(4, 14, 8))
    A[1, :, 3] = A[1, :, 2] * (2 - 1j)
    out["rect_A"] = A
    out["rect_rank"] = np.array([rl.condition_and_rank(a)[1] for a in A])
    out["rect_cond"] = np.array([rl.condition_and_rank(a)[0] for a in A])
    save("linalg_golden", **out)


def gen_track_small():
    p1 = configs.c1()
    save("track_c1", **track_problem(p1, np.arange(p1.paths)))
    p2 = configs.c2()
    save("track_c2", **track_problem(p2, np.arange(p2.paths)))


def gen_track_c5():
    p5 = configs.c5()
    idx = np.sort(np.random.default_rng(3).choice(p5.paths, size=512, replace=False))
    save("track_c5_sample", **track_problem(p5, idx))


def gen_track_c5_large():
    """16,384 seeded uniform C5 paths: pins the finite count and per-path
    statuses at a sample size where the finite fraction (~0.9 %) is measurable.
    Stored compactly: statuses and steps for all, endpoints of finite paths."""
    p5 = configs.c5()
    idx = np.sort(np.random.default_rng(6).choice(p5.paths, size=16384, replace=False))
    d = track_problem(p5, idx)
    fin = np.isin(d["status"], (0, 2))
    save("track_c5_large", index=d["index"], status=d["status"], steps=d["steps"].astype(np.int16),
         fin_x=d["x"][fin], fin_regular=d["regular"][fin])


def gen_track_c3():
    pd = configs.c3()
    p = configs.c3_top(pd)
    idx = np.sort(np.random.default_rng(4).choice(p.paths, size=64, replace=False))
    save("track_c3_sample", **track_problem(p, idx))


def sols_arrays(prefix, sols, n):
    d = {}
    d[prefix + "_x"] = np.array([s.coordinates for s in sols]).reshape(len(sols), n)
    d[prefix + "_res"] = np.array([s.residual for s in sols])
    d[prefix + "_cond"] = np.array([s.condition for s in sols])
    d[prefix + "_reg"] = np.array([s.regularity == "regular" for s in sols])
    return d


def gen_pipeline_c3m():
    """Total-degree top continuation, run_cascade, filter_junk and
    classify_isolated on the n=4 analog of C3 (SURVEY §7 fast fixture)."""
    pd = configs.c3_mini()
    prob = configs.c3_top(pd)
    t0 = time.time()
    top = track_problem(prob, np.arange(prob.paths))
    emb = ref_emb(pd.emb)
    h = rt.LinearHomotopy(ref_sys(prob.start), ref_sys(prob.target), prob.gamma)
    starts = top["starts"]
    results = work_crew(list(starts), PROCS, lambda x0: rt.track(h, x0), mode="process")
    sup = rc.run_cascade(results, emb, PROCS, rt.TrackParams(), "process")
    print("cascade", [lv.counts for lv in sup.levels], time.time() - t0)
    wsets, stages = rf.filter_junk(sup, PROCS, rt.TrackParams(), "process")
    cands = sup.candidates(0)
    reg, sing, st0 = rf.classify_isolated(cands, wsets, emb.base, PROCS, rt.TrackParams(), "process")
    print("witness", [(w.dimension, w.degree) for w in wsets], "isolated", len(reg), len(sing),
          time.time() - t0)
    out = {f"top_{k}": v for k, v in top.items()}
    nv = emb.nvars
    for lv in sup.levels:
        d = lv.dimension
        nvl = emb.n_original + d
        out.update(sols_arrays(f"L{d}_zero", lv.zero_slack, nvl))
        out.update(sols_arrays(f"L{d}_nonzero", lv.nonzero_slack, nvl))
        out[f"L{d}_counts"] = np.array([lv.starts, lv.at_infinity, len(lv.zero_slack),
                                        len(lv.nonzero_slack), lv.failures])
    for w in wsets:
        out.update(sols_arrays(f"W{w.dimension}", w.points, emb.n_original + w.dimension))
    out["witness_dims"] = np.array([w.dimension for w in wsets])
    out["stages"] = np.array([[s.candidate_dimension, s.against_dimension, s.candidates, s.degree,
                               s.paths_tracked, s.removed] for s in stages + st0]).reshape(-1, 6)
    out.update(sols_arrays("iso_regular", reg, emb.n_original))
    out.update(sols_arrays("iso_singular", sing, emb.n_original))
    out["nvars_top"] = np.array(nv)
    save("pipeline_c3m", **out)


def gen_membership_c3m():
    """Membership verdicts on the C3-mini component: on-component points from
    random slices (solved by the reference tracker), off-component points."""
    pd = configs.c3_mini()
    fixture = np.load(os.path.join(HERE, "pipeline_c3m.npz"))
    emb = ref_emb(pd.emb)
    n = emb.n_original
    W = fixture["W2_x"]
    wpts = [rt.Solution(x, 0.0, 1.0) for x in W]
    w = rf.WitnessSet(2, emb, wpts)
    hyper = configs.random_slices(n, 6, 77)
    onpts = []
    for hb in hyper:
        g = configs.component_slice_system(pd, hb)
        prob = configs.total_degree_problem("slice", g, 77)
        hh = rt.LinearHomotopy(ref_sys(prob.start), ref_sys(prob.target), prob.gamma)
        for x0 in systems.total_degree_starts(prob.degrees):
            r = rt.track(hh, x0)
            if r.succeeded:
                onpts.append(r.endpoint.coordinates)
    off = configs.membership_candidates_offcomponent(n, 12, 77)
    cands = np.concatenate([np.array(onpts), off, W[:2, :n]])
    verdict = []
    for q in cands:
        try:
            verdict.append(1 if rf.membership_test(w, q) else 0)
        except rf.MembershipIndeterminate:
            verdict.append(-1)
    print("membership verdicts", verdict)
    save("membership_c3m", witness=W, candidates=cands, verdict=np.array(verdict, np.int8),
         n_on=np.array(len(onpts)), slices=hyper)


def gen_refine():
    """The reference's own known-answer refinement cases (test_tracker.py:109-173)."""
    out = {}
    eq6 = rp.PolySystem(2, (rp.make_poly(2, [((2, 0), 1), ((1, 0), -3), ((0, 0), 2)]),
                            rp.make_poly(2, [((1, 2), 1), ((0, 2), -1)])))
    demo = rs.demo_system()
    cyc4 = rs.cyclic(4)
    rng = np.random.default_rng(5)
    cases = [
        ("demo_exact", demo, np.array([3, 2, 2, 1], complex), 1e-12, 10),
        ("demo_pert", demo, np.array([3, 2, 2, 1], complex) + 1e-4 * rng.normal(size=4), 1e-12, 10),
        ("cyc4_pert", cyc4, np.array([1, 1, -1, -1], complex) + 1e-4 * np.random.default_rng(2).normal(size=4),
         1e-12, 10),
        ("eq6_mult", eq6, np.array([2.0, 0.0], complex), 1e-12, 10),
        ("cyc4_far", cyc4, np.array([10.0, 10, 10, 10], complex), 1e-12, 2),
    ]
    for name, f, x, tol, it in cases:
        s = rt.newton_refine(f, x, tol, it)
        out[name + "_in"] = x
        out[name + "_x"] = s.coordinates
        out[name + "_res"] = np.array(s.residual)
        out[name + "_cond"] = np.array(s.condition)
        out[name + "_reg"] = np.array(s.regularity == "regular")
    x = np.array([2.0 + 1e-5, 1e-5], complex)
    out["eq6_dd_in"] = x
    out["eq6_dd_out"] = rt.refine_dd(eq6, x, steps=12)
    save("refine_golden", **out)


def gen_dd():
    from nidpipe.dd import CDD, DD
    gen = np.random.default_rng(7)
    a = gen.normal(size=(200, 4)) * np.array([1, 1e-17, 1, 1e-17])
    b = gen.normal(size=(200, 4)) * np.array([1, 1e-17, 1, 1e-17])
    outs = {"mul": [], "add": [], "div": []}
    for u, v in zip(a, b):
        A = CDD(DD(u[0], u[1]), DD(u[2], u[3]))
        B = CDD(DD(v[0], v[1]), DD(v[2], v[3]))
        for k, r in (("mul", A * B), ("add", A + B), ("div", A / B)):
            outs[k].append([r.re.hi, r.re.lo, r.im.hi, r.im.lo])
    save("dd_golden", a=a, b=b, **{k: np.array(v) for k, v in outs.items()})


def gen_dedup():
    gen = np.random.default_rng(11)
    base = gen.normal(size=(30, 5)) + 1j * gen.normal(size=(30, 5))
    pts, res = [], []
    for i, p in enumerate(base):
        for j in range(1 + i % 3):
            pts.append(p + (1e-9 if j else 0) * gen.normal(size=5))
            res.append(abs(gen.normal()) * 1e-12)
    pts = np.array(pts)
    sols = [rt.Solution(x, r, 1.0) for x, r in zip(pts, res)]
    kept = rf._dedup(sols)
    idx = [next(i for i, s in enumerate(sols) if s is k) for k in kept]
    save("dedup_golden", x=pts, res=np.array(res), kept=np.array(idx))


GENS = {"eval": gen_eval, "linalg": gen_linalg, "track_small": gen_track_small, "track_c5": gen_track_c5, "track_c5_large": gen_track_c5_large,
        "track_c3": gen_track_c3, "pipeline_c3m": gen_pipeline_c3m, "membership_c3m": gen_membership_c3m,
        "refine": gen_refine, "dd": gen_dd, "dedup": gen_dedup}

if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", nargs="*", default=list(GENS))
    args = ap.parse_args()
    for name in args.only:
        GENS[name]()
