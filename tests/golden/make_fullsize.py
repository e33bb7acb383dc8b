"""Full-size parity fixtures decided by the REFERENCE (nidpipe) itself.

Runs only in the build container, where the reference is importable (long:
hours of CPU on 7 processes; every phase checkpoints to scratch/fullsize/ so
an interrupted run resumes):

    PYTHONPATH=/root/reference/pkg/src:. python tests/golden/make_fullsize.py [--only c4 c3 c5] [--c5-chunks K]

* c5: a seeded uniform sample of C5 paths (chunks of 16,384 indices drawn
  from default_rng(8) over the 3,628,800 total-degree paths), tracked by
  `nidpipe.tracker.track` through `work_crew(mode="process")`.  Stored:
  index, status, steps for every path; endpoints and regularity of the finite
  ones.  -> tests/golden/track_c5_full_sample.npz
* c3: a 2,048-path seeded sample of the C3 top continuation, the reference's
  `_classify_level` of it, then a chain of `cascade_step` calls d = 6 .. 1,
  each from (at most) 256 of the previous level's nonzero-slack solutions
  (cascade.py:249-322).  Stored per level: the input starts, the counts and
  the zero/nonzero-slack endpoints.  -> tests/golden/c3_cascade_chain.npz
* c4: `nidpipe.filtering.membership_test` (filtering.py:92-127) on the C3
  witness set (the 4 witness points recorded in c4_hard.npz) for 200
  on-component candidates (50 random 2-dim slices of {h1 = h2 = 0}, solved
  by the reference tracker), 200 off-component candidates, and the C4 hard
  candidates of c4_hard.npz.  -> tests/golden/c4_membership_ref.npz
"""

from __future__ import annotations

import argparse
import multiprocessing as mp
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)

import nidpipe.cascade as rc  # noqa: E402
import nidpipe.filtering as rf  # noqa: E402
import nidpipe.tracker as rt  # noqa: E402
from nidpipe.parallel import work_crew  # noqa: E402

from make_golden import STATUS, pack_results, ref_emb, ref_sys, save  # noqa: E402
from paper_1804_03807_b200 import configs, systems  # noqa: E402

PROCS = int(os.environ.get("GOLDEN_PROCS", "7"))
SCRATCH = os.path.join(ROOT, "scratch", "fullsize")
C5_CHUNK = 16384


def log(*a):
    print(time.strftime("%H:%M:%S"), *a, flush=True)


# ----------------------------------------------------------------------------- C5

def c5_sample_index(chunks: int) -> np.ndarray:
    """Chunk c is the c-th block of 16,384 draws of a fixed permutation
    prefix, so a longer run extends a shorter one."""
    p5 = configs.c5()
    perm = np.random.default_rng(8).choice(p5.paths, size=64 * C5_CHUNK, replace=False)
    return perm[: chunks * C5_CHUNK]


def gen_c5(chunks: int):
    p5 = configs.c5()
    h = rt.LinearHomotopy(ref_sys(p5.start), ref_sys(p5.target), p5.gamma)
    idx_all = c5_sample_index(chunks)
    os.makedirs(SCRATCH, exist_ok=True)
    parts = []
    for c in range(chunks):
        path = os.path.join(SCRATCH, f"c5_chunk{c:02d}.npz")
        idx = idx_all[c * C5_CHUNK:(c + 1) * C5_CHUNK]
        if not os.path.exists(path):
            starts = np.concatenate([systems.total_degree_starts(p5.degrees, int(i), 1) for i in idx])
            t0 = time.time()
            res = work_crew(list(starts), PROCS, lambda x0: rt.track(h, x0), mode="process")
            d = pack_results(res, p5.n)
            np.savez_compressed(path, index=idx, **d)
            fin = int(np.isin(d["status"], (0, 2)).sum())
            log(f"C5 chunk {c}: {len(idx)} paths in {time.time() - t0:.0f}s, finite {fin}")
        parts.append(np.load(path))
    index = np.concatenate([p["index"] for p in parts])
    status = np.concatenate([p["status"] for p in parts])
    steps = np.concatenate([p["steps"] for p in parts]).astype(np.int16)
    x = np.concatenate([p["x"] for p in parts])
    reg = np.concatenate([p["regular"] for p in parts])
    fin = np.isin(status, (0, 2))
    order = np.argsort(index, kind="stable")
    fin_o = fin[order]
    save("track_c5_full_sample", index=index[order], status=status[order], steps=steps[order],
         fin_x=x[order][fin_o], fin_regular=reg[order][fin_o])
    log("C5 sample", len(index), "finite", int(fin.sum()))


# ----------------------------------------------------------------------------- C3

def sols(prefix, lst, n):
    d = {f"{prefix}_x": np.array([s.coordinates for s in lst], np.complex128).reshape(len(lst), n),
         f"{prefix}_res": np.array([s.residual for s in lst]),
         f"{prefix}_cond": np.array([s.condition for s in lst]),
         f"{prefix}_reg": np.array([s.regularity == "regular" for s in lst], bool)}
    return d


def gen_c3(top_paths: int = 2048, per_level: int = 256):
    pd = configs.c3()
    prob = configs.c3_top(pd)
    emb = ref_emb(pd.emb)
    os.makedirs(SCRATCH, exist_ok=True)
    top_path = os.path.join(SCRATCH, "c3_top.npz")
    idx = np.sort(np.random.default_rng(9).choice(prob.paths, size=top_paths, replace=False))
    starts = np.concatenate([systems.total_degree_starts(prob.degrees, int(i), 1) for i in idx])
    h = rt.LinearHomotopy(ref_sys(prob.start), ref_sys(prob.target), prob.gamma)
    if not os.path.exists(top_path):
        t0 = time.time()
        res = work_crew(list(starts), PROCS, lambda x0: rt.track(h, x0), mode="process")
        np.savez_compressed(top_path, index=idx, starts=starts, **pack_results(res, prob.n))
        log(f"C3 top: {len(idx)} paths in {time.time() - t0:.0f}s")
    top = np.load(top_path)
    inv = {v: k for k, v in STATUS.items()}
    results = []
    for i in range(len(idx)):
        st = inv[int(top["status"][i])]
        ep = None
        if st in ("converged", "singular_endpoint"):
            ep = rt.Solution(top["x"][i], float(top["residual"][i]), float(top["condition"][i]))
        results.append(rt.PathResult(st, ep, int(top["steps"][i]), float(top["t_reached"][i])))
    t0 = time.time()
    level = rc._classify_level(results, emb, emb.k, rt.TrackParams())
    log(f"C3 top classify {level.starts}/{level.at_infinity}/{len(level.zero_slack)}/"
        f"{len(level.nonzero_slack)}/{level.failures} in {time.time() - t0:.0f}s")
    out = {f"top_{k}": top[k] for k in ("index", "starts", "status", "steps", "x", "residual", "condition", "regular")}
    out["top_counts"] = np.array([level.starts, level.at_infinity, len(level.zero_slack), len(level.nonzero_slack),
                                  level.failures])
    nv = emb.n_original + level.dimension
    out.update(sols("top_zero", level.zero_slack, nv))
    out.update(sols("top_nonzero", level.nonzero_slack, nv))
    sel_gen = np.random.default_rng(10)
    while level.dimension > 0:
        d = level.dimension
        nz = level.nonzero_slack
        if len(nz) > per_level:
            keep = np.sort(sel_gen.choice(len(nz), per_level, replace=False))
            nz = [nz[i] for i in keep]
        inp = rc.CascadeLevel(d, level.embedding, starts=level.starts, at_infinity=level.at_infinity,
                              zero_slack=level.zero_slack, nonzero_slack=nz, failures=level.failures)
        out.update(sols(f"in{d}", nz, emb.n_original + d))
        t0 = time.time()
        level = rc.cascade_step(inp, PROCS, rt.TrackParams(), "process")
        nv = emb.n_original + level.dimension
        out[f"out{d}_counts"] = np.array([level.starts, level.at_infinity, len(level.zero_slack),
                                          len(level.nonzero_slack), level.failures])
        out.update(sols(f"out{d}_zero", level.zero_slack, nv))
        out.update(sols(f"out{d}_nonzero", level.nonzero_slack, nv))
        log(f"C3 cascade_step d={d}: {out[f'out{d}_counts'].tolist()} in {time.time() - t0:.0f}s")
        np.savez_compressed(os.path.join(SCRATCH, "c3_chain_partial.npz"), **out)
    save("c3_cascade_chain", **out)


# ----------------------------------------------------------------------------- C4

_W = None


def _decide(q):
    try:
        return 1 if rf.membership_test(_W, q, 1, rt.TrackParams(), "thread") else 0
    except rf.MembershipIndeterminate:
        return -1


def _slice_points(hb):
    pd = configs.c3()
    g = configs.component_slice_system(pd, hb)
    prob = configs.total_degree_problem("slice", g, 45)
    hh = rt.LinearHomotopy(ref_sys(prob.start), ref_sys(prob.target), prob.gamma)
    pts = []
    for x0 in systems.total_degree_starts(prob.degrees):
        r = rt.track(hh, x0)
        if r.succeeded:
            pts.append(r.endpoint.coordinates)
    return pts


def gen_c4(n_slices: int = 50, n_off: int = 200):
    global _W
    pd = configs.c3()
    emb = ref_emb(pd.emb)
    n = emb.n_original
    hard = np.load(os.path.join(HERE, "c4_hard.npz"))
    W = hard["witness"]
    _W = rf.WitnessSet(pd.emb.k, emb, [rt.Solution(x, 0.0, 1.0) for x in W])
    hyper = configs.random_slices(n, n_slices, 45)
    t0 = time.time()
    ctx = mp.get_context("fork")
    with ctx.Pool(PROCS) as pool:
        on = [p for pts in pool.map(_slice_points, list(hyper)) for p in pts]
    log(f"C4 on-component points {len(on)} in {time.time() - t0:.0f}s")
    off = configs.membership_candidates_offcomponent(n, n_off, 45)
    cands = np.concatenate([np.array(on), off, hard["candidates"]])
    labels = np.concatenate([np.ones(len(on), np.int8), np.zeros(n_off, np.int8), hard["labels"].astype(np.int8)])
    t0 = time.time()
    with ctx.Pool(PROCS) as pool:
        verdict = np.array(pool.map(_decide, list(cands), chunksize=1), np.int8)
    log(f"C4 {len(cands)} membership tests in {time.time() - t0:.0f}s; "
        f"disagree with labels: {int(np.sum((verdict == 1) != (labels == 1)))}")
    save("c4_membership_ref", witness=W, candidates=cands, labels=labels, verdict=verdict,
         n_on=np.array(len(on)), n_hard=np.array(len(hard["candidates"])), slices=hyper)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", nargs="*", default=["c4", "c3", "c5"])
    ap.add_argument("--c5-chunks", type=int, default=8)
    a = ap.parse_args()
    for name in a.only:
        {"c4": gen_c4, "c3": gen_c3, "c5": lambda: gen_c5(a.c5_chunks)}[name]()
