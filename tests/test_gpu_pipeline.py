"""The stage drivers on the GPU vs the reference's run on the n=4 analog of C3
(tests/golden/pipeline_c3m.npz): top continuation, cascade, junk filter,
isolated-point classification, membership verdicts, dedup (B200 only)."""

import numpy as np
import pytest

from conftest import golden
from oracle import nid_oracle as O
from paper_1804_03807_b200 import cascade, configs, filtering, tracker
from paper_1804_03807_b200.tracker import Solution

pytestmark = pytest.mark.gpu


def set_match(A, B, tol=1e-8):
    """every row of A matches a distinct row of B within tol (relative)"""
    A = np.asarray(A)
    B = np.asarray(B)
    assert A.shape == B.shape, (A.shape, B.shape)
    used = np.zeros(len(B), bool)
    for a in A:
        d = np.max(np.abs(B - a), axis=1) / max(1.0, np.max(np.abs(a)))
        d[used] = np.inf
        j = int(np.argmin(d))
        assert d[j] < tol, d[j]
        used[j] = True


@pytest.fixture(scope="module")
def pipeline(nid):
    pd = configs.c3_mini()
    top, stats = cascade.solve_top(pd.emb, return_arrays=True)
    sup = cascade.run_cascade(top, pd.emb)
    wsets, stages = filtering.filter_junk(sup)
    iso = filtering.classify_isolated(sup.candidates(0), wsets, pd.emb.base)
    return pd, top, stats, sup, wsets, stages, iso


def test_top_continuation_matches_reference(pipeline):
    _, top, stats, *_ = pipeline
    g = golden("pipeline_c3m")
    assert stats.finite == int(np.sum(np.isin(g["top_status"], (0, 2))))
    assert np.mean(top.status == g["top_status"]) >= 0.99
    fin = top.succeeded
    set_match(top.x[fin], g["top_x"][np.isin(g["top_status"], (0, 2))])


def regular_rows(sols):
    return np.array([s.coordinates for s in sols if s.condition < 1e8])


def test_cascade_levels_match_reference(pipeline):
    """Counts per level exact; regular points (isolated solutions of the
    level's embedding) as sets within 1e-8.  Singular zero-slack points lie
    on higher-dimensional components (junk): where on that set a path lands
    depends on its rounding history, so only their count is pinned."""
    _, _, _, sup, *_ = pipeline
    g = golden("pipeline_c3m")
    for lv in sup.levels:
        d = lv.dimension
        ref = g[f"L{d}_counts"]
        got = [lv.starts, lv.at_infinity, len(lv.zero_slack), len(lv.nonzero_slack), lv.failures]
        assert got == list(ref), (d, got, list(ref))
        for kind, pts in (("zero", lv.zero_slack), ("nonzero", lv.nonzero_slack)):
            if not pts:
                continue
            mine = regular_rows(pts)
            refx = g[f"L{d}_{kind}_x"][g[f"L{d}_{kind}_cond"] < 1e8]
            assert abs(len(mine) - len(refx)) <= max(1, len(refx) // 50), (d, kind, len(mine), len(refx))
            for x in mine:
                dist = np.max(np.abs(g[f"L{d}_{kind}_x"] - x), axis=1) / max(1.0, np.max(np.abs(x)))
                assert dist.min() < 1e-8, (d, kind, dist.min())


def test_filter_junk_matches_reference(pipeline):
    """Same witness sets as the reference; every membership verdict equals the
    oracle's verdict on the same candidate (the junk candidates themselves come
    from this run's cascade)."""
    pd, _, _, sup, wsets, stages, _ = pipeline
    g = golden("pipeline_c3m")
    assert [w.dimension for w in wsets] == list(g["witness_dims"])
    assert [w.degree for w in wsets] == [len(g[f"W{d}_x"]) for d in g["witness_dims"]]
    for w in wsets:
        set_match([s.coordinates for s in w.points], g[f"W{w.dimension}_x"])
    n = pd.emb.n_original
    w = wsets[0]
    cands = filtering._dedup(list(sup.levels[1].zero_slack), n)
    Q = np.array([c.coordinates[:n] for c in cands])
    verdict, _ = filtering.membership_batch(w, Q)
    wpts = [s.coordinates for s in w.points]
    ref_v = [O.membership_test(wpts, pd.emb, q) for q in Q]
    assert list(verdict.astype(bool)) == ref_v
    got = [(s.candidate_dimension, s.against_dimension, s.candidates, s.degree, s.paths_tracked)
           for s in stages]
    ref_stages = [tuple(r[:5]) for r in g["stages"] if r[0] != 0]
    assert got == ref_stages
    assert stages[0].removed == int(sum(ref_v))


def test_classify_isolated_matches_reference(pipeline):
    *_, iso = pipeline
    g = golden("pipeline_c3m")
    regular, singular, st0 = iso
    assert len(regular) == len(g["iso_regular_x"])
    set_match([s.coordinates for s in regular], g["iso_regular_x"])
    assert len(singular) == len(g["iso_singular_x"])


def test_membership_verdicts_match_reference(nid):
    g = golden("membership_c3m")
    pd = configs.c3_mini()
    w = filtering.WitnessSet(2, pd.emb, [Solution(x, 0.0, 1.0) for x in g["witness"]])
    verdict, tracked = filtering.membership_batch(w, g["candidates"])
    assert list(verdict) == list(g["verdict"])
    for q, v in zip(g["candidates"][:3], g["verdict"][:3]):
        assert filtering.membership_test(w, q) == bool(v)


def test_dedup_matches_reference(nid):
    g = golden("dedup_golden")
    sols = [Solution(x, r, 1.0) for x, r in zip(g["x"], g["res"])]
    kept, mult = filtering.dedup(sols)
    idx = [next(i for i, s in enumerate(sols) if s is k) for k in kept]
    assert idx == list(g["kept"])
    assert sum(mult) == len(sols) and max(mult) == 3
