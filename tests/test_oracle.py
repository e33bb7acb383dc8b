"""Pin the CPU oracle to the reference's own outputs (tests/golden, generated
by tests/golden/make_golden.py running nidpipe).  CPU only."""

import numpy as np
import pytest

from conftest import golden
from oracle import dd
from oracle import nid_oracle as O
from paper_1804_03807_b200 import configs, systems
from paper_1804_03807_b200.polys import PolySystem, make_poly

STATUS = {"converged": 0, "at_infinity": 1, "singular_endpoint": 2, "failed": 3}


def problems():
    return {p.name: p for p in (configs.c1(), configs.c2(), configs.c5(), configs.c3_top(configs.c3_mini()),
                                configs.c3_top(configs.c3()))}


@pytest.mark.parametrize("name", ["C1", "C2", "C5", "C3top"])
def test_oracle_eval_matches_reference(name):
    g = golden("eval_golden")
    probs = problems()
    # C3top appears twice in the fixture (mini and full); the full one was written last
    p = probs[name] if name != "C3top" else configs.c3_top(configs.c3())
    h = O.LinearHomotopy(p.start, p.target, p.gamma)
    X, T = g[name + "_x"], g[name + "_t"]
    for i, (x, t) in enumerate(zip(X, T)):
        H = h.eval(x, t)
        J = h.jac(x, t)
        s = h.eval_scale(x, t)
        assert np.max(np.abs(H - g[name + "_H"][i])) <= 1e-14 * max(1.0, s)
        assert np.max(np.abs(J - g[name + "_J"][i])) <= 1e-13 * max(1.0, np.max(np.abs(J)))
        assert abs(s - g[name + "_scale"][i]) <= 1e-14 * max(1.0, s)


@pytest.mark.parametrize("n", [2, 4, 7, 10, 14])
def test_oracle_linalg_matches_reference(n):
    g = golden("linalg_golden")
    J, r = g[f"n{n}_J"], g[f"n{n}_r"]
    for i in range(len(J)):
        dx = O.newton_step(J[i], r[i])
        ref = g[f"n{n}_dx"][i]
        assert np.allclose(dx, ref, rtol=1e-9, atol=1e-9 * np.max(np.abs(ref))), i
        c, k = O.condition_and_rank(J[i])
        assert k == g[f"n{n}_rank"][i]
        assert c == pytest.approx(g[f"n{n}_cond"][i], rel=1e-6)
    A = g["rect_A"]
    for i in range(len(A)):
        assert O.condition_and_rank(A[i])[1] == g["rect_rank"][i]


def test_oracle_dd_bit_exact():
    g = golden("dd_golden")
    for u, v, m, a, q in zip(g["a"], g["b"], g["mul"], g["add"], g["div"]):
        A, B = tuple(u), tuple(v)
        assert dd.c_mul(A, B) == tuple(m)
        assert dd.c_add(A, B) == tuple(a)
        assert dd.c_div(A, B) == tuple(q)


def eq6():
    return PolySystem(2, (make_poly(2, [((2, 0), 1), ((1, 0), -3), ((0, 0), 2)]),
                          make_poly(2, [((1, 2), 1), ((0, 2), -1)])))


def refine_cases():
    return {"demo_exact": (systems.demo_system(), 1e-12, 10), "demo_pert": (systems.demo_system(), 1e-12, 10),
            "cyc4_pert": (systems.cyclic(4), 1e-12, 10), "eq6_mult": (eq6(), 1e-12, 10),
            "cyc4_far": (systems.cyclic(4), 1e-12, 2)}


@pytest.mark.parametrize("name", list(refine_cases()))
def test_oracle_newton_refine(name):
    g = golden("refine_golden")
    f, tol, it = refine_cases()[name]
    s = O.newton_refine(f, g[name + "_in"], tol, it)
    assert np.allclose(s.coordinates, g[name + "_x"], atol=1e-12)
    assert s.residual <= max(10 * float(g[name + "_res"]), 1e-15)
    assert (s.regularity == "regular") == bool(g[name + "_reg"])


def test_oracle_refine_dd_multiple_point():
    g = golden("refine_golden")
    out = O.refine_dd(eq6(), g["eq6_dd_in"], steps=12)
    assert np.allclose(out, g["eq6_dd_out"], atol=1e-14)
    assert abs(out[0] - 2.0) < 1e-8 and abs(out[1]) < 1e-8


def check_track(prob, fixture, idx_subset):
    h = O.LinearHomotopy(prob.start, prob.target, prob.gamma)
    st = fixture["starts"]
    diffs = 0
    for i in idx_subset:
        r = O.track(h, st[i])
        assert STATUS[r.status] == fixture["status"][i] or (r.status in ("at_infinity", "failed") and
                                                          fixture["status"][i] in (1, 3)), i
        if r.endpoint is not None and fixture["status"][i] in (0, 2):
            diffs = max(diffs, np.max(np.abs(r.endpoint.coordinates - fixture["x"][i])) /
                        max(1.0, np.max(np.abs(fixture["x"][i]))))
    assert diffs < 1e-8


def test_oracle_track_c1_all_paths():
    f = golden("track_c1")
    assert int(np.sum(f["status"] == 0)) == 16
    check_track(configs.c1(), f, range(16))


def test_oracle_track_c2_subset():
    f = golden("track_c2")
    # the reference recovers 917 of the 924 (mixed volume) roots on this seed
    assert int(np.sum((f["status"] == 0) | (f["status"] == 2))) == 917
    rng = np.random.default_rng(0)
    conv = np.nonzero(f["status"] == 0)[0]
    idx = np.concatenate([rng.choice(conv, 12, replace=False), rng.choice(len(f["status"]), 12, replace=False)])
    check_track(configs.c2(), f, idx)


def test_oracle_track_c5_subset():
    f = golden("track_c5_sample")
    conv = np.nonzero(f["status"] == 0)[0]
    idx = np.concatenate([conv[:3], np.arange(6)])
    check_track(configs.c5(), f, idx)


def test_total_degree_starts_are_roots():
    p = configs.c5()
    X = systems.total_degree_starts(p.degrees, 123456, 64)
    for x in X:
        assert np.max(np.abs(O.eval_system(p.start, x))) < 1e-13


def test_oracle_dedup_matches_reference():
    g = golden("dedup_golden")
    sols = [O.Solution(x, r, 1.0) for x, r in zip(g["x"], g["res"])]
    kept, mult = O.dedup(sols)
    idx = [next(i for i, s in enumerate(sols) if s is k) for k in kept]
    assert idx == list(g["kept"])
    assert sum(mult) == len(sols)


def test_oracle_cascade_step_subset():
    """cascade_step on a subset of the reference's level-2 nonzero-slack
    points lands on the reference's level-1 points."""
    g = golden("pipeline_c3m")
    pd = configs.c3_mini()
    starts = [O.Solution(x, 0.0, 1.0, "regular", "nonzero_slack") for x in g["L2_nonzero_x"][:6]]
    lv = O.CascadeLevel(2, pd.emb, len(starts), 0, [], starts)
    nxt = O.cascade_step(lv)
    ref = np.concatenate([g["L1_zero_x"], g["L1_nonzero_x"]])
    for s in nxt.zero_slack + nxt.nonzero_slack:
        assert np.min(np.max(np.abs(ref - s.coordinates), axis=1)) < 1e-8


def test_oracle_membership_matches_reference_c4():
    """The oracle's membership test on C4 candidates decided by nidpipe itself
    (tests/golden/c4_hard.npz, c4_membership_ref.npz): the 10 hard
    candidates (stored verdicts, both decided from the same witness points)
    and two seeded candidates re-run here, one on the component and one off."""
    from paper_1804_03807_b200 import configs

    h = golden("c4_hard")
    assert np.array_equal(h["oracle_verdict"], h["reference_verdict"])
    g = golden("c4_membership_ref")
    pd = configs.c3()
    for i in (0, int(g["n_on"])):
        try:
            v = 1 if O.membership_test(list(g["witness"]), pd.emb, g["candidates"][i]) else 0
        except O.MembershipIndeterminate:
            v = -1
        assert v == g["verdict"][i], (i, v, g["verdict"][i])
