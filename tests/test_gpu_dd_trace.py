"""Double-double tracking mode and the per-step trace hook on the GPU
(tracker.py:341-407, 458-497), against fixtures made by
the reference itself (tests/golden/make_dd_trace.py).

Exact: statuses, finite sets.  Endpoints within 1e-8 relative (1e-12 on the
double-double C1 endpoints: both sides polish in double-double).  Traces
(t, step, corrector iterations per accepted step) are discrete decisions of
the step controller: identical to the reference's on every C1 path and on
>= 90 % of the C2 sample (a corrector that converges in 2 vs 3 iterations on
a last-ulp difference of the Newton step shifts the schedule).
"""

import numpy as np
import pytest

from conftest import golden
from paper_1804_03807_b200 import configs, tracker
from paper_1804_03807_b200.homotopy import LinearHomotopy, TrackParams
from paper_1804_03807_b200.polys import PolySystem, make_poly

pytestmark = pytest.mark.gpu


def rel_rows(a, b):
    return np.max(np.abs(a - b), axis=-1) / np.maximum(1.0, np.max(np.abs(b), axis=-1))


def _traces_equal(got, ref_rows, n):
    if len(got) != n:
        return False
    a = np.array(got, float).reshape(-1, 3)
    return bool(np.all(a[:, 2] == ref_rows[:n, 2]) and np.allclose(a[:, :2], ref_rows[:n, :2], rtol=1e-13, atol=0))


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_trace_matches_reference(nid, name):
    g = golden("trace_c1")
    p = getattr(configs, name)()
    h = LinearHomotopy(p.start, p.target, p.gamma)
    res = tracker.track_batch(h, g[f"{name}_starts"], trace=True)
    st_ref = g[f"{name}_status"].astype(int)
    assert np.array_equal(res.status.astype(int), st_ref)
    fin = np.isin(st_ref, (0, 2))
    assert np.all(rel_rows(res.x[fin], g[f"{name}_x"][fin]) < 1e-8)
    same = [_traces_equal(res.traces[i], g[f"{name}_trace"][i], int(g[f"{name}_trace_n"][i]))
            for i in range(len(st_ref))]
    assert np.mean(same) >= (1.0 if name == "c1" else 0.9), same
    # an accepted step is a used step; the snap / finish steps are not traced
    assert all(len(t) <= s for t, s in zip(res.traces, res.steps))
    # untraced tracking of the same starts gives the same records
    plain = tracker.track_batch(h, g[f"{name}_starts"])
    assert np.array_equal(plain.status, res.status) and np.array_equal(plain.steps, res.steps)
    # (the traced run goes through the auxiliary kernel's factor-list evaluator, the
    # plain one through the parameter-bank evaluator: same arithmetic, other order)
    assert np.all(rel_rows(plain.x[fin], res.x[fin]) < 1e-12)


def test_track_single_path_appends_to_the_trace_list(nid):
    """track(h, x0, params, trace=list) (tracker.py:341-346)."""
    g = golden("trace_c1")
    p = configs.c1()
    h = LinearHomotopy(p.start, p.target, p.gamma)
    tr = [("kept", 0, 0)]
    r = tracker.track(h, g["c1_starts"][3], TrackParams(), trace=tr)
    assert r.status == "converged" and tr[0] == ("kept", 0, 0)
    assert _traces_equal(tr[1:], g["c1_trace"][3], int(g["c1_trace_n"][3]))
    assert 1.0 - tr[-1][0] <= 2e-8 and all(  # the last accepted step is within snap_remaining of t = 1
        isinstance(t[2], int) for t in tr[1:])


def test_double_double_mode_c1_c2(nid):
    """TrackParams(precision="double_double") (tracker.py:461-497): every
    evaluation in complex double-double, no noise floor, every endpoint
    polished in double-double."""
    g = golden("track_c1_dd")
    dd = TrackParams(precision="double_double")
    for name in ("c1", "c2"):
        p = getattr(configs, name)()
        h = LinearHomotopy(p.start, p.target, p.gamma)
        res = tracker.track_batch(h, g[f"{name}_starts"], dd)
        st_ref = g[f"{name}_status"].astype(int)
        fin = np.isin(st_ref, (0, 2))
        assert np.array_equal(res.succeeded, fin), (name, res.status, st_ref)
        assert np.mean(res.status.astype(int) == st_ref) >= 0.9
        assert np.all(rel_rows(res.x[fin], g[f"{name}_x"][fin]) < (1e-12 if name == "c1" else 1e-8))
        assert np.array_equal(res.regular[fin], g[f"{name}_regular"][fin])
        c = res.condition[fin] / g[f"{name}_condition"][fin]
        assert np.all((c > 0.99) & (c < 1.01))
        if name == "c1":
            assert np.all(np.abs(res.steps - g["c1_steps"]) <= 2)
            assert res.counters["dd_polished"] == 16  # the final polish always runs and is accepted here


def test_double_double_trace_c1(nid):
    g = golden("trace_c1")
    p = configs.c1()
    h = LinearHomotopy(p.start, p.target, p.gamma)
    res = tracker.track_batch(h, g["c1_starts"], TrackParams(precision="double_double"), trace=True)
    same = [_traces_equal(res.traces[i], g["c1dd_trace"][i], int(g["c1dd_trace_n"][i])) for i in range(16)]
    assert np.mean(same) >= 0.9, same


def test_double_double_small_linear_system(nid):
    """The reference's own dd test (tests/test_tracker.py:176-183): a linear
    2 x 2 homotopy tracked in double-double converges onto the direct solve."""
    def linear_system(rows, nv):
        polys = []
        for row in rows:
            terms = [((0,) * nv, row[0])]
            for j in range(nv):
                terms.append((tuple(1 if k == j else 0 for k in range(nv)), row[j + 1]))
            polys.append(make_poly(nv, terms))
        return PolySystem(nv, tuple(polys))

    gsys = linear_system([[1, 2, 1], [2, -1, 1]], 2)
    fsys = linear_system([[-3, 1, 4], [5, 2, -1]], 2)
    x0 = np.linalg.solve([[2, 1], [-1, 1]], [-1, -2])
    r = tracker.track(LinearHomotopy(gsys, fsys), x0, TrackParams(precision="double_double"))
    assert r.status == "converged"
    direct = np.linalg.solve([[1, 4], [2, -1]], [3, -5])
    assert np.max(np.abs(r.endpoint.coordinates - direct)) < 1e-10


def test_double_double_membership_parameters(nid):
    """Per-path target coefficients (membership homotopies) in dd mode:
    verdicts on the C3-mini candidates equal the double-precision verdicts."""
    from paper_1804_03807_b200 import filtering

    g = golden("membership_c3m")
    pd = configs.c3_mini()
    W = filtering.WitnessSet(pd.emb.k, pd.emb, [tracker.Solution(x, 0.0, 1.0) for x in g["witness"]])
    Q = g["candidates"][:8]
    v1, _ = filtering.membership_batch(W, Q)
    v2, _ = filtering.membership_batch(W, Q, params=TrackParams(precision="double_double"))
    assert np.array_equal(v1, v2)
    assert np.array_equal(v1 == 1, g["verdict"][:8].astype(bool))


def test_decompose_in_double_double(nid):
    """decompose(precision="dd") (blackbox.py:57-60: TrackParams(precision=
    "double_double") through every stage; the mixed cells of the polyhedral
    start are tracked in double, see polyhedral._cell_params) on the C3-mini
    system: the same witness-set degrees as the double-precision run, every
    start accounted for at every level, and isolated points that are all among
    the double-precision ones.  Counts are not equal to the double run's: without
    the evaluation-noise floor (tracker.py:177-181 through `_DDView`) a path
    whose coordinates grow cannot meet the fixed corrector tolerance and ends
    FAILED instead of at infinity (test_double_double_diverging_paths pins that
    to the reference), and a few finite paths are lost with them."""
    from paper_1804_03807_b200 import blackbox
    from test_polyhedral import _cells_from

    g = golden("decompose_c3m")
    pd = configs.c3_mini()
    cells = _cells_from(g, int(g["n"]), pd.emb.system)
    a = blackbox.decompose(pd.f, top_dimension=pd.emb.k, seed=pd.seed, cells=cells)
    b = blackbox.decompose(pd.f, top_dimension=pd.emb.k, seed=pd.seed, cells=cells, precision="dd")
    assert b.precision == "dd" and a.precision == "double"
    assert a.degrees == b.degrees == {2: 4}
    for c in b.cascade_counts:
        assert c["starts"] == c["at_infinity"] + c["zero_slack"] + c["nonzero_slack"] + c["failures"]
    assert b.cascade_counts[0]["starts"] == a.cascade_counts[0]["starts"] == 256
    assert 0.9 * len(a.isolated) <= len(b.isolated) <= len(a.isolated) == 80
    A = np.array([s.coordinates for s in a.isolated])
    B = np.array([s.coordinates for s in b.isolated])
    d = np.abs(A[:, None, :] - B[None, :, :]).max(axis=2)
    assert d.min(axis=0).max() < 1e-8  # every dd isolated point is a double-precision one


def test_double_double_diverging_paths(nid):
    """16 paths of the C3-mini top continuation tracked by the reference in
    double and in double-double (tests/golden/make_dd_c3m.py): finite sets equal
    in both modes, and the paths the reference fails in double-double (for lack
    of a noise floor) fail here too -- statuses agree on >= 14 of 16."""
    from paper_1804_03807_b200 import cascade

    g = golden("track_c3m_dd")
    pd = configs.c3_mini()
    h, _ = cascade.top_homotopy(pd.emb)
    for name, prm in (("double", TrackParams()), ("dd", TrackParams(precision="double_double"))):
        res = tracker.track_batch(h, g["starts"], prm)
        st = g[f"{name}_status"].astype(int)
        fin = np.isin(st, (0, 2))
        assert np.array_equal(res.succeeded, fin), (name, res.status, st)
        assert int(np.sum(res.status.astype(int) == st)) >= 14, (name, res.status, st)
        assert np.all(rel_rows(res.x[fin], g[f"{name}_x"][fin]) < 1e-8)
    # the two modes really differ on this sample
    assert np.sum(g["dd_status"] == 3) > np.sum(g["double_status"] == 3)
