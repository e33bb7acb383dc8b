"""Per-cell polyhedral tracking: the reference's
`solve_cell` (polyhedral.py:794-811) on every fine mixed cell of the C1 and
C2 supports, pinned by tests/golden/polyhedral_{c1,c2}.npz (made by running
the reference, tests/golden/make_polyhedral.py).

CPU tests pin the oracle restatement (oracle/polyhedral.py) and the host-side
binomial start solver against the reference's outputs; GPU tests compare the
CUDA tracker (start_kind 2 of the C-ABI) with the same fixtures.  Bar:
statuses and finite counts exact per cell, endpoints matched as sets within
1e-8 relative, evaluation within 1e-13 of the oracle.
"""

import numpy as np
import pytest

from conftest import golden
from oracle import nid_oracle as O
from oracle import polyhedral as OP
from paper_1804_03807_b200 import polyhedral as PH
from paper_1804_03807_b200.polys import PolySystem, make_poly

STATUS = {"converged": 0, "at_infinity": 1, "singular_endpoint": 2, "failed": 3}


def load(name):
    g = golden(f"polyhedral_{name}")
    n = int(g["n"])
    off = g["row_off"]
    sup = g["support"]
    supports = tuple(tuple(tuple(int(v) for v in sup[k]) for k in range(off[i], off[i + 1])) for i in range(n))
    polys = tuple(make_poly(n, [(supports[i][j], g["coef"][off[i] + j]) for j in range(off[i + 1] - off[i])])
                  for i in range(n))
    gs = PolySystem(n, polys)
    cells = []
    for c in range(int(g["ncells"])):
        pr = g[f"c{c}_pairs"]
        tx = g[f"c{c}_texps"]
        cells.append(PH.Cell(tuple((tuple(map(int, pr[i, 0])), tuple(map(int, pr[i, 1]))) for i in range(n)),
                             tuple(tuple(tx[off[i]:off[i + 1]]) for i in range(n)), int(g[f"c{c}_volume"])))
    return g, gs, supports, cells


def match_sets(A, B, rel=1e-8):
    """Every row of A has a distinct partner in B within rel * max(1, |b|)."""
    A, B = np.asarray(A), np.asarray(B)
    assert len(A) == len(B)
    used = np.zeros(len(B), bool)
    for a in A:
        d = np.max(np.abs(B - a[None]), axis=1)
        d[used] = np.inf
        j = int(np.argmin(d))
        assert d[j] <= rel * max(1.0, np.max(np.abs(B[j]))), (a, B[j], d[j])
        used[j] = True


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_mixed_volume_and_cells(name):
    g, gs, supports, cells = load(name)
    assert sum(c.volume for c in cells) == {"c1": 16, "c2": 924}[name]
    assert PH.supports_of(gs) == supports


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_binomial_starts_match_reference(name):
    """Host solver and oracle against the reference's binomial_solutions."""
    g, gs, supports, cells = load(name)
    for c, cell in enumerate(cells):
        ref = g[f"c{c}_starts"]
        host = PH.cell_starts(cell, gs)
        assert host.shape == ref.shape == (cell.volume, gs.nvars)
        match_sets(host, ref, 1e-12)
        match_sets(np.array(OP.cell_starts(gs, cell.pairs)), ref, 1e-12)


def test_binomial_solutions_solve_the_system():
    V = [[3, 1, 0], [-2, 2, 1], [0, -1, 4]]
    beta = [0.3 + 1.1j, -2.0 + 0.5j, 0.7 - 0.2j]
    Y = PH.binomial_solutions(V, beta)
    assert len(Y) == abs(round(np.linalg.det(np.array(V, float))))
    for y in Y:
        for i in range(3):
            assert abs(np.prod(y ** np.array(V[i])) - beta[i]) <= 1e-12 * abs(beta[i])
    match_sets(Y, np.array(OP.binomial_solutions(V, beta)), 1e-12)


def test_rescaled_texps_and_lowering():
    g, gs, supports, cells = load("c2")
    cell = cells[0]
    w = PH.rescaled_texps(cell)
    raw = np.concatenate([np.asarray(t) for t in cell.texps])
    assert np.all(w[raw <= PH.SLACK_MARGIN] == 0.0)
    assert np.isclose(w[raw > PH.SLACK_MARGIN].min(), 1.0)
    np.testing.assert_array_equal(w, OP.rescale_texps(raw))
    low = PH.lower_polyhedral(gs, cell, supports)
    assert low.nterms == sum(len(s) for s in supports) and low.texp.shape == (low.nterms,)
    assert not np.any(low.cs) and low.start_degrees is None
    bad = PH.Cell(cell.pairs, (cell.texps[0][:-1],) + cell.texps[1:])
    with pytest.raises(ValueError):
        PH.lower_polyhedral(gs, bad, supports)


def test_oracle_solve_cell_matches_reference_c1():
    """Pins the oracle: its per-cell tracking reproduces the reference."""
    g, gs, supports, cells = load("c1")
    for c, cell in enumerate(cells):
        res = OP.solve_cell(gs, cell.pairs, np.concatenate([np.asarray(t) for t in cell.texps]), supports)
        st = np.array([STATUS[r.status] for r in res])
        assert np.array_equal(np.sort(st), np.sort(g[f"c{c}_status"]))
        ok = g[f"c{c}_status"] == 0
        match_sets(np.array([r.endpoint.coordinates for r in res if r.status == "converged"]), g[f"c{c}_x"][ok])


# ------------------------------------------------------------------ GPU


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["c1", "c2"])
def test_gpu_polyhedral_eval_matches_oracle(nid, name):
    g, gs, supports, cells = load(name)
    gen = np.random.default_rng(5)
    for cell in cells[:6]:
        h = PH.PolyhedralHomotopy(gs, cell, supports)
        ho = OP.PolyhedralHomotopy(gs, np.concatenate([np.asarray(t) for t in cell.texps]), supports)
        X = gen.normal(size=(5, gs.nvars)) + 1j * gen.normal(size=(5, gs.nvars))
        T = np.array([0.0, 0.01, 0.37, 0.9, 1.0])
        H, J, S = h.evaluate(X, T)
        for i in range(5):
            s = ho.eval_scale(X[i], T[i])
            assert abs(S[i] - s) <= 1e-13 * max(1.0, s)
            assert np.max(np.abs(H[i] - ho.eval(X[i], T[i]))) <= 1e-13 * max(1.0, s)
            Jo = ho.jac(X[i], T[i])
            assert np.max(np.abs(J[i] - Jo)) <= 1e-13 * max(1.0, np.max(np.abs(Jo)))


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["c1", "c2"])
def test_gpu_solve_cell_matches_reference(nid, name):
    g, gs, supports, cells = load(name)
    total = 0
    for c, cell in enumerate(cells):
        res = PH.solve_cell(cell, gs, supports)
        assert len(res) == cell.volume
        st = np.array([STATUS[r.status] for r in res])
        assert np.array_equal(np.sort(st), np.sort(g[f"c{c}_status"])), c
        ok = g[f"c{c}_status"] == 0
        X = np.array([r.endpoint.coordinates for r in res if r.status == "converged"]).reshape(-1, gs.nvars)
        match_sets(X, g[f"c{c}_x"][ok])
        total += int(ok.sum())
    assert total == {"c1": 16, "c2": 924}[name]


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["c1", "c2"])
def test_gpu_batched_cells_match_reference(nid, name):
    """All cells in one launch (nid_track_cells): per-cell parity with the
    reference, and every root solves g."""
    g, gs, supports, cells = load(name)
    res, counts = PH.track_cells(cells, gs, supports)
    assert counts == [c.volume for c in cells]
    pos = 0
    for c, k in enumerate(counts):
        st = res.status[pos:pos + k]
        assert np.array_equal(np.sort(st), np.sort(g[f"c{c}_status"])), c
        ok = g[f"c{c}_status"] == 0
        match_sets(res.x[pos:pos + k][st == 0], g[f"c{c}_x"][ok])
        pos += k
    X = res.x[res.status == 0]
    assert len(X) == {"c1": 16, "c2": 924}[name]
    for x in X[::7]:
        assert np.max(np.abs(O.eval_system(gs, x))) <= 1e-8
    assert len(PH.solve_cells(cells, gs, supports)) == sum(counts)


@pytest.mark.parametrize("name,seed", [("c1", 11), ("c2", 12)])
def test_random_coefficient_system_matches_reference(name, seed):
    """g from the START_COEFFS stream equals the reference's g (polyhedral.py:645-652)."""
    g, gs, supports, cells = load(name)
    mine = PH.random_coefficient_system(supports, gs.nvars, seed)
    for pa, pb in zip(mine.polys, gs.polys):
        assert [e for e, _ in pa.terms] == [e for e, _ in pb.terms]
        np.testing.assert_array_equal([c for _, c in pa.terms], [c for _, c in pb.terms])


def load_top(name):
    g = golden(f"polyhedral_top_{name}")
    n = int(g["n"])
    cells = []
    for c in range(int(g["ncells"])):
        pr = g[f"c{c}_pairs"]
        tx = g[f"c{c}_texps"]
        # split the concatenated t-exponents by each support's size (the
        # support of row i has len(cell.texps[i]) points)
        cells.append((pr, tx, int(g[f"c{c}_volume"])))
    return g, n, cells


@pytest.mark.gpu
@pytest.mark.parametrize("p", [1, 2])
def test_gpu_solve_top_polyhedral_matches_reference(nid, p):
    """solve_top with the reference's default polyhedral start on the C3-mini
    embedding (6 variables, 20 cells, mixed volume 256): cell counts, the
    continuation's finite / at-infinity / failed counts exact, finite
    endpoints matched as sets within 1e-8."""
    from paper_1804_03807_b200 import cascade, configs

    g, n, raw = load_top("c3m")
    pd = configs.c3_mini()
    system = pd.emb.system
    supports = PH.supports_of(system)
    sizes = [len(s) for s in supports]
    off = np.concatenate([[0], np.cumsum(sizes)])
    cells = [PH.Cell(tuple((tuple(map(int, pr[i, 0])), tuple(map(int, pr[i, 1]))) for i in range(n)),
                     tuple(tuple(tx[off[i]:off[i + 1]]) for i in range(n)), vol) for pr, tx, vol in raw]
    # p = 2: the cells stream through the producer -> GPU consumer pipeline
    res, stats = cascade.solve_top(pd.emb, p=p, cells=iter(cells), return_arrays=True)
    assert stats.cells == int(g["cells"]) and stats.mixed_volume == int(g["mixed_volume"])
    assert stats.start_failures == int(g["start_failures"])
    assert (stats.finite, stats.at_infinity, stats.failures) == (int(g["finite"]), int(g["at_infinity"]),
                                                                  int(g["failures"]))
    ref_ok = (g["top_status"] == 0) | (g["top_status"] == 2)
    match_sets(res.x[res.succeeded], g["top_x"][ref_ok])


# ------------------------------------------------------------- pipeline


class _FakeResults:
    def __init__(self, rows):
        self.rows = rows

    def path_results(self):
        return self.rows


def _fake_track(delay=0.0, fail_on=None):
    calls = []

    def track(cells, g, supports, params):
        import time

        calls.append(len(cells))
        if fail_on is not None and any(c == fail_on for c in cells):
            raise ValueError("boom")
        time.sleep(delay)
        rows = [(c, j) for c in cells for j in range(c % 3 + 1)]
        return _FakeResults(rows), [c % 3 + 1 for c in cells]

    return track, calls


def test_pipeline_keeps_cell_order_and_batches():
    import time

    def slow_cells():
        for c in range(40):
            time.sleep(0.002)
            yield c

    track, calls = _fake_track(delay=0.01)
    res, counts, st = PH.pipeline_cells(slow_cells(), None, (), track=track, queue_capacity=4)
    assert counts == [c % 3 + 1 for c in range(40)]
    assert res == [(c, j) for c in range(40) for j in range(c % 3 + 1)]
    assert st.produced == st.consumed == 40 and sum(calls) == 40 and st.batches == len(calls)
    assert st.first_consume_before_last_produce and st.producer_error is None


def test_pipeline_producer_error_is_reported_and_drained():
    def bad_cells():
        yield 1
        yield 2
        raise RuntimeError("lp failed")

    track, _ = _fake_track()
    res, counts, st = PH.pipeline_cells(bad_cells(), None, (), track=track)
    assert st.produced == 2 and st.consumed == 2 and counts == [2, 3]
    assert "lp failed" in st.producer_error


def test_pipeline_consumer_error_raises():
    track, _ = _fake_track(fail_on=5)
    with pytest.raises(RuntimeError, match="GPU consumer failed"):
        PH.pipeline_cells(iter(range(200)), None, (), track=track, queue_capacity=2, max_batch_cells=1)


@pytest.mark.gpu
def test_gpu_pipeline_matches_reference_c2(nid):
    """C2's 115 cells streamed by a producer thread (with the pauses of a
    CPU enumeration) through the GPU consumer: per-cell parity."""
    import time

    g, gs, supports, cells = load("c2")

    def producer():
        for c in cells:
            time.sleep(0.001)
            yield c

    res, counts, st = PH.pipeline_cells(producer(), gs, supports, queue_capacity=16)
    assert counts == [c.volume for c in cells] and st.consumed == len(cells) and st.batches >= 2
    pos = 0
    for c, k in enumerate(counts):
        st_c = np.array([STATUS[r.status] for r in res[pos:pos + k]])
        assert np.array_equal(np.sort(st_c), np.sort(g[f"c{c}_status"])), c
        ok = g[f"c{c}_status"] == 0
        match_sets(np.array([r.endpoint.coordinates for r in res[pos:pos + k] if r.status == "converged"]),
                   g[f"c{c}_x"][ok])
        pos += k


# ------------------------------------------------------------- decompose


def _cells_from(g, n, system):
    supports = PH.supports_of(system)
    off = np.concatenate([[0], np.cumsum([len(s) for s in supports])])
    cells = []
    for c in range(int(g["ncells"])):
        pr = g[f"c{c}_pairs"]
        tx = g[f"c{c}_texps"]
        cells.append(PH.Cell(tuple((tuple(map(int, pr[i, 0])), tuple(map(int, pr[i, 1]))) for i in range(n)),
                             tuple(tuple(tx[off[i]:off[i + 1]]) for i in range(n)), int(g[f"c{c}_volume"])))
    return cells


def test_decompose_argument_checks():
    from paper_1804_03807_b200 import blackbox, configs

    f = configs.c3_mini().f
    with pytest.raises(ValueError):
        blackbox.decompose(f, top_dimension=f.nvars, cells=[])
    with pytest.raises(ValueError):
        blackbox.decompose(f, top_dimension=2, precision="quad", cells=[])
    with pytest.raises(ValueError):
        blackbox.decompose(f, top_dimension=2, mode="fpga", cells=[])
    nonsquare = PolySystem(f.nvars, f.polys[:-1])
    with pytest.raises(ValueError):
        blackbox.decompose(nonsquare, top_dimension=2, cells=[])


@pytest.mark.gpu
def test_gpu_decompose_matches_reference_c3m(nid):
    """decompose(mode="gpu") from the polyhedral start (the reference's cell
    log) on the C3-mini base system against the reference's own decompose:
    witness-set degrees, cascade counts, filter stages and isolated points."""
    from paper_1804_03807_b200 import blackbox, configs

    g = golden("decompose_c3m")
    pd = configs.c3_mini()
    cells = _cells_from(g, int(g["n"]), pd.emb.system)
    rep = blackbox.decompose(pd.f, top_dimension=pd.emb.k, seed=pd.seed, cells=cells)
    assert sorted(rep.degrees.items()) == [tuple(r) for r in g["degrees"].tolist()]
    keys = ("dimension", "starts", "at_infinity", "zero_slack", "nonzero_slack", "failures")
    assert [[c[k] for k in keys] for c in rep.cascade_counts] == g["cascade"].tolist()
    # stage shapes exact; junk removal checked as in test_gpu_pipeline.py: the
    # junk candidates lie on a positive-dimensional set, so where a cascade
    # path lands on it depends on rounding history -- every GPU verdict must
    # equal the CPU oracle's verdict on the same candidate
    assert [[s.candidate_dimension, s.against_dimension, s.candidates]
            for s in rep.filter_stages] == [r[:3] for r in g["stages"].tolist()]
    from paper_1804_03807_b200 import filtering

    n = pd.emb.n_original
    wpts = [s.coordinates for s in rep.witness_sets[0].points]
    for st in rep.filter_stages:
        if st.candidate_dimension == 0:
            continue
        lv = [lv for lv in rep.superset.levels if lv.dimension == st.candidate_dimension][0]
        Q = [c.coordinates[:n] for c in filtering._dedup(list(lv.zero_slack), n)]
        assert st.removed == sum(O.membership_test(wpts, pd.emb, q) for q in Q)
    ref0 = [r for r in g["stages"].tolist() if r[0] == 0]
    assert [[s.candidate_dimension, s.against_dimension, s.candidates, s.removed]
            for s in rep.filter_stages if s.candidate_dimension == 0] == ref0
    assert len(rep.suspects) == int(g["suspects"])
    iso = np.array([s.coordinates for s in rep.isolated]).reshape(-1, pd.f.nvars)
    match_sets(iso, g["isolated"])


# ------------------------------------------------------------- edge cases


@pytest.mark.gpu
def test_gpu_polyhedral_univariate_cell(nid):
    """n = 1: g = a x^3 + b, one cell (volume 3) whose binomial system is g
    itself -- the three roots of g, each converged."""
    a, b = 0.6 - 0.8j, -1.3 + 0.4j
    g = PolySystem(1, (make_poly(1, [((0,), b), ((3,), a)]),))
    supports = PH.supports_of(g)
    cell = PH.Cell((((0,), (3,)),), ((0.0, 0.0),), 3)
    res = PH.solve_cell(cell, g, supports)
    roots = np.roots([a, 0, 0, b])
    X = np.array([r.endpoint.coordinates for r in res if r.status == "converged"])
    assert len(X) == 3
    match_sets(X, roots.reshape(-1, 1), 1e-12)


@pytest.mark.gpu
def test_gpu_polyhedral_argument_errors(nid):
    from paper_1804_03807_b200 import _lib
    from paper_1804_03807_b200.homotopy import LinearHomotopy

    g, gs, supports, cells = load("c1")
    with pytest.raises(ValueError):
        PH.track_cells([], gs, supports)
    low = PH.lower_polyhedral(gs, cells[0], supports)
    bad = type(low)(**{**low.__dict__, "texp": -np.ones_like(low.texp)})
    with pytest.raises(_lib.NidError, match="term_texp"):
        PH.DeviceHomotopy(bad)
    # a linear homotopy handle refuses per-cell t-exponent rows
    h = LinearHomotopy(gs, gs, 1.0 + 0j)
    import ctypes as C

    L = _lib.lib()
    st = np.zeros((1, gs.nvars), np.complex128)
    tw = np.zeros((1, low.nterms))
    out = np.zeros((1, gs.nvars), np.complex128)
    o = _lib.PathOutC(_lib.ptr(out), *[None] * 6)
    rc = L.nid_track_cells(h.device().handle, C.byref(PH.TrackParams().to_c()), 1, _lib.ptr(st), _lib.ptr(tw),
                           C.byref(o), 0, None)
    assert rc != 0 and b"polyhedral" in L.nid_last_error()
