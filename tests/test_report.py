"""Report / text-format adjacency: the deterministic
JSON report (report.py:81-128), the text summary (:131-170) and the plain
text system format (polytext.py:111-160).

Fixtures are the reference's own outputs (tests/golden/make_polyhedral.py
writes report_c3m.json / summary_c3m.txt from nidpipe's decompose of the
C3-mini base system; tests/golden/make_polytext.py runs nidpipe.polytext).
CPU: the serialiser reproduces the reference's bytes from the same records;
the parser returns the same terms, bit for bit, and refuses the same inputs.
GPU: decompose(mode="gpu") serialises to the reference's report on every
seed-stable field, points within 1e-8.
"""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, golden
from paper_1804_03807_b200 import polytext, refbridge
from paper_1804_03807_b200 import report as R


def _ref_json():
    with open(os.path.join(GOLDEN, "report_c3m.json"), encoding="utf-8") as fh:
        return fh.read()


def test_report_json_is_byte_identical_to_the_reference():
    """Rebuilding the records of the reference's report and serialising them
    here gives the reference's file, byte for byte (key order, canonical
    point order, float repr, indent, trailing newline)."""
    txt = _ref_json()
    rep = R.report_from_jsonable(json.loads(txt))
    assert R.report_to_json(rep) == txt
    # canonical order does not depend on the order the points arrive in
    rep.isolated.reverse()
    rep.witness_sets[0].points.reverse()
    assert R.report_to_json(rep) == txt
    assert rep.degrees == {2: 4}


def test_summary_text_matches_the_reference():
    rep = R.report_from_jsonable(json.loads(_ref_json()))
    with open(os.path.join(GOLDEN, "summary_c3m.txt"), encoding="utf-8") as fh:
        want = fh.read()
    got = R.summary_text(rep)
    assert got.split("timings:")[0] == want
    rows = got.split("timings:\n")[1].splitlines()
    assert [r.split("  ")[0].strip() for r in rows] == ["start system", "continuation", "top total", "cascade",
                                                         "filter", "grand total"]


def test_timings_totals():
    t = R.Timings(1.0, 2.0, 3.0, 4.0)
    assert t.top_total == 3.0 and t.grand_total == 10.0
    assert t.table().splitlines()[-1] == "grand total " + "  " + "    10.000" + " s"  # name:<12, sec:10.3f


def test_polytext_matches_the_reference_parser():
    with open(os.path.join(GOLDEN, "polytext_cases.json"), encoding="utf-8") as fh:
        cases = json.load(fh)
    assert sum(1 for c in cases if "error" in c) >= 10
    for c in cases:
        if "error" in c:
            with pytest.raises(polytext.ParseError):
                polytext.parse_system(c["text"])
            continue
        f = polytext.parse_system(c["text"])
        assert f.nvars == c["nvars"]
        got = [[[list(e), [repr(z.real), repr(z.imag)]] for e, z in p.terms] for p in f.polys]
        assert got == c["polys"], c["text"]
        assert polytext.format_system(f) == c["formatted"]


def test_polytext_round_trip_c1(tmp_path):
    """format -> parse reproduces every coefficient to the last ulp, and the
    printed C1 system equals the reference's print of it."""
    from paper_1804_03807_b200 import configs

    f = configs.c1().target
    with open(os.path.join(GOLDEN, "polytext_c1.txt"), encoding="utf-8") as fh:
        want = fh.read()
    assert polytext.format_system(f) == want
    g = polytext.parse_system(want)
    assert [p.terms for p in g.polys] == [p.terms for p in f.polys]
    path = tmp_path / "c1.txt"
    polytext.save_system(f, path)
    assert [p.terms for p in polytext.load_system(path).polys] == [p.terms for p in f.polys]


def test_mode_strings():
    """mode="gpu" runs here, "thread"/"process" are the reference's work crew
    (delegated), anything else is refused as in parallel.py:109."""
    assert refbridge.check_mode("gpu") is True
    assert refbridge.check_mode("thread") is False and refbridge.check_mode("process") is False
    with pytest.raises(ValueError):
        refbridge.check_mode("cuda")
    from paper_1804_03807_b200 import cascade, configs

    with pytest.raises(ValueError):
        cascade.solve_top(configs.c3_mini().emb, mode="fpga")


def test_cpu_modes_delegate_to_the_reference_when_importable():
    """With nidpipe importable (the build container), mode="thread" runs the
    reference's own driver on converted inputs and returns its records."""
    pytest.importorskip("nidpipe")
    from paper_1804_03807_b200 import cascade, configs, filtering
    from paper_1804_03807_b200.tracker import Solution

    pd = configs.c3_mini()
    g = golden("pipeline_c3m")
    # one cascade step from two of the reference's own nonzero-slack solutions
    keys = [k for k in g.files if k.endswith("nonzero_x")]
    assert keys
    X = g[keys[0]][:2]
    d = X.shape[1] - pd.emb.n_original
    lv = cascade.CascadeLevel(d, pd.emb.level(d), starts=len(X), at_infinity=0,
                              nonzero_slack=[Solution(x, 0.0, 1.0) for x in X])
    nxt = cascade.cascade_step(lv, 1, mode="thread")
    assert type(nxt).__module__.startswith("nidpipe.")
    assert nxt.dimension == d - 1 and nxt.starts == 2
    with pytest.raises(ValueError):
        filtering.membership_test(filtering.WitnessSet(d, pd.emb.level(d), []), np.zeros(3), mode="thread")


@pytest.mark.gpu
def test_gpu_decompose_report_matches_reference_json(nid):
    """decompose(mode="gpu") from the reference's cell log: its JSON report
    equals the reference's on every field except the point coordinates
    (within 1e-8, same canonical order up to ties) and the junk-removal count
    of the dimension-1 stage, which is pinned to the oracle in
    test_gpu_decompose_matches_reference_c3m."""
    from paper_1804_03807_b200 import blackbox, configs
    from test_polyhedral import _cells_from

    g = golden("decompose_c3m")
    pd = configs.c3_mini()
    cells = _cells_from(g, int(g["n"]), pd.emb.system)
    rep = blackbox.decompose(pd.f, top_dimension=pd.emb.k, seed=pd.seed, cells=cells)
    got = json.loads(R.report_to_json(rep))
    want = json.loads(_ref_json())
    assert list(got) == list(want)  # same keys in the same (sorted) order

    def pts(a):
        return np.array([[complex(re, im) for re, im in p] for p in a]).reshape(len(a), -1)

    def same_set(a, b, tol=1e-8):
        A, B = pts(a), pts(b)
        assert A.shape == B.shape
        if len(A):
            d = np.abs(A[:, None, :] - B[None, :, :]).max(axis=2) / np.maximum(1.0, np.abs(B).max(axis=1))[None, :]
            assert d.min(axis=1).max() < tol and d.min(axis=0).max() < tol

    same_set(got.pop("isolated"), want.pop("isolated"))
    # a suspect is an isolated *singular* point: its coordinates carry the
    # square-root-of-precision error of a multiple root, so it is compared with
    # the reference's own points_match tolerance (1e-6 relative, filtering.py:34)
    same_set(got.pop("suspects"), want.pop("suspects"), 1e-6)
    gw, ww = got.pop("witness_sets"), want.pop("witness_sets")
    assert list(gw) == list(ww)
    for k in gw:
        assert gw[k]["degree"] == ww[k]["degree"]
        same_set(gw[k]["points"], ww[k]["points"])
    gs, wsn = got["counts"].pop("filter_stages"), want["counts"].pop("filter_stages")
    assert len(gs) == len(wsn)
    for a, b in zip(gs, wsn):
        if a["candidate_dimension"] != 0:
            a, b = dict(a), dict(b)
            a.pop("removed"), b.pop("removed")
        assert a == b
    assert got == want
    assert R.summary_text(rep).startswith("seed 33, top dimension 2, 1 task(s), double precision\n")
