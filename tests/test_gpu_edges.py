"""Edge cases of the tracking path on the GPU: empty and one-variable
batches, every TrackParams field away from its default (against the CPU
oracle, the restatement of tracker.py:109-407), the status a path gets when it
runs out of steps, and the C-ABI's argument errors."""

import ctypes as C

import numpy as np
import pytest

from oracle import nid_oracle as O
from paper_1804_03807_b200 import _lib, configs, systems, tracker
from paper_1804_03807_b200.homotopy import LinearHomotopy, TrackParams, params_c
from paper_1804_03807_b200.polys import PolySystem, make_poly

pytestmark = pytest.mark.gpu


def test_empty_batch(nid):
    p = configs.c1()
    h = LinearHomotopy(p.start, p.target, p.gamma)
    r = tracker.track_batch(h, np.zeros((0, p.n), np.complex128))
    assert len(r) == 0 and r.x.shape == (0, p.n) and r.counts() == dict.fromkeys(tracker.STATUS_NAMES, 0)
    r = tracker.track_batch(h, None, degrees=p.degrees, count=0)
    assert len(r) == 0
    assert tracker.refine_batch(p.target, np.zeros((0, p.n))).x.shape == (0, p.n)
    assert tracker.track_batch(h, np.zeros((0, p.n)), trace=True).traces == []


def test_one_variable(nid):
    """n = 1: x^3 = c from the total-degree start x^3 - 1: the three cube roots."""
    c = 2.0 - 1.5j
    f = PolySystem(1, (make_poly(1, [((3,), 1.0), ((0,), -c)]),))
    g = systems.total_degree_start(f)
    r = tracker.track_batch(LinearHomotopy(g, f, 0.8 + 0.6j), None, degrees=(3,), count=3)
    assert np.all(r.status == 0)
    roots = np.sort_complex(np.roots([1, 0, 0, -c]))
    assert np.allclose(np.sort_complex(r.x[:, 0]), roots, atol=1e-12)


PARAM_SETS = [
    dict(max_steps=5),
    dict(max_steps=40, endgame_start=0.5),
    dict(initial_step=0.01, max_step=0.05, min_step=1e-6),
    dict(corrector_tol=1e-12, max_corrector_iters=2),
    dict(max_corrector_iters=1),
    dict(endgame_contraction=0.25, snap_remaining=1e-6),
    dict(final_newton_iters=1),
    dict(infinity_threshold=3.0, soft_infinity=2.0),
    dict(dd_refine_singular=0),
    dict(min_step=1e-3, initial_step=0.1),
]


@pytest.mark.parametrize("kw", PARAM_SETS, ids=[",".join(k) for k in map(list, PARAM_SETS)])
def test_every_track_param_is_honoured(nid, kw):
    """Non-default TrackParams on all 16 C1 paths and 24 C2 paths: statuses,
    step counts and t_reached equal the oracle's path by path (steps within 1
    on <= 10 % of the paths: SURVEY §7's rounding-sensitive decisions),
    endpoints within 1e-8."""
    for prob, idx in ((configs.c1(), np.arange(16)), (configs.c2(), np.arange(7, 5040, 210))):
        starts = systems.total_degree_starts_at(prob.degrees, idx)
        res = tracker.track_batch(LinearHomotopy(prob.start, prob.target, prob.gamma), starts, TrackParams(**kw))
        oh = O.LinearHomotopy(prob.start, prob.target, prob.gamma)
        ref = [O.track(oh, x0, O.TrackParams(**kw)) for x0 in starts]
        st = np.array([tracker.STATUS_CODES[r.status] for r in ref])
        assert np.array_equal(np.isin(res.status, (0, 2)), np.isin(st, (0, 2))), (kw, res.status, st)
        assert np.mean(res.status == st) >= 0.9, (kw, res.status, st)
        steps = np.array([r.steps_used for r in ref])
        assert np.mean(res.steps == steps) >= 0.9 and np.max(np.abs(res.steps - steps)) <= max(2, steps.max() // 20)
        same = res.status == st
        tr = np.array([r.t_reached for r in ref])
        # a tolerance at the evaluation-noise floor makes accept / reject decisions
        # rounding-sensitive: equal step counts, slightly different schedules
        tol_t = dict(rtol=0, atol=1e-2) if kw.get("corrector_tol", 1.0) < 1e-11 else dict(rtol=1e-12, atol=0)
        assert np.allclose(res.t_reached[same & (res.steps == steps)], tr[same & (res.steps == steps)], **tol_t)
        for i, r in enumerate(ref):
            if r.succeeded:
                d = np.max(np.abs(res.x[i] - r.endpoint.coordinates)) / max(1.0, np.max(np.abs(r.endpoint.coordinates)))
                assert d < 1e-8, (kw, i, d)


def test_out_of_steps_is_failed_before_the_endgame(nid):
    """max_steps exhausted at t < endgame_start: FAILED with steps_used =
    max_steps and no endpoint (tracker.py:404-407)."""
    p = configs.c1()
    starts = systems.total_degree_starts(p.degrees)
    r = tracker.track_batch(LinearHomotopy(p.start, p.target, p.gamma), starts, TrackParams(max_steps=3))
    assert np.all(r.status == 3) and np.all(r.steps == 3)
    assert np.all(np.isnan(r.x.real)) and np.all(r.regular == -1) and np.all(r.t_reached < 0.9)


def test_c_abi_argument_errors(nid):
    L = nid
    p = configs.c1()
    h = LinearHomotopy(p.start, p.target, p.gamma).device()
    pc = params_c(TrackParams())
    P = 4
    st = systems.total_degree_starts(p.degrees, 0, P)
    out = tracker.TrackResults(np.empty((P, p.n), np.complex128), np.empty(P, np.int8), np.empty(P, np.int32),
                               np.empty(P), np.empty(P), np.empty(P), np.empty(P, np.int8), {})
    o = _lib.PathOutC(_lib.ptr(out.x), _lib.ptr(out.status), _lib.ptr(out.steps), _lib.ptr(out.t_reached),
                      _lib.ptr(out.residual), _lib.ptr(out.condition), _lib.ptr(out.regular))

    def call(handle=h.handle, prm=C.byref(pc), count=P, starts=_lib.ptr(st), stride=1, deg=None, outp=C.byref(o),
             dev=0):
        return L.nid_track_batch_strided(handle, prm, count, starts, 0, stride, deg, None, 1, outp, dev, None)

    assert call() == 0
    for bad, needle in ((dict(handle=None), b"null"), (dict(prm=None), b"null"), (dict(outp=None), b"null"),
                        (dict(count=-1), b"negative"), (dict(stride=0), b"index_stride"),
                        (dict(starts=None), b"starts"), (dict(starts=C.c_void_p(8), dev=1), b"aligned")):
        assert call(**bad) != 0
        assert needle in L.nid_last_error(), (bad, L.nid_last_error())
    bad_prec = params_c(TrackParams())
    bad_prec.precision = 7
    assert call(prm=C.byref(bad_prec)) != 0 and b"precision" in L.nid_last_error()
    tr = np.zeros((P, 4, 3))
    tn = np.zeros(P, np.int32)
    assert L.nid_track_trace(h.handle, C.byref(pc), P, None, None, 1, C.byref(o), 4, _lib.ptr(tr), _lib.ptr(tn)) != 0
    assert L.nid_track_trace(h.handle, C.byref(pc), P, _lib.ptr(st), None, 1, C.byref(o), 0, _lib.ptr(tr),
                             _lib.ptr(tn)) != 0
    # a trace buffer smaller than the path: counts keep counting, rows stop at the capacity
    assert L.nid_track_trace(h.handle, C.byref(pc), P, _lib.ptr(st), None, 1, C.byref(o), 4, _lib.ptr(tr),
                             _lib.ptr(tn)) == 0
    assert np.all(tn > 4) and np.all(tr[:, :, 0] > 0)
    assert call() == 0 and np.all(out.status == 0)  # the handle is still usable after the errors
