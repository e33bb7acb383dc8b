"""Multi-rank stage drivers on CPU (gloo, world_size 2): SURVEY §8(e).

Under `parallel.activate(ctx)` every rank runs the same host logic, tracks
its strided share of each stage's paths and gets the whole stage back from one
all_gather, in job order.  Here the per-rank GPU calls (`tracker._track_local`,
`_refine_local`, `filtering.match_pairs`) are replaced by the CPU oracle (test
infrastructure), so the sharding, the gathers, the per-level re-sharding and
the rank-0 dedup run for real on two processes.  Bar: the two-rank records
equal the one-rank records exactly, on both ranks.
"""

import multiprocessing as mp
import os
import socket

import numpy as np
import pytest

from conftest import golden
from oracle import nid_oracle as O
from paper_1804_03807_b200 import _lib, cascade, configs, filtering, parallel, systems, tracker
from paper_1804_03807_b200.homotopy import LinearHomotopy, TrackParams
from paper_1804_03807_b200.tracker import RefineResults, Solution, TrackResults

STATUS = {"converged": 0, "at_infinity": 1, "singular_endpoint": 2, "failed": 3}
SLACK = {"at_infinity": _lib.CLS_AT_INFINITY, "zero_slack": _lib.CLS_ZERO, "nonzero_slack": _lib.CLS_NONZERO}


def oracle_track_local(h, starts=None, params=TrackParams(), *, degrees=None, first_index=0, count=None,
                       index_stride=1, target_params=None, param_div=1, out=None, trace=False):
    if starts is None:
        starts = systems.total_degree_starts(degrees, first_index, count, index_stride)
    starts = np.asarray(starts, np.complex128)
    P, n = starts.shape
    res = TrackResults(np.full((P, n), np.nan + 0j), np.zeros(P, np.int8), np.zeros(P, np.int32), np.zeros(P),
                       np.full(P, np.nan), np.full(P, np.nan), np.full(P, -1, np.int8),
                       {"evals": 0, "jacs": 0, "scales": 0, "paths": P, "dd_polished": 0, "lstsq_fallbacks": 0,
                        "kernel_ms_track": 0.0, "kernel_ms_endpoint": 0.0})
    if target_params is not None:  # plumbing fake for per-group parameters: a deterministic function of (start, param)
        tp = np.asarray(target_params, np.complex128).reshape(P // param_div, -1)
        for i in range(P):
            res.x[i] = starts[i] * 2 + tp[i // param_div].sum()
            res.status[i] = 2 if starts[i][0].real > 0 else 0
            res.steps[i] = int(abs(tp[i // param_div][0]) * 100) % 97
            res.residual[i] = float(abs(starts[i][0]))
        return res
    oh = O.LinearHomotopy(h.start, h.target, h.gamma)
    for i, x0 in enumerate(starts):
        r = O.track(oh, x0)
        res.status[i], res.steps[i], res.t_reached[i] = STATUS[r.status], r.steps_used, r.t_reached
        if r.endpoint is not None:
            res.x[i] = r.endpoint.coordinates
            res.residual[i], res.condition[i] = r.endpoint.residual, r.endpoint.condition
            res.regular[i] = 1 if r.endpoint.regularity == "regular" else 0
        res.counters["evals"] += r.steps_used
    return res


def oracle_refine_local(f, X, tol=1e-12, max_iters=10, n_original=None, infinity_threshold=1e8, h=None):
    X = np.array(X, np.complex128).reshape(-1, f.nvars)
    P = len(X)
    rr = RefineResults(X, np.zeros(P), np.zeros(P), np.zeros(P, np.int8), np.zeros(P, np.int32), np.zeros(P, np.int8))
    for i in range(P):
        s = O.newton_refine(f, X[i], tol, max_iters)
        rr.x[i], rr.residual[i], rr.condition[i] = s.coordinates, s.residual, s.condition
        rr.regular[i] = 1 if s.regularity == "regular" else 0
        rr.rank[i] = O.condition_and_rank(O.jacobian(f, s.coordinates))[1]
        rr.slack[i] = SLACK[O.classify(s.coordinates, f.nvars if n_original is None else n_original,
                                       infinity_threshold)]
    return rr


def oracle_match_pairs(X, ncmp=None):
    X = np.asarray(X)
    return np.array([(i, j) for i in range(len(X)) for j in range(i + 1, len(X)) if O.points_match(X[j], X[i])],
                    np.int32).reshape(-1, 2)


def _patch():
    tracker._track_local = oracle_track_local
    tracker._refine_local = oracle_refine_local
    filtering.match_pairs = oracle_match_pairs


def stages():
    """C2: 40 device-generated total-degree paths (strided index shards);
    C3-mini: one cascade step from 14 of the reference's nonzero-slack
    solutions (explicit starts, refine + classify re-gathered), the dedup of
    its endpoints decided on rank 0; membership-style groups of 3 paths with
    per-group parameters."""
    out = {}
    p2 = configs.c2()
    r = tracker.track_batch(LinearHomotopy(p2.start, p2.target, p2.gamma), None, degrees=p2.degrees, count=40,
                            first_index=100, index_stride=7)
    out["c2"] = (r.x, r.status, r.steps, r.t_reached, r.residual, r.condition, r.regular, r.counters["paths"],
                 r.counters["evals"])
    pd = configs.c3_mini()
    g = golden("pipeline_c3m")
    sols = [Solution(x, 0.0, 1.0) for x in g["L2_nonzero_x"][:14]]
    lv = cascade.CascadeLevel(2, pd.emb.level(2), starts=len(sols), at_infinity=0, nonzero_slack=sols)
    nxt = cascade.cascade_step(lv)
    out["c3m_counts"] = nxt.counts
    out["c3m_nonzero"] = np.array([s.coordinates for s in nxt.nonzero_slack])
    out["c3m_zero"] = np.array([s.coordinates for s in nxt.zero_slack])
    pts = nxt.nonzero_slack + nxt.zero_slack + nxt.nonzero_slack[:3]
    kept, mult = filtering.dedup(pts, pd.emb.n_original)
    out["dedup"] = (np.array([s.coordinates for s in kept]), mult)
    rng = np.random.default_rng(5)
    st = rng.normal(size=(7 * 3, 4)) + 1j * rng.normal(size=(7 * 3, 4))
    tp = rng.normal(size=(7, 2)) + 1j * rng.normal(size=(7, 2))
    r = tracker.track_batch(LinearHomotopy(pd.emb.base, pd.emb.base), st, target_params=tp, param_div=3)
    out["groups"] = (r.x, r.status, r.steps, r.residual)
    return out


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    _patch()
    ctx = parallel.DistContext.from_env(world, backend="gloo")
    parallel.activate(ctx)
    try:
        q.put((rank, stages()))
        ctx.barrier()
    finally:
        parallel.activate(None)
        ctx.close()


def _same(a, b):
    if isinstance(a, (tuple, list)):
        return len(a) == len(b) and all(_same(x, y) for x, y in zip(a, b))
    if isinstance(a, np.ndarray):
        return a.shape == b.shape and a.dtype == b.dtype and np.array_equal(a, b, equal_nan=True)
    return a == b


def test_two_rank_stage_drivers_equal_one_rank():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mpc = mp.get_context("spawn")
    q = mpc.Queue()
    procs = [mpc.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    saved = (tracker._track_local, tracker._refine_local, filtering.match_pairs)
    try:
        _patch()
        one = stages()  # the one-rank records, computed while the two ranks run
    finally:
        tracker._track_local, tracker._refine_local, filtering.match_pairs = saved
    got = dict(q.get(timeout=600) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert one["c2"][7] == 40 and int(np.isin(one["c2"][1], (0, 2)).sum()) >= 1
    assert one["c3m_counts"]["starts"] == 14
    for rank in (0, 1):
        for key in one:
            assert _same(one[key], got[rank][key]), (rank, key)


def test_group_shard_and_on_root_single_rank():
    assert parallel.group_shard(7, 1, 3).tolist() == [1, 4]
    assert parallel.group_shard(2, 2, 3).tolist() == []
    assert parallel.active() is None
    assert parallel.on_root(lambda a, b: a + b, 2, 3) == 5
    with pytest.raises(ValueError):
        parallel.shard_strided(10, 3, 3)


def test_torchrun_two_ranks_gloo():
    """The launch line of the driver (`python -m torch.distributed.run --nnodes=1
    --nproc-per-node 2 --master-addr 127.0.0.1 --master-port P ...`) on CPU / gloo:
    both shapes of the multi-rank path (per-rank shard + gather to rank 0, and the
    sharded stage driver) agree with the one-rank records."""
    import json
    import subprocess
    import sys

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    here = os.path.dirname(os.path.abspath(__file__))
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port),
                        os.path.join(here, "mr_torchrun_worker.py")], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    p2 = configs.c2()
    one = oracle_track_local(LinearHomotopy(p2.start, p2.target, p2.gamma), None, degrees=p2.degrees, count=48)
    assert line["world"] == 2 and line["max"] == 2.0
    assert line["finite"] == line["gathered"] == line["full_finite"] == int(one.succeeded.sum())
    assert line["full_paths"] == 48 and line["status"] == one.status.tolist()
