"""Host-side logic on the CPU: lowering, systems, configs, FLOP model, the
C-ABI library's exports, sharding and the 2-rank gloo endpoint gather."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT, golden
from paper_1804_03807_b200 import _lib, configs, flops, parallel, rng, systems
from paper_1804_03807_b200.homotopy import LinearHomotopy, TrackParams, lower
from paper_1804_03807_b200.polys import PolySystem, make_poly, poly_diff


def test_track_params_validation_mirrors_reference():
    with pytest.raises(ValueError):
        TrackParams(initial_step=0.3, max_step=0.2)
    with pytest.raises(ValueError):
        TrackParams(min_step=0.5)
    with pytest.raises(ValueError):
        TrackParams(corrector_tol=0.0)
    c = TrackParams().to_c()
    assert c.max_steps == 2000 and c.final_newton_iters == 40 and c.dd_refine_singular == 3


def test_linear_homotopy_shape_check():
    with pytest.raises(ValueError):
        LinearHomotopy(systems.cyclic(3), systems.cyclic(4))


def test_lowering_merges_rows():
    p = configs.c5()
    low = lower(p.start, p.target, p.gamma)
    # the total-degree start is recognised and evaluated in closed form
    assert list(low.start_degrees) == list(range(1, 11))
    assert low.n == 10 and low.nterms == 92 and not np.any(low.cs)
    for i in range(10):
        seg = slice(low.row_off[i], low.row_off[i + 1])
        ex = [tuple(e[:10]) for e in low.expo[seg]]
        assert ex == sorted(ex)
        assert {e: c for e, c in zip(ex, low.ct[seg]) if c != 0} == dict(p.target.polys[i].terms)
    # a generic start is merged term by term
    pd = configs.c3_mini()
    E = pd.emb.system
    g = PolySystem(E.nvars, tuple(make_poly(E.nvars, [(e, 2 * c) for e, c in q.terms]) for q in E.polys))
    low = lower(g, E, 0.5j)
    assert low.start_degrees is None
    for i in range(E.nvars):
        seg = slice(low.row_off[i], low.row_off[i + 1])
        ex = [tuple(e[:E.nvars]) for e in low.expo[seg]]
        assert {e: c for e, c in zip(ex, low.cs[seg]) if c != 0} == dict(g.polys[i].terms)
        assert {e: c for e, c in zip(ex, low.ct[seg]) if c != 0} == dict(E.polys[i].terms)


def test_lowering_param_slots_for_membership():
    pd = configs.c3_mini()
    E = pd.emb.system
    n, k = pd.emb.n_original, pd.emb.k
    zero = (0,) * E.nvars
    low = lower(E, E, 1.0, {(n + j, zero): j for j in range(k)})
    assert low.nparam == k
    assert int(np.sum(low.pslot >= 0)) == k
    for j in range(k):
        kk = int(np.nonzero(low.pslot == j)[0][0])
        assert low.row_off[n + j] <= kk < low.row_off[n + j + 1]
        assert not low.expo[kk].any()


def test_lowering_rejects_unsupported():
    with pytest.raises(ValueError):
        f = PolySystem(17, tuple(make_poly(17, [((1,) + (0,) * 16, 1.0)]) for _ in range(17)))
        lower(f, f)
    f = PolySystem(3, tuple(make_poly(3, [((1, 0, 0), 1.0)]) for _ in range(2)))
    with pytest.raises(ValueError):
        lower(f, f)


def test_flop_model_matches_survey_table():
    m = flops.flop_model(lower(configs.c5().start, configs.c5().target))
    assert (m.T_H, m.nnzJ_H, m.M, m.M_J) == (110, 469, 90, 253)
    m3 = flops.flop_model(lower(configs.c3_top(configs.c3()).start, configs.c3_top(configs.c3()).target))
    assert (m3.T_H, m3.nnzJ_H, m3.M) == (4068, 10662, 486)


def test_gamma_and_embedding_streams_match_reference_fixture():
    g = golden("pipeline_c3m")
    pd = configs.c3_mini()
    # top-level starts in the fixture were generated with our start builder
    prob = configs.c3_top(pd)
    assert np.allclose(g["top_starts"], systems.total_degree_starts(prob.degrees))
    assert rng.gamma_for(5) == complex(np.exp(1j * np.random.default_rng(
        np.random.SeedSequence(5, spawn_key=(4,))).uniform(0, 2 * np.pi)))


def test_total_degree_start_indexing():
    X = systems.total_degree_starts((2, 3), 0)
    assert X.shape == (6, 2)
    assert np.allclose(X[1], [1.0, np.exp(2j * np.pi / 3)])  # last variable fastest
    assert np.allclose(X[3], [-1.0, 1.0])


def test_poly_diff_and_make_poly():
    p = make_poly(2, [((2, 1), 3.0), ((2, 1), 1.0), ((0, 0), 0.0)])
    assert p.terms == (((2, 1), 4.0 + 0j),)
    assert poly_diff(p, 0).terms == (((1, 1), 8.0 + 0j),)


def test_library_exports_every_declared_symbol():
    """libnid.so loads without a GPU and exports every function include/nid.h declares."""
    L = _lib.load_library()
    header = open(os.path.join(ROOT, "include", "nid.h")).read()
    declared = set(re.findall(r"\b(nid_[a-z_]+)\s*\(", header))
    assert declared, "no declarations found"
    for name in declared:
        assert hasattr(L, name), name
    assert set(_lib.EXPORTS) <= declared


def test_no_gpu_means_loud_failure():
    try:
        import torch

        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    with pytest.raises(_lib.NidUnavailable):
        _lib.lib()


def test_ctypes_struct_layout_matches_header():
    assert ctypes.sizeof(_lib.TrackParamsC) == 4 * 8 + 2 * 4 + 4 * 8 + 2 * 4 + 8 + 2 * 4
    # ..., start_kind(+pad), degrees, term_texp
    assert ctypes.sizeof(_lib.HomotopyDescC) == 4 + 4 + 5 * 8 + 8 + 16 + 8 + 8 + 8


@pytest.mark.parametrize("total,world", [(3628800, 8), (5040, 3), (7, 4), (0, 2)])
def test_shard_range_covers_exactly(total, world):
    spans = [parallel.shard_range(total, r, world) for r in range(world)]
    assert spans[0][0] == 0 and spans[-1][1] == total
    for (a, b), (c, d) in zip(spans, spans[1:]):
        assert b == c
    sizes = [b - a for a, b in spans]
    assert max(sizes) - min(sizes) <= 1


@pytest.mark.parametrize("total,world", [(3628800, 8), (5040, 3), (7, 4), (0, 2)])
def test_shard_strided_partitions(total, world):
    got = []
    for r in range(world):
        first, stride, count = parallel.shard_strided(min(total, 100000), r, world)
        got.append(first + stride * np.arange(count))
    allidx = np.sort(np.concatenate(got)) if got else np.array([])
    assert np.array_equal(allidx, np.arange(min(total, 100000)))
    sizes = [len(g) for g in got]
    assert max(sizes) - min(sizes) <= 1


def test_strided_total_degree_starts_are_a_subset():
    from paper_1804_03807_b200 import systems

    deg = [1, 2, 3, 4]
    full = systems.total_degree_starts(deg)
    for r in range(3):
        sub = systems.total_degree_starts(deg, r, None, 3)
        assert np.array_equal(sub, full[r::3])


def _gloo_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import torch

    ctx = parallel.DistContext.from_env(world, backend="gloo")
    lo, hi = ctx.shard(10)
    x = torch.arange(lo, hi, dtype=torch.float64).reshape(-1, 1, 1).repeat(1, 3, 2)
    status = torch.tensor([(i % 3) for i in range(lo, hi)], dtype=torch.int8)  # 0 conv, 1 inf, 2 singular
    got = parallel.gather_finite(ctx, x, status)
    mx = ctx.max_over_ranks(float(rank))
    sm = ctx.sum_over_ranks(hi - lo)
    if rank == 0:
        q.put((got[:, 0, 0].tolist(), mx, sm))
    ctx.barrier()
    ctx.close()


def test_two_rank_gloo_gather_and_reductions():
    import multiprocessing as mp
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got, mx, sm = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert got == [0.0, 2.0, 3.0, 5.0, 6.0, 8.0, 9.0]  # indices with status 0 or 2, rank order
    assert mx == 1.0 and sm == 10
