"""The multi-device C-ABI (nid_init_devices / nid_use_device /
nid_compact_finite / nid_gather_endpoints, SURVEY §8(b),(e)) on the one GPU
this pool offers: the device list names GPU 0 twice, so two shards go through
the per-device handles, the per-shard compaction kernels and the peer copies
exactly as on two GPUs (cudaMemcpyPeer with equal source and destination
device is a plain device copy)."""

import ctypes as C

import numpy as np
import pytest

from paper_1804_03807_b200 import _lib, configs, tracker
from paper_1804_03807_b200.homotopy import DeviceHomotopy, LinearHomotopy, TrackParams

pytestmark = pytest.mark.gpu


def test_two_shards_gathered_equal_one_launch(nid):
    import torch

    L = nid
    p = configs.c2()
    h = LinearHomotopy(p.start, p.target, p.gamma)
    full = tracker.track_batch(h, None, degrees=p.degrees, count=p.paths)
    fin = np.nonzero(full.succeeded)[0]
    assert len(fin) == 917

    devs = (C.c_int * 2)(0, 0)
    _lib.check(L.nid_init_devices(2, devs), L)
    n, W = p.n, 2
    shards = []
    for r in range(W):
        _lib.check(L.nid_use_device(r), L)
        dh = DeviceHomotopy(h.lowered())  # a handle on "device" r
        Pl = (p.paths - r + W - 1) // W
        out = {"x_end": torch.empty((Pl, n, 2), dtype=torch.float64, device="cuda"),
               "status": torch.empty(Pl, dtype=torch.int8, device="cuda"),
               "steps": torch.empty(Pl, dtype=torch.int32, device="cuda"),
               "t_reached": torch.empty(Pl, dtype=torch.float64, device="cuda"),
               "residual": torch.empty(Pl, dtype=torch.float64, device="cuda"),
               "condition": torch.empty(Pl, dtype=torch.float64, device="cuda"),
               "regular": torch.empty(Pl, dtype=torch.int8, device="cuda")}
        tracker.track_batch_device(dh, TrackParams(), Pl, {k: v.data_ptr() for k, v in out.items()},
                                   degrees=p.degrees, first_index=r, index_stride=W)
        shards.append((dh, Pl, out))
    torch.cuda.synchronize()

    cap = p.paths
    x_out = torch.zeros((cap, n, 2), dtype=torch.float64, device="cuda")
    idx_out = torch.full((cap,), -1, dtype=torch.int64, device="cuda")
    part_dev = (C.c_int * W)(0, 1)
    xs = (C.c_void_p * W)(*[s[2]["x_end"].data_ptr() for s in shards])
    sts = (C.c_void_p * W)(*[s[2]["status"].data_ptr() for s in shards])
    counts = (C.c_longlong * W)(*[s[1] for s in shards])
    first = (C.c_longlong * W)(0, 1)
    stride = (C.c_longlong * W)(W, W)
    total = C.c_longlong(0)
    _lib.check(L.nid_gather_endpoints(W, part_dev, xs, sts, counts, first, stride, n, 0,
                                      C.c_void_p(x_out.data_ptr()), C.c_void_p(idx_out.data_ptr()), cap,
                                      C.byref(total)), L)
    assert total.value == len(fin)
    idx = idx_out[: total.value].cpu().numpy()
    X = x_out[: total.value].cpu().numpy().view(np.complex128).reshape(-1, n)
    # part after part, each in path order
    assert np.array_equal(idx, np.concatenate([fin[fin % W == r] for r in range(W)]))
    assert np.array_equal(X, full.x[idx])

    # single-shard compaction, no indices, and the capacity check
    cnt = C.c_longlong(0)
    s0 = shards[0]
    _lib.check(L.nid_compact_finite(n, s0[1], C.c_void_p(s0[2]["x_end"].data_ptr()),
                                    C.c_void_p(s0[2]["status"].data_ptr()), 0, 1, C.c_void_p(x_out.data_ptr()), None,
                                    cap, C.byref(cnt), None), L)
    assert cnt.value == int(np.sum(fin % W == 0))
    assert L.nid_compact_finite(n, s0[1], C.c_void_p(s0[2]["x_end"].data_ptr()),
                                C.c_void_p(s0[2]["status"].data_ptr()), 0, 1, C.c_void_p(x_out.data_ptr()), None,
                                3, C.byref(cnt), None) != 0
    assert b"capacity" in L.nid_last_error()
    assert L.nid_use_device(5) != 0 and L.nid_init_devices(0, devs) != 0
    bad = (C.c_int * 1)(99)
    assert L.nid_init_devices(1, bad) != 0
    _lib.check(L.nid_use_device(0), L)


def test_empty_shard_and_all_failed(nid):
    import torch

    L = nid
    devs = (C.c_int * 1)(0)
    _lib.check(L.nid_init_devices(1, devs), L)
    n = 3
    x = torch.zeros((5, n, 2), dtype=torch.float64, device="cuda")
    st = torch.tensor([1, 3, 1, 3, 3], dtype=torch.int8, device="cuda")
    out = torch.zeros((5, n, 2), dtype=torch.float64, device="cuda")
    cnt = C.c_longlong(-1)
    _lib.check(L.nid_compact_finite(n, 5, C.c_void_p(x.data_ptr()), C.c_void_p(st.data_ptr()), 0, 1,
                                    C.c_void_p(out.data_ptr()), None, 5, C.byref(cnt), None), L)
    assert cnt.value == 0
    _lib.check(L.nid_compact_finite(n, 0, C.c_void_p(x.data_ptr()), C.c_void_p(st.data_ptr()), 0, 1,
                                    C.c_void_p(out.data_ptr()), None, 5, C.byref(cnt), None), L)
    assert cnt.value == 0


def test_compact_finite_tensor_path(nid):
    """parallel.compact_finite on CUDA tensors (what bench.py's endpoint gather
    uses) equals the boolean-mask compaction, for shapes [P, n, 2]."""
    import torch

    from paper_1804_03807_b200 import parallel

    g = torch.Generator(device="cpu").manual_seed(3)
    for P in (0, 1, 255, 256, 257, 5000):
        x = torch.randn((P, 7, 2), generator=g, dtype=torch.float64)
        st = torch.randint(0, 4, (P,), generator=g, dtype=torch.int8)
        want = x[(st == 0) | (st == 2)]
        got = parallel.compact_finite(x.cuda(), st.cuda())
        assert got.shape == want.shape and torch.equal(got.cpu(), want)
        assert torch.equal(parallel.compact_finite(x, st), want)
    ctx = parallel.DistContext()
    x = torch.randn((100, 4, 2), generator=g, dtype=torch.float64).cuda()
    st = torch.randint(0, 4, (100,), generator=g, dtype=torch.int8).cuda()
    assert torch.equal(parallel.gather_finite(ctx, x, st), x[(st == 0) | (st == 2)])
