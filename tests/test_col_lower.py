"""Host lowering of the column-owner stream (csrc/col_lower.h) through the
host-only hook nid_col_lower: the stream is decoded here exactly as
csrc/track_col.cuh walks it (run descriptors, ring rule for record positions,
headers, coefficient pieces, blend classes) and must reproduce H, J and the abs
sums of the term table it was built from -- every cell once, nothing twice.
No GPU needed."""

import ctypes as C

import numpy as np
import pytest

from paper_1804_03807_b200 import _lib
from paper_1804_03807_b200.homotopy import lower
from paper_1804_03807_b200.polys import PolySystem, make_poly

RP = 128  # ring pieces (col::RP): a record never straddles a multiple of it


def _system(rng, n, shared_rows, nmono, extra_rows_terms, same_as=None, perturb_rows=()):
    """n rows: the first `shared_rows` on one random support of `nmono` monomials
    of degree <= 4, the others sparse linear rows."""
    expos = set()
    while len(expos) < nmono:
        deg = int(rng.integers(0, 5))
        e = [0] * n
        for _ in range(deg):
            e[int(rng.integers(0, n))] += 1
        expos.add(tuple(e))
    expos = sorted(expos)
    polys = []
    for i in range(n):
        if same_as is not None and i not in perturb_rows:
            polys.append(same_as.polys[i])
            continue
        if i < shared_rows:
            terms = [(e, complex(rng.normal(), rng.normal())) for e in expos]
        else:
            terms = [(tuple(0 for _ in range(n)), complex(rng.normal(), rng.normal()))]
            for v in rng.choice(n, size=extra_rows_terms, replace=False):
                e = [0] * n
                e[int(v)] = 1
                terms.append((tuple(e), complex(rng.normal(), rng.normal())))
        polys.append(make_poly(n, terms))
    return PolySystem(n, tuple(polys))


def _lower_stream(low, groups):
    L = _lib.load_library()
    kind = 0 if low.start_degrees is None else 1
    d = _lib.HomotopyDescC(low.n, low.nterms, _lib.ptr(low.row_off), _lib.ptr(low.expo), _lib.ptr(low.cs),
                           _lib.ptr(low.ct), _lib.ptr(low.pslot), low.nparam, low.gamma.real, low.gamma.imag, kind,
                           _lib.ptr(low.start_degrees), None)
    npc, nrn, ok = C.c_longlong(0), C.c_longlong(0), C.c_int(0)
    cgrun = (C.c_int * 17)()
    cgbase = (C.c_int * 17)()
    _lib.check(L.nid_col_lower(C.byref(d), groups, None, 0, C.byref(npc), None, 0, C.byref(nrn), cgrun, cgbase,
                               C.byref(ok)), L)
    if not ok.value:
        return None
    pieces = np.zeros((npc.value, 4), dtype=np.uint32)
    runs = np.zeros((nrn.value, 4), dtype=np.uint32)
    _lib.check(L.nid_col_lower(C.byref(d), groups, pieces.ctypes.data_as(C.c_void_p), npc.value, C.byref(npc),
                               runs.ctypes.data_as(C.c_void_p), nrn.value, C.byref(nrn), cgrun, cgbase,
                               C.byref(ok)), L)
    return pieces, runs, list(cgrun), list(cgbase)


def _decode_eval(low, stream, groups, x, t, prm):
    """Walk the stream as eval_cols does; returns H, J, sS, sT and the per-cell write counts."""
    pieces, runs, cgrun, cgbase = stream
    n = low.n
    td = low.start_degrees is not None
    alpha = (1.0 - t) * low.gamma
    beta = alpha + t
    ax = np.abs(x)
    H = np.zeros(n, dtype=complex)
    J = np.zeros((n, n), dtype=complex)
    sS = np.zeros(n)
    sT = np.zeros(n)
    wrote = np.zeros((n, n + 2), dtype=int)  # cells flushed (J columns, H column n, abs column n+1)
    as_c = lambda p: complex(p[:2].view(np.float64)[0], p[2:].view(np.float64)[0])
    for w in range(groups):
        base = cgbase[w]
        acc = np.zeros(8, dtype=complex)
        for u in range(cgrun[w], cgrun[w + 1]):
            rx, ry, rz, rw = (int(v) for v in runs[u])
            col, row0, nr = rx & 0xff, (rx >> 8) & 0xff, (rx >> 16) & 0xff
            first, last, kind = (rx >> 24) & 1, (rx >> 25) & 1, (rx >> 26) & 3
            D, mask, cls, ln = ry & 0xff, (ry >> 8) & 0xff, (ry >> 16) & 0xf, (ry >> 20) & 0x3f
            if first:
                acc[:] = 0
            q = rz
            for _ in range(rw):
                if (q % RP) + ln > RP:
                    q = (q + RP - 1) // RP * RP
                hd = pieces[base + q]
                fac = int(hd[0]) | (int(hd[1]) << 32)
                vs = [(fac >> (4 * j)) & 15 for j in range(D)]
                em = (fac >> 48) & 0xff
                ps = list(hd[2:].view(np.int8))
                cq = q + 1
                if kind == 1:  # abs sums
                    m = float(np.prod(ax[vs])) if D else 1.0
                    for i in range(8):
                        if (mask >> i) & 1:
                            a = as_c(pieces[base + cq])
                            acc[i] += complex(0.0 if td else a.real * m, a.imag * m)
                            cq += 1
                else:
                    p = complex(np.prod(x[vs])) if D else 1.0 + 0j
                    for i in range(8):
                        if not (mask >> i) & 1:
                            continue
                        if cls >= 3:  # start and target coefficients, multiplier in the header
                            cs_, ct_ = as_c(pieces[base + cq]), as_c(pieces[base + cq + 1])
                            if cls == 4 and ps[i] >= 0:
                                ct_ = prm[ps[i]]
                            acc[i] += (cs_ * alpha + ct_ * t) * p * em
                            cq += 2
                        else:  # one coefficient (multiplier folded), blend scalar by class
                            sc = (t, alpha, beta)[cls]
                            acc[i] += as_c(pieces[base + cq]) * sc * p
                            cq += 1
                assert cq - q == ln
                q += ln
            if last:
                for i in range(nr):
                    r = row0 + i
                    if kind == 1:
                        sS[r] += acc[i].real
                        sT[r] += acc[i].imag
                        wrote[r, n + 1] += 1
                    elif col == n:
                        H[r] += acc[i]  # per-warp partial sums, added after the barrier
                        wrote[r, n] += 1
                    else:
                        J[r, col] += acc[i]
                        wrote[r, col] += 1
    return H, J, sS, sT, wrote


def _direct(low, x, t, prm):
    n = low.n
    alpha = (1.0 - t) * low.gamma
    H = np.zeros(n, dtype=complex)
    J = np.zeros((n, n), dtype=complex)
    sS = np.zeros(n)
    sT = np.zeros(n)
    for i in range(n):
        for k in range(low.row_off[i], low.row_off[i + 1]):
            e = low.expo[k, :n].astype(int)
            ct = low.ct[k]
            if low.pslot is not None and low.pslot[k] >= 0:
                ct = prm[low.pslot[k]]
            c = alpha * low.cs[k] + t * ct
            H[i] += c * np.prod(x ** e)
            m = float(np.prod(np.abs(x) ** e))
            sS[i] += abs(low.cs[k]) * m
            sT[i] += abs(low.ct[k]) * m
            for v in range(n):
                if e[v]:
                    e2 = e.copy()
                    e2[v] -= 1
                    J[i, v] += c * e[v] * np.prod(x ** e2)
    return H, J, sS, sT


@pytest.mark.parametrize("n,groups,shared,case", [(8, 4, 3, "shared"), (14, 8, 8, "shared"), (11, 8, 5, "blend"),
                                                  (9, 4, 4, "param"), (12, 8, 6, "td")])
def test_stream_reproduces_the_term_table(n, groups, shared, case):
    rng = np.random.default_rng(100 + n)
    target = _system(rng, n, shared, 40 if n < 14 else 120, 3)
    param_terms = None
    if case == "shared":  # every row the same in start and target
        start = target
    elif case == "blend":  # the last rows differ (cascade / membership slices)
        start = _system(rng, n, shared, 40, 3, same_as=target, perturb_rows=(n - 1, n - 2))
    elif case == "param":  # per-path constants on the last row
        start = _system(rng, n, shared, 40, 3, same_as=target, perturb_rows=(n - 1,))
        param_terms = {(n - 1, tuple(0 for _ in range(n))): 0}
    else:  # total-degree start: the table holds the target only
        start = PolySystem(n, tuple(make_poly(n, [(tuple(4 if v == i else 0 for v in range(n)), 1.0 + 0j),
                                                  (tuple(0 for _ in range(n)), -1.0 + 0j)]) for i in range(n)))
    low = lower(start, target, 0.6 - 0.8j, param_terms)
    stream = _lower_stream(low, groups)
    assert stream is not None
    pieces, runs, cgrun, cgbase = stream
    assert all(b % 32 == 0 for b in cgbase[:groups]) and len(runs) <= 256
    x = rng.normal(size=n) + 1j * rng.normal(size=n)
    t = 0.37
    prm = np.array([0.3 - 1.1j])
    H, J, sS, sT, wrote = _decode_eval(low, stream, groups, x, t, prm)
    H0, J0, sS0, sT0 = _direct(low, x, t, prm)
    if low.start_degrees is not None:
        sS0[:] = 0.0  # closed form on the device, not in the stream
    # every Jacobian cell and every abs sum flushed exactly once, every value once per warp
    assert (wrote[:, :n] == 1).all() and (wrote[:, n + 1] == 1).all() and (wrote[:, n] == groups).all()
    scale = max(1.0, np.abs(J0).max())
    assert np.abs(H - H0).max() <= 1e-12 * max(1.0, np.abs(H0).max())
    assert np.abs(J - J0).max() <= 1e-12 * scale
    assert np.abs(sS - sS0).max() <= 1e-12 * max(1.0, sS0.max()) and np.abs(sT - sT0).max() <= 1e-12 * max(1.0, sT0.max())


def test_ineligible_table_is_reported():
    # a term of total degree 13 does not fit a record's factor list
    n = 8
    e = [0] * n
    e[0], e[1] = 7, 6
    f = PolySystem(n, tuple(make_poly(n, [(tuple(e), 1.0 + 0j), (tuple(0 for _ in range(n)), 1.0 + 0j)]) for _ in range(n)))
    assert _lower_stream(lower(f, f, 1.0 + 0j), 4) is None
