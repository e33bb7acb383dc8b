"""Homotopy membership tests, junk removal and isolated-point classification
on the GPU (mode="gpu"), with the reference's signatures and records
(pkg/src/nidpipe/filtering.py:34-256).

K8 (`membership_batch`): every candidate x witness-point path of a stage is
one launch.  Each path carries its candidate's hyperplane constants
c0_j = -a_j . q as per-path target coefficients of a single uploaded term
table, so the 400,000-path C4 stage is one `track_batch` call.
K7 (`dedup`): all-pairs `points_match` on the GPU, greedy keep in
ascending-residual order on the host over the (sparse) match list;
multiplicity = cluster size.
"""

from __future__ import annotations

from dataclasses import dataclass

import ctypes as C

import numpy as np

from . import _lib
from . import parallel, refbridge
from .cascade import WitnessSuperset, _check_mode
from .homotopy import LinearHomotopy, TrackParams, lower
from .homotopy import DeviceHomotopy
from .polys import PolySystem, make_poly
from .systems import EmbeddedSystem, slice_to_zero
from .tracker import (
    REGULAR,
    SINGULAR,
    Solution,
    condition_and_rank,
    refine_batch,
    refine_dd_batch,
    singular_values,
    track_batch,
)

MATCH_TOL = 1e-6
MATCH_FLOOR = 1e-8


class MembershipIndeterminate(RuntimeError):
    """Every membership path failed (filtering.py:38-39)."""


@dataclass
class WitnessSet:
    """filtering.py:42-58"""

    dimension: int
    embedding: EmbeddedSystem
    points: list
    label: str = ""

    @property
    def degree(self) -> int:
        return len(self.points)

    def original_points(self) -> np.ndarray:
        n = self.embedding.n_original
        return np.array([s.coordinates[:n] for s in self.points])


@dataclass
class FilterStage:
    """filtering.py:61-70"""

    candidate_dimension: int
    against_dimension: int
    candidates: int
    degree: int
    paths_tracked: int
    removed: int


def points_match(a, b, tol: float = MATCH_TOL, floor: float = MATCH_FLOOR) -> bool:
    """filtering.py:73-78"""
    a = np.asarray(a, dtype=np.complex128)
    b = np.asarray(b, dtype=np.complex128)
    scale = max(1.0, float(np.max(np.abs(b))))
    return float(np.max(np.abs(a - b))) <= max(floor, tol * scale)


def _match_rows(A: np.ndarray, B: np.ndarray) -> np.ndarray:
    """points_match(A[i], B[i]) row-wise (vectorised bookkeeping)."""
    scale = np.maximum(1.0, np.max(np.abs(B), axis=1))
    return np.max(np.abs(A - B), axis=1) <= np.maximum(MATCH_FLOOR, MATCH_TOL * scale)


def membership_targets(w: WitnessSet, q) -> EmbeddedSystem:
    """filtering.py:81-89"""
    q = np.asarray(q, dtype=np.complex128)
    consts = [-np.dot(np.asarray(row[1:], dtype=np.complex128), q) for row in w.embedding.hyper_coeffs]
    return w.embedding.with_hyper_constants(consts)


class MembershipHomotopy:
    """LinearHomotopy(E, E_q) for every candidate q at once: the hyperplane
    constant terms of the target are per-path parameters (filtering.py:112-113)."""

    def __init__(self, w: WitnessSet):
        emb = w.embedding
        self.emb = emb
        E = emb.system
        n, k = emb.n_original, emb.k
        zero = (0,) * E.nvars
        slots = {(n + j, zero): j for j in range(k)}
        self.low = lower(E, E, 1.0 + 0j, slots)
        self.dev = DeviceHomotopy(self.low)
        self.A = np.array([row[1:] for row in emb.hyper_coeffs], dtype=np.complex128)  # (k, n)

    def constants(self, Q: np.ndarray) -> np.ndarray:
        return -(np.asarray(Q, dtype=np.complex128) @ self.A.T)  # (C, k)


def membership_batch(w: WitnessSet, Q, p: int = 1, params: TrackParams = TrackParams(), mode: str = "gpu",
                     mh: MembershipHomotopy | None = None):
    """Membership verdicts for many candidates in one launch.

    Returns (verdict int8 [C]: 1 member, 0 not, -1 indeterminate;
    paths_tracked)."""
    if not _check_mode(mode):  # the reference decides candidate by candidate
        v = np.zeros(len(Q), np.int8)
        for i, q in enumerate(np.asarray(Q, dtype=np.complex128)):
            try:
                v[i] = 1 if refbridge.membership_test(w, q, p, params, mode) else 0
            except Exception as e:  # the reference's MembershipIndeterminate
                if type(e).__name__ != "MembershipIndeterminate":
                    raise
                v[i] = -1
        return v, len(Q) * len(w.points)
    Q = np.asarray(Q, dtype=np.complex128)
    n = w.embedding.n_original
    if Q.ndim != 2 or Q.shape[1] != n:
        raise ValueError(f"candidates must have shape (C, {n})")
    Cn = Q.shape[0]
    verdict = np.zeros(Cn, np.int8)
    W = np.array([s.coordinates for s in w.points], dtype=np.complex128)
    d = W.shape[0]
    if Cn == 0:
        return verdict, 0
    # shortcut: q already on a witness point (filtering.py:109-111)
    short = np.zeros(Cn, bool)
    for j in range(d):
        short |= _match_rows(np.broadcast_to(W[j, :n], Q.shape), Q)
    verdict[short] = 1
    todo = np.nonzero(~short)[0]
    if len(todo) == 0 or d == 0:
        return verdict, 0
    mh = mh or MembershipHomotopy(w)
    prm = mh.constants(Q[todo])  # (len(todo), k)
    starts = np.tile(W, (len(todo), 1))  # path c*d + j starts at witness point j
    res = track_batch(mh.dev, starts, params, target_params=prm, param_div=d)
    ok = res.succeeded.reshape(len(todo), d)
    xe = res.x.reshape(len(todo), d, -1)[:, :, :n]
    hit = np.zeros((len(todo), d), bool)
    for j in range(d):
        hit[:, j] = ok[:, j] & _match_rows(np.nan_to_num(xe[:, j], nan=np.inf), Q[todo])
    member = hit.any(axis=1)
    verdict[todo] = np.where(member, 1, np.where(ok.any(axis=1), 0, -1))
    return verdict, len(todo) * d


def membership_test(w: WitnessSet, q, p: int = 1, params: TrackParams = TrackParams(), mode: str = "gpu") -> bool:
    """filtering.py:92-127"""
    if not _check_mode(mode):
        return refbridge.membership_test(w, q, p, params, mode)
    q = np.asarray(q, dtype=np.complex128)
    n = w.embedding.n_original
    if q.shape != (n,):
        raise ValueError(f"candidate has dimension {q.shape}, expected {n}")
    v, _ = membership_batch(w, q[None], p, params, mode)
    if v[0] < 0:
        raise MembershipIndeterminate(f"all {w.degree} membership paths failed for dimension {w.dimension}")
    return bool(v[0] == 1)


def _restricted_regular_batch(emb: EmbeddedSystem, X: np.ndarray) -> np.ndarray:
    """Full column rank of the slice_to_zero Jacobian at x[:n] (filtering.py:130-137).
    The (n+k) x n Jacobian is evaluated on the GPU as the leading columns of a
    square system padded with k unused variables."""
    n, k = emb.n_original, emb.k
    sl = slice_to_zero(emb)
    m = n + k
    pad = PolySystem(m, tuple(make_poly(m, [(tuple(e) + (0,) * k, c) for e, c in p.terms]) for p in sl.polys))
    h = LinearHomotopy(pad, pad)
    Xp = np.zeros((len(X), m), np.complex128)
    Xp[:, :n] = np.asarray(X)[:, :n]
    _, J, _ = h.evaluate(Xp, np.ones(len(X)))
    out = np.zeros(len(X), bool)
    A = np.ascontiguousarray(J[:, :, :n])
    fin = np.all(np.isfinite(A.view(np.float64).reshape(len(X), -1)), axis=1)
    if fin.any():
        sv = singular_values(A[fin])
        smax = sv[:, 0]
        rank = np.sum(sv > 1e-8 * smax[:, None], axis=1)
        rank[smax == 0.0] = 0
        out[np.nonzero(fin)[0]] = rank == n
    return out


def _restricted_regular(emb: EmbeddedSystem, sol: Solution) -> bool:
    return bool(_restricted_regular_batch(emb, np.asarray(sol.coordinates)[None])[0])


def match_pairs(X: np.ndarray, ncmp: int | None = None) -> np.ndarray:
    """All (i, j), i < j, with points_match(X[j][:ncmp], X[i][:ncmp]) -- GPU."""
    X = np.ascontiguousarray(X, dtype=np.complex128)
    P, n = X.shape
    ncmp = n if ncmp is None else ncmp
    if P < 2:
        return np.zeros((0, 2), np.int32)
    L = _lib.lib()
    cap = 1 << 16
    while True:
        pairs = np.empty((cap, 2), np.int32)
        cnt = C.c_longlong(0)
        _lib.check(L.nid_match_pairs(n, ncmp, P, _lib.ptr(X), _lib.ptr(pairs), cap, C.byref(cnt)), L)
        if cnt.value <= cap:
            return pairs[: cnt.value]
        cap = int(cnt.value)


def dedup(points: list, n: int | None = None) -> tuple[list, list]:
    """_dedup (filtering.py:140-150) with multiplicities: kept points in
    ascending-residual order, and each kept point's cluster size."""
    if not points:
        return [], []
    order = sorted(range(len(points)), key=lambda i: points[i].residual)
    X = np.array([points[i].coordinates if n is None else points[i].coordinates[:n] for i in order])
    # a global view: decided on rank 0's GPU and broadcast
    pairs = parallel.on_root(match_pairs, X)
    by_j: dict[int, list] = {}
    for i, j in pairs:
        by_j.setdefault(int(j), []).append(int(i))
    kept_pos: dict[int, int] = {}
    mult: list[int] = []
    for j in range(len(order)):
        owners = [kept_pos[i] for i in sorted(by_j.get(j, [])) if i in kept_pos]
        if owners:
            mult[min(owners)] += 1
        else:
            kept_pos[j] = len(mult)
            mult.append(1)
    kept = [points[order[j]] for j in sorted(kept_pos, key=lambda j: kept_pos[j])]
    return kept, mult


def _dedup(points: list, n: int | None = None) -> list:
    return dedup(points, n)[0]


def filter_junk(superset: WitnessSuperset, p: int = 1, params: TrackParams = TrackParams(), mode: str = "gpu"):
    """Top-down junk removal (filtering.py:153-201)."""
    if not _check_mode(mode):
        return refbridge.filter_junk(superset, p, params, mode)
    witness_sets: list[WitnessSet] = []
    stages: list[FilterStage] = []
    n = superset.embedding.n_original
    for level in superset.levels:
        d = level.dimension
        if d == 0:
            continue
        cands = _dedup(list(level.zero_slack), n)
        for w in witness_sets:
            if not cands:
                break
            Q = np.array([c.coordinates[:n] for c in cands])
            verdict, tracked = membership_batch(w, Q, p, params, mode)
            kept = [c for c, v in zip(cands, verdict) if v != 1]  # indeterminate keeps the candidate
            stages.append(FilterStage(d, w.dimension, len(cands), w.degree, tracked, len(cands) - len(kept)))
            cands = kept
        if cands:
            reg = _restricted_regular_batch(level.embedding, np.array([c.coordinates for c in cands]))
            survivors = [c for c, r in zip(cands, reg) if r]
        else:
            survivors = []
        if survivors:
            witness_sets.append(WitnessSet(d, level.embedding, survivors, label=f"dimension-{d}"))
    return witness_sets, stages


def classify_isolated(candidates: list, witness_sets: list, base_system, p: int = 1,
                      params: TrackParams = TrackParams(), mode: str = "gpu"):
    """Regular vs singular dimension-0 points, then the membership chain
    for the singular ones (filtering.py:204-256)."""
    if not _check_mode(mode):
        return refbridge.classify_isolated(candidates, witness_sets, base_system, p, params, mode)
    stages: list[FilterStage] = []
    regular: list[Solution] = []
    singular: list[Solution] = []
    if candidates:
        X = np.array([c.coordinates for c in candidates])
        r1 = refine_batch(base_system, X, tol=1e-13, max_iters=8)
        pol, _ = refine_dd_batch(base_system, r1.x.copy(), steps=12)
        r2 = refine_batch(base_system, pol, tol=0.0, max_iters=0)
        nv = base_system.nvars
        for i in range(len(candidates)):
            if r2.residual[i] <= max(r1.residual[i] * 10, 1e-12):
                sol, rank = r2.solution(i), int(r2.rank[i])
            else:
                sol, rank = r1.solution(i), int(r1.rank[i])
            (regular if rank == nv else singular).append(sol)
    regular = _dedup(regular)
    singular = _dedup(singular)
    for w in sorted(witness_sets, key=lambda w: -w.dimension):
        if not singular:
            stages.append(FilterStage(0, w.dimension, 0, w.degree, 0, 0))
            continue
        Q = np.array([c.coordinates for c in singular])
        verdict, tracked = membership_batch(w, Q, p, params, mode)
        kept = [c for c, v in zip(singular, verdict) if v != 1]
        stages.append(FilterStage(0, w.dimension, len(singular), w.degree, tracked, len(singular) - len(kept)))
        singular = kept
    return regular, singular, stages
