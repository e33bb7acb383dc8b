"""Seeded synthetic inputs for the five BASELINE.json configs.

Every coefficient comes from `rng.stream(seed, CONFIG_COEFFS)`; gamma for the
total-degree continuation is the reference's own `stream(seed, GAMMA)` draw
(cascade.py:226); embeddings use `embed(f, k, seed)` (systems.py:228-240).
The seeds are fixed here and recorded in DESIGN.md.

C1  dense quadrics, n=4 (16 paths)
C2  cyclic support, n=7 (5,040 paths)
C3  h1*p_i + h2*r_i, n=8, embedded with 6 slacks (65,536 top paths + cascade)
C3m the n=4 analog of C3 embedded with 2 slacks (256 top paths): CI stand-in
C4  membership on the C3 component (100,000 candidates x 4 paths)
C5  cyclic support, n=10 (3,628,800 paths)
"""

from __future__ import annotations

from dataclasses import dataclass
from itertools import product

import numpy as np

from . import rng as rngmod
from .polys import PolySystem, make_poly, poly_add, poly_mul
from .systems import EmbeddedSystem, embed, total_degree_start

SEEDS = {"C1": 1, "C2": 2, "C3": 3, "C3m": 33, "C4": 3, "C5": 5}


def quadric_exponents(n: int):
    return sorted(e for e in product(range(3), repeat=n) if sum(e) <= 2)


def dense_quadric(n: int, gen: np.random.Generator):
    ex = quadric_exponents(n)
    c = gen.normal(size=len(ex)) + 1j * gen.normal(size=len(ex))
    return make_poly(n, zip(ex, c))


def dense_quadrics(n: int, seed: int) -> PolySystem:
    """C1: n rows, each with every monomial of degree <= 2, N(0,1)+iN(0,1)."""
    gen = rngmod.stream(seed, rngmod.CONFIG_COEFFS)
    return PolySystem(n, tuple(dense_quadric(n, gen) for _ in range(n)))


def cyclic_support(n: int, seed: int) -> PolySystem:
    """C2/C5: row k = sum_i c_{k,i} prod_{j<k} x_{(i+j) mod n} (k=1..n-1),
    row n = c_n x_0...x_{n-1} - c_0, every c uniform on the unit circle."""
    gen = rngmod.stream(seed, rngmod.CONFIG_COEFFS)
    rows = []
    for k in range(1, n):
        c = rngmod.unit_complex(gen, n)
        terms = []
        for i in range(n):
            e = [0] * n
            for j in range(k):
                e[(i + j) % n] += 1
            terms.append((e, c[i]))
        rows.append(make_poly(n, terms))
    cn, c0 = rngmod.unit_complex(gen, 2)
    rows.append(make_poly(n, [((1,) * n, cn), ((0,) * n, -c0)]))
    return PolySystem(n, tuple(rows))


@dataclass(frozen=True)
class PositiveDimensional:
    """f_i = h1 p_i + h2 r_i; the component {h1 = h2 = 0} has dimension n-2
    and degree 4."""

    f: PolySystem
    h1: object
    h2: object
    emb: EmbeddedSystem
    seed: int


def positive_dimensional(n: int, seed: int, k: int | None = None) -> PositiveDimensional:
    gen = rngmod.stream(seed, rngmod.CONFIG_COEFFS)
    h1 = dense_quadric(n, gen)
    h2 = dense_quadric(n, gen)
    rows = []
    for _ in range(n):
        p = dense_quadric(n, gen)
        r = dense_quadric(n, gen)
        rows.append(poly_add(poly_mul(h1, p), poly_mul(h2, r)))
    f = PolySystem(n, tuple(rows))
    k = n - 2 if k is None else k
    return PositiveDimensional(f, h1, h2, embed(f, k, seed), seed)


@dataclass(frozen=True)
class TotalDegreeProblem:
    """A square target F with its total-degree start G and gamma."""

    name: str
    target: PolySystem
    start: PolySystem
    gamma: complex
    degrees: tuple

    @property
    def n(self) -> int:
        return self.target.nvars

    @property
    def paths(self) -> int:
        return int(np.prod(self.degrees, dtype=np.int64))


def total_degree_problem(name: str, target: PolySystem, seed: int) -> TotalDegreeProblem:
    g = total_degree_start(target)
    return TotalDegreeProblem(name, target, g, rngmod.gamma_for(seed), tuple(target.degrees()))


def c1() -> TotalDegreeProblem:
    return total_degree_problem("C1", dense_quadrics(4, SEEDS["C1"]), SEEDS["C1"])


def c2() -> TotalDegreeProblem:
    return total_degree_problem("C2", cyclic_support(7, SEEDS["C2"]), SEEDS["C2"])


def c5() -> TotalDegreeProblem:
    return total_degree_problem("C5", cyclic_support(10, SEEDS["C5"]), SEEDS["C5"])


def c3() -> PositiveDimensional:
    return positive_dimensional(8, SEEDS["C3"], 6)


def c3_mini() -> PositiveDimensional:
    return positive_dimensional(4, SEEDS["C3m"], 2)


def c3_top(pd: PositiveDimensional) -> TotalDegreeProblem:
    """Total-degree continuation onto the top embedding."""
    return total_degree_problem("C3top", pd.emb.system, pd.seed)


def component_slice_system(pd: PositiveDimensional, hyper) -> PolySystem:
    """{h1 = h2 = 0} cut by n-2 affine hyperplanes (rows of `hyper`, each
    [c0, a_1..a_n]): a square system in the n original variables whose 4
    roots lie on the component."""
    n = pd.f.nvars
    rows = [pd.h1, pd.h2]
    for c in hyper:
        terms = [((0,) * n, c[0])]
        for l in range(n):
            e = [0] * n
            e[l] = 1
            terms.append((e, c[l + 1]))
        rows.append(make_poly(n, terms))
    return PolySystem(n, tuple(rows))


def membership_candidates_offcomponent(n: int, count: int, seed: int) -> np.ndarray:
    gen = rngmod.stream(seed, rngmod.CONFIG_CANDIDATES, 1)
    return gen.normal(size=(count, n)) + 1j * gen.normal(size=(count, n))


def random_slices(n: int, count: int, seed: int) -> np.ndarray:
    """count random (n-2) x (n+1) hyperplane blocks (each cuts a 2-dim
    affine slice of C^n) for the on-component sampler (SURVEY §7 open
    decision 2)."""
    gen = rngmod.stream(seed, rngmod.CONFIG_CANDIDATES, 2)
    return rngmod.random_complex(gen, count * (n - 2) * (n + 1)).reshape(count, n - 2, n + 1)


def slice_homotopy(pd: PositiveDimensional, gamma_seed: int = 0):
    """Total-degree homotopy onto {h1 = h2 = 0} cut by n-2 hyperplanes whose
    coefficients are per-path parameters (one slice per 2^2 = 4 paths): the
    C4 on-component sampler as a single launch."""
    from .homotopy import LinearHomotopy, lower

    n = pd.f.nvars
    template = component_slice_system(pd, np.ones((n - 2, n + 1)))
    start = total_degree_start(template)
    slots = {}
    for j in range(n - 2):
        for l in range(n + 1):
            e = [0] * n
            if l:
                e[l - 1] = 1
            slots[(2 + j, tuple(e))] = j * (n + 1) + l
    gamma = rngmod.gamma_for(gamma_seed if gamma_seed else pd.seed, 7)
    low = lower(start, template, gamma, slots)
    return low, tuple(template.degrees())


def c4_candidates(pd: PositiveDimensional, n_on: int, n_off: int, seed: int, params=None):
    """n_on points on the component (random 2-dim slices, 4 points each,
    tracked on the GPU) and n_off iid complex N(0,1) points; returns
    (candidates [n_on + n_off, n], labels)."""
    from .homotopy import DeviceHomotopy, TrackParams
    from .tracker import track_batch

    n = pd.f.nvars
    n_slices = (n_on + 3) // 4
    low, degrees = slice_homotopy(pd)
    dev = DeviceHomotopy(low)
    hyper = random_slices(n, n_slices, seed)  # (slices, n-2, n+1)
    prm = hyper.reshape(n_slices, -1)
    paths = 4 * n_slices
    starts = np.tile(total_degree_starts_np(degrees), (n_slices, 1))
    res = track_batch(dev, starts, params or TrackParams(), target_params=prm, param_div=4)
    ok = res.succeeded
    on = res.x[ok][:n_on]
    off = membership_candidates_offcomponent(n, n_off, seed)
    cands = np.concatenate([on, off])
    labels = np.concatenate([np.ones(len(on), np.int8), np.zeros(len(off), np.int8)])
    return cands, labels, {"slices": n_slices, "slice_paths": paths, "slice_finite": int(ok.sum())}


def total_degree_starts_np(degrees):
    from .systems import total_degree_starts

    return total_degree_starts(degrees)
