"""Sparse complex polynomials and systems: the host-side objects the path
tracker consumes.

Mirrors the term model of the reference (`pkg/src/nidpipe/polynomials.py:24-171`):
a polynomial is a sorted tuple of (exponent tuple, complex coefficient) with
no repeated exponents and no zero coefficients.  Evaluation never happens
here -- points are evaluated on the GPU (`csrc/eval.cuh`) or, for parity
checks only, by the CPU oracle under `oracle/`.  This module only builds and
lowers term lists.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Iterable, Sequence

import numpy as np


class DimensionMismatch(ValueError):
    """Point or polynomial variable count disagrees (polynomials.py:20-21)."""


@dataclass(frozen=True)
class SparsePolynomial:
    nvars: int
    terms: tuple  # ((exponent tuple, complex), ...) sorted by exponent

    def __post_init__(self):
        for e, _ in self.terms:
            if len(e) != self.nvars:
                raise ValueError(f"exponent vector {e} has wrong length")

    @property
    def is_zero(self) -> bool:
        return len(self.terms) == 0

    def degree(self) -> int:
        return max((sum(e) for e, _ in self.terms), default=0)


def make_poly(nvars: int, terms: Iterable[tuple[Sequence[int], complex]]) -> SparsePolynomial:
    """Merge equal exponents, drop zero coefficients, sort (polynomials.py:51-62)."""
    acc: dict[tuple, complex] = {}
    for e, c in terms:
        key = tuple(int(v) for v in e)
        if len(key) != nvars:
            raise ValueError(f"exponent vector {key} has length {len(key)}, expected {nvars}")
        if min(key, default=0) < 0:
            raise ValueError("negative exponent")
        acc[key] = acc.get(key, 0j) + complex(c)
    return SparsePolynomial(nvars, tuple(sorted((k, v) for k, v in acc.items() if v != 0)))


def constant_poly(nvars: int, value: complex) -> SparsePolynomial:
    return make_poly(nvars, [((0,) * nvars, value)])


def variable_poly(nvars: int, index: int) -> SparsePolynomial:
    e = [0] * nvars
    e[index] = 1
    return make_poly(nvars, [(e, 1.0 + 0j)])


def poly_add(p: SparsePolynomial, q: SparsePolynomial) -> SparsePolynomial:
    if p.nvars != q.nvars:
        raise DimensionMismatch("cannot add polynomials in different variable counts")
    return make_poly(p.nvars, list(p.terms) + list(q.terms))


def poly_scale(p: SparsePolynomial, c: complex) -> SparsePolynomial:
    return make_poly(p.nvars, [(e, c * a) for e, a in p.terms])


def poly_mul(p: SparsePolynomial, q: SparsePolynomial) -> SparsePolynomial:
    if p.nvars != q.nvars:
        raise DimensionMismatch("cannot multiply polynomials in different variable counts")
    out = []
    for ea, ca in p.terms:
        for eb, cb in q.terms:
            out.append((tuple(a + b for a, b in zip(ea, eb)), ca * cb))
    return make_poly(p.nvars, out)


def poly_diff(p: SparsePolynomial, var: int) -> SparsePolynomial:
    """d/dx_var, exact (polynomials.py:95-105)."""
    out = []
    for e, c in p.terms:
        k = e[var]
        if k:
            d = list(e)
            d[var] = k - 1
            out.append((tuple(d), c * k))
    return make_poly(p.nvars, out)


def extend_vars(p: SparsePolynomial, nvars: int) -> SparsePolynomial:
    if nvars < p.nvars:
        raise ValueError("cannot shrink variable count")
    pad = (0,) * (nvars - p.nvars)
    return SparsePolynomial(nvars, tuple((e + pad, c) for e, c in p.terms))


@dataclass(frozen=True)
class PolySystem:
    """A tuple of polynomials in one variable set (polynomials.py:134-171)."""

    nvars: int
    polys: tuple
    names: tuple = ()
    _cache: dict = field(default_factory=dict, repr=False, compare=False)

    def __post_init__(self):
        for p in self.polys:
            if p.nvars != self.nvars:
                raise DimensionMismatch("polynomial variable count differs from system")
        if not self.names:
            object.__setattr__(self, "names", tuple(f"x{i + 1}" for i in range(self.nvars)))
        elif len(self.names) != self.nvars:
            raise ValueError("need one name per variable")

    def __len__(self):
        return len(self.polys)

    @property
    def npolys(self) -> int:
        return len(self.polys)

    @property
    def is_square(self) -> bool:
        return len(self.polys) == self.nvars

    def degrees(self) -> list[int]:
        return [p.degree() for p in self.polys]

    def __getstate__(self):
        return (self.nvars, self.polys, self.names)

    def __setstate__(self, state):
        object.__setattr__(self, "nvars", state[0])
        object.__setattr__(self, "polys", state[1])
        object.__setattr__(self, "names", state[2])
        object.__setattr__(self, "_cache", {})


def as_term_rows(system) -> list[list[tuple[tuple, complex]]]:
    """Duck-typed view of any system object exposing ``.polys[i].terms``
    (ours or the reference's), as plain lists."""
    return [[(tuple(int(v) for v in e), complex(c)) for e, c in p.terms] for p in system.polys]


def system_from_rows(nvars: int, rows) -> PolySystem:
    return PolySystem(nvars, tuple(make_poly(nvars, r) for r in rows))
