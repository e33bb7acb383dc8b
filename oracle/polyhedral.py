"""ORACLE -- CPU restatement of the reference's per-cell polyhedral homotopy.

Test infrastructure only (see oracle/nid_oracle.py): used by `tests/` as the
checker of the GPU per-cell tracker, never by the product path.  Pinned
against the reference's own `solve_cell` outputs in
`tests/golden/polyhedral_{c1,c2}.npz` (tests/golden/make_polyhedral.py).

Restates:
  * PolyhedralHomotopy   polyhedral.py:730-791 (coefficients weighted by
    t^(rescaled lifted slack); the Jacobian terms carry the weight of the
    term they come from; eval_scale over |c| with the same weights)
  * binomial_solutions   polyhedral.py:696-727 (column Hermite reduction,
    then the triangular binomial system root by root)
  * solve_cell           polyhedral.py:794-811
"""

from __future__ import annotations

import cmath

import numpy as np

from . import nid_oracle as O

SLACK_MARGIN = 1e-9  # polyhedral.py:30


def rescale_texps(texps):
    """Exponents > SLACK_MARGIN divided by the smallest of them, else 0
    (polyhedral.py:784-789)."""
    raw = np.asarray(texps, dtype=float)
    pos = raw[raw > SLACK_MARGIN]
    scale = 1.0 / pos.min() if pos.size else 1.0
    return np.where(raw > SLACK_MARGIN, raw * scale, 0.0)


class _WBlock:
    """Rows of (exponent, coefficient, weight index) terms; evaluates
    sum_k c_k w_k x^a_k per row for a weight vector w."""

    def __init__(self, rows, nvars):
        self.nrows = len(rows)
        self.rows = rows
        self.nvars = nvars

    def __call__(self, x, w):
        out = np.zeros(self.nrows, dtype=np.complex128)
        for i, terms in enumerate(self.rows):
            s = 0j
            for e, c, k in terms:
                m = 1.0 + 0j
                for v, a in enumerate(e):
                    if a:
                        m *= x[v] ** a
                s += c * w[k] * m
            out[i] = s
        return out


class PolyhedralHomotopy:
    """polyhedral.py:730-791.  `supports[i]` lists row i's exponents in the
    order of g.polys[i].terms; `texps` is the concatenation of the cell's
    per-row lifted slacks (one per support point)."""

    def __init__(self, g, texps, supports):
        n = g.nvars
        self.g = g
        self.dim = n
        rows, jrows, arows = [], [], []
        k = 0
        for i, p in enumerate(g.polys):
            pts = supports[i]
            if len(p.terms) != len(pts):
                raise ValueError("start system terms must align with the support")
            row = []
            for e, (_, c) in zip(pts, p.terms):
                row.append((tuple(e), complex(c), k))
                k += 1
            rows.append(row)
            arows.append([(e, abs(c), kk) for e, c, kk in row])
            for j in range(n):
                d = []
                for e, c, kk in row:
                    if e[j]:
                        de = list(e)
                        de[j] -= 1
                        d.append((tuple(de), c * e[j], kk))
                jrows.append(d)
        self.texp = rescale_texps(texps)
        if self.texp.size != k:
            raise ValueError("one t-exponent per support point")
        self._ev = _WBlock(rows, n)
        self._jev = _WBlock(jrows, n)
        self._aev = _WBlock(arows, n)

    def _w(self, t):
        return float(t) ** self.texp

    def eval(self, x, t):
        return self._ev(np.asarray(x, dtype=np.complex128), self._w(t))

    def jac(self, x, t):
        return self._jev(np.asarray(x, dtype=np.complex128), self._w(t)).reshape(self.dim, self.dim)

    def eval_scale(self, x, t):
        xa = np.abs(np.asarray(x, dtype=np.complex128)).astype(np.complex128)
        v = self._aev(xa, self._w(t))
        return float(np.max(v.real)) if v.size else 0.0

    # double-double polishing only happens at t = 1: the plain start system
    def eval_generic(self, x, t):
        assert t == 1.0
        return O.eval_cdd(self.g, x)

    def jac_generic(self, x, t):
        assert t == 1.0
        return O.jacobian_cdd(self.g, x)


def _column_hermite(V):
    """Unimodular U with V U lower triangular, positive diagonal (Euclid on
    columns; the restatement of polyhedral.py:658-693)."""
    n = len(V)
    M = [list(map(int, r)) for r in V]
    U = [[int(i == j) for j in range(n)] for i in range(n)]

    def colop(j, k, q):
        for r in range(n):
            M[r][j] -= q * M[r][k]
            U[r][j] -= q * U[r][k]

    def swap(j, k):
        for r in range(n):
            M[r][j], M[r][k] = M[r][k], M[r][j]
            U[r][j], U[r][k] = U[r][k], U[r][j]

    for k in range(n):
        while True:
            nz = [j for j in range(k, n) if M[k][j] != 0]
            if not nz:
                raise ValueError("singular binomial exponent matrix")
            p = min(nz, key=lambda j: abs(M[k][j]))
            if p != k:
                swap(p, k)
            done = True
            for j in range(k + 1, n):
                if M[k][j]:
                    colop(j, k, M[k][j] // M[k][k])
                    if M[k][j]:
                        done = False
            if done:
                break
        if M[k][k] < 0:
            for r in range(n):
                M[r][k] = -M[r][k]
                U[r][k] = -U[r][k]
    return M, U


def binomial_solutions(V, beta):
    """All torus solutions of y^(rows of V) = beta (polyhedral.py:696-727)."""
    n = len(V)
    L, U = _column_hermite(V)
    sols = []
    w = [0j] * n

    def descend(k):
        if k == n:
            sols.append(np.array([np.prod([w[j] ** U[l][j] for j in range(n)]) for l in range(n)],
                                 dtype=np.complex128))
            return
        rhs = complex(beta[k])
        for j in range(k):
            rhs = rhs / w[j] ** L[k][j]
        m = L[k][k]
        r = abs(rhs) ** (1.0 / m)
        th = cmath.phase(rhs)
        for l in range(m):
            w[k] = r * cmath.exp(1j * (th + 2.0 * cmath.pi * l) / m)
            descend(k + 1)

    descend(0)
    return sols


def cell_starts(g, pairs):
    """The cell's binomial start points (polyhedral.py:800-808)."""
    n = g.nvars
    coeff_of = [dict((tuple(int(v) for v in e), complex(c)) for e, c in p.terms) for p in g.polys]
    V, beta = [], []
    for i, (a, b) in enumerate(pairs):
        a, b = tuple(int(v) for v in a), tuple(int(v) for v in b)
        V.append([b[j] - a[j] for j in range(n)])
        beta.append(-coeff_of[i][a] / coeff_of[i][b])
    return binomial_solutions(V, beta)


def solve_cell(g, pairs, texps, supports, params=O.TrackParams()):
    """polyhedral.py:794-811"""
    h = PolyhedralHomotopy(g, texps, supports)
    return [O.track(h, y0, params) for y0 in cell_starts(g, pairs)]
