"""Algorithmic FLOP accounting for the roofline.

Unit of work: one tracked path.  Complex mul = 6, complex FMA = 8, real
FMA = 2 FLOP.  For the merged homotopy term table:
  F_eval  = 8 T_H + 6 M            (M: distinct monomials of degree >= 2)
  F_jac   = 8 nnzJ_H + 6 M_J       (M_J: new degree >= 2 monomials of dH)
  F_LU    = (8/3) n^3 + 8 n^2      (LU + two triangular solves)
  F_scale = 2 T_H + M
FLOP/path = N_eval F_eval + N_jac (F_jac + F_LU) + N_scale F_scale with
the executed call counts the kernel reports (the reference's h.eval /
h.jac / h.eval_scale calls).
"""

from __future__ import annotations

from dataclasses import dataclass

from .homotopy import Lowered


@dataclass(frozen=True)
class FlopModel:
    n: int
    T_H: int
    nnzJ_H: int
    M: int
    M_J: int

    @property
    def F_eval(self) -> float:
        return 8 * self.T_H + 6 * self.M

    @property
    def F_jac(self) -> float:
        return 8 * self.nnzJ_H + 6 * self.M_J

    @property
    def F_LU(self) -> float:
        n = self.n
        return 8.0 / 3.0 * n ** 3 + 8 * n ** 2

    @property
    def F_scale(self) -> float:
        return 2 * self.T_H + self.M

    def total(self, evals: float, jacs: float, scales: float) -> float:
        return evals * self.F_eval + jacs * (self.F_jac + self.F_LU) + scales * self.F_scale

    def as_dict(self) -> dict:
        return {"n": self.n, "T_H": self.T_H, "nnzJ_H": self.nnzJ_H, "M": self.M, "M_J": self.M_J,
                "F_eval": self.F_eval, "F_jac": self.F_jac, "F_LU": self.F_LU, "F_scale": self.F_scale}


def flop_model(low: Lowered) -> FlopModel:
    """Counts over the merged start+target term table (a closed-form
    total-degree start is counted as its two terms per row, as in §8(d))."""
    n = low.n
    ex = []
    for i in range(n):
        row = {tuple(int(v) for v in e[:n]) for e in low.expo[low.row_off[i]:low.row_off[i + 1]]}
        if low.start_degrees is not None:
            e = [0] * n
            e[i] = int(low.start_degrees[i])
            row |= {tuple(e), (0,) * n}
        ex.extend(sorted(row))
    mono = {e for e in ex if sum(e) >= 2}
    dmono = set()
    nnz = 0
    for e in ex:
        for v in range(n):
            if e[v]:
                nnz += 1
                d = list(e)
                d[v] -= 1
                d = tuple(d)
                if sum(d) >= 2:
                    dmono.add(d)
    return FlopModel(n, len(ex), nnz, len(mono), len(dmono - mono))
