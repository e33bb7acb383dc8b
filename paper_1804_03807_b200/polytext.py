"""The reference's plain-text polynomial system format
(`nidpipe/polytext.py:1-160`): what `nidpipe solve FILE --mode gpu` reads.

    nvars npolys
    (1.0+0.5*i)*x1^2*x3 - 2*x2 + (0.0-1.0*i);
    ...

One `;`-terminated polynomial per entry, variables x1..xN, coefficients as
parenthesised complex literals `(re+im*i)` or plain real numbers; floats are
printed with shortest-repr decimals so a print/parse round trip is exact.

The parser here is a small tokenizer + recursive descent (the reference
splits strings on top-level signs and `*`); it accepts the same language and
multiplies a term's coefficient factors in the same left-to-right order, so
parsed coefficients are bit-identical to the reference's.
"""

from __future__ import annotations

import re

from .polys import PolySystem, SparsePolynomial, make_poly


class ParseError(ValueError):
    """polytext.py:19-20"""


_TOKEN = re.compile(r"""
    (?P<ws>\s+)
  | (?P<num>(?:\d+\.?\d*|\.\d+)(?:[eE][+-]?\d+)?)
  | (?P<ident>[A-Za-z_][A-Za-z0-9_]*)
  | (?P<group>\([^()]*\))
  | (?P<op>[*^+\-])
""", re.X)


def _tokens(text: str) -> list:
    out, pos = [], 0
    while pos < len(text):
        m = _TOKEN.match(text, pos)
        if not m:
            if text[pos] in "()":
                raise ParseError(f"unbalanced parentheses in {text!r}")
            raise ParseError(f"bad character {text[pos]!r} in {text!r}")
        pos = m.end()
        if m.lastgroup != "ws":
            out.append((m.lastgroup, m.group()))
    return out


def _complex_literal(body: str) -> complex:
    s = body.replace(" ", "").replace("*i", "j").replace("i", "j")
    try:
        return complex(s)
    except ValueError as exc:
        raise ParseError(f"bad complex literal {body!r}") from exc


class _Terms:
    """term { (+|-) term } over one polynomial's token list."""

    def __init__(self, toks: list, nvars: int, src: str):
        self.t, self.i, self.n, self.src = toks, 0, nvars, src

    def peek(self):
        return self.t[self.i] if self.i < len(self.t) else (None, None)

    def take(self):
        tok = self.peek()
        self.i += 1
        return tok

    def signs(self) -> float:
        s = 1.0
        while self.peek() in (("op", "+"), ("op", "-")):
            if self.take()[1] == "-":
                s = -s
        return s

    def factor(self, coef: complex, expo: list) -> complex:
        # a real factor may carry its own sign after '*' ("2*-3*x1")
        neg = ""
        if self.peek() in (("op", "+"), ("op", "-")):
            neg = self.take()[1]
            if self.peek()[0] != "num":
                raise ParseError(f"bad factor after {neg!r} in {self.src!r}")
        kind, val = self.take()
        if kind == "group":
            return coef * _complex_literal(val[1:-1])
        if kind == "num":
            return coef * float(neg + val)
        if kind == "ident":
            m = re.fullmatch(r"x(\d+)", val)
            if not m:
                raise ParseError(f"unknown variable {val!r} (expected x1..x{self.n})")
            idx = int(m.group(1)) - 1
            if not 0 <= idx < self.n:
                raise ParseError(f"variable {val!r} out of range for {self.n} variables")
            power = 1
            if self.peek() == ("op", "^"):
                self.take()
                k, p = self.take()
                if k != "num" or not p.isdigit():
                    raise ParseError(f"bad exponent in {self.src!r}")
                power = int(p)
            expo[idx] += power
            return coef
        raise ParseError(f"empty factor in term of {self.src!r}" if kind is None or kind == "op"
                         else f"bad factor {val!r}")

    def term(self):
        coef = complex(self.signs())
        if self.peek()[0] is None:
            raise ParseError("empty term")
        expo = [0] * self.n
        coef = self.factor(coef, expo)
        while self.peek() == ("op", "*"):
            self.take()
            coef = self.factor(coef, expo)
        return tuple(expo), coef

    def poly(self) -> list:
        terms = [self.term()]
        while self.peek()[0] is not None:
            if self.peek() not in (("op", "+"), ("op", "-")):
                raise ParseError(f"expected + or - before {self.peek()[1]!r} in {self.src!r}")
            terms.append(self.term())
        return terms


def parse_system(text: str) -> PolySystem:
    """polytext.py:111-132"""
    lines = text.strip().splitlines()
    if not lines:
        raise ParseError("empty input")
    head = lines[0].split()
    if len(head) != 2:
        raise ParseError(f"first line must be 'nvars npolys', got {lines[0]!r}")
    try:
        nvars, npolys = int(head[0]), int(head[1])
    except ValueError as exc:
        raise ParseError(f"bad header {lines[0]!r}") from exc
    if nvars < 1 or npolys < 0:
        raise ParseError("nvars must be >= 1 and npolys >= 0")
    entries = [e.strip() for e in "\n".join(lines[1:]).split(";")]
    entries = [e for e in entries if e]
    if len(entries) != npolys:
        raise ParseError(f"expected {npolys} polynomials, found {len(entries)}")
    return PolySystem(nvars, tuple(make_poly(nvars, _Terms(_tokens(e), nvars, e).poly()) for e in entries))


def _coef_text(c: complex) -> str:
    """polytext.py:135-138: shortest-repr parts, the sign of the imaginary part explicit"""
    neg = c.imag < 0
    return f"({c.real!r}{'-' if neg else '+'}{(-c.imag if neg else c.imag)!r}*i)"


def format_poly(p: SparsePolynomial) -> str:
    if not p.terms:
        return "(0.0+0.0*i)"
    return " + ".join("*".join([_coef_text(c)] + [f"x{j + 1}" if e == 1 else f"x{j + 1}^{e}"
                                                  for j, e in enumerate(expo) if e >= 1])
                      for expo, c in p.terms)


def format_system(f: PolySystem) -> str:
    return "".join([f"{f.nvars} {len(f.polys)}\n"] + [format_poly(p) + ";\n" for p in f.polys])


def load_system(path) -> PolySystem:
    with open(path, "r", encoding="utf-8") as fh:
        return parse_system(fh.read())


def save_system(f: PolySystem, path) -> None:
    with open(path, "w", encoding="utf-8") as fh:
        fh.write(format_system(f))
