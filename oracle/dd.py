"""ORACLE (test infrastructure only; never shipped, never on the product path).

Double-double and complex double-double arithmetic, restating the
error-free transformations of the reference `pkg/src/nidpipe/dd.py`:
two_sum (:16-21), quick_two_sum (:24-28), Dekker two_prod with the 2^27+1
splitter (:31-44), DD add/mul/div (:84-133), CDD mul and Smith division
(:217-240), |CDD| = hypot of the rounded parts (:251-252).

Values are plain (hi, lo) tuples; complex values are (re_hi, re_lo, im_hi,
im_lo) tuples.  Only what the endpoint polish needs is provided.
"""

from __future__ import annotations

import math

_SPLIT = 134217729.0


def two_sum(a, b):
    s = a + b
    bb = s - a
    return s, (a - (s - bb)) + (b - bb)


def quick_two_sum(a, b):
    s = a + b
    return s, b - (s - a)


def _split(a):
    c = _SPLIT * a
    hi = c - (c - a)
    return hi, a - hi


def two_prod(a, b):
    p = a * b
    ah, al = _split(a)
    bh, bl = _split(b)
    return p, ((ah * bh - p) + ah * bl + al * bh) + al * bl


def dd_add(x, y):
    s, e = two_sum(x[0], y[0])
    t, f = two_sum(x[1], y[1])
    e += t
    s, e = quick_two_sum(s, e)
    e += f
    return quick_two_sum(s, e)


def dd_neg(x):
    return (-x[0], -x[1])


def dd_sub(x, y):
    return dd_add(x, (-y[0], -y[1]))


def dd_mul(x, y):
    p, e = two_prod(x[0], y[0])
    e += x[0] * y[1] + x[1] * y[0]
    return quick_two_sum(p, e)


def dd_div(x, y):
    q1 = x[0] / y[0]
    r = dd_sub(x, dd_mul(y, (q1, 0.0)))
    q2 = r[0] / y[0]
    r = dd_sub(r, dd_mul(y, (q2, 0.0)))
    q3 = r[0] / y[0]
    s, e = quick_two_sum(q1, q2)
    e += q3
    return quick_two_sum(s, e)


ZERO = (0.0, 0.0, 0.0, 0.0)


def c_from(z: complex):
    return (float(z.real), 0.0, float(z.imag), 0.0)


def c_to(z) -> complex:
    return complex(z[0] + z[1], z[2] + z[3])


def c_add(a, b):
    r = dd_add((a[0], a[1]), (b[0], b[1]))
    i = dd_add((a[2], a[3]), (b[2], b[3]))
    return (r[0], r[1], i[0], i[1])


def c_sub(a, b):
    r = dd_sub((a[0], a[1]), (b[0], b[1]))
    i = dd_sub((a[2], a[3]), (b[2], b[3]))
    return (r[0], r[1], i[0], i[1])


def c_neg(a):
    return (-a[0], -a[1], -a[2], -a[3])


def c_conj(a):
    return (a[0], a[1], -a[2], -a[3])


def c_mul(a, b):
    ar, ai, br, bi = (a[0], a[1]), (a[2], a[3]), (b[0], b[1]), (b[2], b[3])
    r = dd_sub(dd_mul(ar, br), dd_mul(ai, bi))
    i = dd_add(dd_mul(ar, bi), dd_mul(ai, br))
    return (r[0], r[1], i[0], i[1])


def c_div(a, b):
    ar, ai, br, bi = (a[0], a[1]), (a[2], a[3]), (b[0], b[1]), (b[2], b[3])
    if abs(br[0]) >= abs(bi[0]):
        r = dd_div(bi, br)
        den = dd_add(br, dd_mul(bi, r))
        re = dd_div(dd_add(ar, dd_mul(ai, r)), den)
        im = dd_div(dd_sub(ai, dd_mul(ar, r)), den)
    else:
        r = dd_div(br, bi)
        den = dd_add(bi, dd_mul(br, r))
        re = dd_div(dd_add(dd_mul(ar, r), ai), den)
        im = dd_div(dd_sub(dd_mul(ai, r), ar), den)
    return (re[0], re[1], im[0], im[1])


def c_abs(a) -> float:
    return math.hypot(a[0] + a[1], a[2] + a[3])


def c_add_real(a, x: float):
    r = dd_add((a[0], a[1]), (x, 0.0))
    i = dd_add((a[2], a[3]), (0.0, 0.0))
    return (r[0], r[1], i[0], i[1])
