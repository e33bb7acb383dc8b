// Complex double-double arithmetic for the endpoint polish (K5).
// Same error-free transformations and operation order as the reference
// (pkg/src/nidpipe/dd.py:16-252): two_sum, quick_two_sum, exact two_prod
// (here via FMA, which yields the same exact error term as Dekker's split),
// the accurate DD add, DD mul/div, CDD Smith division, |CDD| = hypot of the
// rounded parts.  __dadd_rn/__dmul_rn keep nvcc from contracting steps
// that the reference rounds separately.
#pragma once
#include "nid_common.cuh"

struct dd {
  double hi, lo;
};
struct cdd {
  dd re, im;
};

NID_D dd two_sum(double a, double b) {
  double s = __dadd_rn(a, b);
  double bb = __dsub_rn(s, a);
  double e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
  return dd{s, e};
}
NID_D dd quick_two_sum(double a, double b) {
  double s = __dadd_rn(a, b);
  return dd{s, __dsub_rn(b, __dsub_rn(s, a))};
}
NID_D dd two_prod(double a, double b) {
  double p = __dmul_rn(a, b);
  return dd{p, fma(a, b, -p)};
}
NID_D dd dd_add(dd x, dd y) {
  dd s = two_sum(x.hi, y.hi);
  dd t = two_sum(x.lo, y.lo);
  double e = __dadd_rn(s.lo, t.hi);
  dd u = quick_two_sum(s.hi, e);
  e = __dadd_rn(u.lo, t.lo);
  return quick_two_sum(u.hi, e);
}
NID_D dd dd_neg(dd x) { return dd{-x.hi, -x.lo}; }
NID_D dd dd_sub(dd x, dd y) { return dd_add(x, dd_neg(y)); }
NID_D dd dd_mul(dd x, dd y) {
  dd p = two_prod(x.hi, y.hi);
  double e = __dadd_rn(p.lo, __dadd_rn(__dmul_rn(x.hi, y.lo), __dmul_rn(x.lo, y.hi)));
  return quick_two_sum(p.hi, e);
}
NID_D dd dd_div(dd x, dd y) {
  double q1 = __ddiv_rn(x.hi, y.hi);
  dd r = dd_sub(x, dd_mul(y, dd{q1, 0.0}));
  double q2 = __ddiv_rn(r.hi, y.hi);
  r = dd_sub(r, dd_mul(y, dd{q2, 0.0}));
  double q3 = __ddiv_rn(r.hi, y.hi);
  dd s = quick_two_sum(q1, q2);
  double e = __dadd_rn(s.lo, q3);
  return quick_two_sum(s.hi, e);
}

NID_D cdd cdd_from(cd z) { return cdd{dd{z.re, 0.0}, dd{z.im, 0.0}}; }
NID_D cd cdd_to(cdd z) { return cd{__dadd_rn(z.re.hi, z.re.lo), __dadd_rn(z.im.hi, z.im.lo)}; }
NID_D cdd cdd_zero() { return cdd{dd{0.0, 0.0}, dd{0.0, 0.0}}; }
NID_D cdd cdd_add(cdd a, cdd b) { return cdd{dd_add(a.re, b.re), dd_add(a.im, b.im)}; }
NID_D cdd cdd_sub(cdd a, cdd b) { return cdd{dd_sub(a.re, b.re), dd_sub(a.im, b.im)}; }
NID_D cdd cdd_neg(cdd a) { return cdd{dd_neg(a.re), dd_neg(a.im)}; }
NID_D cdd cdd_conj(cdd a) { return cdd{a.re, dd_neg(a.im)}; }
NID_D cdd cdd_mul(cdd a, cdd b) {
  return cdd{dd_sub(dd_mul(a.re, b.re), dd_mul(a.im, b.im)),
             dd_add(dd_mul(a.re, b.im), dd_mul(a.im, b.re))};
}
NID_D cdd cdd_div(cdd a, cdd b) {
  if (fabs(b.re.hi) >= fabs(b.im.hi)) {
    dd r = dd_div(b.im, b.re);
    dd den = dd_add(b.re, dd_mul(b.im, r));
    return cdd{dd_div(dd_add(a.re, dd_mul(a.im, r)), den), dd_div(dd_sub(a.im, dd_mul(a.re, r)), den)};
  }
  dd r = dd_div(b.re, b.im);
  dd den = dd_add(b.im, dd_mul(b.re, r));
  return cdd{dd_div(dd_add(dd_mul(a.re, r), a.im), den), dd_div(dd_sub(dd_mul(a.im, r), a.re), den)};
}
NID_D double cdd_abs(cdd a) { return hypot(__dadd_rn(a.re.hi, a.re.lo), __dadd_rn(a.im.hi, a.im.lo)); }
NID_D cdd cdd_add_real(cdd a, double x) { return cdd{dd_add(a.re, dd{x, 0.0}), dd_add(a.im, dd{0.0, 0.0})}; }
