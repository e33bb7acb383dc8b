// K1: evaluation of a lowered LinearHomotopy, one lane per row.
//
// Replaces LinearHomotopy.eval/.jac/.eval_scale (tracker.py:81-92) and the
// stacked evaluator underneath (polynomials.py:202-256, eval_magnitude
// :282-287).  Start and target rows are merged into one term table; a term
// contributes c(t) * x^a with c(t) = (1-t) gamma c_start + t c_target, so
// rows shared by both systems cost one monomial pass instead of two.
//
// Lane i of a path group owns row i: it forms each term's monomial and all
// of its partial derivatives from one prefix pass and one suffix pass over
// the exponent vector (shared factors: the leave-one-out product of every
// variable), accumulating H_i and the full Jacobian row i in registers.
// The point x is held, complete, by every lane of the group.
#pragma once
#include "nid_common.cuh"

struct HomDev {
  int n, nterms, nparam, maxdeg;
  const int* row_off;     // [n+1]
  const uint4* expo;      // [nterms], 16 exponent bytes
  const cd* cs;           // start coefficients
  const cd* ct;           // target coefficients
  const double* acs;      // |cs|
  const double* act;      // |ct|
  const int8_t* pslot;    // per-path target coefficient slot or null
  cd gamma;
};

NID_D cd ldg_c(const cd* p) {
  double2 v = __ldg(reinterpret_cast<const double2*>(p));
  return cd{v.x, v.y};
}

NID_D int expo_at(const unsigned (&w)[4], int v) { return (w[v >> 2] >> (8 * (v & 3))) & 0xff; }

NID_D cd cpow_small(cd x, int a) {  // x^a, a >= 1, by repeated products like the reference's power table
  cd r = x;
  for (int e = 1; e < a; ++e) r = r * x;
  return r;
}

// Row `row` of H(x, t), its Jacobian row, and the start/target abs sums
// (sum |c| |x|^a) when want_scale.  Rows >= n evaluate to zero.
template <int N>
NID_D void eval_row(const HomDev& H, int row, const cd (&x)[N], double t, const cd* prm, cd& hv,
                    cd (&J)[N], double& sS, double& sT, bool want_scale) {
  const cd alpha = (1.0 - t) * H.gamma;
  hv = cd{0.0, 0.0};
#pragma unroll
  for (int v = 0; v < N; ++v) J[v] = cd{0.0, 0.0};
  sS = 0.0;
  sT = 0.0;
  int k0 = 0, k1 = 0;
  if (row < H.n) {
    k0 = __ldg(H.row_off + row);
    k1 = __ldg(H.row_off + row + 1);
  }
  for (int k = k0; k < k1; ++k) {
    uint4 ew = __ldg(H.expo + k);
    const unsigned w[4] = {ew.x, ew.y, ew.z, ew.w};
    cd cs = ldg_c(H.cs + k), ct = ldg_c(H.ct + k);
    if (H.pslot != nullptr) {
      int s = H.pslot[k];
      if (s >= 0) ct = prm[s];
    }
    const cd c = alpha * cs + t * ct;
    // prefix products P[v] = prod_{u<v} x_u^{a_u}
    cd P[N];
    cd p = cd{1.0, 0.0};
#pragma unroll
    for (int v = 0; v < N; ++v) {
      P[v] = p;
      int a = expo_at(w, v);
      if (a == 1) p = p * x[v];
      else if (a > 1) p = p * cpow_small(x[v], a);
    }
    hv = cfma(c, p, hv);
    // suffix sweep: d/dx_v = a_v x_v^{a_v-1} * P[v] * S[v]
    cd s = cd{1.0, 0.0};
#pragma unroll
    for (int v = N - 1; v >= 0; --v) {
      int a = expo_at(w, v);
      if (a == 1) {
        J[v] = cfma(P[v] * s, c, J[v]);
        s = s * x[v];
      } else if (a > 1) {
        cd q = cpow_small(x[v], a - 1);
        J[v] = cfma(P[v] * s, (double)a * (c * q), J[v]);
        s = s * (q * x[v]);
      }
    }
  }
  if (want_scale) {
    double ax[N];
#pragma unroll
    for (int v = 0; v < N; ++v) ax[v] = cabsd(x[v]);
    for (int k = k0; k < k1; ++k) {
      uint4 ew = __ldg(H.expo + k);
      const unsigned w[4] = {ew.x, ew.y, ew.z, ew.w};
      double m = 1.0;
#pragma unroll
      for (int v = 0; v < N; ++v) {
        int a = expo_at(w, v);
        double pv = 1.0;
        for (int e = 0; e < a; ++e) pv = __dmul_rn(pv, ax[v]);
        m = __dmul_rn(m, pv);
      }
      sS = __dadd_rn(sS, __dmul_rn(__ldg(H.acs + k), m));
      sT = __dadd_rn(sT, __dmul_rn(__ldg(H.act + k), m));
    }
  }
}

// Value-only variant (no Jacobian), used where only residuals are needed.
template <int N>
NID_D cd eval_row_value(const HomDev& H, int row, const cd (&x)[N], double t, const cd* prm) {
  const cd alpha = (1.0 - t) * H.gamma;
  cd hv = cd{0.0, 0.0};
  int k0 = 0, k1 = 0;
  if (row < H.n) {
    k0 = __ldg(H.row_off + row);
    k1 = __ldg(H.row_off + row + 1);
  }
  for (int k = k0; k < k1; ++k) {
    uint4 ew = __ldg(H.expo + k);
    const unsigned w[4] = {ew.x, ew.y, ew.z, ew.w};
    cd cs = ldg_c(H.cs + k), ct = ldg_c(H.ct + k);
    if (H.pslot != nullptr) {
      int s = H.pslot[k];
      if (s >= 0) ct = prm[s];
    }
    const cd c = alpha * cs + t * ct;
    cd p = cd{1.0, 0.0};
#pragma unroll
    for (int v = 0; v < N; ++v) {
      int a = expo_at(w, v);
      if (a == 1) p = p * x[v];
      else if (a > 1) p = p * cpow_small(x[v], a);
    }
    hv = cfma(c, p, hv);
  }
  return hv;
}
