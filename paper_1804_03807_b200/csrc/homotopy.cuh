// K1: evaluation of a lowered LinearHomotopy, one lane per row.
//
// Replaces LinearHomotopy.eval/.jac/.eval_scale (tracker.py:81-92) and the
// stacked evaluator underneath (polynomials.py:202-256, eval_magnitude
// :282-287).  Start and target rows are merged into one term table; a term
// contributes c(t) * x^a with c(t) = (1-t) gamma c_start + t c_target, so
// rows shared by both systems cost one monomial pass instead of two.  A
// total-degree start system G_i = x_i^{d_i} - 1 is not stored as terms: lane
// i evaluates it in closed form.
//
// Lane i of a path group owns row i: it forms each term's monomial and all
// of its partial derivatives from one prefix pass and one suffix pass over
// the exponent vector (shared factors: the leave-one-out product of every
// variable), accumulating H_i and the full Jacobian row i in registers.
// The per-variable work is branch-free (selects, not branches): lanes of a
// warp evaluate different rows with different exponent patterns and must
// not diverge.  Tables whose exponents are all 0/1 (multilinear, e.g. the
// cyclic systems) take a cheaper path; otherwise powers up to the table's
// maximum degree are formed with predicated products.
// The point x is held, complete, by every lane of the group.
#pragma once
#include "nid_common.cuh"

// One term of the streamed record table (track_rec.cuh), 64 bytes: target
// and start coefficients, |ct|, |cs|, and the factor list -- 4 bits per
// position (every variable once per unit of exponent, ascending), bits 48-51
// the factor count K, bits 52-63 the repeat mask (bit j: position j repeats
// position j-1's variable) -- and the per-path coefficient slot (-1: none).
struct __align__(16) TermRec {
  double ctr, cti, csr, csi, acs, act;
  unsigned long long meta;
  int pslot, pad;
};

struct HomDev {
  int n, nterms, nparam, maxdeg;
  int multilinear;        // every table exponent is 0 or 1
  int td;                 // start system is total degree (closed form)
  int tddeg[NID_MAX_VARS];
  // rows of each warp group of the tracker, cost balanced on the host:
  // group g evaluates rows grow[goff[g] .. goff[g+1])
  int grow[NID_MAX_VARS];
  int goff[17];
  const int* row_off;     // [n+1]
  const uint4* expo;      // [nterms], 16 exponent bytes
  // factor lists (tracker evaluator): x,y = indices of the term's variables,
  // ascending, 4 bits each; z = their count.  fex: their exponents, 8 bits each
  const uint4* fac;
  const uint4* fex;
  const cd* cs;           // start coefficients
  const cd* ct;           // target coefficients
  const double* acs;      // |cs|
  const double* act;      // |ct|
  const int8_t* pslot;    // per-path target coefficient slot or null
  cd gamma;
  // per-cell polyhedral homotopy (start_kind 2): coefficient k is
  // ct[k] * t^tw[k] (polyhedral.py:764-781); null for a linear homotopy
  const double* tw;
  // streamed records (n > 10, every term of total degree <= 12) or null:
  // group g evaluates runs [grun[g], grun[g+1]) of `runs` = {row, factor
  // count, first record, records}, whose records are contiguous
  const TermRec* rec;
  const uint4* runs;
  int grun[17];
  // column-owner stream (track_col.cuh) or null: group g walks the runs
  // [cgrun[g], cgrun[g+1]) of the launch's run descriptors over the pieces
  // that start at crec + cgbase[g]
  const uint4* crec;
  int cgrun[17];
  int cgbase[17];
  int dd;  // evaluate in complex double-double (auxiliary kernel, track_aux.cuh); set per launch
};

NID_D cd ldg_c(const cd* p) {
  double2 v = __ldg(reinterpret_cast<const double2*>(p));
  return cd{v.x, v.y};
}

NID_D int expo_at(const unsigned (&w)[4], int v) { return (w[v >> 2] >> (8 * (v & 3))) & 0xff; }

NID_D cd csel(bool c, cd a, cd b) { return cd{c ? a.re : b.re, c ? a.im : b.im}; }

// x^a and a*x^(a-1) for 0 <= a <= maxdeg, branch-free across lanes
// (repeated products like the reference's power table)
NID_D void cpow_pair(cd x, int a, int maxdeg, cd& f, cd& d) {
  cd pw = x, prev = cd{1.0, 0.0};
#pragma unroll 1
  for (int e = 2; e <= maxdeg; ++e) {
    const bool m = e <= a;
    const cd nx = pw * x;
    prev = csel(m, pw, prev);
    pw = csel(m, nx, pw);
  }
  f = csel(a > 0, pw, cd{1.0, 0.0});
  d = csel(a > 0, (double)a * prev, cd{0.0, 0.0});
}

NID_D double rpow_small(double x, int a, int maxdeg) {
  double p = 1.0;
#pragma unroll 1
  for (int e = 1; e <= maxdeg; ++e) p = (e <= a) ? __dmul_rn(p, x) : p;
  return p;
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
  const bool ml = H.multilinear != 0;
  const int maxdeg = H.maxdeg;
  cd xl[N], Jl[N];
#pragma unroll
  for (int v = 0; v < N; ++v) {
    xl[v] = x[v];
    Jl[v] = cd{0.0, 0.0};
  }
  for (int k = k0; k < k1; ++k) {
    uint4 ew = __ldg(H.expo + k);
    const unsigned w[4] = {ew.x, ew.y, ew.z, ew.w};
    cd ct = ldg_c(H.ct + k);
    if (H.pslot != nullptr) {
      int s = H.pslot[k];
      if (s >= 0) ct = prm[s];
    }
    const double tp = H.tw ? pow(t, __ldg(H.tw + k)) : 1.0;
    const cd c = H.tw ? tp * ct : (H.td ? t * ct : alpha * ldg_c(H.cs + k) + t * ct);
    cd P[N];
    cd p = cd{1.0, 0.0};
    if (ml) {
      // prefix products P[v] = prod_{u<v} x_u^{a_u}
#pragma unroll
      for (int v = 0; v < N; ++v) {
        P[v] = p;
        p = csel(expo_at(w, v) != 0, p * x[v], p);
      }
      hv = cfma(c, p, hv);
      // suffix sweep: d/dx_v = P[v] * S[v]
      cd s = cd{1.0, 0.0};
#pragma unroll
      for (int v = N - 1; v >= 0; --v) {
        const bool on = expo_at(w, v) != 0;
        J[v] = csel(on, cfma(P[v] * s, c, J[v]), J[v]);
        s = csel(on, s * x[v], s);
      }
    } else {
      // factor list of the term (its variables ascending, with exponents):
      // the same products in the same order as the variable-by-variable sweep
      // (absent variables multiply by one), without its N-wide predicated work.
      // xl / Jl are indexed per lane (lanes walk different rows): local memory.
      const uint4 fl = __ldg(H.fac + k);
      const uint4 fe = __ldg(H.fex + k);
      const int K = (int)fl.z;
      cd F[N], D[N];
#pragma unroll 1
      for (int q = 0; q < K; ++q) {
        const int v = ((q < 8 ? fl.x : fl.y) >> (4 * (q & 7))) & 15;
        const int a = ((q < 4 ? fe.x : (q < 8 ? fe.y : (q < 12 ? fe.z : fe.w))) >> (8 * (q & 3))) & 255;
        const cd xv = xl[v];
        cd pw = xv, prev = cd{1.0, 0.0};
#pragma unroll 1
        for (int e = 2; e <= a; ++e) {
          prev = pw;
          pw = pw * xv;
        }
        P[q] = p;
        F[q] = pw;
        D[q] = (double)a * prev;
        p = p * pw;
      }
      hv = cfma(c, p, hv);
      cd s = cd{1.0, 0.0};
#pragma unroll 1
      for (int q = K - 1; q >= 0; --q) {
        const int v = ((q < 8 ? fl.x : fl.y) >> (4 * (q & 7))) & 15;
        Jl[v] = cfma(P[q] * s, c * D[q], Jl[v]);
        s = s * F[q];
      }
    }
  }
  if (!ml) {
#pragma unroll
    for (int v = 0; v < N; ++v) J[v] = Jl[v];
  }
  // total-degree start row: G_i = x_i^{d_i} - 1, dG_i/dx_i = d_i x_i^{d_i - 1}
  double xa_td = 0.0;
  if (H.td && row < H.n) {
    const int d = H.tddeg[row];
    const cd xi = pick<N>(x, row);
    cd q = cd{1.0, 0.0};
    for (int e = 1; e < d; ++e) q = q * xi;
    const cd f = q * xi;
    hv = cfma(alpha, f - cd{1.0, 0.0}, hv);
    const cd dj = alpha * ((double)d * q);
#pragma unroll
    for (int v = 0; v < N; ++v) J[v] = csel(v == row, J[v] + dj, J[v]);
    if (want_scale) {
      const double ax = cabsd(xi);
      double m = 1.0;
      for (int e = 0; e < d; ++e) m = __dmul_rn(m, ax);
      xa_td = m;
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
      for (int v = 0; v < N; ++v) m = __dmul_rn(m, rpow_small(ax[v], expo_at(w, v), maxdeg));
      if (H.tw) m = __dmul_rn(m, pow(t, __ldg(H.tw + k)));
      if (!H.td) sS = __dadd_rn(sS, __dmul_rn(__ldg(H.acs + k), m));
      sT = __dadd_rn(sT, __dmul_rn(__ldg(H.act + k), m));
    }
    // |G_i| terms sorted as the reference stores them: constant, then x_i^d
    if (H.td && row < H.n) sS = __dadd_rn(1.0, xa_td);
    // polyhedral: one weighted system, scale = its own abs sum whatever t
    if (H.tw) sS = sT;
  }
}

// Value-only variant (no Jacobian), used where only residuals are needed.
template <int N>
NID_D cd eval_row_value(const HomDev& H, int row, const cd (&x)[N], double t, const cd* prm) {
  cd J[N];
  cd hv;
  double sS, sT;
  eval_row<N>(H, row, x, t, prm, hv, J, sS, sT, false);
  return hv;
}
