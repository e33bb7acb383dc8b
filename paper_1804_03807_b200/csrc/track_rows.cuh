// Row-split evaluation helpers of the tracker (csrc/track_ctl.cuh): warp g
// of a block evaluates the rows of group g for the block's 32 path slots,
// writing each slot's augmented matrix [J | -H] into shared memory laid out
// [element][slot].
#pragma once
#include "homotopy.cuh"
#include "linalg.cuh"
#include "track_common.cuh"

namespace rows {

constexpr int SLOTS = 32;  // paths per block
#ifndef NID_G10
#define NID_G10 4
#endif

// G: warps per block = threads per path (rows split G ways)
NID_HD constexpr int groups_for(int n) { return n <= 3 ? 1 : (n <= 6 ? 2 : (n <= 10 ? NID_G10 : 8)); }
template <int N>
constexpr int groups() {
  return groups_for(N);
}

// shared-memory layout (complex units unless noted), each [item][slot]
template <int N>
struct Layout {
  static constexpr int G = groups<N>();
  static constexpr int AUG = N * (N + 1);     // augmented matrix
  static constexpr int XO = AUG;              // accepted point
  static constexpr int XS = XO + N;           // x_prev / damped-Newton base
  static constexpr int DS = XS + N;           // damped-Newton direction
  static constexpr int DXS = DS + N;          // Newton step exchange (fallback)
  static constexpr int CPLX = DXS + N;
  // doubles after the complex area: per-group partial maxima
  static constexpr int R2 = 0;                // G entries: max |H_i|^2
  static constexpr int SS = G;                // G entries: max start abs sums
  static constexpr int ST = 2 * G;            // G entries: max target abs sums
  static constexpr int PK = 3 * G;            // G entries: pivot key
  static constexpr int PP = 4 * G;            // G entries: pivot logical position (as double)
  static constexpr int DBL = 5 * G;
  static constexpr size_t bytes() { return (size_t)SLOTS * (CPLX * sizeof(cd) + DBL * sizeof(double) + 8); }
};

template <int N>
NID_D cd& A(cd* base, int i, int j) {  // augmented matrix element of this slot
  return base[(i * (N + 1) + j) * SLOTS];
}

NID_D cd upow(cd x, int a) {
  cd r = x;
#pragma unroll 1
  for (int e = 1; e < a; ++e) r = r * x;
  return r;
}

// ---------------------------------------------------------------------------
// Factor-list evaluator (the tracker's default): a term loops over the K
// variables it contains (K = its factor count, dispatched to a fully
// unrolled body per K) instead of over all n with predicated bodies; the
// point is read from the slot's shared-memory copy and the Jacobian row is
// accumulated in place in the augmented matrix.  The arithmetic -- prefix
// products in ascending variable order, one suffix pass for the partials,
// abs-sum scale -- follows polynomials.py:236-256 (`_StackedEvaluator`).
template <int N, int K, bool ML>
NID_D void fterm(const HomDev& H, int k, const uint4 f, const cd* xs, const double* axs, bool ws, cd c, cd* row,
                 cd& hv, double& m) {
  // A term's variables are distinct, so every Jacobian entry it touches is
  // read up front (overlapping the prefix chain) and written once at the
  // end -- no load-after-store chain through shared memory.  x (and for
  // exponents > 1 the powers) stay in registers between the two passes.
  // Wide non-multilinear terms (K > 6) keep only the prefix products live.
  constexpr bool BATCH = ML || K <= 6;
  cd P[K];
  cd Xr[BATCH ? K : 1];
  cd Qr[(!ML && BATCH) ? K : 1];
  cd Jv[BATCH ? K : 1];
  uint4 fe = make_uint4(0u, 0u, 0u, 0u);
  if (!ML) fe = __ldg(H.fex + k);
  if (BATCH) {
#pragma unroll
    for (int j = 0; j < K; ++j) Jv[j] = row[(((j < 8 ? f.x : f.y) >> (4 * (j & 7))) & 15) * SLOTS];
  }
  cd p = cd{1.0, 0.0};
  m = 1.0;
#pragma unroll
  for (int j = 0; j < K; ++j) {
    const int v = ((j < 8 ? f.x : f.y) >> (4 * (j & 7))) & 15;
    const cd x = xs[v * SLOTS];
    P[j] = p;
    if (ML) {
      Xr[j] = x;
      p = p * x;
      if (ws) m = __dmul_rn(m, axs[v * SLOTS]);
    } else {
      const int a = ((j < 4 ? fe.x : (j < 8 ? fe.y : (j < 12 ? fe.z : fe.w))) >> (8 * (j & 3))) & 255;
      if (BATCH) {
        // x^a = x^(a-1) * x, the same products as upow(x, a)
        const cd q = a == 1 ? cd{1.0, 0.0} : upow(x, a - 1);
        const cd xa = a == 1 ? x : q * x;
        Qr[j] = q;
        Xr[j] = xa;
        p = p * xa;
      } else {
        p = p * (a == 1 ? x : upow(x, a));
      }
      if (ws) {
        const double ax = axs[v * SLOTS];
        double pv = ax;
#pragma unroll 1
        for (int e = 1; e < a; ++e) pv = __dmul_rn(pv, ax);
        m = __dmul_rn(m, pv);
      }
    }
  }
  hv = cfma(c, p, hv);
  cd s = c;
#pragma unroll
  for (int j = K - 1; j >= 0; --j) {
    if (ML) {
      Jv[j] = cfma(P[j], s, Jv[j]);
      s = s * Xr[j];
    } else if (BATCH) {
      const int a = ((j < 4 ? fe.x : (j < 8 ? fe.y : (j < 12 ? fe.z : fe.w))) >> (8 * (j & 3))) & 255;
      if (a == 1) {
        Jv[j] = cfma(P[j], s, Jv[j]);
      } else {
        Jv[j] = cfma(P[j] * ((double)a * Qr[j]), s, Jv[j]);
      }
      s = s * Xr[j];
    } else {
      const int v = ((j < 8 ? f.x : f.y) >> (4 * (j & 7))) & 15;
      const cd x = xs[v * SLOTS];
      cd* const J = row + v * SLOTS;
      const int a = ((j < 4 ? fe.x : (j < 8 ? fe.y : (j < 12 ? fe.z : fe.w))) >> (8 * (j & 3))) & 255;
      if (a == 1) {
        *J = cfma(P[j], s, *J);
        s = s * x;
      } else {
        const cd q = upow(x, a - 1);
        *J = cfma(P[j] * ((double)a * q), s, *J);
        s = s * (q * x);
      }
    }
  }
  if (BATCH) {
#pragma unroll
    for (int j = 0; j < K; ++j) row[(((j < 8 ? f.x : f.y) >> (4 * (j & 7))) & 15) * SLOTS] = Jv[j];
  }
}

// Terms k, k+1, ... of a row while their factor count is K (the host keeps
// rows in table order; equal-count runs are the common case, e.g. every row
// of the cyclic systems): one dispatch per run.  Returns the next term.
template <int N, int K, bool ML>
NID_D int fterm_run(const HomDev& H, int k, int k1, uint4 f, const cd* xs, const double* axs, bool ws, cd alpha,
                    double t, const cd* prm, cd* row, cd& hv, double& sS, double& sT, const double* tws) {
  const int kend = (int)f.w;  // the run's end, precomputed on the host
#pragma unroll 1
  for (;;) {
    // the next term's factor list is fetched while this term computes
    const uint4 fn = k + 1 < kend ? __ldg(H.fac + k + 1) : f;
    cd ct = ldg_c(H.ct + k);
    if (H.pslot != nullptr) {
      const int sl = __ldg(H.pslot + k);
      if (sl >= 0) ct = prm[sl];
    }
    // tws: polyhedral t-exponents (coefficient ct t^w, polyhedral.py:764-781)
    const double tp = tws ? pow(t, __ldg(tws + k)) : 1.0;
    const cd c = tws ? tp * ct : (H.td ? t * ct : alpha * ldg_c(H.cs + k) + t * ct);
    double m;
    fterm<N, K, ML>(H, k, f, xs, axs, ws, c, row, hv, m);
    if (ws) {
      if (tws) m = __dmul_rn(m, tp);
      if (!H.td) sS = __dadd_rn(sS, __dmul_rn(__ldg(H.acs + k), m));
      sT = __dadd_rn(sT, __dmul_rn(__ldg(H.act + k), m));
    }
    if (++k >= kend) break;
    f = fn;
  }
  return k;
}

template <int N, bool ML>
NID_D int fterm_dispatch(const HomDev& H, int k, int k1, const cd* xs, const double* axs, bool ws, cd alpha, double t,
                         const cd* prm, cd* row, cd& hv, double& sS, double& sT, const double* tws) {
  const uint4 f = __ldg(H.fac + k);
  switch (f.z) {
#define NID_FT(KK) \
  case KK:         \
    if (KK <= N) return fterm_run<N, (KK <= N ? KK : 1), ML>(H, k, k1, f, xs, axs, ws, alpha, t, prm, row, hv, sS, sT, tws); \
    break;
    NID_FT(1) NID_FT(2) NID_FT(3) NID_FT(4) NID_FT(5) NID_FT(6) NID_FT(7) NID_FT(8)
    NID_FT(9) NID_FT(10) NID_FT(11) NID_FT(12) NID_FT(13) NID_FT(14) NID_FT(15) NID_FT(16)
#undef NID_FT
    default:
      break;
  }
  // constant term
  cd ct = ldg_c(H.ct + k);
  if (H.pslot != nullptr) {
    const int sl = __ldg(H.pslot + k);
    if (sl >= 0) ct = prm[sl];
  }
  const double tp = tws ? pow(t, __ldg(tws + k)) : 1.0;
  const cd c = tws ? tp * ct : (H.td ? t * ct : alpha * ldg_c(H.cs + k) + t * ct);
  hv = cfma(c, cd{1.0, 0.0}, hv);
  if (ws) {
    if (!H.td) sS = __dadd_rn(sS, __dmul_rn(__ldg(H.acs + k), tp));
    sT = __dadd_rn(sT, __dmul_rn(__ldg(H.act + k), tp));
  }
  return k + 1;
}

// Rows of warp group g into the slot's augmented matrix (as eval_rows).
// xs: the slot's evaluation point in shared memory (stride SLOTS); axw: this
// warp's |x_v| scratch for the slot.
template <int N>
NID_D void eval_rows_fac(const HomDev& H, int g, const cd* xs, double t, const cd* prm, cd* aug, double* dbl,
                         bool want_scale, double* axw, const double* tws = nullptr) {
  using L = Layout<N>;
  const cd alpha = (1.0 - t) * H.gamma;
  const bool ws = __any_sync(__activemask(), want_scale);
  // axw: |x_v|, written by the tracker (track_body) before the evaluation barrier
  double r2 = 0.0, mS = 0.0, mT = 0.0;
#pragma unroll 1
  for (int gi = H.goff[g]; gi < H.goff[g + 1]; ++gi) {
    const int i = H.grow[gi];
    cd* const row = aug + i * (N + 1) * SLOTS;
#pragma unroll
    for (int v = 0; v < N; ++v) row[v * SLOTS] = cd{0.0, 0.0};
    cd hv = cd{0.0, 0.0};
    const int k0 = __ldg(H.row_off + i), k1 = __ldg(H.row_off + i + 1);
    double sS = 0.0, sT = 0.0;
#pragma unroll 1
    for (int k = k0; k < k1;) {
      if (H.multilinear) {
        k = fterm_dispatch<N, true>(H, k, k1, xs, axw, ws, alpha, t, prm, row, hv, sS, sT, tws);
      } else {
        k = fterm_dispatch<N, false>(H, k, k1, xs, axw, ws, alpha, t, prm, row, hv, sS, sT, tws);
      }
    }
    if (H.td) {  // G_i = x_i^{d_i} - 1 in closed form
      const int d = H.tddeg[i];
      const cd xi = xs[i * SLOTS];
      cd q = cd{1.0, 0.0};
#pragma unroll 1
      for (int e = 1; e < d; ++e) q = q * xi;
      hv = cfma(alpha, q * xi - cd{1.0, 0.0}, hv);
      const cd dj = alpha * ((double)d * q);
      row[i * SLOTS] = row[i * SLOTS] + dj;
      if (ws) {
        const double axi = axw[i * SLOTS];
        double m = 1.0;
#pragma unroll 1
        for (int e = 0; e < d; ++e) m = __dmul_rn(m, axi);
        sS = __dadd_rn(1.0, m);
      }
    }
    row[N * SLOTS] = -hv;
    r2 = nanmax(r2, cabs2(hv));
    mS = fmax(mS, tws ? sT : sS);  // polyhedral: one weighted system, (1-t) mT + t mT
    mT = fmax(mT, sT);
  }
  dbl[(L::R2 + g) * SLOTS] = r2;
  dbl[(L::SS + g) * SLOTS] = mS;
  dbl[(L::ST + g) * SLOTS] = mT;
}

// combine the G partial maxima (after a barrier): residual max|H_i| and scale
template <int N>
NID_D double combine_resid(const cd* aug, const double* dbl, double t, double& scale, bool poly = false) {
  using L = Layout<N>;
  double r2 = 0.0, mS = 0.0, mT = 0.0;
#pragma unroll
  for (int g = 0; g < L::G; ++g) {
    r2 = nanmax(r2, dbl[(L::R2 + g) * SLOTS]);
    mS = fmax(mS, dbl[(L::SS + g) * SLOTS]);
    mT = fmax(mT, dbl[(L::ST + g) * SLOTS]);
  }
  scale = poly ? mT : (1.0 - t) * mS + t * mT;  // polyhedral: one weighted system
  if (r2 < 1e290) return sqrt(r2);  // NaN takes the exact path as well
  double resid = 0.0;
#pragma unroll 1
  for (int i = 0; i < N; ++i) resid = nanmax(resid, cabsd(A<N>(const_cast<cd*>(aug), i, N)));  // exact hypot
  return resid;
}

template <int N>
NID_D double norm_inf(const cd (&v)[N]) {
  double m = 0.0;
#pragma unroll
  for (int i = 0; i < N; ++i) m = nanmax(m, cabsd(v[i]));
  return m;
}

template <int N>
NID_D bool all_finite(const cd (&v)[N]) {
  bool f = true;
#pragma unroll
  for (int i = 0; i < N; ++i) f = f && cfinite(v[i]);
  return f;
}

}  // namespace rows

