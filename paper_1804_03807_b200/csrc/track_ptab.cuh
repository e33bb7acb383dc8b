// Parameter-space term table: the tracker's evaluator for homotopies whose
// merged table fits the kernel's parameter bank (C1, C2, C5: up to
// PT_MAXT terms and PT_MAXF variable occurrences, no per-path coefficients).
//
// The table travels with the launch as a __grid_constant__ argument, so every
// table word a warp reads is a uniform constant-bank load: a term's variable
// byte offsets land in uniform registers and address the slot's point and
// Jacobian row as [lane base + UR] (no per-lane decode or address
// arithmetic), and its coefficients are uniform FP64 operands.  The
// arithmetic is the factor-list evaluator's (track_rows.cuh) with the
// coefficient folded into the prefix chain: P_0 = c, P_{q+1} = P_q x_q, value
// = P_K, d/dx_q = P_q * (x_{q+1} ... x_{K-1}) -- the shared-factor
// leave-one-out products of polynomials.py:236-256 (`_StackedEvaluator`)
// without the reference's power table.  Each Jacobian entry a term touches is
// read once and written once.
#pragma once
#include "track_common.cuh"
#include "track_rows.cuh"

constexpr int PT_MAXT = 256;   // terms (incl. constants)
constexpr int PT_MAXF = 1536;  // variable occurrences over all terms
constexpr int PT_MAXR = 256;   // runs of equal factor count

struct PTab {
  unsigned short row_run[NID_MAX_VARS + 1];  // runs of row i: [row_run[i], row_run[i+1])
  unsigned short run_k0[PT_MAXR];            // first term of the run
  unsigned short run_f0[PT_MAXR];            // first variable occurrence of the run
  unsigned char run_K[PT_MAXR];              // factor count of the run's terms (0: constants)
  unsigned char run_n[PT_MAXR];              // terms in the run
  cd ct[PT_MAXT];                            // target coefficients
  cd cs[PT_MAXT];                            // start coefficients (unused for a total-degree start)
  double act[PT_MAXT];                       // |ct|
  double acs[PT_MAXT];                       // |cs|
  unsigned foff[PT_MAXF];                    // v * SLOTS * sizeof(cd): byte offset of variable v
  unsigned char fexp[PT_MAXF];               // its exponent
  double tw[PT_MAXT];                        // polyhedral t-exponents (start_kind 2)
  int poly;                                  // coefficient k is ct[k] * t^tw[k]
};

struct TrackArgsPT {
  TrackArgs a;
  PTab t;
};

namespace ptab {

using rows::SLOTS;

NID_D const cd& at(const cd* base, unsigned off) {
  return *reinterpret_cast<const cd*>(reinterpret_cast<const char*>(base) + off);
}
NID_D cd& at(cd* base, unsigned off) { return *reinterpret_cast<cd*>(reinterpret_cast<char*>(base) + off); }
NID_D double atd(const double* base, unsigned off) {  // |x_v| scratch: stride SLOTS doubles = off / 2
  return *reinterpret_cast<const double*>(reinterpret_cast<const char*>(base) + (off >> 1));
}

// the terms of one run (factor count K) of a row
template <int N, int K, bool ML, bool PO>
NID_D void run(const PTab& T, int r, const cd* xs, const double* axs, bool ws, bool td, cd alpha, double t, cd* row,
               cd& hv, double& sS, double& sT, const double* tws) {
  const int k0 = T.run_k0[r], cnt = T.run_n[r], f0 = T.run_f0[r];
#pragma unroll 1
  for (int j = 0; j < cnt; ++j) {
    const int k = k0 + j, fb = f0 + j * K;
    const cd ct = T.ct[k];
    const double tp = PO ? pow(t, tws ? __ldg(tws + k) : T.tw[k]) : 1.0;  // polyhedral.py:764-781
    const cd c = PO ? tp * ct : (td ? t * ct : alpha * T.cs[k] + t * ct);
    // x (and the powers) stay in registers between the two passes for
    // narrow terms; wide terms re-read x in the suffix pass (register budget)
    constexpr bool KEEPX = K <= 6;
    unsigned off[K];
    cd Jv[K], P[K];
    cd X[KEEPX ? K : 1];
    cd Q[(!ML && KEEPX) ? K : 1];
#pragma unroll
    for (int q = 0; q < K; ++q) off[q] = T.foff[fb + q];
#pragma unroll
    for (int q = 0; q < K; ++q) Jv[q] = at(row, off[q]);
    cd p = c;
    double m = 1.0;
#pragma unroll
    for (int q = 0; q < K; ++q) {
      const cd x = at(xs, off[q]);
      P[q] = p;
      cd xa = x;
      if (ML) {
        if (ws) m = __dmul_rn(m, atd(axs, off[q]));
      } else {
        const int a = T.fexp[fb + q];
        const cd qq = a == 1 ? cd{1.0, 0.0} : rows::upow(x, a - 1);
        if (KEEPX) Q[q] = qq;
        xa = a == 1 ? x : qq * x;
        if (ws) {
          const double ax = atd(axs, off[q]);
          double pv = ax;
#pragma unroll 1
          for (int e = 1; e < a; ++e) pv = __dmul_rn(pv, ax);
          m = __dmul_rn(m, pv);
        }
      }
      if (KEEPX) X[q] = xa;
      p = p * xa;
    }
    hv = hv + p;
    cd s = cd{1.0, 0.0};
#pragma unroll
    for (int q = K - 1; q >= 0; --q) {
      cd d = P[q];
      cd xa, qq = cd{1.0, 0.0};
      int a = 1;
      if (KEEPX) {
        xa = X[q];
        if (!ML) qq = Q[q];
      } else {
        xa = at(xs, off[q]);
        if (!ML) {
          a = T.fexp[fb + q];
          if (a != 1) {
            qq = rows::upow(xa, a - 1);
            xa = qq * xa;
          }
        }
      }
      if (!ML) {
        a = T.fexp[fb + q];
        if (a != 1) d = d * ((double)a * qq);
      }
      Jv[q] = (q == K - 1) ? Jv[q] + d : cfma(d, s, Jv[q]);
      if (q > 0) s = (q == K - 1) ? xa : s * xa;
    }
#pragma unroll
    for (int q = 0; q < K; ++q) at(row, off[q]) = Jv[q];
    if (ws) {
      if (PO) m = __dmul_rn(m, tp);
      if (!td) sS = __dadd_rn(sS, __dmul_rn(T.acs[k], m));
      sT = __dadd_rn(sT, __dmul_rn(T.act[k], m));
    }
  }
}

template <int N, bool ML, bool PO>
NID_D void dispatch(const PTab& T, int r, const cd* xs, const double* axs, bool ws, bool td, cd alpha, double t,
                    cd* row, cd& hv, double& sS, double& sT, const double* tws = nullptr) {
  switch (T.run_K[r]) {
#define NID_PT(KK)                                                                                   \
  case KK:                                                                                           \
    if (KK <= N) run<N, (KK <= N ? KK : 1), ML, PO>(T, r, xs, axs, ws, td, alpha, t, row, hv, sS, sT, tws); \
    return;
    NID_PT(1) NID_PT(2) NID_PT(3) NID_PT(4) NID_PT(5) NID_PT(6) NID_PT(7) NID_PT(8)
    NID_PT(9) NID_PT(10) NID_PT(11) NID_PT(12) NID_PT(13) NID_PT(14) NID_PT(15) NID_PT(16)
#undef NID_PT
    default:
      break;
  }
  // constant terms
  const int k0 = T.run_k0[r], cnt = T.run_n[r];
#pragma unroll 1
  for (int k = k0; k < k0 + cnt; ++k) {
    const cd ct = T.ct[k];
    const double tp = PO ? pow(t, tws ? __ldg(tws + k) : T.tw[k]) : 1.0;
    hv = hv + (PO ? tp * ct : (td ? t * ct : alpha * T.cs[k] + t * ct));
    if (ws) {
      if (!td) sS = __dadd_rn(sS, PO ? __dmul_rn(T.acs[k], tp) : T.acs[k]);
      sT = __dadd_rn(sT, PO ? __dmul_rn(T.act[k], tp) : T.act[k]);
    }
  }
}

}  // namespace ptab

// evaluator policy of track_pt_kernel (same contract as TableEval::rows);
// PO: coefficients weighted by t^tw (per-cell polyhedral homotopy)
template <int N, bool PO = false>
struct PTEval {
  static NID_D void rows(const HomDev& H, const PTab& T, int g, double t, cd* aug, double* dbl, bool want_scale,
                         const cd* xs, double* axw, const double* tws = nullptr) {
    using L = rows::Layout<N>;
    constexpr int S = rows::SLOTS;
    const cd alpha = (1.0 - t) * H.gamma;
    const bool ws = __any_sync(__activemask(), want_scale);
    const bool td = H.td != 0;
    // axw: |x_v|, written by the tracker before the evaluation barrier
    double r2 = 0.0, mS = 0.0, mT = 0.0;
    // the warp's group index through a shuffle: the compiler then treats it
    // (and every table word addressed from it) as warp-uniform, so the table
    // is read by uniform constant loads into uniform registers
    // (called in a divergent region: only the lanes whose slot evaluates)
    const unsigned am = __activemask();
    const int gu = __shfl_sync(am, g, __ffs(am) - 1);
#pragma unroll 1
    for (int gi = H.goff[gu]; gi < H.goff[gu + 1]; ++gi) {
      const int i = H.grow[gi];
      cd* const row = aug + i * (N + 1) * S;
#pragma unroll
      for (int v = 0; v < N; ++v) row[v * S] = cd{0.0, 0.0};
      cd hv = cd{0.0, 0.0};
      double sS = 0.0, sT = 0.0;
#pragma unroll 1
      for (int r = T.row_run[i]; r < T.row_run[i + 1]; ++r) {
        if constexpr (PO)  // per-cell polyhedral homotopy (start_kind 2)
          ptab::dispatch<N, false, true>(T, r, xs, axw, ws, td, alpha, t, row, hv, sS, sT, tws);
        else if (H.multilinear)
          ptab::dispatch<N, true, false>(T, r, xs, axw, ws, td, alpha, t, row, hv, sS, sT);
        else
          ptab::dispatch<N, false, false>(T, r, xs, axw, ws, td, alpha, t, row, hv, sS, sT);
      }
      if (td) {  // G_i = x_i^{d_i} - 1 in closed form
        const int d = H.tddeg[i];
        const cd xi = xs[i * S];
        cd q = cd{1.0, 0.0};
#pragma unroll 1
        for (int e = 1; e < d; ++e) q = q * xi;
        hv = cfma(alpha, q * xi - cd{1.0, 0.0}, hv);
        const cd dj = alpha * ((double)d * q);
        row[i * S] = row[i * S] + dj;
        if (ws) {
          const double axi = axw[i * S];
          double m = 1.0;
#pragma unroll 1
          for (int e = 0; e < d; ++e) m = __dmul_rn(m, axi);
          sS = __dadd_rn(1.0, m);
        }
      }
      row[N * S] = -hv;
      r2 = nanmax(r2, cabs2(hv));
      mS = fmax(mS, sS);
      mT = fmax(mT, sT);
    }
    dbl[(L::R2 + g) * S] = r2;
    dbl[(L::SS + g) * S] = mS;
    dbl[(L::ST + g) * S] = mT;
  }
};
