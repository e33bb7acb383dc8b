// The auxiliary tracker kernel: the same state machine as track_ctl_kernel
// (track_body), instantiated once more per size for the two modes that are
// kept out of the throughput kernels' instruction streams:
//
//   * double-double tracking (TrackParams.precision = "double_double",
//     tracker.py:458-497 `_DDView` / `_track_dd`): every H and J evaluation
//     runs in complex double-double arithmetic at the double point and is
//     rounded to double; the correction steps are solved in double; there is
//     no evaluation-noise floor (`_DDView` has no eval_scale, so
//     `_effective_tol` returns the requested tolerance, tracker.py:177-181);
//   * the per-step trace hook of `track(..., trace=list)` (tracker.py:345,
//     393-394): (t, step, corrector iterations) of every accepted step.
//
// The evaluator walks the merged term table through L1 like the factor-list
// evaluator (no streamed records, no per-slot latency mode).
#pragma once
#include "dd.cuh"
#include "track_ctl.cuh"

namespace aux {

using rows::SLOTS;

NID_D cdd cdd_scale_int(cdd a, int k) {  // k * a, k a small integer (exact factor)
  const dd kk = dd{(double)k, 0.0};
  return cdd{dd_mul(a.re, kk), dd_mul(a.im, kk)};
}

// H rows of warp group g at the slot's point in complex double-double:
// term k contributes c_k(t) x^a with c_k(t) = gamma (1 - t) cs_k + t ct_k
// formed in double-double (LinearHomotopy.eval_generic / jac_generic,
// tracker.py:94-106, over eval_poly_generic, polynomials.py:293-314: the
// reference sums the start and the target system separately and combines the
// sums; the difference is of double-double rounding size).  Partial
// derivatives come from one prefix and one suffix pass over the term's
// variables.  Results are rounded to double into the augmented matrix.
template <int N>
NID_D void dd_rows(const HomDev& H, int g, const cd* xs, double t, const cd* prm, cd* aug, double* dbl) {
  using L = rows::Layout<N>;
  cdd x[N];
#pragma unroll
  for (int v = 0; v < N; ++v) x[v] = cdd_from(xs[v * SLOTS]);
  const cdd gam = cdd_from((1.0 - t) * H.gamma);
  const cdd tt = cdd_from(cd{t, 0.0});
  double r2 = 0.0;
#pragma unroll 1
  for (int gi = H.goff[g]; gi < H.goff[g + 1]; ++gi) {
    const int i = H.grow[gi];
    cd* const row = aug + i * (N + 1) * SLOTS;
    cdd hv = cdd_zero();
    cdd Jr[N];
#pragma unroll
    for (int v = 0; v < N; ++v) Jr[v] = cdd_zero();
    const int k0 = __ldg(H.row_off + i), k1 = __ldg(H.row_off + i + 1);
#pragma unroll 1
    for (int k = k0; k < k1; ++k) {
      cd ct = ldg_c(H.ct + k);
      if (H.pslot != nullptr) {
        const int sl = __ldg(H.pslot + k);
        if (sl >= 0) ct = prm[sl];
      }
      cdd c = cdd_mul(tt, cdd_from(ct));
      if (!H.td) c = cdd_add(cdd_mul(gam, cdd_from(ldg_c(H.cs + k))), c);
      const uint4 ew = __ldg(H.expo + k);
      const unsigned w[4] = {ew.x, ew.y, ew.z, ew.w};
      // the term's variables: full power x^a and derivative factor a x^(a-1)
      cdd F[N], D[N], P[N];
      int var[N];
      int K = 0;
#pragma unroll 1
      for (int u = 0; u < N; ++u) {
        const int a = expo_at(w, u);
        if (a == 0) continue;
        cdd pw = cdd_from(cd{1.0, 0.0});
        for (int e = 1; e < a; ++e) pw = cdd_mul(pw, x[u]);
        F[K] = a == 1 ? x[u] : cdd_mul(pw, x[u]);
        D[K] = a == 1 ? pw : cdd_scale_int(pw, a);
        var[K] = u;
        ++K;
      }
      cdd p = c;
#pragma unroll 1
      for (int q = 0; q < K; ++q) {
        P[q] = p;
        p = cdd_mul(p, F[q]);
      }
      hv = cdd_add(hv, p);
      cdd s = cdd_from(cd{1.0, 0.0});
#pragma unroll 1
      for (int q = K - 1; q >= 0; --q) {
        const int u = var[q];
        cdd d = cdd_mul(cdd_mul(P[q], D[q]), s);
        // Jr is indexed dynamically: keep the update in one place
#pragma unroll
        for (int v = 0; v < N; ++v)
          if (v == u) Jr[v] = cdd_add(Jr[v], d);
        s = cdd_mul(s, F[q]);
      }
    }
    if (H.td) {  // G_i = x_i^{d_i} - 1
      const int d = H.tddeg[i];
      cdd q = cdd_from(cd{1.0, 0.0});
      for (int e = 1; e < d; ++e) q = cdd_mul(q, x[i]);
      const cdd gi_ = cdd_sub(cdd_mul(q, x[i]), cdd_from(cd{1.0, 0.0}));
      hv = cdd_add(hv, cdd_mul(gam, gi_));
      const cdd dj = cdd_mul(gam, cdd_scale_int(q, d));
#pragma unroll
      for (int v = 0; v < N; ++v)
        if (v == i) Jr[v] = cdd_add(Jr[v], dj);
    }
#pragma unroll
    for (int v = 0; v < N; ++v) row[v * SLOTS] = cdd_to(Jr[v]);
    const cd h = cdd_to(hv);
    row[N * SLOTS] = -h;
    r2 = nanmax(r2, cabs2(h));
  }
  dbl[(L::R2 + g) * SLOTS] = r2;
  dbl[(L::SS + g) * SLOTS] = 0.0;  // no noise floor in double-double mode
  dbl[(L::ST + g) * SLOTS] = 0.0;
}

}  // namespace aux

// evaluator policy of the auxiliary kernel (no kTable flag: the streamed-record
// and per-slot paths of track_body are compiled out)
template <int N>
struct AuxEval {
  static NID_D void rows(const HomDev& H, int g, const cd (&x)[N], double t, const cd* prm, cd* aug, double* part,
                         bool want_scale, const cd* xs, double* axw) {
    if (H.dd) {
      aux::dd_rows<N>(H, g, xs, t, prm, aug, part);
    } else {
      rows::eval_rows_fac<N>(H, g, xs, t, prm, aug, part, want_scale, axw);
    }
  }
};

template <int N>
__global__ void __launch_bounds__(rows::groups<N>() * 32, 1) track_aux_kernel(const __grid_constant__ TrackArgs Ar) {
  track_body<N, AuxEval<N>, void, false, true>(Ar, nullptr);
}
