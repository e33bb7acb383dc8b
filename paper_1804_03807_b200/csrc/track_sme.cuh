// Shared-monomial evaluator of the large-system tracker (n > 10, G = 8
// warps): the rows of C3/C4's embedding share their monomials (the eight
// heavy rows f_i = h1 p_i + h2 r_i all have the same 495-monomial support),
// so each distinct monomial is formed once per slot -- the shared-factor
// products of polynomials.py:236-256 -- instead of once per row.
//
// Monomials are grouped by degree into chunks of at most 8, one per warp.
// Per chunk: every warp forms its monomial for the block's 32 slots (value
// and the leave-one-out partials, repeated variables folded) into a
// double-buffered exchange area in shared memory; one block barrier; every
// warp then streams the consumer records of its own rows for that chunk
// (coefficients, the monomial's slot in the chunk, the local row) through
// its cp.async ring (track_rec.cuh) and accumulates coefficient x value into
// the row and coefficient x partial into the Jacobian entries.  The barrier
// of chunk c+1 also guarantees that chunk c-1's buffer has been consumed
// before it is overwritten.
#pragma once
#include "track_rec.cuh"

namespace sme {

using rows::SLOTS;
constexpr int G = 8;
constexpr int KM = SME_KM;
constexpr int ENT = KM + 1;  // value + partials per monomial and slot

// exchange area per block: [buf][warp][entry][slot] complex, then |m| [buf][warp][slot]
constexpr size_t bytes() { return (size_t)2 * G * ENT * SLOTS * sizeof(cd) + (size_t)2 * G * SLOTS * sizeof(double); }

// the monomial (factor list `meta`, K factors with repeats) at the slot's
// point: value, partials at each run's first position, |value| of |x|
template <int K>
NID_D void produce(unsigned long long meta, const cd* xs, const double* axs, cd* out, double* oabs) {
  int v[K];
#pragma unroll
  for (int j = 0; j < K; ++j) v[j] = (int)((meta >> (4 * j)) & 15);
  const unsigned dup = (unsigned)(meta >> 52);
  cd X[K], P[K];
  cd p = cd{1.0, 0.0};
  double m = 1.0;
#pragma unroll
  for (int j = 0; j < K; ++j) {
    X[j] = xs[v[j] * SLOTS];
    m = __dmul_rn(m, axs[v[j] * SLOTS]);
    P[j] = p;
    p = (j == 0) ? X[0] : p * X[j];
  }
  cd d[K];
  cd s = cd{1.0, 0.0};
#pragma unroll
  for (int j = K - 1; j >= 0; --j) {
    d[j] = (j == K - 1) ? P[j] : (j == 0 ? s : P[j] * s);
    if (j > 0) s = (j == K - 1) ? X[j] : s * X[j];
  }
  if (K > 1 && dup) {
#pragma unroll
    for (int j = K - 1; j > 0; --j)
      if (dup & (1u << j)) d[j - 1] = d[j - 1] + d[j];
  }
  out[0] = p;
#pragma unroll
  for (int j = 0; j < K; ++j) out[(1 + j) * SLOTS] = d[j];
  *oabs = m;
}

// the warp's consumer records of one chunk (factor count K of the chunk's
// monomials) through the ring
template <int N, int K>
NID_D void consume(const HomDev& H, long long base, long long& kr, long long kend, long long& cnext, TermRec* ring,
                   int lane, const cd* ex, const double* eabs, bool ws, bool td, cd alpha, double t, const cd* prm,
                   cd* row0, cd* row1, bool active, cd (&hv)[2], double (&sS)[2], double (&sT)[2]) {
#pragma unroll 1
  for (; kr < kend; ++kr) {
    const int pos = (int)((kr - base) & (2 * rec::CHUNK - 1));
    if ((pos & (rec::CHUNK - 1)) == 0) {
      rec::wait_one();
      __syncwarp();
    }
    const TermRec& R = ring[pos];
    const unsigned pad = (unsigned)R.pad;
    const int li = (pad >> 4) & 15;
    cd ct = cd{R.ctr, R.cti};
    if (prm) {
      const int ps = R.pslot;
      if (ps >= 0) ct = prm[ps];
    }
    const cd c = td ? t * ct : alpha * cd{R.csr, R.csi} + t * ct;
    double m = 1.0;
    cd val;
    if (pad & 0x100) {  // constant term
      val = c;
    } else {
      const int w = pad & 15;
      const cd* e = ex + (size_t)w * ENT * SLOTS;
      val = c * e[0];
      m = eabs[w * SLOTS];
      const unsigned long long meta = R.meta;
      const unsigned dup = (unsigned)(meta >> 52);
      cd* const rowp = li ? row1 : row0;
      if (active) {
#pragma unroll
        for (int j = 0; j < K; ++j) {
          if (!(dup & (1u << j))) {
            cd& J = rowp[(int)((meta >> (4 * j)) & 15) * SLOTS];
            J = cfma(c, e[(1 + j) * SLOTS], J);
          }
        }
      }
    }
    if (li) {
      hv[1] = hv[1] + val;
      if (ws) {
        if (!td) sS[1] = __dadd_rn(sS[1], __dmul_rn(R.acs, m));
        sT[1] = __dadd_rn(sT[1], __dmul_rn(R.act, m));
      }
    } else {
      hv[0] = hv[0] + val;
      if (ws) {
        if (!td) sS[0] = __dadd_rn(sS[0], __dmul_rn(R.acs, m));
        sT[0] = __dadd_rn(sT[0], __dmul_rn(R.act, m));
      }
    }
    if ((pos & (rec::CHUNK - 1)) == rec::CHUNK - 1) {
      __syncwarp();
      rec::fetch(H.srec, cnext, ring + (pos & ~(rec::CHUNK - 1)), lane);
      cnext += rec::CHUNK;
    }
  }
}

}  // namespace sme

// The rows of warp group g (at most two) by shared monomials (same contract
// as eval_rows_rec; called by every lane of every warp: it holds block
// barriers).  xbuf: the block's exchange area (sme::bytes()).
template <int N>
NID_D void eval_rows_sme(const HomDev& H, int g, const cd* xs, double t, const cd* prm, cd* aug, double* dbl,
                         bool want_scale, bool active, double* axw, TermRec* ring, unsigned char* xbuf) {
  using L = rows::Layout<N>;
  constexpr int S = rows::SLOTS;
  constexpr int G = sme::G;
  const int lane = threadIdx.x & 31;
  const cd alpha = (1.0 - t) * H.gamma;
  const bool ws = __any_sync(0xffffffffu, want_scale && active);
  const bool td = H.td != 0;
  cd* const ex = reinterpret_cast<cd*>(xbuf);
  double* const eabs = reinterpret_cast<double*>(xbuf + (size_t)2 * G * sme::ENT * S * sizeof(cd));
  const int gr0 = H.goff[g], nr = H.goff[g + 1] - gr0;
  const int ri0 = nr > 0 ? H.grow[gr0] : 0, ri1 = nr > 1 ? H.grow[gr0 + 1] : ri0;
  cd* const row0 = aug + ri0 * (N + 1) * S;
  cd* const row1 = aug + ri1 * (N + 1) * S;
  if (active) {
#pragma unroll
    for (int v = 0; v < N; ++v) {
      if (nr > 0) row0[v * S] = cd{0.0, 0.0};
      if (nr > 1) row1[v * S] = cd{0.0, 0.0};
    }
  }
  cd hv[2] = {cd{0.0, 0.0}, cd{0.0, 0.0}};
  double sS[2] = {0.0, 0.0}, sT[2] = {0.0, 0.0};
  const long long base = H.sbase[g], send = H.sbase[g + 1];
  long long cnext = base, kr = base;
  if (send > base) {
    rec::fetch(H.srec, cnext, ring, lane);
    cnext += rec::CHUNK;
    rec::fetch(H.srec, cnext, ring + rec::CHUNK, lane);
    cnext += rec::CHUNK;
  }
#pragma unroll 1
  for (int c = 0; c < H.snchunk; ++c) {
    const uint4 ch = __ldg(&H.schunk[c]);
    const int buf = c & 1;
    cd* const exb = ex + (size_t)buf * G * sme::ENT * S;
    double* const eab = eabs + (size_t)buf * G * S;
    if (g < (int)ch.z) {
      const unsigned long long meta = __ldg(&H.smono[ch.y + g]);
      cd* const out = exb + (size_t)g * sme::ENT * S + lane;
      switch (ch.x) {
#define NID_SP(KK)                                                                 \
  case KK:                                                                         \
    sme::produce<KK>(meta, xs, axw, out, eab + g * S + lane);                      \
    break;
        NID_SP(1) NID_SP(2) NID_SP(3) NID_SP(4)
#undef NID_SP
        default:
          break;
      }
    }
    __syncthreads();
    const long long kend = kr + __ldg(&H.scnt[c * G + g]);
    switch (ch.x) {
#define NID_SC(KK)                                                                                                   \
  case KK:                                                                                                           \
    sme::consume<N, KK>(H, base, kr, kend, cnext, ring, lane, exb + lane, eab + lane, ws, td, alpha, t, prm, row0,  \
                        row1, active, hv, sS, sT);                                                                   \
    break;
      NID_SC(1) NID_SC(2) NID_SC(3) NID_SC(4)
#undef NID_SC
      default:
        break;
    }
  }
  if (send > base) {
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    __syncwarp();
  }
  // close the rows: start system in closed form, -H, partial maxima
  double r2 = 0.0, mS = 0.0, mT = 0.0;
#pragma unroll 1
  for (int li = 0; li < nr; ++li) {
    const int ri = li ? ri1 : ri0;
    cd* const row = li ? row1 : row0;
    cd h = li ? hv[1] : hv[0];
    double s0 = li ? sS[1] : sS[0];
    const double s1 = li ? sT[1] : sT[0];
    if (td) {
      const int d = H.tddeg[ri];
      const cd xi = xs[ri * S];
      cd q = cd{1.0, 0.0};
#pragma unroll 1
      for (int e = 1; e < d; ++e) q = q * xi;
      h = cfma(alpha, q * xi - cd{1.0, 0.0}, h);
      if (active) row[ri * S] = row[ri * S] + alpha * ((double)d * q);
      if (ws) {
        const double axi = axw[ri * S];
        double m = 1.0;
#pragma unroll 1
        for (int e = 0; e < d; ++e) m = __dmul_rn(m, axi);
        s0 = __dadd_rn(1.0, m);
      }
    }
    if (active) row[N * S] = -h;
    r2 = nanmax(r2, cabs2(h));
    mS = fmax(mS, s0);
    mT = fmax(mT, s1);
  }
  if (active) {
    dbl[(L::R2 + g) * S] = r2;
    dbl[(L::SS + g) * S] = mS;
    dbl[(L::ST + g) * S] = mT;
  }
}
