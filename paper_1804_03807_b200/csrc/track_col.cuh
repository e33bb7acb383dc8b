// Column-owner evaluator of the table-driven tracker for large systems whose
// rows share monomials (C3/C4: eight dense quartics on one 495-monomial
// support; cascade and membership homotopies of the same system).
//
// The row-per-warp evaluator (track_rec.cuh) forms every monomial and its
// leave-one-out partials once per ROW that contains it.  Here the work is cut
// the other way, as the reference's stacked evaluator does (polynomials.py:
// 202-256, `_StackedEvaluator`: one monomial table, then a coefficient
// product): a warp owns COLUMNS of the augmented matrix [J | -H].  For column
// v it walks the monomials m that contain x_v, forms d m / d x_v once for its
// lane's slot, and adds c[r][m] * (d m / d x_v) to a register accumulator per
// row r of the unit's row block (at most eight rows); each cell of the column
// is written once, by its owner -- no read-modify-write of the Jacobian in
// shared memory and no monomial formed more than once per column.  The values
// H_r are the column v = N (the partial is the monomial itself); that column
// is split by monomial ranges over all warps, each warp leaving its partial
// sums in its own scratch area, and the warp that controls a slot adds the
// partial sums in warp order after the evaluation barrier (fixed order:
// results do not depend on the schedule).  The abs-sum noise scale
// (polynomials.py:282-287) is one more unit per row block at the end of a
// warp's stream, skipped when no slot of the block wants it.
//
// Stream format (built in capi.cu): 16-byte pieces.  A record is a header
// {factor list: 4 bits per position, every variable once per unit of
// exponent; bits 48..55 the integer multiplier a_v of the partial; bytes 8..15
// per-row parameter slots} followed by one coefficient piece per row of the
// run's row mask (two, start and target, for runs whose rows blend
// differently).  Runs are described by uint4 words that travel in the
// launch's parameter bank (uniform loop bounds, factor counts, row masks).
// A warp pulls its stream through a four-chunk cp.async ring (32 pieces per
// chunk, one per lane); records may straddle chunks but not the ring's end.
#pragma once
#include "track_rows.cuh"

namespace col {

using rows::SLOTS;

constexpr int RCH = 4;         // ring chunks
constexpr int CP = 32;         // pieces per chunk
constexpr int RP = RCH * CP;   // ring pieces
constexpr int RMAX = 8;        // rows per unit

// run descriptor fields
//  x: column | row0 << 8 | nrows << 16 | first << 24 | last << 25 | kind << 26
//  y: D | mask << 8 | cls << 16 | pieces per record << 20
//  z: first piece (relative to the warp's stream), w: records
enum : int { K_JH = 0, K_ABS = 1 };
enum : int { C_T = 0, C_S = 1, C_B = 2, C_TWO = 3, C_PRM = 4 };

NID_D unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

NID_D void fetch(const uint4* src, uint4* ring, int chunk, int lane) {
  const unsigned dst = smem_u32(ring + (chunk & (RCH - 1)) * CP + lane);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src + (long long)chunk * CP + lane)
               : "memory");
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}

NID_D cd as_cd(const uint4& u) {
  return cd{__hiloint2double((int)u.y, (int)u.x), __hiloint2double((int)u.w, (int)u.z)};
}

// A record never straddles the end of the ring (the host pads to the next
// multiple of RP pieces, same rule), so its pieces are contiguous in shared
// memory: rb[0] the header, rb[1 ...] the coefficients.
// Entering chunk c, chunk c-2's slot is refilled with chunk c+2 (the record in
// hand may still lie in chunk c-1: the pipelined loops below read one record
// ahead), and chunks <= c+1 are waited for.
NID_D void advance(int& q, int len, int& cur, const uint4* src, uint4* ring, int lane) {
  if ((q & (RP - 1)) + len > RP) q = (q + RP - 1) & ~(RP - 1);
  const int c = q >> 5;
  if (c != cur) {
    __syncwarp();
    fetch(src, ring, c + 2, lane);
    asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    __syncwarp();
    cur = c;
  }
}

NID_D const cd* as_cdp(const uint4* p) { return reinterpret_cast<const cd*>(p); }
NID_D int fidx(const uint4& hd, int j) { return (int)(((j < 8 ? hd.x : hd.y) >> (4 * (j & 7))) & 15u) * SLOTS; }

// One-coefficient runs whose FM rows are all present (the bulk: C3's dense
// rows), software pipelined: the next record's header and coefficients are
// loaded while the current record's factors are multiplied.
//   ABS = false: acc[i] += c[i] * (sc * product of the factors)   (the host has
//                folded the partial's integer multiplier into c)
//   ABS = true:  acc[i] += (|cs|, |ct|)[i] * product of the moduli
// DD: the factor count when it is one of 0..4 (unrolled), else -1 (loop over D).
// one record held in (hd, C) while the next is loaded into (hdn, Cn)
template <bool ABS, int DD, int FM>
NID_D void full_stage(const uint4& hd, const cd (&C)[FM], uint4& hdn, cd (&Cn)[FM], bool more, uint4* ring, int& q,
                      int len, int D, const cd* xs, const double* axs, cd sc, bool td, cd (&acc)[RMAX],
                      const uint4* src, int& cur, int lane) {
  // the current record's factors
  cd X[DD > 0 ? DD : 1];
  double A[DD > 0 ? DD : 1];
  if (DD > 0) {
#pragma unroll
    for (int j = 0; j < DD; ++j) {
      if (ABS) A[j] = axs[fidx(hd, j)];
      else X[j] = xs[fidx(hd, j)];
    }
  }
  // the next record's header and coefficients
  q += len;
  if (more) {
    advance(q, len, cur, src, ring, lane);
    const uint4* const rb = ring + (q & (RP - 1));
    hdn = rb[0];
#pragma unroll
    for (int i = 0; i < FM; ++i) Cn[i] = as_cdp(rb)[1 + i];
  }
  if (ABS) {
    double m = 1.0;
    if (DD >= 0) {
#pragma unroll
      for (int j = 0; j < DD; ++j) m = __dmul_rn(m, A[j]);
    } else {
#pragma unroll 1
      for (int j = 0; j < D; ++j) m = __dmul_rn(m, axs[fidx(hd, j)]);
    }
#pragma unroll
    for (int i = 0; i < FM; ++i) {
      if (!td) acc[i].re = __dadd_rn(acc[i].re, __dmul_rn(C[i].re, m));
      acc[i].im = __dadd_rn(acc[i].im, __dmul_rn(C[i].im, m));
    }
  } else {
    cd p = sc;
    if (DD >= 0) {
#pragma unroll
      for (int j = 0; j < DD; ++j) p = p * X[j];
    } else {
#pragma unroll 1
      for (int j = 0; j < D; ++j) p = p * xs[fidx(hd, j)];
    }
#pragma unroll
    for (int i = 0; i < FM; ++i) acc[i] = cfma(C[i], p, acc[i]);
  }
}

template <bool ABS, int DD, int FM>
NID_D void run_full(uint4* ring, int& q, int cnt, int len, int D, const cd* xs, const double* axs, cd sc, bool td,
                    cd (&acc)[RMAX], const uint4* src, int& cur, int lane) {
  if (cnt <= 0) return;
  advance(q, len, cur, src, ring, lane);
  uint4 hdA, hdB;
  cd CA[FM], CB[FM];
  {
    const uint4* const rb = ring + (q & (RP - 1));
    hdA = rb[0];
    hdB = hdA;
#pragma unroll
    for (int i = 0; i < FM; ++i) CB[i] = CA[i] = as_cdp(rb)[1 + i];
  }
  // two records per trip: the buffers swap roles without register moves
  int r = 0;
#pragma unroll 1
  while (true) {
    full_stage<ABS, DD, FM>(hdA, CA, hdB, CB, r + 1 < cnt, ring, q, len, D, xs, axs, sc, td, acc, src, cur, lane);
    if (++r >= cnt) break;
    full_stage<ABS, DD, FM>(hdB, CB, hdA, CA, r + 1 < cnt, ring, q, len, D, xs, axs, sc, td, acc, src, cur, lane);
    if (++r >= cnt) break;
  }
}

template <bool ABS, int FM>
NID_D void run_full_d(uint4* ring, int& q, int cnt, int len, int D, const cd* xs, const double* axs, cd sc, bool td,
                      cd (&acc)[RMAX], const uint4* src, int& cur, int lane) {
  switch (D) {
    case 0: run_full<ABS, 0, FM>(ring, q, cnt, len, D, xs, axs, sc, td, acc, src, cur, lane); break;
    case 1: run_full<ABS, 1, FM>(ring, q, cnt, len, D, xs, axs, sc, td, acc, src, cur, lane); break;
    case 2: run_full<ABS, 2, FM>(ring, q, cnt, len, D, xs, axs, sc, td, acc, src, cur, lane); break;
    case 3: run_full<ABS, 3, FM>(ring, q, cnt, len, D, xs, axs, sc, td, acc, src, cur, lane); break;
    case 4: run_full<ABS, 4, FM>(ring, q, cnt, len, D, xs, axs, sc, td, acc, src, cur, lane); break;
    default: run_full<ABS, -1, FM>(ring, q, cnt, len, D, xs, axs, sc, td, acc, src, cur, lane); break;
  }
}

// Any row mask, any blend class (the slice rows, per-path coefficients): one
// record at a time.  CLS C_T stands for the three one-coefficient classes (sc
// is the blend scalar); C_TWO / C_PRM multiply by the partial's integer
// multiplier here (header bits 48..55), the one-coefficient classes carry it
// in the coefficient.
template <int CLS>
NID_D void run(uint4* ring, int& q, int cnt, int len, int D, unsigned mask, const cd* xs, cd sc, cd alpha, double t,
               const cd* prm, cd (&acc)[RMAX], const uint4* src, int& cur, int lane) {
#pragma unroll 1
  for (int r = 0; r < cnt; ++r) {
    advance(q, len, cur, src, ring, lane);
    const uint4* const rb = ring + (q & (RP - 1));
    const uint4 hd = rb[0];
    cd p = (CLS >= C_TWO) ? cd{1.0, 0.0} : sc;
    if (CLS >= C_TWO) {
      const int em = (int)(hd.y >> 16) & 0xff;
      if (em != 1) p = (double)em * p;
    }
#pragma unroll 1
    for (int j = 0; j < D; ++j) p = p * xs[fidx(hd, j)];
    cd pa, pt;
    if (CLS >= C_TWO) {
      pa = alpha * p;
      pt = t * p;
    }
    int cq = 1;
#pragma unroll
    for (int i = 0; i < RMAX; ++i) {
      if ((mask >> i) & 1u) {
        if (CLS >= C_TWO) {
          const cd cs = as_cdp(rb)[cq];
          cd ct = as_cdp(rb)[cq + 1];
          if (CLS == C_PRM && prm) {
            const int ps = (int)(signed char)(((i < 4 ? hd.z : hd.w) >> (8 * (i & 3))) & 0xffu);
            if (ps >= 0) ct = prm[ps];
          }
          acc[i] = cfma(cs, pa, cfma(ct, pt, acc[i]));
          cq += 2;
        } else {
          acc[i] = cfma(as_cdp(rb)[cq], p, acc[i]);
          cq += 1;
        }
      }
    }
    q += len;
  }
}

// abs sums, any row mask: acc[i] = (sum |cs| |m|, sum |ct| |m|)
NID_D void run_abs(uint4* ring, int& q, int cnt, int len, int D, unsigned mask, const double* axs, bool td,
                   cd (&acc)[RMAX], const uint4* src, int& cur, int lane) {
#pragma unroll 1
  for (int r = 0; r < cnt; ++r) {
    advance(q, len, cur, src, ring, lane);
    const uint4* const rb = ring + (q & (RP - 1));
    const uint4 hd = rb[0];
    double m = 1.0;
#pragma unroll 1
    for (int j = 0; j < D; ++j) m = __dmul_rn(m, axs[fidx(hd, j)]);
    int cq = 1;
#pragma unroll
    for (int i = 0; i < RMAX; ++i) {
      if ((mask >> i) & 1u) {
        const cd a = as_cdp(rb)[cq];  // (|cs|, |ct|)
        if (!td) acc[i].re = __dadd_rn(acc[i].re, __dmul_rn(a.re, m));
        acc[i].im = __dadd_rn(acc[i].im, __dmul_rn(a.im, m));
        cq += 1;
      }
    }
    q += len;
  }
}

}  // namespace col

// The units of warp group g (same outputs as eval_rows_rec, except that the
// values H_r are left as per-warp partial sums in `hpart` [row][slot] and the
// residual partial maxima are zero: col_reduce completes them).  Called by
// every lane of the warp; `active` lanes own an evaluating slot.
// Out of line, like eval_slot_rec: its accumulators get registers of their own
// (inlined into the 255-register block loop they were placed in local memory).
template <int N>
NID_D void eval_cols(const HomDev& H, const uint4* runs, int g, const cd* xs, double t, const cd* prm, cd* aug,
                     double* dbl, bool want_scale, bool active, const double* axw, uint4* ring, cd* hpart) {
  using L = rows::Layout<N>;
  constexpr int S = rows::SLOTS;
  const int lane = threadIdx.x & 31;
  const cd alpha = (1.0 - t) * H.gamma;
  const cd beta = cd{alpha.re + t, alpha.im};
  const bool ws = __any_sync(0xffffffffu, want_scale && active);
  const bool td = H.td != 0;
  double mS = 0.0, mT = 0.0;
  const int gu = __shfl_sync(0xffffffffu, g, 0);
  const int u0 = H.cgrun[gu], u1 = H.cgrun[gu + 1];
  const uint4* const src = H.crec + H.cgbase[gu];
  col::fetch(src, ring, 0, lane);
  col::fetch(src, ring, 1, lane);
  col::fetch(src, ring, 2, lane);
  asm volatile("cp.async.wait_group 1;\n" ::: "memory");
  __syncwarp();
  int cur = 0, q = 0;
  // defined on every path from here (a register first written under the unit's
  // `first` flag would count as live around the whole block loop and be spilled)
  cd acc[col::RMAX];
#pragma unroll
  for (int i = 0; i < col::RMAX; ++i) acc[i] = cd{0.0, 0.0};
#pragma unroll 1
  for (int u = u0; u < u1; ++u) {
    const uint4 run = runs[u];
    const int kind = (int)((run.x >> 26) & 3u);
    if (kind == col::K_ABS && !ws) break;  // the abs units close the stream
    if ((run.x >> 24) & 1u) {
#pragma unroll
      for (int i = 0; i < col::RMAX; ++i) acc[i] = cd{0.0, 0.0};
    }
    const int D = (int)(run.y & 0xffu);
    const unsigned mask = (run.y >> 8) & 0xffu;
    const int cls = (int)((run.y >> 16) & 0xfu);
    const int len = (int)((run.y >> 20) & 0x3fu);
    const int cnt = (int)run.w;
    q = (int)run.z;
    if (kind == col::K_ABS) {
      if (mask == 0x0fu) col::run_full_d<true, 4>(ring, q, cnt, len, D, xs, axw, alpha, td, acc, src, cur, lane);
      else col::run_abs(ring, q, cnt, len, D, mask, axw, td, acc, src, cur, lane);
    } else if (cls == col::C_TWO) {
      col::run<col::C_TWO>(ring, q, cnt, len, D, mask, xs, alpha, alpha, t, prm, acc, src, cur, lane);
    } else if (cls == col::C_PRM) {
      col::run<col::C_PRM>(ring, q, cnt, len, D, mask, xs, alpha, alpha, t, prm, acc, src, cur, lane);
    } else {
      const cd sc = cls == col::C_T ? cd{t, 0.0} : (cls == col::C_S ? alpha : beta);
      if (mask == 0xffu) col::run_full_d<false, 8>(ring, q, cnt, len, D, xs, axw, sc, td, acc, src, cur, lane);
      else col::run<col::C_T>(ring, q, cnt, len, D, mask, xs, sc, alpha, t, prm, acc, src, cur, lane);
    }
    if ((run.x >> 25) & 1u) {  // the unit's last run: write its cells
      const int v = (int)(run.x & 0xffu), row0 = (int)((run.x >> 8) & 0xffu), nr = (int)((run.x >> 16) & 0xffu);
      if (kind == col::K_ABS) {
#pragma unroll
        for (int i = 0; i < col::RMAX; ++i)
          if (i < nr) {
            double s0 = acc[i].re;
            if (td) {  // start system x_i^{d_i} - 1: abs sum 1 + |x_i|^{d_i}
              const double axi = axw[(row0 + i) * S];
              double m = 1.0;
#pragma unroll 1
              for (int e = 0; e < H.tddeg[row0 + i]; ++e) m = __dmul_rn(m, axi);
              s0 = __dadd_rn(1.0, m);
            }
            mS = fmax(mS, s0);
            mT = fmax(mT, acc[i].im);
          }
      } else if (v == N) {  // values: this warp's partial sums
        if (active) {
#pragma unroll
          for (int i = 0; i < col::RMAX; ++i)
            if (i < nr) hpart[(row0 + i) * S] = acc[i];
        }
      } else {
#pragma unroll
        for (int i = 0; i < col::RMAX; ++i)
          if (i < nr) {
            cd cell = acc[i];
            if (td && row0 + i == v) {  // d/dx_v of alpha (x_v^{d_v} - 1)
              const int d = H.tddeg[v];
              const cd xi = xs[v * S];
              cd qq = cd{1.0, 0.0};
#pragma unroll 1
              for (int e = 1; e < d; ++e) qq = qq * xi;
              cell = cell + alpha * ((double)d * qq);
            }
            if (active) aug[((row0 + i) * (N + 1) + v) * S] = cell;
          }
      }
    }
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  __syncwarp();
  if (active) {
    dbl[(L::R2 + g) * S] = 0.0;
    dbl[(L::SS + g) * S] = mS;
    dbl[(L::ST + g) * S] = mT;
  }
}

// After the evaluation barrier: the warp that controls CPW slots adds the G
// warps' partial sums of H_r in warp order, adds the closed-form start system,
// writes -H_r into the augmented column and max |H_r|^2 into the slot's
// residual entry (group 0's; the others were left zero).  lane = q * CPW + sl:
// slot g * CPW + sl, rows q, q + G, ...  `doit`: the slot was evaluated by
// eval_cols this iteration (uniform over the slot's G lanes).
template <int N, int G, int CPW>
NID_D void col_reduce(const HomDev& H, int g, int lane, bool doit, cd* cb, double* part, const cd* xe, double t,
                      const unsigned char* scr0, size_t warp_stride) {
  using L = rows::Layout<N>;
  constexpr int S = rows::SLOTS;
  const int sl = lane % CPW, q = lane / CPW;
  const int ss = g * CPW + sl;
  double r2 = 0.0;
  if (doit) {
    const cd alpha = (1.0 - t) * H.gamma;
#pragma unroll
    for (int r = q; r < N; r += G) {
      cd h = reinterpret_cast<const cd*>(scr0)[r * S + ss];
#pragma unroll
      for (int w = 1; w < G; ++w) h = h + reinterpret_cast<const cd*>(scr0 + w * warp_stride)[r * S + ss];
      if (H.td) {
        const int d = H.tddeg[r];
        const cd xi = xe[r * S + ss];
        cd qq = cd{1.0, 0.0};
#pragma unroll 1
        for (int e = 1; e < d; ++e) qq = qq * xi;
        h = cfma(alpha, qq * xi - cd{1.0, 0.0}, h);
      }
      cb[(r * (N + 1) + N) * S + ss] = -h;
      r2 = nanmax(r2, cabs2(h));
    }
  }
#pragma unroll
  for (int o = CPW; o < 32; o <<= 1) r2 = nanmax(r2, __shfl_xor_sync(0xffffffffu, r2, o));
  if (doit && q == 0) part[(L::R2 + 0) * S + ss] = r2;
}
