// Streamed term-record evaluator of the table-driven tracker for large
// systems (n > 10: C3/C4's 14-variable embedding, 4,068 terms).
//
// The table is too large for the parameter bank or L1, so every warp streams
// its rows' terms from L2.  The host lays each warp group's terms out as one
// contiguous run of 64-byte records (coefficients, |c|, factor list),
// grouped per row by factor count (tracker row groups, capi.cu), and a warp
// pulls them through a double-buffered ring in shared memory with cp.async:
// 8 records (512 B, one 16-byte piece per lane) per chunk, the next chunk in
// flight while the current one is evaluated -- the L2 latency is paid once
// per 8 terms instead of once or twice per term.
//
// A term's factor list holds every variable once per unit of exponent
// (x^2 y -> x, x, y), so every term is a product of K factors and the
// partials are the leave-one-out products of polynomials.py:236-256
// (`_StackedEvaluator`) with no exponent logic: for a repeated variable the
// leave-one-out products of its positions sum to a * x^(a-1) * rest.  A
// position that repeats the previous variable folds its partial into the
// first position of the run, which alone updates the Jacobian entry.
//
// Runs (capi.cu): a row's terms are grouped by factor count and, up to four
// factors, by repeat pattern (run descriptor y: count | 0x100 | pattern << 9),
// so those runs' term bodies are instantiated per pattern: repeats fold
// statically and each distinct variable is loaded once.  Inside a run the
// records are laid out as [lead single][pairs of terms with disjoint
// variables][singles] (y bit 28, bits 16..27): a pair is told by its position
// and its two product chains are interleaved.  y bit 30 marks runs with
// per-path coefficients (membership targets); other runs skip that test.
#pragma once
#include "track_rows.cuh"

namespace rec {

using rows::SLOTS;

constexpr int CHUNK = 8;  // records per chunk (32 lanes x 16 bytes)
constexpr int KMAX = 12;  // factors per record
constexpr int PAIRK = 6;  // terms of at most this many factors are paired (register budget)

NID_D unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

// one chunk of records [r0, r0 + 8) into the ring slot `buf` (every lane one
// 16-byte piece), committed as its own group
NID_D void fetch(const TermRec* recs, int r0, TermRec* buf, int lane) {
  const char* src = reinterpret_cast<const char*>(recs + r0) + lane * 16;
  const unsigned dst = smem_u32(reinterpret_cast<char*>(buf) + lane * 16);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src) : "memory");
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}
NID_D void wait_one() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }

// One term of factor count K, record `R` (in shared memory), at the slot's
// point xs (|x| in axs), in three phases so two terms with disjoint
// variables can be interleaved (term2): load (coefficient, Jacobian entries,
// point), compute (prefix products, leave-one-out partials, repeat folding),
// commit (active lanes add into the slot's Jacobian row).
template <int K>
struct TermState {
  static constexpr int KK = K > 0 ? K : 1;
  int v[KK];
  cd Jv[KK], X[KK], d[KK];
  cd p;
  double m;
  unsigned dup;
  double acs, act;
};

// DUP: the run's repeat pattern when the host has grouped the run by it (bit j:
// position j repeats position j-1's variable; K <= SDUPK), or -1 for a run whose
// records carry their own pattern.  A static pattern loads each distinct
// variable's point, modulus and Jacobian entry once and folds the repeats'
// partials without selects; the products are the same in the same order.
constexpr int SDUPK = 4;
template <int DUP>
NID_D constexpr bool rep(int j) {
  return DUP >= 0 && j > 0 && ((DUP >> j) & 1);
}

template <int N, int K, int DUP = -1>
NID_D void t_load(TermState<K>& S, const TermRec& R, const cd* xs, const double* axs, bool ws, bool td, cd alpha,
                  double t, const cd* prm, const cd* row) {
  const unsigned long long meta = R.meta;
  cd ct = cd{R.ctr, R.cti};
  if (prm) {  // per-path coefficients (membership tests): warp-uniform test first
    const int ps = R.pslot;
    if (ps >= 0) ct = prm[ps];
  }
  S.p = td ? t * ct : alpha * cd{R.csr, R.csi} + t * ct;  // the coefficient heads the prefix chain
  S.dup = (unsigned)(meta >> 52) & ~1u;                    // bit 0: the pairing flag, not a repeat
  S.acs = R.acs;
  S.act = R.act;
  S.m = 1.0;
#pragma unroll
  for (int j = 0; j < K; ++j) S.v[j] = (int)((meta >> (4 * j)) & 15);
#pragma unroll
  for (int j = 0; j < K; ++j)
    if (!rep<DUP>(j)) S.Jv[j] = row[S.v[j] * SLOTS];
  double ax = 1.0;
#pragma unroll
  for (int j = 0; j < K; ++j) {
    if (rep<DUP>(j)) {
      S.X[j] = S.X[j - 1];
    } else {
      S.X[j] = xs[S.v[j] * SLOTS];
      if (ws) ax = axs[S.v[j] * SLOTS];
    }
    if (ws) S.m = __dmul_rn(S.m, ax);
  }
}

template <int K>
NID_D void t_compute(TermState<K>& S) {
  cd P[TermState<K>::KK];
  cd p = S.p;
#pragma unroll
  for (int j = 0; j < K; ++j) {
    P[j] = p;
    p = p * S.X[j];
  }
  S.p = p;  // the term's value
  cd s = cd{1.0, 0.0};
#pragma unroll
  for (int j = K - 1; j >= 0; --j) {
    S.d[j] = (j == K - 1) ? P[j] : P[j] * s;
    if (j > 0) s = (j == K - 1) ? S.X[j] : s * S.X[j];
  }
}

template <int K, int DUP = -1>
NID_D void t_commit(TermState<K>& S, cd* row, bool active, bool ws, bool td, cd& hv, double& sS, double& sT) {
  hv = hv + S.p;
  if (DUP >= 0) {  // static repeat pattern
#pragma unroll
    for (int j = K - 1; j > 0; --j)
      if (rep<DUP>(j)) S.d[j - 1] = S.d[j - 1] + S.d[j];
    if (active) {
#pragma unroll
      for (int j = 0; j < K; ++j)
        if (!rep<DUP>(j)) row[S.v[j] * SLOTS] = S.Jv[j] + S.d[j];
    }
  } else if (K > 1 && S.dup) {  // repeated variables (uniform): fold into each run's first position
#pragma unroll
    for (int j = K - 1; j > 0; --j)
      if (S.dup & (1u << j)) S.d[j - 1] = S.d[j - 1] + S.d[j];
    if (active) {
#pragma unroll
      for (int j = 0; j < K; ++j)
        if (!(S.dup & (1u << j))) row[S.v[j] * SLOTS] = S.Jv[j] + S.d[j];
    }
  } else if (active) {
#pragma unroll
    for (int j = 0; j < K; ++j) row[S.v[j] * SLOTS] = S.Jv[j] + S.d[j];
  }
  if (ws) {
    if (!td) sS = __dadd_rn(sS, __dmul_rn(S.acs, S.m));
    sT = __dadd_rn(sT, __dmul_rn(S.act, S.m));
  }
}

template <int N, int K, int DUP = -1>
NID_D void term(const TermRec& R, const cd* xs, const double* axs, bool ws, bool td, cd alpha, double t,
                const cd* prm, cd* row, bool active, cd& hv, double& sS, double& sT) {
  TermState<K> A;
  t_load<N, K, DUP>(A, R, xs, axs, ws, td, alpha, t, prm, row);
  t_compute<K>(A);
  t_commit<K, DUP>(A, row, active, ws, td, hv, sS, sT);
}

// two terms whose variable sets are disjoint (paired on the host): every
// load first, the two product chains interleaved, then both commits
template <int N, int K, int DUP = -1>
NID_D void term2(const TermRec& RA, const TermRec& RB, const cd* xs, const double* axs, bool ws, bool td, cd alpha,
                 double t, const cd* prm, cd* row, bool active, cd& hv, double& sS, double& sT) {
  TermState<K> A, B;
  t_load<N, K, DUP>(A, RA, xs, axs, ws, td, alpha, t, prm, row);
  t_load<N, K, DUP>(B, RB, xs, axs, ws, td, alpha, t, prm, row);
  t_compute<K>(A);
  t_compute<K>(B);
  t_commit<K, DUP>(A, row, active, ws, td, hv, sS, sT);
  t_commit<K, DUP>(B, row, active, ws, td, hv, sS, sT);
}

// the records [kr, kend) of one run (factor count K) through the ring:
// wait for a chunk when the first of its records is reached, refill its
// slot two chunks ahead once all of its records are consumed
template <int N, int K, int DUP = -1>
NID_D void run(const HomDev& H, int base, int& kr, int kend, int p0, int p1, int& cnext, TermRec* ring,
               int lane, const cd* xs, const double* axs, bool ws, bool td, cd alpha, double t, const cd* prm,
               cd* row, bool active, cd& hv, double& sS, double& sT) {
#pragma unroll 1
  while (kr < kend) {
    const int pos = (int)((kr - base) & (2 * CHUNK - 1));
    if ((pos & (CHUNK - 1)) == 0) {  // the chunk holding kr has landed (the next may be in flight)
      wait_one();
      __syncwarp();
    }
    // records [p0, p1) of the run are pairs at even offsets whose two terms share
    // no variable (capi.cu lays a run out as lead single, pairs, singles)
    if (K > 0 && K <= PAIRK && kr >= p0 && kr < p1) {
      term2<N, (K <= PAIRK ? K : 1), (K <= PAIRK ? DUP : -1)>(ring[pos], ring[pos + 1], xs, axs, ws, td, alpha, t, prm,
                                                              row, active, hv, sS, sT);
      kr += 2;
    } else {
      term<N, K, DUP>(ring[pos], xs, axs, ws, td, alpha, t, prm, row, active, hv, sS, sT);
      kr += 1;
    }
    if (((kr - base) & (CHUNK - 1)) == 0) {  // chunk consumed by every lane: refill its slot
      __syncwarp();
      fetch(H.rec, cnext, ring + ((pos & ~(CHUNK - 1))), lane);
      cnext += CHUNK;
    }
  }
}

}  // namespace rec

// The rows of warp group g from the streamed records (same contract as
// rows::eval_rows_fac).  Called by every lane of the warp (the ring needs all
// 32 lanes); `active` lanes own an evaluating slot and alone write it.
// ring: this warp's 2 x 8 records of shared memory.
template <int N>
NID_D void eval_rows_rec(const HomDev& H, const uint4* runs, int g, const cd* xs, double t, const cd* prm, cd* aug,
                         double* dbl, bool want_scale, bool active, double* axw, TermRec* ring) {
  using L = rows::Layout<N>;
  constexpr int S = rows::SLOTS;
  const int lane = threadIdx.x & 31;
  const cd alpha = (1.0 - t) * H.gamma;
  const bool ws = __any_sync(0xffffffffu, want_scale && active);
  const bool td = H.td != 0;
  double r2 = 0.0, mS = 0.0, mT = 0.0;
  // the warp's group index through a shuffle: the compiler then knows it is uniform
  const int gu = __shfl_sync(0xffffffffu, g, 0);
  const int u0 = H.grun[gu], u1 = H.grun[gu + 1];
  if (u0 < u1) {
    // record indices fit 32 bits (a table of 2^31 records would be 128 GB)
    const int base = (int)runs[u0].z;  // the group's first record
    int cnext = base;                             // next chunk to fetch
    rec::fetch(H.rec, cnext, ring, lane);
    cnext += rec::CHUNK;
    rec::fetch(H.rec, cnext, ring + rec::CHUNK, lane);
    cnext += rec::CHUNK;
    int kr = base;  // the next record to evaluate
    int row_i = -1;
    cd* row = aug;
    cd hv = cd{0.0, 0.0};
    double sS = 0.0, sT = 0.0;
#pragma unroll 1
    for (int u = u0; u <= u1; ++u) {
      const uint4 run = u < u1 ? runs[u] : make_uint4(0xffffffffu, 0u, 0u, 0u);
      if ((int)run.x != row_i) {
        if (row_i >= 0) {  // close the previous row: start system, -H, partial maxima
          if (td) {  // G_i = x_i^{d_i} - 1 in closed form
            const int d = H.tddeg[row_i];
            const cd xi = xs[row_i * S];
            cd q = cd{1.0, 0.0};
#pragma unroll 1
            for (int e = 1; e < d; ++e) q = q * xi;
            hv = cfma(alpha, q * xi - cd{1.0, 0.0}, hv);
            if (active) row[row_i * S] = row[row_i * S] + alpha * ((double)d * q);
            if (ws) {
              const double axi = axw[row_i * S];
              double m = 1.0;
#pragma unroll 1
              for (int e = 0; e < d; ++e) m = __dmul_rn(m, axi);
              sS = __dadd_rn(1.0, m);
            }
          }
          if (active) row[N * S] = -hv;
          r2 = nanmax(r2, cabs2(hv));
          mS = fmax(mS, sS);
          mT = fmax(mT, sT);
        }
        if (u == u1) break;
        row_i = (int)run.x;
        row = aug + row_i * (N + 1) * S;
        if (active) {
#pragma unroll
          for (int v = 0; v < N; ++v) row[v * S] = cd{0.0, 0.0};
        }
        hv = cd{0.0, 0.0};
        sS = 0.0;
        sT = 0.0;
      }
      // run.y: factor count K, and for a run grouped by repeat pattern
      // (K <= rec::SDUPK) 0x100 | pattern << 9
      const int K = (int)(run.y & 0xffu);
      const int key = (int)((run.y >> 8) & 0xffu);  // 0: records carry their own pattern
      const cd* const prm_run = ((run.y >> 30) & 1u) ? prm : nullptr;  // runs without parameter slots skip the test
      const int kend = (int)(run.z + run.w);
      const int p0 = (int)run.z + (int)((run.y >> 28) & 1u);          // first pair
      const int p1 = p0 + 2 * (int)((run.y >> 16) & 0xfffu);          // one past the last pair
#define NID_RD(KK, DD)                                                                                       \
  case (KK) | 0x100 | ((DD) << 9):                                                                           \
    rec::run<N, KK, DD>(H, base, kr, kend, p0, p1, cnext, ring, lane, xs, axw, ws, td, alpha, t, prm_run, row, active, hv, \
                        sS, sT);                                                                             \
    break;
#define NID_RT(KK)                                                                                       \
  case KK:                                                                                               \
    rec::run<N, KK>(H, base, kr, kend, p0, p1, cnext, ring, lane, xs, axw, ws, td, alpha, t, prm_run, row, active, hv, \
                    sS, sT);                                                                             \
    break;
      switch (K | (key << 8)) {
        NID_RD(1, 0)
        NID_RD(2, 0) NID_RD(2, 2)
        NID_RD(3, 0) NID_RD(3, 2) NID_RD(3, 4) NID_RD(3, 6)
        NID_RD(4, 0) NID_RD(4, 2) NID_RD(4, 4) NID_RD(4, 6) NID_RD(4, 8) NID_RD(4, 10) NID_RD(4, 12) NID_RD(4, 14)
        NID_RT(0) NID_RT(1) NID_RT(2) NID_RT(3) NID_RT(4) NID_RT(5) NID_RT(6) NID_RT(7) NID_RT(8)
        NID_RT(9) NID_RT(10) NID_RT(11) NID_RT(12)
        default:
          break;
      }
#undef NID_RT
#undef NID_RD
    }
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    __syncwarp();
  }
  if (active) {
    dbl[(L::R2 + g) * S] = r2;
    dbl[(L::SS + g) * S] = mS;
    dbl[(L::ST + g) * S] = mT;
  }
}

// ---------------------------------------------------------------------------
// Per-slot ("latency") evaluation of the streamed records.  The row-per-warp
// evaluator above serves 32 slots per pass, one term at a time per lane: a
// block iteration lasts as long as a warp's walk over its rows' terms (~500
// for C3's heavy rows) whether 32 slots are active or one.  In the tail of a
// small launch (a cascade level of ~5k paths whose slowest path takes 30x the
// mean number of steps) almost every slot is idle, so when at most
// TrackArgs::lat_slots of the block's slots evaluate, each is evaluated here instead: the warp's
// 32 lanes split its rows' terms (lane l takes records l, l+32, ...), each
// lane accumulates into its own row of a per-warp shared-memory scratch, and
// the rows are summed in lane order.  The term arithmetic is t_load /
// t_compute / t_commit's; only the summation order differs, and the switch is
// a function of the path's own step count, so results stay deterministic.
namespace lat {

// per-warp scratch: the slot's point and moduli, then 32 lane rows of NP
// complex (J_v for v < N, H at N, the two abs sums at N+1; NP odd so lane
// rows start in different banks)
template <int N>
constexpr int NP() {
  return (N + 2) | 1;
}
template <int N>
constexpr size_t warp_bytes() {  // xb[N] cd, 32 lane rows of NP cd, axb[N] double; 16-byte multiple
  return ((size_t)N * sizeof(cd) + (size_t)32 * NP<N>() * sizeof(cd) + (size_t)N * sizeof(double) + 15) & ~(size_t)15;
}

template <int N, int K>
NID_D void lane_terms(const TermRec* recs, long long r, long long r1, const cd* xb, const double* axb, bool ws,
                      bool td, cd alpha, double t, const cd* prm, cd* jl, cd& hv, double& sS, double& sT) {
  // (defined on every path: a record first written under `r < r1` counts as live
  // from the function's entry in each of the 13 instantiations, and is spilled)
  TermRec Rn;
  memset(&Rn, 0, sizeof(Rn));
  if (r < r1) Rn = recs[r];
#pragma unroll 1
  for (; r < r1; r += 32) {
    const TermRec R = Rn;
    if (r + 32 < r1) Rn = recs[r + 32];  // the next record's L2 trip overlaps this term
    rec::TermState<(K > 0 ? K : 1)> S;
    cd ct = cd{R.ctr, R.cti};
    if (prm && R.pslot >= 0) ct = prm[R.pslot];
    const cd c = td ? t * ct : alpha * cd{R.csr, R.csi} + t * ct;
    if (K == 0) {
      hv = hv + c;
      if (ws) {
        if (!td) sS = __dadd_rn(sS, R.acs);
        sT = __dadd_rn(sT, R.act);
      }
      continue;
    }
    const unsigned long long meta = R.meta;
    S.p = c;
    S.dup = (unsigned)(meta >> 52) & ~1u;
    S.acs = R.acs;
    S.act = R.act;
    S.m = 1.0;
#pragma unroll
    for (int j = 0; j < K; ++j) S.v[j] = (int)((meta >> (4 * j)) & 15);
#pragma unroll
    for (int j = 0; j < K; ++j) {
      S.Jv[j] = jl[S.v[j]];
      S.X[j] = xb[S.v[j]];
      if (ws) S.m = __dmul_rn(S.m, axb[S.v[j]]);
    }
    rec::t_compute<(K > 0 ? K : 1)>(S);
    // t_commit on the lane's row (stride 1 instead of SLOTS)
    hv = hv + S.p;
    if (K > 1 && S.dup) {
#pragma unroll
      for (int j = K - 1; j > 0; --j)
        if (S.dup & (1u << j)) S.d[j - 1] = S.d[j - 1] + S.d[j];
#pragma unroll
      for (int j = 0; j < K; ++j)
        if (!(S.dup & (1u << j))) jl[S.v[j]] = S.Jv[j] + S.d[j];
    } else {
#pragma unroll
      for (int j = 0; j < K; ++j) jl[S.v[j]] = S.Jv[j] + S.d[j];
    }
    if (ws) {
      if (!td) sS = __dadd_rn(sS, __dmul_rn(S.acs, S.m));
      sT = __dadd_rn(sT, __dmul_rn(S.act, S.m));
    }
  }
}

}  // namespace lat

// The rows of warp group g for ONE slot s (warp-uniform), every lane taking
// part.  xs / axs / aug / dbl: the block's arrays at slot s (stride SLOTS);
// scr: this warp's lat::warp_bytes<N>() of shared memory.
// Out of line: its registers are allocated apart from the block loop's (inlined, it
// pushed the n = 14 kernel into 1.1 KB of spills and cost the row-per-warp pass 14 %).
template <int N>
__device__ __noinline__ void eval_slot_rec(const HomDev& H, int g, const cd* xs, double t, const cd* prm, cd* aug, double* dbl, bool ws,
                         const double* axs, unsigned char* scr) {
  using L = rows::Layout<N>;
  constexpr int S = rows::SLOTS;
  constexpr int NP = lat::NP<N>();
  const int lane = threadIdx.x & 31;
  cd* const xb = reinterpret_cast<cd*>(scr);
  cd* const rowsl = xb + N;  // 32 lane rows of NP
  double* const axb = reinterpret_cast<double*>(rowsl + 32 * NP);
  cd* const jl = rowsl + lane * NP;
  __syncwarp();  // the previous slot's readers are done with the scratch
  if (lane < N) {
    xb[lane] = xs[lane * S];
    axb[lane] = ws ? axs[lane * S] : 0.0;
  }
  const cd alpha = (1.0 - t) * H.gamma;
  const bool td = H.td != 0;
  double r2 = 0.0, mS = 0.0, mT = 0.0;
  const int u0 = H.grun[g], u1 = H.grun[g + 1];
  int row_i = -1;
  cd hv = cd{0.0, 0.0};
  double sS = 0.0, sT = 0.0;
#pragma unroll
  for (int v = 0; v < N; ++v) jl[v] = cd{0.0, 0.0};
  __syncwarp();
#pragma unroll 1
  for (int u = u0; u <= u1; ++u) {
    const uint4 run = u < u1 ? __ldg(&H.runs[u]) : make_uint4(0xffffffffu, 0u, 0u, 0u);
    if ((int)run.x != row_i) {
      if (row_i >= 0) {  // close the row: sum the lane rows in lane order
        jl[N] = hv;
        jl[N + 1] = cd{sS, sT};
        __syncwarp();
        if (lane <= N + 1) {
          cd acc = rowsl[lane];
#pragma unroll 4
          for (int l = 1; l < 32; ++l) acc = acc + rowsl[l * NP + lane];
          if (lane < N) {
            if (td && lane == row_i) {  // start system G_i = x_i^{d_i} - 1, Jacobian term
              const int d = H.tddeg[row_i];
              const cd xi = xb[row_i];
              cd q = cd{1.0, 0.0};
#pragma unroll 1
              for (int e = 1; e < d; ++e) q = q * xi;
              acc = acc + alpha * ((double)d * q);
            }
            aug[(row_i * (N + 1) + lane) * S] = acc;
          } else if (lane == N) {
            cd h = acc;
            if (td) {
              const int d = H.tddeg[row_i];
              const cd xi = xb[row_i];
              cd q = cd{1.0, 0.0};
#pragma unroll 1
              for (int e = 1; e < d; ++e) q = q * xi;
              h = cfma(alpha, q * xi - cd{1.0, 0.0}, h);
            }
            aug[(row_i * (N + 1) + N) * S] = -h;
            r2 = nanmax(r2, cabs2(h));
          } else {  // lane N + 1: the abs sums
            double s0 = acc.re;
            if (td && ws) {
              const double axi = axb[row_i];
              double m = 1.0;
#pragma unroll 1
              for (int e = 0; e < H.tddeg[row_i]; ++e) m = __dmul_rn(m, axi);
              s0 = __dadd_rn(1.0, m);
            }
            mS = fmax(mS, s0);
            mT = fmax(mT, acc.im);
          }
        }
        __syncwarp();
#pragma unroll
        for (int v = 0; v < N; ++v) jl[v] = cd{0.0, 0.0};
        hv = cd{0.0, 0.0};
        sS = 0.0;
        sT = 0.0;
        __syncwarp();
      }
      if (u == u1) break;
      row_i = (int)run.x;
    }
    const int K = (int)(run.y & 0xffu);
    const long long r0 = (long long)run.z + lane;
    long long r1 = (long long)run.z + run.w;
    // runs of the same row and factor count that differ only in their repeat
    // pattern are contiguous: one pass over all of them (each record carries
    // its own pattern), so the 32 lanes stay filled
    while (u + 1 < u1) {
      const uint4 nx = __ldg(&H.runs[u + 1]);
      if ((int)nx.x != row_i || (int)(nx.y & 0xffu) != K) break;
      r1 += nx.w;
      ++u;
    }
    switch (K) {
#define NID_LT(KK)                                                                                          \
  case KK:                                                                                                  \
    lat::lane_terms<N, KK>(H.rec, r0, r1, xb, axb, ws, td, alpha, t, prm, jl, hv, sS, sT);                \
    break;
      NID_LT(0) NID_LT(1) NID_LT(2) NID_LT(3) NID_LT(4) NID_LT(5) NID_LT(6) NID_LT(7) NID_LT(8)
      NID_LT(9) NID_LT(10) NID_LT(11) NID_LT(12)
#undef NID_LT
      default:
        break;
    }
  }
  // partial maxima of this warp's rows for the slot (lanes N and N+1 hold them)
  r2 = __shfl_sync(0xffffffffu, r2, N);
  mS = __shfl_sync(0xffffffffu, mS, N + 1);
  mT = __shfl_sync(0xffffffffu, mT, N + 1);
  if (lane == 0) {
    dbl[(L::R2 + g) * S] = r2;
    dbl[(L::SS + g) * S] = mS;
    dbl[(L::ST + g) * S] = mT;
  }
}
