// K3 + K4: the persistent path tracker -- controller warp + row-split workers.
//
// A block serves 32 path slots (slot l = lane l) with G warps.  Warp g
// evaluates and eliminates the rows i == g (mod G) of all 32 slots, so every
// warp walks ONE row's term table for 32 different paths: the evaluation
// loops are warp-uniform (coefficients and exponents are broadcast loads,
// absent variables are skipped by uniform branches, the point sits in
// registers).  Each path's augmented Jacobian [J | -H] lives in shared
// memory laid out [element][slot] -- every warp access is one conflict-free
// 512-byte transaction whatever each path's row permutation.
//
// Lanes 0..32/G-1 of every warp are controllers: each runs one slot's state
// machine, whose state lives in shared memory (struct of arrays), claims new
// paths from a global atomic counter -- the GPU form of the reference's
// claim-guarded work crew (parallel.py:37-109) -- publishes the next
// evaluation point and back-substitutes its slot's Newton step.  Per block
// iteration: control -> [barrier] evaluation (all warps, row groups) ->
// [barrier] control -> LU of the warp's own slots (warp-local) -> back
// substitution + control.  Only the two block barriers couple the warps.
// The state machine replays, branch for branch,
//   track           tracker.py:341-407  (secant predictor, step control,
//                                        endgame, snap, infinity test)
//   _correct        tracker.py:184-207  (residual-judged Newton, noise floor)
//   _finish         tracker.py:305-338  (t=1 polish + endpoint verdict)
//   _damped_newton  tracker.py:210-238  (8 halvings, never accept increase)
// newton_step (linalg.py:35-51) is an LU with LAPACK's partial pivoting
// (izamax on |Re|+|Im| in row-swap order, unfused updates) with the zgelsd
// min-norm fallback (solved by the controller lane on a global scratch copy).
#pragma once
#include "track_ptab.cuh"
#include "track_rec.cuh"
#include "track_col.cuh"
#include "track_rows.cuh"

namespace ctl {

using rows::A;
template <class T>
struct is_ptab {
  static constexpr bool value = false;
};
template <>
struct is_ptab<PTab> {
  static constexpr bool value = true;
};
using rows::SLOTS;

// slot state, struct of arrays [field][slot]
enum DField {
  D_TE, D_CTOL, D_CTOLEFF, D_DNLAM, D_DNRES, D_T, D_STEP, D_PREV, D_HSTEP, D_TTRY, D_ENTRY, D_NORMNOW,
  D_MOVECAP, D_TFROM, D_OUTT, D_OUTRES, D_RESID, D_SCALE, D_COUNT
};
enum IField {
  I_ACT, I_MODE, I_CTX, I_CITERS, I_CIT, I_CPHASE, I_CITS, I_DNIT, I_DNTRIAL, I_USED, I_OUTST, I_FLAGS, I_BAD,
  I_COUNT
};
enum Flag { F_COK = 1, F_HAVEPREV = 2, F_ENDGAME = 4, F_NEEDSCALE = 8, F_HASX = 16, F_FALLBACK = 32 };

template <int N>
struct Lay {
  static constexpr int G = rows::groups<N>();
  // complex [item][slot]
  static constexpr int AUG = 0;              // N*(N+1) augmented matrix
  static constexpr int XE = N * (N + 1);     // evaluation point
  static constexpr int CPLX = XE + N;
  // the accepted point, x_prev / damped-Newton base and damped-Newton
  // direction (touched once per step, not per Newton iteration) live in
  // global memory, [block][item][slot] (TrackArgs::gstate): 3 blocks per SM
  static constexpr int GXO = 0, GXS = N, GDS = 2 * N, GITEMS = 3 * N;
  // doubles [item][slot]: slot state + per-group partial maxima / pivot exchange
  static constexpr int DST = 0;
  static constexpr int PART = D_COUNT;       // 3*G: r2, sS, sT per group (reused for pivot key/pos)
  // N: |x_v| of the evaluation point (evaluator scratch; every warp writes
  // the same values for its lane's slot before reading them)
  static constexpr int AXW = PART + 3 * G;
  static constexpr int DBL = AXW + N;
  // long long [item][slot]: path index, parameter row, LU row permutation
  static constexpr int LLN = 3;
  static constexpr size_t bytes() {
    return (size_t)SLOTS * (CPLX * sizeof(cd) + DBL * sizeof(double) + LLN * sizeof(long long) +
                            I_COUNT * sizeof(int));
  }
};

// zgetf2's multiplier and rank-1 update, fused (NID_LU_UNFUSED: zgetf2's
// separately rounded products, as the parity-hook kernels use)
NID_D cd lu_mul(cd a, cd inv) {
#ifdef NID_LU_UNFUSED
  return cmul_nf(a, inv);
#else
  return a * inv;
#endif
}
NID_D cd lu_upd(cd a, cd l, cd p) {
#ifdef NID_LU_UNFUSED
  return csub_nf(a, cmul_nf(l, p));
#else
  return cfms(a, l, p);
#endif
}

// The pivot search of step k over the slot's G lanes (izamax as in lu_step):
// the winning logical position, or k with bad set when no pivot is usable.
template <int N, int G, int CPW, int PB>
NID_D int lu_pivot(const cd* augs, int k, int q, unsigned long long perm, bool& bad) {
  unsigned long long best = 0ull;
#pragma unroll
  for (int m = 0; m < PB; ++m) {
    const int pos = k + q + m * G;
    if (pos < N) {
      const int r = (perm >> (4 * pos)) & 15;
      const double key = cabs1(rows::A<N>(const_cast<cd*>(augs), r, k));
      const unsigned long long u =
          key > 0.0 ? ((unsigned long long)__double_as_longlong(key) & ~15ull) | (unsigned long long)(15 - pos) : 0ull;
      best = u > best ? u : best;
    }
  }
#pragma unroll
  for (int m = CPW; m < 32; m <<= 1) {
    const unsigned long long o = __shfl_xor_sync(0xffffffffu, best, m);
    best = o > best ? o : best;
  }
  if (best == 0ull) bad = true;
  return best == 0ull ? k : 15 - (int)(best & 15ull);
}

NID_D int perm_swap(unsigned long long& perm, int k, int pk) {
  const unsigned long long rk = (perm >> (4 * k)) & 15, rp = (perm >> (4 * pk)) & 15;
  perm &= ~((15ull << (4 * k)) | (15ull << (4 * pk)));
  perm |= (rp << (4 * k)) | (rk << (4 * pk));
  return (int)rp;
}

// One elimination step k of the warp-local column-split LU (track_body):
// pivot search over the slot's G lanes, implicit row swap, multipliers and
// the rank-1 update of the remaining rows.  MCK = ceil((N-k)/G), the most
// columns (and candidate pivot rows) a lane owns at this k: the k loop is
// split into runs of equal MCK so no predicated-off column update is issued.
template <int N, int G, int CPW, int MCK>
NID_D void lu_step(cd* augs, int k, int q, bool solving, unsigned long long& perm, bool& bad, int& pk) {
  // pk: this step's pivot position (izamax of column k, found by the
  // previous step's row loop or, for k = 0, by lu_pivot); on return, the
  // next step's
  const int r0 = perm_swap(perm, k, pk);
  const cd inv = crecip_fast(rows::A<N>(augs, r0, k));
  // column slots past the last column read column N (valid, unused): the
  // arrays are written unconditionally and stay in registers
  cd prow[MCK];
#pragma unroll
  for (int m = 0; m < MCK; ++m) prow[m] = rows::A<N>(augs, r0, min(k + 1 + q + m * G, N));
  // the next pivot: the lane owning column k+1 (q = 0, first column slot)
  // keys each updated entry of it as the row loop produces it -- izamax in
  // logical order, packed as in lu_pivot -- so step k+1 needs no search
  unsigned long long nbest = 0ull;
  if (solving && k + 1 < N) {
    // column k is not written in step k: the next row's multiplier
    // source is loaded before this row's stores
    const bool lastok = k + 1 + q + (MCK - 1) * G <= N;  // only the last column slot can fall off the end
    int r = (perm >> (4 * (k + 1))) & 15;
    cd ark = rows::A<N>(augs, r, k);
#pragma unroll 1
    for (int pos = k + 1; pos < N; ++pos) {
      const int rn = pos + 1 < N ? (int)((perm >> (4 * (pos + 1))) & 15) : r;
      const cd arkn = rows::A<N>(augs, rn, k);
      const cd l = lu_mul(ark, inv);
#pragma unroll
      for (int m = 0; m < MCK; ++m)
        if (m < MCK - 1 || lastok) {
          cd& a = rows::A<N>(augs, r, k + 1 + q + m * G);
          const cd an = lu_upd(a, l, prow[m]);
          a = an;
          if (m == 0) {
            const double key = cabs1(an);
            const unsigned long long u =
                key > 0.0 ? ((unsigned long long)__double_as_longlong(key) & ~15ull) | (unsigned long long)(15 - pos)
                          : 0ull;
            nbest = u > nbest ? u : nbest;
          }
        }
      r = rn;
      ark = arkn;
    }
  }
  __syncwarp();
  // the pivot's reciprocal replaces it (the back substitution multiplies)
  if (solving && q == 0) rows::A<N>(augs, r0, k) = inv;
  if (k + 1 < N) {
    const unsigned long long b = __shfl_sync(0xffffffffu, nbest, threadIdx.x & (CPW - 1));  // from q = 0
    if (b == 0ull) bad = true;
    pk = b == 0ull ? k + 1 : 15 - (int)(b & 15ull);
  }
}

// the k range [k0, N) split into runs of equal ceil((N-k)/G)
template <int N, int G, int CPW, int MCK>
NID_D void lu_run(cd* augs, int q, bool solving, unsigned long long& perm, bool& bad, int& pk) {
  constexpr int kb = N - MCK * G > 0 ? N - MCK * G : 0;  // first k with ceil((N-k)/G) == MCK
  constexpr int ke = N - (MCK - 1) * G;                   // one past the last
#pragma unroll 1
  for (int k = kb; k < ke; ++k) lu_step<N, G, CPW, MCK>(augs, k, q, solving, perm, bad, pk);
  if constexpr (MCK > 1) lu_run<N, G, CPW, MCK - 1>(augs, q, solving, perm, bad, pk);
}

// the table kernel streams term records (track_rec.cuh) for n >= 8 (tables
// too large for the parameter bank: C3's cascade levels n = 8..14, C4)
template <int N>
constexpr bool rec_on() {
  return N >= 8;
}
// dynamic shared memory of the table kernel: the slot layout, each warp's
// ring of streamed term records and per-slot evaluation scratch;
// the parameter-bank kernel needs the slot layout only
template <int N>
constexpr size_t ring_bytes() {
  // (the row-per-warp ring needs 2 x 8 records of 64 bytes, the column-owner
  // ring of track_col.cuh four chunks of 32 pieces: the larger of the two)
  return rec_on<N>() ? (size_t)rows::groups<N>() * (size_t)col::RP * sizeof(uint4) : 0;
}
// per-slot evaluation of long paths, where its scratch fits beside the slot
// layout and the rings (n = 8 .. 14; not n = 15, 16)
template <int N>
constexpr bool lat_on() {
  return rec_on<N>() && Lay<N>::bytes() + ring_bytes<N>() + (size_t)rows::groups<N>() * lat::warp_bytes<N>() +
                            1024 <= (size_t)227 * 1024;
}
// the host builds the column-owner stream for n = 8 .. 14 (capi.cu) and then
// passes its run descriptors with the launch: the kernel must take that path
static_assert(lat_on<8>() && lat_on<9>() && lat_on<10>() && lat_on<11>() && lat_on<12>() && lat_on<13>() &&
                  lat_on<14>(),
              "column-owner evaluator needs the per-slot scratch for n = 8 .. 14");
template <int N>
constexpr size_t lat_bytes() {
  return lat_on<N>() ? (size_t)rows::groups<N>() * lat::warp_bytes<N>() : 0;
}
template <int N>
constexpr size_t smem_bytes() {
  return Lay<N>::bytes() + ring_bytes<N>() + lat_bytes<N>();
}

// blocks per SM the register budget is sized for: as many as the shared
// memory admits (228 KB per SM, 1 KB reserved per block), at most 3
template <int N>
constexpr int blocks_for_smem(size_t smem) {
  const int fit = (int)((228u * 1024u) / (smem + 1024u));
  const int cap = Lay<N>::G <= 4 ? 3 : 2;
  return fit < 1 ? 1 : (fit > cap ? cap : fit);
}
template <int N>
constexpr int min_blocks() {  // table kernel
  return blocks_for_smem<N>(smem_bytes<N>());
}
template <int N>
constexpr int min_blocks_pt() {  // parameter-bank kernel
  return blocks_for_smem<N>(Lay<N>::bytes());
}

}  // namespace ctl


namespace ctl {

// per-slot shared-memory views for the controller lane
struct SlotView {
  cd *xes, *xos, *xss, *dss;
  double* dsl;
  int* isl;
  long long* lsl;
  int slot;
};

#define DS_(f) V.dsl[(f) * SLOTS]
#define IS_(f) V.isl[(f) * SLOTS]
#define HAS(fl) ((IS_(I_FLAGS) & (fl)) != 0)
#define SETF(fl, on) (IS_(I_FLAGS) = (on) ? (IS_(I_FLAGS) | (fl)) : (IS_(I_FLAGS) & ~(fl)))

// the start point of path `path` into the slot's evaluation point: an
// explicit start list, or a total-degree root generated from the path index
// (mixed radix, last variable fastest).  Out of line: once per path, and the
// 64-bit divisions would otherwise sit in the hot loop's instruction stream.
#ifdef NID_CLAIM_INLINE
#define NID_CLAIM_ATTR __forceinline__
#else
#define NID_CLAIM_ATTR __noinline__
#endif
template <int N>
__device__ NID_CLAIM_ATTR void load_start(const TrackArgs& Ar, long long path, cd* xes) {
  constexpr int S = SLOTS;
  if (Ar.starts) {
    for (int v = 0; v < N; ++v) xes[v * S] = Ar.starts[path * N + v];
  } else {
    long long rem = Ar.first_index + path * Ar.index_stride;
    if (rem < (1ll << 32)) {  // 32-bit digits (every config here)
      unsigned r32 = (unsigned)rem;
      for (int v = N - 1; v >= 0; --v) {
        const unsigned d = (unsigned)Ar.deg[v];
        const unsigned k = r32 % d;
        r32 /= d;
        xes[v * S] = Ar.roots[Ar.root_off[v] + (int)k];
      }
    } else {
      for (int v = N - 1; v >= 0; --v) {
        const int d = Ar.deg[v];
        const long long k = rem % d;
        rem /= d;
        xes[v * S] = Ar.roots[Ar.root_off[v] + (int)k];
      }
    }
  }
}

// The controller: runs slot transitions until the slot needs an evaluation
// or a solve, or goes idle.  dxv: the Newton step just solved (A_ON_SOLVE),
// left by the back substitution in the augmented matrix's last column
// (stride (N+1)*SLOTS).  Called from one site only (the top of the block
// loop), so inlining it costs no code duplication.
#ifdef NID_CTL_NOINLINE
#define NID_CTL_ATTR __noinline__
#else
#define NID_CTL_ATTR __forceinline__
#endif
template <int N, bool TR = false>
__device__ NID_CTL_ATTR void control(const TrackArgs& Ar, const SlotView& V, const cd* dxv) {
  constexpr int S = SLOTS;
  constexpr int DXST = (N + 1) * SLOTS;
  const NidTrackParams& q = Ar.prm;
  cd* const xes = V.xes;
  cd* const xos = V.xos;
  cd* const xss = V.xss;
  cd* const dss = V.dss;
  long long* const lsl = V.lsl;
  int act = IS_(I_ACT);
  while (true) {
    if (act == A_EVAL || act == A_SOLVE || act == A_IDLE) break;

      if (act == A_CLAIM) {
        // A launch that fits the grid's slots (P <= blocks x 32) takes path
        // slot * blocks + block, once: paths are dealt round the blocks, so a small
        // launch spreads over the SMs with few slots per block (the streamed-record
        // kernel then evaluates per slot, track_rec.cuh), and which paths share a
        // block is the same on every run -- and so is every record.
        // Larger launches claim from the counter -- the reference's
        // claim-guarded job queue (parallel.py:37-59).
        unsigned long long idx;
        if (Ar.static_claim) {
          idx = lsl[0] == -1 ? (unsigned long long)V.slot * gridDim.x + blockIdx.x : (unsigned long long)Ar.P;
        } else {
          idx = atomicAdd(Ar.next, 1ull);
        }
        if ((long long)idx >= Ar.P) {
          act = A_IDLE;
          break;
        }
        const long long path = (long long)idx;
        lsl[0] = path;
        lsl[S] = Ar.params ? (path / Ar.param_div) * Ar.H.nparam : (Ar.ptw ? path * Ar.H.nterms : -1);
        load_start<N>(Ar, path, xes);
        DS_(D_TE) = 0.0;
        IS_(I_USED) = 0;
        IS_(I_FLAGS) = F_NEEDSCALE;
        IS_(I_MODE) = M_CORR;  // precondition _correct(h, x0, 0, tol*10, 3) (tracker.py:356)
        IS_(I_CTX) = CTX_PRE;
        DS_(D_CTOL) = q.corrector_tol * 10.0;
        IS_(I_CITERS) = 3;
        IS_(I_CIT) = 0;
        IS_(I_CPHASE) = 0;
        act = A_EVAL;
        break;
      }
      if (act == A_ON_EVAL) {
        const double resid = DS_(D_RESID), scale = DS_(D_SCALE);
        if (IS_(I_MODE) == M_CORR) {  // _correct loop body (tracker.py:191-207)
          const int ph = IS_(I_CPHASE);
          if (ph == 0) DS_(D_CTOLEFF) = fmax(DS_(D_CTOL), NOISE_ULPS * scale);
          if (ph == 2 || (ph == 0 && IS_(I_CITERS) == 0)) {
            SETF(F_COK, resid <= fmax(DS_(D_CTOL), NOISE_ULPS * scale));
            IS_(I_CITS) = IS_(I_CITERS);
            act = A_CORR_DONE;
          } else if (!isfinite(resid)) {
            SETF(F_COK, false);
            IS_(I_CITS) = IS_(I_CIT);
            act = A_CORR_DONE;
          } else if (resid <= DS_(D_CTOLEFF)) {
            SETF(F_COK, true);
            IS_(I_CITS) = IS_(I_CIT);
            act = A_CORR_DONE;
          } else {
            act = A_SOLVE;
            break;
          }
        } else {  // _damped_newton (tracker.py:216-238)
          if (IS_(I_DNTRIAL) < 0) {
            DS_(D_DNRES) = resid;
            act = A_DN_CONT;
          } else if (isfinite(resid) && resid < DS_(D_DNRES)) {
            for (int v = 0; v < N; ++v) xss[v * S] = xes[v * S];  // accepted trial = new base
            DS_(D_DNRES) = resid;
            IS_(I_DNIT) += 1;
            IS_(I_DNTRIAL) = -1;
            act = A_DN_CONT;
          } else {
            const double lam = DS_(D_DNLAM) * 0.5;
            DS_(D_DNLAM) = lam;
            IS_(I_DNTRIAL) += 1;
            if (IS_(I_DNTRIAL) < 8) {
              for (int v = 0; v < N; ++v) xes[v * S] = xss[v * S] + cd{lam, 0.0} * dss[v * S];
              act = A_EVAL;
              break;
            }
            IS_(I_DNIT) += 1;  // not improved: break
            act = A_DECIDE;
          }
        }
        continue;
      }
      if (act == A_ON_SOLVE) {  // tracker.py:200-205 / 223-233
        if (IS_(I_MODE) == M_CORR) {
          bool fin = true;
          for (int v = 0; v < N; ++v) {
            const cd x = xes[v * S] + dxv[v * DXST];
            xes[v * S] = x;
            fin = fin && cfinite(x);
          }
          if (!fin) {
            SETF(F_COK, false);
            IS_(I_CITS) = IS_(I_CIT) + 1;
            act = A_CORR_DONE;
            continue;
          }
          IS_(I_CIT) += 1;
          IS_(I_CPHASE) = (IS_(I_CIT) >= IS_(I_CITERS)) ? 2 : 1;
          SETF(F_NEEDSCALE, IS_(I_CPHASE) == 2);
          act = A_EVAL;
          break;
        }
        DS_(D_DNLAM) = 1.0;
        IS_(I_DNTRIAL) = 0;
        for (int v = 0; v < N; ++v) {
          dss[v * S] = dxv[v * DXST];
          xes[v * S] = xss[v * S] + dxv[v * DXST];
        }
        act = A_EVAL;
        break;
      }
      if (act == A_CORR_DONE) {
        if (IS_(I_CTX) == CTX_PRE) {
          if (!HAS(F_COK)) {
            IS_(I_OUTST) = NID_FAILED;
            SETF(F_HASX, false);
            DS_(D_OUTT) = 0.0;
            act = A_WRITE;
            continue;
          }
          double m = 0.0;
          for (int v = 0; v < N; ++v) {
            const cd x = xes[v * S];
            xos[v * S] = x;
            m = nanmax(m, cabs_fast(x));
          }
          DS_(D_T) = 0.0;
          DS_(D_STEP) = q.initial_step;
          SETF(F_HAVEPREV, false);
          SETF(F_ENDGAME, false);
          DS_(D_PREV) = 0.0;
          IS_(I_USED) = 0;
          DS_(D_ENTRY) = m;
          act = A_LOOP_TOP;
          continue;
        }
        if (HAS(F_COK)) {
          // ||x||_inf > threshold, decided on squared moduli (no square roots);
          // the exact moduli only within 1e-12 of the threshold
          double m2 = 0.0;
          for (int v = 0; v < N; ++v) m2 = nanmax(m2, cabs2(xes[v * S]));
          const double th2 = q.infinity_threshold * q.infinity_threshold;
          bool inf_x = m2 > th2 * (1.0 + 1e-12) || isnan(m2);
          if (!inf_x && m2 >= th2 * (1.0 - 1e-12)) {
            double m = 0.0;
            for (int v = 0; v < N; ++v) m = nanmax(m, cabs_fast(xes[v * S]));
            inf_x = m > q.infinity_threshold;
          }
          if (inf_x) {
            IS_(I_OUTST) = NID_AT_INFINITY;
            SETF(F_HASX, false);
            DS_(D_OUTT) = DS_(D_TTRY);
            act = A_WRITE;
            continue;
          }
          for (int v = 0; v < N; ++v) {
            xss[v * S] = xos[v * S];  // x_prev <- x
            xos[v * S] = xes[v * S];  // x <- x_new
          }
          DS_(D_PREV) = DS_(D_HSTEP);
          SETF(F_HAVEPREV, true);
          DS_(D_T) = DS_(D_TTRY);
          if constexpr (TR) {  // trace.append((t, hstep, iters)) (tracker.py:393-394)
            if (Ar.trace) {
              const long long path = lsl[0];
              const int k = Ar.trace_n[path];
              if (k < Ar.trace_cap) {
                double* rec = Ar.trace + ((size_t)path * Ar.trace_cap + k) * 3;
                rec[0] = DS_(D_TTRY);
                rec[1] = DS_(D_HSTEP);
                rec[2] = (double)IS_(I_CITS);
              }
              Ar.trace_n[path] = k + 1;
            }
          }
          if (DS_(D_T) >= 1.0) {
            act = A_FINISH;
            continue;
          }
          if (IS_(I_CITS) <= 2) DS_(D_STEP) = fmin(DS_(D_STEP) * 2.0, q.max_step);
          act = A_LOOP_TOP;
        } else {
          const double st = DS_(D_HSTEP) * 0.5;
          DS_(D_STEP) = st;
          if (st < q.min_step) {
            if (HAS(F_ENDGAME)) {
              act = A_FINISH;
            } else {
              IS_(I_OUTST) = NID_FAILED;
              SETF(F_HASX, false);
              DS_(D_OUTT) = DS_(D_T);
              act = A_WRITE;
            }
            continue;
          }
          act = A_LOOP_TOP;
        }
        continue;
      }
      if (act == A_LOOP_TOP) {  // tracker.py:367-387
        if (IS_(I_USED) >= q.max_steps) {
          if (HAS(F_ENDGAME)) {
            act = A_FINISH;
          } else {
            IS_(I_OUTST) = NID_FAILED;
            SETF(F_HASX, false);
            DS_(D_OUTT) = DS_(D_T);
            act = A_WRITE;
          }
          continue;
        }
        const double t = DS_(D_T);
        const double rem = 1.0 - t;
        if (!HAS(F_ENDGAME) && t >= q.endgame_start) {
          SETF(F_ENDGAME, true);
          double m = 0.0;
          for (int v = 0; v < N; ++v) m = nanmax(m, cabs_fast(xos[v * S]));
          DS_(D_ENTRY) = m;
        }
        if (rem <= q.snap_remaining) {
          act = A_FINISH;
          continue;
        }
        IS_(I_USED) += 1;
        double hs = fmin(fmin(DS_(D_STEP), q.max_step), rem);
        if (HAS(F_ENDGAME)) hs = fmin(hs, q.endgame_contraction * rem);
        double tt = t + hs;
        if (1.0 - tt < 1e-14) tt = 1.0;
        DS_(D_HSTEP) = hs;
        DS_(D_TTRY) = tt;
        const double prev = DS_(D_PREV);
        if (HAS(F_HAVEPREV) && prev > 0.0) {
          const cd ratio = cd{hs / prev, 0.0};
          for (int v = 0; v < N; ++v) {
            const cd xo = xos[v * S];
            xes[v * S] = xo + (xo - xss[v * S]) * ratio;
          }
        } else {
          for (int v = 0; v < N; ++v) xes[v * S] = xos[v * S];
        }
        DS_(D_TE) = tt;
        IS_(I_MODE) = M_CORR;
        IS_(I_CTX) = CTX_STEP;
        DS_(D_CTOL) = q.corrector_tol;
        IS_(I_CITERS) = q.max_corrector_iters;
        IS_(I_CIT) = 0;
        IS_(I_CPHASE) = 0;
        SETF(F_NEEDSCALE, true);
        act = A_EVAL;
        break;
      }
      if (act == A_FINISH) {  // tracker.py:315-317
        bool fin = true;
        double m = 0.0;
        for (int v = 0; v < N; ++v) {
          const cd x = xos[v * S];
          fin = fin && cfinite(x);
          m = nanmax(m, cabs_fast(x));
          xss[v * S] = x;  // damped-Newton base x1 <- x
          xes[v * S] = x;
        }
        const double nn = fin ? m : INFINITY;
        DS_(D_NORMNOW) = nn;
        DS_(D_MOVECAP) = 0.05 * (1.0 + nn);
        DS_(D_TFROM) = DS_(D_T);
        IS_(I_MODE) = M_DN;
        IS_(I_DNIT) = 0;
        IS_(I_DNTRIAL) = -1;
        DS_(D_TE) = 1.0;
        SETF(F_NEEDSCALE, false);
        act = A_EVAL;
        break;
      }
      if (act == A_DN_CONT) {  // loop head of _damped_newton
        const double r = DS_(D_DNRES);
        if (IS_(I_DNIT) >= q.final_newton_iters || !isfinite(r) || r <= q.corrector_tol) {
          act = A_DECIDE;
          continue;
        }
        act = A_SOLVE;
        break;
      }
      if (act == A_DECIDE) {  // tracker.py:318-338
        const double res = DS_(D_DNRES);
        bool finb = true;
        double moved = 0.0;
        for (int v = 0; v < N; ++v) {
          const cd xb = xss[v * S];
          finb = finb && cfinite(xb);
          moved = nanmax(moved, cabs_fast(xb - xos[v * S]));
        }
        if (!finb) moved = INFINITY;
        const double cap = DS_(D_MOVECAP), nn = DS_(D_NORMNOW);
        SETF(F_HASX, false);
        DS_(D_OUTRES) = NAN;
        if (isfinite(res) && res <= CONVERGED_RESIDUAL && moved <= cap) {
          IS_(I_OUTST) = NID_CONVERGED;
          SETF(F_HASX, true);
          DS_(D_OUTT) = 1.0;
          DS_(D_OUTRES) = res;
        } else if (nn > q.soft_infinity || (nn + 1e-6) / (DS_(D_ENTRY) + 1e-6) >= 8.0) {
          IS_(I_OUTST) = NID_AT_INFINITY;
          DS_(D_OUTT) = DS_(D_TFROM);
        } else if (isfinite(res) && res <= 1e-4 && moved <= cap) {
          IS_(I_OUTST) = NID_SINGULAR_ENDPOINT;
          SETF(F_HASX, true);
          DS_(D_OUTT) = DS_(D_TFROM);
          DS_(D_OUTRES) = res;
        } else {
          IS_(I_OUTST) = NID_FAILED;
          DS_(D_OUTT) = DS_(D_TFROM);
        }
        act = A_WRITE;
        continue;
      }
      if (act == A_WRITE) {
        const long long path = lsl[0];
        const bool hx = HAS(F_HASX);
        Ar.status[path] = (int8_t)IS_(I_OUTST);
        Ar.steps[path] = IS_(I_USED);
        Ar.t_reached[path] = DS_(D_OUTT);
        Ar.resid[path] = hx ? DS_(D_OUTRES) : NAN;
        for (int v = 0; v < N; ++v) Ar.x_end[path * N + v] = hx ? xss[v * S] : cd{NAN, NAN};
        act = A_CLAIM;
        continue;
      }
      act = A_IDLE;  // A_IDLE / unknown
      break;
    }
    IS_(I_ACT) = act;
}

#undef DS_
#undef IS_
#undef HAS
#undef SETF

}  // namespace ctl

// The table kernel's evaluator: the factor-list term-table interpreter
// (rows::eval_rows_fac).
template <int N>
struct TableEval {
  static constexpr bool kTable = true;
  static NID_D void rows(const HomDev& H, int g, const cd (&x)[N], double t, const cd* prm, cd* aug, double* part,
                         bool want_scale, const cd* xs, double* axw) {
    rows::eval_rows_fac<N>(H, g, xs, t, prm, aug, part, want_scale, axw);
  }
  // per-cell polyhedral homotopy: tws = the slot's t-exponent row
  static NID_D void rows(const HomDev& H, int g, const cd (&x)[N], double t, const cd* prm, cd* aug, double* part,
                         bool want_scale, const cd* xs, double* axw, const double* tws) {
    rows::eval_rows_fac<N>(H, g, xs, t, prm, aug, part, want_scale, axw, tws);
  }
};

// true for the table evaluator (the streamed-record path replaces it for n > 10)
template <class E, class = void>
struct has_table_flag {
  static constexpr bool value = false;
};
template <class E>
struct has_table_flag<E, decltype((void)E::kTable)> {
  static constexpr bool value = true;
};

// Optional phase timers (-DNID_PHASE_TIMERS): per-warp clock64 cycles spent
// in each phase of the block loop, summed into TrackArgs::counters[8..15].
#ifdef NID_PHASE_TIMERS
#define NID_T0() long long t_ph_ = clock64()
#define NID_TP(i)                                   \
  do {                                              \
    const long long t1_ = clock64();                \
    if (lane == 0) ph_cyc[i] += (t1_ - t_ph_);      \
    t_ph_ = t1_;                                    \
  } while (0)
#else
#define NID_T0()
#define NID_TP(i)
#endif

// The kernel body, shared by the table-driven kernel (track_ctl_kernel: term
// table in global memory, read through L1) and the parameter-table kernel
// (track_pt_kernel: csrc/track_ptab.cuh, the table in the launch's constant
// bank).  Tab = void selects Eval; Tab = PTab selects PTEval.
template <int N, class Eval, class Tab, bool PO = false, bool TR = false>
__device__ __forceinline__ void track_body(const TrackArgs& Ar, const Tab* tab) {
  using namespace ctl;
  using L = Lay<N>;
  constexpr int G = L::G;
  constexpr int S = SLOTS;
  constexpr int CPW = S / G;  // controller slots per warp
  extern __shared__ __align__(16) unsigned char smem_ctl[];
  const int lane = threadIdx.x & 31;
  const int g = threadIdx.x >> 5;
  cd* const cb = reinterpret_cast<cd*>(smem_ctl);
  double* const db = reinterpret_cast<double*>(cb + (size_t)L::CPLX * S);
  long long* const lb = reinterpret_cast<long long*>(db + (size_t)L::DBL * S);
  int* const ib = reinterpret_cast<int*>(lb + (size_t)L::LLN * S);
  // worker view: this thread evaluates/eliminates rows of slot `lane`
  cd* const aug = cb + lane;
  double* const part = db + L::PART * S + lane;
  // controller view: lanes < CPW of warp g run the state machine of slot cs
  const bool is_ctl = lane < CPW;
  const int cs = g * CPW + (lane % CPW);
  cd* const augc = cb + cs;
  double* const partc = db + L::PART * S + cs;
  cd* const gs = Ar.gstate + (size_t)blockIdx.x * L::GITEMS * S + cs;
  const SlotView V{cb + L::XE * S + cs, gs + L::GXO * S, gs + L::GXS * S, gs + L::GDS * S, db + cs,
                   ib + cs, lb + cs, cs};
  unsigned long long n_eval = 0, n_jac = 0, n_scale = 0, n_fb = 0;
#ifdef NID_PHASE_TIMERS
  unsigned long long ph_cyc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#endif

#define W_IS(f) ib[(f) * S + lane]   // worker's slot
#define W_DS(f) db[(f) * S + lane]
#define C_IS(f) V.isl[(f) * S]       // controller's slot
#define C_DS(f) V.dsl[(f) * S]

  if (is_ctl) {
    C_IS(I_ACT) = A_CLAIM;
    V.lsl[0] = -1;  // no path yet (static claims take one path per slot)
  }

  while (true) {
    NID_T0();
    if (is_ctl) control<N, TR>(Ar, V, augc + N * S);
    __syncwarp();
    {
      // |x_v| of the evaluation points of this warp's slots that need the
      // noise scale, spread over all 32 lanes (slot g*CPW + lane % CPW,
      // variables lane / CPW + j * G); the evaluator reads them after the
      // barrier instead of every warp recomputing all N moduli
      const int sl = g * CPW + lane % CPW;
      if (ib[I_ACT * S + sl] == A_EVAL && (ib[I_FLAGS * S + sl] & (F_NEEDSCALE | F_FALLBACK))) {
#pragma unroll
        for (int v = lane / CPW; v < N; v += G) db[(L::AXW + v) * S + sl] = cabs_fast(cb[(L::XE + v) * S + sl]);
      }
    }
    NID_TP(0);  // control (top)
    // ------------------------------------------------------------ evaluation
    if (!__syncthreads_or(W_IS(I_ACT) != A_IDLE)) break;
    NID_TP(1);  // barrier before the evaluation
    bool rec_done = false;
    bool col_done = false;  // block-uniform: this round's block pass was the column-owner one
    if constexpr (rec_on<N>() && !ctl::is_ptab<Tab>::value && has_table_flag<Eval>::value) {
      if (Ar.H.rec) {  // streamed records: every lane of the warp takes part
        const bool act0 = W_IS(I_ACT) == A_EVAL;
        // Few evaluating slots in the block (the tail of a launch, or a launch
        // smaller than the machine): the row-per-warp pass would run with most
        // lanes idle, so each slot is evaluated on its own with its rows' terms
        // split over the warp's 32 lanes.  Every warp sees the same 32 slots,
        // so the decision is block-uniform without a barrier.
        const int nact = __popc(__ballot_sync(0xffffffffu, act0));  // (every lane votes: no short circuit)
        const bool lat = lat_on<N>() && act0 && nact <= Ar.lat_slots;
        const bool act = act0 && !lat;  // slots of the row-per-warp pass
        const bool want = act && (W_IS(I_FLAGS) & (F_NEEDSCALE | F_FALLBACK)) != 0;
        const long long pr = lb[S + lane];
        const cd* prm = (act && pr >= 0) ? Ar.params + pr : nullptr;
        unsigned char* const ringb = smem_ctl + L::bytes() + (size_t)g * col::RP * sizeof(uint4);
        unsigned char* scr = smem_ctl + L::bytes() + ring_bytes<N>() + (size_t)g * lat::warp_bytes<N>();
        if (__any_sync(0xffffffffu, act)) {
          if (lat_on<N>() && Ar.H.crec) {
            // column-owner pass (track_col.cuh): the values are left as per-warp
            // partial sums in this warp's scratch, completed after the barrier
            eval_cols<N>(Ar.H, Ar.runs_c, g, cb + L::XE * S + lane, W_DS(D_TE), prm, aug, part, want, act,
                         db + L::AXW * S + lane, reinterpret_cast<uint4*>(ringb), reinterpret_cast<cd*>(scr) + lane);
            col_done = true;
          } else {
#ifndef NID_COL_ONLY
            eval_rows_rec<N>(Ar.H, Ar.runs_c, g, cb + L::XE * S + lane, W_DS(D_TE), prm, aug, part, want, act,
                             db + L::AXW * S + lane, reinterpret_cast<TermRec*>(ringb));
#endif
          }
        }
        // few evaluating slots: one slot at a time, the warp's lanes split the terms
        unsigned lm = __ballot_sync(0xffffffffu, lat);
#pragma unroll 1
        while (lat_on<N>() && lm) {
          const int s = __ffs(lm) - 1;
          lm &= lm - 1;
          const long long ps = lb[S + s];
          const bool ws = (ib[I_FLAGS * S + s] & (F_NEEDSCALE | F_FALLBACK)) != 0;
          eval_slot_rec<N>(Ar.H, g, cb + L::XE * S + s, db[D_TE * S + s], (Ar.params && ps >= 0) ? Ar.params + ps : nullptr,
                           cb + s, db + L::PART * S + s, ws, db + L::AXW * S + s, scr);
        }
        rec_done = true;
      }
    }
    if (!rec_done && W_IS(I_ACT) == A_EVAL) {
      const bool want = (W_IS(I_FLAGS) & (F_NEEDSCALE | F_FALLBACK)) != 0;
      if constexpr (ctl::is_ptab<Tab>::value) {
        // batched cells: the slot's own t-exponent row (else the table's)
        const double* tws = nullptr;
        if constexpr (PO) tws = Ar.ptw ? Ar.ptw + lb[S + lane] : nullptr;
        PTEval<N, PO>::rows(Ar.H, *tab, g, W_DS(D_TE), aug, part, want, cb + L::XE * S + lane, db + L::AXW * S + lane,
                            tws);
      } else {
        cd x[N];
#pragma unroll
        for (int v = 0; v < N; ++v) x[v] = cb[(L::XE + v) * S + lane];
        const long long pr = lb[S + lane];
        const cd* prm = (Ar.params && pr >= 0) ? Ar.params + pr : nullptr;
        const double* tws = Ar.H.tw ? (Ar.ptw ? Ar.ptw + pr : Ar.H.tw) : nullptr;
        if constexpr (has_table_flag<Eval>::value) {
          if (tws) {
            Eval::rows(Ar.H, g, x, W_DS(D_TE), prm, aug, part, want, cb + L::XE * S + lane, db + L::AXW * S + lane, tws);
          } else {
            Eval::rows(Ar.H, g, x, W_DS(D_TE), prm, aug, part, want, cb + L::XE * S + lane, db + L::AXW * S + lane);
          }
        } else {
          Eval::rows(Ar.H, g, x, W_DS(D_TE), prm, aug, part, want, cb + L::XE * S + lane, db + L::AXW * S + lane);
        }
      }
    }
    NID_TP(2);  // evaluation
    __syncthreads();
    NID_TP(3);  // barrier after the evaluation
    if constexpr (lat_on<N>() && !ctl::is_ptab<Tab>::value && has_table_flag<Eval>::value) {
      if (col_done) {
        const int ss = g * CPW + lane % CPW;
        col_reduce<N, G, CPW>(Ar.H, g, lane, ib[I_ACT * S + ss] == A_EVAL, cb, db + L::PART * S, cb + L::XE * S,
                              db[D_TE * S + ss], smem_ctl + L::bytes() + ring_bytes<N>(), lat::warp_bytes<N>());
        __syncwarp();
      }
    }
    if (is_ctl && C_IS(I_ACT) == A_EVAL) {
      double sc = 0.0;
      const double r = rows::combine_resid<N>(augc, partc, C_DS(D_TE), sc, PO);
      if (C_IS(I_FLAGS) & F_FALLBACK) {
        // zgesv failed at this point: min-norm least squares (zgelsd) on the
        // re-evaluated augmented matrix
        C_IS(I_FLAGS) &= ~F_FALLBACK;
        cd* sc2 = Ar.scratch + (size_t)(blockIdx.x * S + cs) * (3 * N * N + 2 * N);
        for (int i = 0; i < N; ++i) {
          for (int j = 0; j < N; ++j) sc2[i * N + j] = A<N>(augc, i, j);
          sc2[N * N + i] = A<N>(augc, i, N);
        }
        double sv[N];
        lstsq_minnorm(sc2, N, N, N, sc2 + N * N, sc2 + N * N + N, sv, sc2 + 2 * N * N + N);
        for (int i = 0; i < N; ++i) A<N>(augc, i, N) = sc2[2 * N * N + N + i];
        C_IS(I_ACT) = A_ON_SOLVE;  // consumed by the next control round
      } else {
        n_eval += 1;
        n_scale += (C_IS(I_FLAGS) & F_NEEDSCALE) ? 1 : 0;
        C_DS(D_RESID) = r;
        C_DS(D_SCALE) = sc;
        // inline fast path of the commonest transition: the corrector's
        // residual is above its tolerance -> Newton step (tracker.py:194-199)
        bool fast = false;
        const int ph = C_IS(I_CPHASE);
        if (C_IS(I_MODE) == M_CORR && ph != 2 && !(ph == 0 && C_IS(I_CITERS) == 0) && isfinite(r)) {
          double tol_eff;
          if (ph == 0) {
            tol_eff = fmax(C_DS(D_CTOL), NOISE_ULPS * sc);
            C_DS(D_CTOLEFF) = tol_eff;
          } else {
            tol_eff = C_DS(D_CTOLEFF);
          }
          if (!(r <= tol_eff)) {
            C_IS(I_ACT) = A_SOLVE;
            fast = true;
          }
        }
        if (!fast) C_IS(I_ACT) = A_ON_EVAL;  // consumed by the next control round
      }
    }
    NID_TP(4);  // combine + control after the evaluation
    // ------------------------------------------------------------ LU (warp-local)
    // Warp g factorizes the CPW slots it controls: lane = q * CPW + sl (slot
    // sl, row group q; physical rows r == q (mod G)).  Slot-minor lanes keep
    // every quarter-warp on 8 different slots, i.e. different banks of the
    // [element][slot] layout.  Pivots are reduced over the slot's G lanes
    // (stride CPW) by shuffles; __syncwarp orders the shared-memory updates.
    __syncwarp();
    {
      const int sl = lane % CPW, q = lane / CPW;
      const int ss = g * CPW + sl;  // slot factorized by this lane
      cd* const augs = cb + ss;
      const bool solving = ib[I_ACT * S + ss] == A_SOLVE;
      if (__any_sync(0xffffffffu, solving)) {
        // Column-split LU over the slot's G lanes: logical row order is an
        // implicit permutation (perm: position -> physical row, swapped
        // exactly as zgetf2 swaps rows), so every lane runs the same row loop
        // (uniform trip count N-1-k) and owns columns j == k+1+q (mod G).
        unsigned long long perm = 0;
#pragma unroll
        for (int i = 0; i < N; ++i) perm |= (unsigned long long)i << (4 * i);
        bool bad = false;
        int pk = lu_pivot<N, G, CPW, (N + G - 1) / G>(augs, 0, q, perm, bad);
        lu_run<N, G, CPW, (N + G - 1) / G>(augs, q, solving, perm, bad, pk);
        if (solving && q == 0) {
          lb[2 * S + ss] = (long long)perm;
          ib[I_BAD * S + ss] = bad ? 1 : 0;
        }
      }
    }
    __syncwarp();
    NID_TP(5);  // LU
    if (is_ctl && C_IS(I_ACT) == A_SOLVE) {  // back substitution by the slot's controller
      n_jac += 1;
      const unsigned long long pm = (unsigned long long)V.lsl[2 * S];
      cd dx[N];
      bool fin = true;
#pragma unroll
      for (int k = N - 1; k >= 0; --k) {
        const int r = (pm >> (4 * k)) & 15;
        cd s = A<N>(augc, r, N);
#pragma unroll
        for (int j = k + 1; j < N; ++j) s = lu_upd(s, A<N>(augc, r, j), dx[j]);
        dx[k] = lu_mul(s, A<N>(augc, r, k));
        fin = fin && cfinite(dx[k]);
      }
      if (!C_IS(I_BAD) && fin) {
        bool fast = false;
        if (C_IS(I_MODE) == M_CORR) {  // inline: x += dx, next corrector evaluation (tracker.py:200-205)
          bool xfin = true;
          cd xn[N];
#pragma unroll
          for (int v = 0; v < N; ++v) {
            xn[v] = V.xes[v * S] + dx[v];
            xfin = xfin && cfinite(xn[v]);
          }
          if (xfin) {
#pragma unroll
            for (int v = 0; v < N; ++v) V.xes[v * S] = xn[v];
            const int it = C_IS(I_CIT) + 1;
            C_IS(I_CIT) = it;
            const int ph = (it >= C_IS(I_CITERS)) ? 2 : 1;
            C_IS(I_CPHASE) = ph;
            if (ph == 2) C_IS(I_FLAGS) |= F_NEEDSCALE;
            else C_IS(I_FLAGS) &= ~F_NEEDSCALE;
            C_IS(I_ACT) = A_EVAL;
            fast = true;
          }
        }
        if (!fast) {
#pragma unroll
          for (int v = 0; v < N; ++v) A<N>(augc, v, N) = dx[v];
          C_IS(I_ACT) = A_ON_SOLVE;  // consumed by the next control round
        }
      } else {
        n_fb += 1;
        C_IS(I_FLAGS) |= F_FALLBACK;
        C_IS(I_ACT) = A_EVAL;  // re-evaluate the same point, then lstsq
      }
    }
    NID_TP(6);  // back substitution + control
  }
#ifdef NID_PHASE_TIMERS
  if (lane == 0)
    for (int i = 0; i < 7; ++i) atomicAdd(Ar.counters + 8 + i, ph_cyc[i]);
#endif
#undef W_IS
#undef W_DS
#undef C_IS
#undef C_DS
  if (is_ctl) {
    atomicAdd(Ar.counters + 0, n_eval);
    atomicAdd(Ar.counters + 1, n_jac);
    atomicAdd(Ar.counters + 2, n_scale);
    atomicAdd(Ar.counters + 3, n_fb);
  }
}

template <int N, class Eval = TableEval<N>>
__global__ void __launch_bounds__(rows::groups<N>() * 32, ctl::min_blocks<N>())
    track_ctl_kernel(const __grid_constant__ TrackArgs Ar) {
  track_body<N, Eval, void>(Ar, nullptr);
}

template <int N, bool PO>  // PO: per-cell polyhedral homotopy (start_kind 2)
__global__ void __launch_bounds__(rows::groups<N>() * 32, ctl::min_blocks_pt<N>())
    track_pt_kernel(const __grid_constant__ TrackArgsPT A) {
  track_body<N, TableEval<N>, PTab, PO>(A.a, &A.t);
}
