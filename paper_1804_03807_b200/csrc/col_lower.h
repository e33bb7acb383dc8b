// Host lowering of a term table into the column-owner stream of
// csrc/track_col.cuh (included by capi.cu after NidHomotopy is defined).
//
// Monomials are merged across rows (one entry per distinct exponent vector,
// with the rows that hold it and their coefficients: the reference's stacked
// evaluator, polynomials.py:202-256).  Units: (column v < n, row block) walks
// the monomials containing x_v; (column n, row block, warp) walks that warp's
// range of the monomials for the values H_r; (abs, row block) the abs sums.
// A unit's records are grouped into runs by (factor count, row mask, blend
// class); units are dealt to the warps by longest processing time.
#pragma once

#include <array>
#include <map>
#include <tuple>
#include <vector>

namespace colhost {

struct Rec {
  int mono, em, var;
};
struct Run {
  int D, cls;
  unsigned mask;
  std::vector<Rec> recs;
};
struct Unit {
  int col, row0, nr, kind;
  std::vector<Run> runs;
  double cost = 0.0;
};

inline int popc(unsigned m) {
  int c = 0;
  for (; m; m &= m - 1) ++c;
  return c;
}

// Returns false when the table is not eligible (the caller keeps the
// row-per-warp records); on success fills pieces, runs, cgrun, cgbase.
inline bool build(const NidHomotopyDesc* d, int n, int T, const std::vector<int>& off, const std::vector<double>& acs,
                  const std::vector<double>& act, int G, bool td, std::vector<uint4>& pieces,
                  std::vector<uint4>& runs_out, int (&cgrun)[17], int (&cgbase)[17]) {
  struct Mono {
    std::array<unsigned char, 16> e;
    int deg;
    int term_of_row[16];
  };
  std::vector<Mono> monos;
  std::map<std::array<unsigned char, 16>, int> index;
  for (int i = 0; i < n; ++i)
    for (int k = off[i]; k < off[i + 1]; ++k) {
      std::array<unsigned char, 16> key;
      int deg = 0;
      for (int v = 0; v < 16; ++v) {
        key[v] = d->expo[k * NID_MAX_VARS + v];
        deg += key[v];
      }
      if (deg > 12) return false;
      auto it = index.find(key);
      int m;
      if (it == index.end()) {
        m = (int)monos.size();
        index[key] = m;
        Mono mo;
        mo.e = key;
        mo.deg = deg;
        for (int r = 0; r < 16; ++r) mo.term_of_row[r] = -1;
        monos.push_back(mo);
      } else {
        m = it->second;
      }
      if (monos[m].term_of_row[i] >= 0) return false;  // a row holds the exponent twice
      monos[m].term_of_row[i] = k;
    }
  const int M = (int)monos.size();
  auto cls_of = [&](int k) {
    if (td) return (int)col::C_T;
    if (d->param_slot && d->param_slot[k] >= 0) return (int)col::C_PRM;
    const double sr = d->coef_start[2 * k], si = d->coef_start[2 * k + 1];
    const double tr = d->coef_target[2 * k], ti = d->coef_target[2 * k + 1];
    if (sr == 0.0 && si == 0.0) return (int)col::C_T;
    if (tr == 0.0 && ti == 0.0) return (int)col::C_S;
    if (sr == tr && si == ti) return (int)col::C_B;
    return (int)col::C_TWO;
  };
  // records of monomials [m0, m1) for (col, row block) grouped into runs
  // experiment knob: NID_COL_W="abs weight,values weight" scales the cost model
  double w_abs = 1.0, w_val = 1.0;
  if (const char* wv = getenv("NID_COL_W")) sscanf(wv, "%lf,%lf", &w_abs, &w_val);
  auto make_unit = [&](int colv, int row0, int nr, int kind, int m0, int m1) {
    const double wscale = kind == col::K_ABS ? w_abs : (colv == n ? w_val : 1.0);
    Unit u;
    u.col = colv;
    u.row0 = row0;
    u.nr = nr;
    u.kind = kind;
    std::map<std::tuple<int, unsigned, int>, std::vector<Rec>> by;
    for (int m = m0; m < m1; ++m) {
      const Mono& mo = monos[m];
      if (colv < n && kind == col::K_JH && mo.e[colv] == 0) continue;
      unsigned mask = 0;
      int cls = -1;
      for (int i = 0; i < nr; ++i) {
        const int k = mo.term_of_row[row0 + i];
        if (k < 0) continue;
        mask |= 1u << i;
        const int c = cls_of(k);
        if (cls < 0) cls = c;
        else if (cls != c) cls = (cls == col::C_PRM || c == col::C_PRM) ? (int)col::C_PRM : (int)col::C_TWO;
      }
      if (!mask) continue;
      const bool jcol = kind == col::K_JH && colv < n;
      const int D = jcol ? mo.deg - 1 : mo.deg;
      if (kind == col::K_ABS) cls = 0;
      by[std::make_tuple(D, mask, cls)].push_back(Rec{m, jcol ? (int)mo.e[colv] : 1, jcol ? colv : -1});
    }
    for (auto& kv : by) {
      Run r;
      r.D = std::get<0>(kv.first);
      r.mask = std::get<1>(kv.first);
      r.cls = std::get<2>(kv.first);
      r.recs = kv.second;
      const int pc = popc(r.mask);
      // instructions per record (SASS counts of the run bodies)
      const double per = kind == col::K_ABS ? 16.0 + 6.0 * r.D + 5.0 * pc
                                            : 12.0 + 9.0 * r.D + pc * (r.cls >= col::C_TWO ? 11.0 : 5.0);
      u.cost += 10.0 + per * wscale * (double)r.recs.size();
      u.runs.push_back(r);
    }
    u.cost += 20.0;
    return u;
  };
  std::vector<std::vector<Unit>> hw(G), jw(G), aw(G);
  std::vector<double> load(G, 0.0);
  const int NB = (n + col::RMAX - 1) / col::RMAX;
  // Jacobian columns (eight-row blocks) and abs sums (four-row blocks: the abs
  // unit of a dense block is the largest unit otherwise): longest processing
  // time first
  std::vector<Unit> rest;
  for (int b = 0; b < NB; ++b) {
    const int row0 = b * col::RMAX, nr = std::min(col::RMAX, n - row0);
    for (int v = 0; v < n; ++v) rest.push_back(make_unit(v, row0, nr, col::K_JH, 0, M));
    for (int r4 = row0; r4 < row0 + nr; r4 += 4)
      rest.push_back(make_unit(n + 1, r4, std::min(4, row0 + nr - r4), col::K_ABS, 0, M));
  }
  std::stable_sort(rest.begin(), rest.end(), [](const Unit& a, const Unit& b) { return a.cost > b.cost; });
  for (const Unit& u : rest) {
    int best = 0;
    for (int w = 1; w < G; ++w)
      if (load[w] < load[best]) best = w;
    load[best] += u.cost;
    (u.kind == col::K_ABS ? aw : jw)[best].push_back(u);
  }
  // values: every warp takes a contiguous range of each row block's monomials,
  // sized to level the warps' loads (water filling over the loads so far)
  for (int b = 0; b < NB; ++b) {
    const int row0 = b * col::RMAX, nr = std::min(col::RMAX, n - row0);
    std::vector<double> pre(M + 1, 0.0);
    for (int m = 0; m < M; ++m) pre[m + 1] = pre[m] + make_unit(n, row0, nr, col::K_JH, m, m + 1).cost - 20.0;
    const double total = pre[M];
    // level L with sum_w max(0, L - load[w]) = total
    double lo = 0.0, hi = total;
    for (int w = 0; w < G; ++w) hi = std::max(hi, load[w] + total);
    for (int it = 0; it < 100; ++it) {
      const double mid = 0.5 * (lo + hi);
      double fill = 0.0;
      for (int w = 0; w < G; ++w) fill += std::max(0.0, mid - load[w]);
      (fill < total ? lo : hi) = mid;
    }
    int m0 = 0;
    double given = 0.0;
    for (int w = 0; w < G; ++w) {
      given += std::max(0.0, hi - load[w]);
      int m1 = m0;
      while (m1 < M && pre[m1 + 1] <= given + 1e-9) ++m1;
      if (w == G - 1) m1 = M;
      Unit u = make_unit(n, row0, nr, col::K_JH, m0, m1);
      load[w] += u.cost;
      hw[w].push_back(u);
      m0 = m1;
    }
  }
  // emit
  pieces.clear();
  runs_out.clear();
  auto put_cd = [&](double re, double im) {
    uint4 p;
    memcpy(&p.x, &re, 8);
    memcpy(&p.z, &im, 8);
    pieces.push_back(p);
  };
  for (int w = 0; w <= 16; ++w) cgrun[w] = cgbase[w] = 0;
  for (int w = 0; w < G; ++w) {
    while (pieces.size() % col::CP) pieces.push_back(make_uint4(0, 0, 0, 0));
    cgrun[w] = (int)runs_out.size();
    cgbase[w] = (int)pieces.size();
    const size_t base = pieces.size();
    std::vector<const Unit*> order;
    for (const Unit& u : hw[w]) order.push_back(&u);
    for (const Unit& u : jw[w]) order.push_back(&u);
    for (const Unit& u : aw[w]) order.push_back(&u);
    for (const Unit* up : order) {
      const Unit& u = *up;
      const unsigned x0 = (unsigned)u.col | ((unsigned)u.row0 << 8) | ((unsigned)u.nr << 16) | ((unsigned)u.kind << 26);
      if (u.runs.empty()) {
        runs_out.push_back(make_uint4(x0 | (1u << 24) | (1u << 25), 0u, (unsigned)(pieces.size() - base), 0u));
        continue;
      }
      for (size_t ri = 0; ri < u.runs.size(); ++ri) {
        const Run& r = u.runs[ri];
        const int pc = popc(r.mask);
        const int len = 1 + pc * ((u.kind == col::K_JH && r.cls >= col::C_TWO) ? 2 : 1);
        if (len > col::CP) return false;
        const unsigned x = x0 | (ri == 0 ? (1u << 24) : 0u) | (ri + 1 == u.runs.size() ? (1u << 25) : 0u);
        const unsigned y = (unsigned)r.D | (r.mask << 8) | ((unsigned)r.cls << 16) | ((unsigned)len << 20);
        runs_out.push_back(make_uint4(x, y, (unsigned)(pieces.size() - base), (unsigned)r.recs.size()));
        for (const Rec& rc : r.recs) {
          // a record never straddles the end of the ring (col::advance applies the same rule)
          if (((pieces.size() - base) % col::RP) + (size_t)len > (size_t)col::RP)
            while ((pieces.size() - base) % col::RP) pieces.push_back(make_uint4(0, 0, 0, 0));
          const Mono& mo = monos[rc.mono];
          unsigned long long fac = 0;
          int npos = 0;
          for (int v = 0; v < n; ++v) {
            int a = mo.e[v];
            if (v == rc.var) a -= 1;
            for (int q = 0; q < a; ++q) fac |= (unsigned long long)v << (4 * npos++);
          }
          fac |= (unsigned long long)rc.em << 48;
          unsigned char ps[8];
          for (int i = 0; i < 8; ++i) ps[i] = 0xff;
          for (int i = 0; i < u.nr; ++i) {
            const int k = mo.term_of_row[u.row0 + i];
            if (k >= 0 && d->param_slot && d->param_slot[k] >= 0) ps[i] = (unsigned char)d->param_slot[k];
          }
          uint4 hd;
          hd.x = (unsigned)fac;
          hd.y = (unsigned)(fac >> 32);
          memcpy(&hd.z, ps, 4);
          memcpy(&hd.w, ps + 4, 4);
          pieces.push_back(hd);
          for (int i = 0; i < u.nr; ++i) {
            if (!((r.mask >> i) & 1u)) continue;
            const int k = mo.term_of_row[u.row0 + i];
            const double sr = td ? 0.0 : d->coef_start[2 * k], si = td ? 0.0 : d->coef_start[2 * k + 1];
            const double tr = d->coef_target[2 * k], ti = d->coef_target[2 * k + 1];
            if (u.kind == col::K_ABS) {
              put_cd(acs[k], act[k]);
            } else if (r.cls >= col::C_TWO) {
              put_cd(sr, si);
              put_cd(tr, ti);
            } else if (r.cls == col::C_S) {  // one-coefficient classes carry the partial's multiplier
              put_cd(sr * rc.em, si * rc.em);
            } else {
              put_cd(tr * rc.em, ti * rc.em);
            }
          }
        }
      }
    }
  }
  if (getenv("NID_COL_DEBUG")) {
    for (int w = 0; w < G; ++w) {
      size_t nrec = 0;
      for (int u = cgrun[w]; u < (w + 1 < G ? cgrun[w + 1] : (int)runs_out.size()); ++u) nrec += runs_out[u].w;
      fprintf(stderr, "[col] warp %d: load %.0f, records %zu, runs %d, units H %zu J %zu A %zu\n", w, load[w], nrec,
              (w + 1 < G ? cgrun[w + 1] : (int)runs_out.size()) - cgrun[w], hw[w].size(), jw[w].size(), aw[w].size());
    }
    fprintf(stderr, "[col] monomials %d, pieces %zu, runs %zu\n", M, pieces.size(), runs_out.size());
  }
  for (int w = G; w <= 16; ++w) {
    cgrun[w] = (int)runs_out.size();
    cgbase[w] = (int)pieces.size();
  }
  for (int z = 0; z < (col::RCH + 1) * col::CP; ++z) pieces.push_back(make_uint4(0, 0, 0, 0));
  return runs_out.size() <= (size_t)NID_MAX_RUNS;
}

}  // namespace colhost
