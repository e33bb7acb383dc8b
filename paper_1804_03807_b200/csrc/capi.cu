// libnid.so: the C-ABI boundary (declared in include/nid.h).
// Host-side plumbing only: uploads lowered homotopies, stages host buffers,
// sizes the persistent grids and dispatches to the per-size kernels.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "aux_kernels.cuh"
#include "endpoint.cuh"
#include "launch.h"
#include "track_common.cuh"
#include "track_ctl.cuh"

static thread_local std::string g_err;
// per host thread: one thread per device may track concurrently (nid_init_devices)
static thread_local NidCounters g_counters = {};
static thread_local unsigned long long g_phase[7] = {};
static int g_device = -1;          // the process default (nid_init)
static thread_local int t_device = -1;  // this host thread's choice (nid_use_device / a handle's device)
static int g_devs[16];
static int g_ndev = 0;
static int cur_device() { return t_device >= 0 ? t_device : g_device; }

#define FAIL(msg)          \
  do {                     \
    g_err = (msg);         \
    return 1;              \
  } while (0)
#define CK(call)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess) {                                                              \
      g_err = std::string(#call) + ": " + cudaGetErrorString(e_);                          \
      return 2;                                                                           \
    }                                                                                     \
  } while (0)

// the ABI the ctypes mirror (paper_1804_03807_b200/_lib.py) and tests/test_host.py pin
static_assert(sizeof(NidHomotopyDesc) == 96, "NidHomotopyDesc layout changed");
static_assert(sizeof(NidTrackParams) == 96, "NidTrackParams layout changed");

struct NidHomotopy {
  int device = -1;  // the CUDA device the table lives on (every call on the handle runs there)
  int n, nterms, nparam, maxdeg, multilinear, td;
  int tddeg[NID_MAX_VARS];
  int grow[NID_MAX_VARS];
  int goff[17];
  cd gamma;
  int* row_off;
  uint4* expo;
  uint4 *fac, *fex;
  cd *cs, *ct;
  double *acs, *act;
  int8_t* pslot;
  double* tw = nullptr;  // polyhedral t-exponents (start_kind 2) or null
  PTab* ptab = nullptr;  // host copy of the parameter-bank table (null: table too large / per-path params)
  TermRec* rec = nullptr;  // streamed records (csrc/track_rec.cuh), n > 10
  uint4* runs = nullptr;
  std::vector<uint4> hruns;  // host copy: travels with every launch (TrackArgs::runs_c)
  int grun[17] = {0};
  uint4* crec = nullptr;      // column-owner stream (csrc/track_col.cuh) or null
  std::vector<uint4> hcruns;  // its run descriptors: travel with the launch instead of hruns
  int cgrun[17] = {0};
  int cgbase[17] = {0};
  HomDev dev() const {
    HomDev h;
    h.n = n;
    h.nterms = nterms;
    h.nparam = nparam;
    h.maxdeg = maxdeg;
    h.multilinear = multilinear;
    h.td = td;
    for (int v = 0; v < NID_MAX_VARS; ++v) h.tddeg[v] = tddeg[v];
    for (int v = 0; v < NID_MAX_VARS; ++v) h.grow[v] = grow[v];
    for (int v = 0; v <= 16; ++v) h.goff[v] = goff[v];
    h.row_off = row_off;
    h.expo = expo;
    h.fac = fac;
    h.fex = fex;
    h.cs = cs;
    h.ct = ct;
    h.acs = acs;
    h.act = act;
    h.pslot = pslot;
    h.gamma = gamma;
    h.tw = tw;
    h.rec = rec;
    h.runs = runs;
    for (int v = 0; v <= 16; ++v) h.grun[v] = grun[v];
    h.crec = crec;
    for (int v = 0; v <= 16; ++v) h.cgrun[v] = cgrun[v];
    for (int v = 0; v <= 16; ++v) h.cgbase[v] = cgbase[v];
    h.dd = 0;
    return h;
  }
};

#include "col_lower.h"

// grow-only device workspace slots
struct Buf {
  void* p = nullptr;
  size_t cap = 0;
};
static Buf g_bufs[16][32];  // per CUDA device
template <class T>
static T* ws(int slot, size_t count) {
  size_t bytes = count * sizeof(T) + 16;
  const int d = cur_device();
  Buf& b = g_bufs[(d >= 0 && d < 16) ? d : 0][slot];
  if (b.cap < bytes) {
    if (b.p) cudaFree(b.p);
    b.p = nullptr;
    b.cap = 0;
    if (cudaMalloc(&b.p, bytes) != cudaSuccess) return nullptr;
    b.cap = bytes;
  }
  return reinterpret_cast<T*>(b.p);
}

#define NID_TABLE(fn)                                                                                    \
  {nullptr,  nid::fn##1,  nid::fn##2,  nid::fn##3,  nid::fn##4,  nid::fn##5,  nid::fn##6, nid::fn##7, \
   nid::fn##8, nid::fn##9, nid::fn##10, nid::fn##11, nid::fn##12, nid::fn##13, nid::fn##14, nid::fn##15, \
   nid::fn##16}

typedef int (*TrackFn)(const TrackArgs&, int, cudaStream_t);
typedef int (*EndpointFn)(const EndpointArgs&, int, cudaStream_t);
typedef int (*RefineFn)(const RefineArgs&, int, cudaStream_t);
typedef int (*DDRefineFn)(const DDRefineArgs&, int, cudaStream_t);
typedef int (*EvalFn)(const EvalArgs&, int, cudaStream_t);
typedef int (*NewtonFn)(const NewtonArgs&, int, cudaStream_t);
typedef int (*RegsFn)();
static const TrackFn k_track[17] = NID_TABLE(launch_track_);
typedef int (*TrackPTFn)(const TrackArgsPT&, int, cudaStream_t);
static const TrackPTFn k_track_pt[17] = NID_TABLE(launch_track_pt_);
static const TrackFn k_track_aux[17] = NID_TABLE(launch_track_aux_);
static const RegsFn k_pt_regs[17] = NID_TABLE(track_pt_regs_);
static const EndpointFn k_endpoint[17] = NID_TABLE(launch_endpoint_);
static const RefineFn k_refine[17] = NID_TABLE(launch_refine_);
static const DDRefineFn k_ddrefine[17] = NID_TABLE(launch_ddrefine_);
static const EvalFn k_eval[17] = NID_TABLE(launch_eval_);
static const NewtonFn k_newton[17] = NID_TABLE(launch_newton_);
static const RegsFn k_regs[17] = NID_TABLE(track_regs_);
static const RegsFn k_tthreads[17] = NID_TABLE(track_threads_);

// The CUDA current device is per host thread: every entry point that touches
// the device re-binds the device nid_init chose, so calls from another host
// thread (e.g. the cell-pipeline consumer, polyhedral.pipeline_cells) land on
// the same GPU as the workspaces and handles.
#define BIND()                                                        \
  do {                                                                \
    if (cur_device() >= 0) {                                          \
      cudaError_t be_ = cudaSetDevice(cur_device());                  \
      if (be_ != cudaSuccess) {                                       \
        g_err = std::string("cudaSetDevice: ") + cudaGetErrorString(be_); \
        return 2;                                                     \
      }                                                               \
    }                                                                 \
  } while (0)

// entry points that take a handle run on the handle's device
#define BIND_H(h)                                            \
  do {                                                       \
    if ((h) && (h)->device >= 0) t_device = (h)->device;     \
    BIND();                                                  \
  } while (0)

// CUDA events destroyed on every exit path
struct Events {
  cudaEvent_t e[3] = {nullptr, nullptr, nullptr};
  ~Events() {
    for (auto& x : e)
      if (x) cudaEventDestroy(x);
  }
};

static int sm_count() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

// number of 128-thread blocks for a grid-stride group kernel over P points
static int grid_for(long long P, int n, int per_sm) {
  long long groups_per_block = 4 * (32 / n);
  long long need = (P + groups_per_block - 1) / groups_per_block;
  long long cap = (long long)sm_count() * per_sm;
  if (need > cap) need = cap;
  return need < 1 ? 1 : (int)need;
}

static long long groups_of(int blocks, int n) { return (long long)blocks * 4 * (32 / n); }

extern "C" {

const char* nid_last_error(void) { return g_err.c_str(); }

int nid_device_count(int* count) {
  CK(cudaGetDeviceCount(count));
  return 0;
}

int nid_init(int device) {
  CK(cudaSetDevice(device));
  CK(cudaFree(0));
  g_device = device;
  return 0;
}

int nid_shutdown(void) {
  for (int d = 0; d < 16; ++d) {
    bool any = false;
    for (auto& b : g_bufs[d]) any = any || b.p;
    if (!any) continue;
    CK(cudaSetDevice(d));
    for (auto& b : g_bufs[d]) {
      if (b.p) cudaFree(b.p);
      b.p = nullptr;
      b.cap = 0;
    }
  }
  BIND();
  return 0;
}

int nid_init_devices(int ndev, const int* devs) {
  if (ndev < 1 || ndev > 16 || !devs) FAIL("nid_init_devices: 1..16 devices");
  int have = 0;
  CK(cudaGetDeviceCount(&have));
  for (int i = 0; i < ndev; ++i)
    if (devs[i] < 0 || devs[i] >= have || devs[i] >= 16) FAIL("nid_init_devices: no such device");
  for (int i = 0; i < ndev; ++i) {
    CK(cudaSetDevice(devs[i]));
    CK(cudaFree(0));
    g_devs[i] = devs[i];
    // peer access for the endpoint gather (NVLink / NVSwitch P2P); already-enabled is fine
    for (int j = 0; j < ndev; ++j) {
      if (devs[j] == devs[i]) continue;
      int can = 0;
      cudaDeviceCanAccessPeer(&can, devs[i], devs[j]);
      if (can) {
        cudaError_t e = cudaDeviceEnablePeerAccess(devs[j], 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) CK(e);
        cudaGetLastError();
      }
    }
  }
  g_ndev = ndev;
  g_device = devs[0];
  t_device = devs[0];
  CK(cudaSetDevice(devs[0]));
  return 0;
}

int nid_use_device(int i) {
  if (g_ndev == 0) FAIL("nid_use_device: call nid_init_devices first");
  if (i < 0 || i >= g_ndev) FAIL("nid_use_device: index out of range");
  t_device = g_devs[i];
  CK(cudaSetDevice(t_device));
  return 0;
}

int nid_track_regs(int n) {
  if (n < 1 || n > 16) return -1;
  return k_regs[n]();
}

int nid_homotopy_create(const NidHomotopyDesc* d, NidHomotopy** out) {
  BIND();
  if (!d || !out) FAIL("null argument");
  if (d->n < 1 || d->n > NID_MAX_VARS) FAIL("n must be in 1..16");
  if (d->nterms < 0) FAIL("negative term count");
  const int n = d->n, T = d->nterms;
  int here_ = 0;
  CK(cudaGetDevice(&here_));
  std::vector<int> off(d->row_off, d->row_off + n + 1);
  if (off[0] != 0 || off[n] != T) FAIL("row offsets do not cover the term table");
  for (int i = 0; i < n; ++i)
    if (off[i + 1] < off[i]) FAIL("row offsets not monotone");
  std::vector<double> acs(T), act(T);
  int maxdeg = 0;
  for (int k = 0; k < T; ++k) {
    acs[k] = hypot(d->coef_start[2 * k], d->coef_start[2 * k + 1]);
    act[k] = hypot(d->coef_target[2 * k], d->coef_target[2 * k + 1]);
    for (int v = 0; v < NID_MAX_VARS; ++v) {
      int a = d->expo[k * NID_MAX_VARS + v];
      if (v >= n && a) FAIL("exponent set on a variable >= n");
      if (a > maxdeg) maxdeg = a;
    }
  }
  if (d->start_kind < 0 || d->start_kind > 2) FAIL("unknown start_kind");
  if (d->start_kind == 2) {  // per-cell polyhedral homotopy (polyhedral.py:730-791)
    if (!d->term_texp) FAIL("polyhedral homotopy needs term_texp");
    if (d->param_slot) FAIL("polyhedral homotopy takes no per-path coefficients");
    for (int k = 0; k < T; ++k)
      if (!(d->term_texp[k] >= 0.0) || !std::isfinite(d->term_texp[k])) FAIL("term_texp must be finite and >= 0");
    for (int k = 0; k < 2 * T; ++k)
      if (d->coef_start[k] != 0.0) FAIL("polyhedral homotopy: the term table must hold only the start system g");
  }
  if (d->start_kind == 1) {
    if (!d->start_degrees) FAIL("total-degree start needs start_degrees");
    for (int v = 0; v < n; ++v)
      if (d->start_degrees[v] < 1) FAIL("total-degree start degrees must be >= 1");
    for (int k = 0; k < 2 * T; ++k)
      if (d->coef_start[k] != 0.0) FAIL("total-degree start: the term table must hold only the target");
  }
  NidHomotopy* h = new NidHomotopy();
  h->device = here_;
  h->n = n;
  h->nterms = T;
  h->nparam = d->nparam;
  h->maxdeg = maxdeg;
  h->multilinear = maxdeg <= 1 ? 1 : 0;
  h->td = d->start_kind == 1 ? 1 : 0;
  for (int v = 0; v < NID_MAX_VARS; ++v) h->tddeg[v] = (h->td && v < n) ? d->start_degrees[v] : 0;
  // tracker row groups (rows::groups<n>()): longest-processing-time assignment
  // of rows to warp groups by evaluation cost (terms x their variable count)
  {
    const int G = rows::groups_for(n);
    std::vector<std::pair<double, int>> cost;
    for (int i = 0; i < n; ++i) {
      double c = h->td ? 2.0 + h->tddeg[i] : 0.0;
      for (int k = off[i]; k < off[i + 1]; ++k) {
        int nz = 0;
        for (int v = 0; v < n; ++v) nz += d->expo[k * NID_MAX_VARS + v] ? 1 : 0;
        c += 4.0 + 3.0 * nz;
      }
      cost.push_back({c, i});
    }
    std::sort(cost.begin(), cost.end(), [](const std::pair<double, int>& a, const std::pair<double, int>& b) {
      return a.first > b.first || (a.first == b.first && a.second < b.second);
    });
    std::vector<std::vector<int>> grp(G);
    std::vector<double> load(G, 0.0);
    for (auto& cr : cost) {
      int best = 0;
      for (int gg = 1; gg < G; ++gg)
        if (load[gg] < load[best]) best = gg;
      grp[best].push_back(cr.second);
      load[best] += cr.first;
    }
    if (const char* ov = getenv("NID_ROW_GROUPS")) {  // experiment knob: "g(row 0),g(row 1),..."
      std::vector<int> gi;
      for (const char* c = ov; *c;) {
        gi.push_back(atoi(c));
        while (*c && *c != ',') ++c;
        if (*c == ',') ++c;
      }
      if ((int)gi.size() == n) {
        for (int gg = 0; gg < G; ++gg) grp[gg].clear();
        for (int i = 0; i < n; ++i) grp[(gi[i] % G + G) % G].push_back(i);
      }
    }
    int pos = 0;
    for (int gg = 0; gg <= 16; ++gg) h->goff[gg] = 0;
    for (int gg = 0; gg < G; ++gg) {
      h->goff[gg] = pos;
      std::sort(grp[gg].begin(), grp[gg].end());
      for (int r : grp[gg]) h->grow[pos++] = r;
    }
    for (int gg = G; gg <= 16; ++gg) h->goff[gg] = pos;
  }
  h->gamma = cd{d->gamma_re, d->gamma_im};
  const size_t Tp = T > 0 ? T : 1;
  cudaError_t e = cudaSuccess;
  e = e ? e : cudaMalloc(&h->row_off, (n + 1) * sizeof(int));
  e = e ? e : cudaMalloc(&h->expo, Tp * sizeof(uint4));
  e = e ? e : cudaMalloc(&h->fac, Tp * sizeof(uint4));
  e = e ? e : cudaMalloc(&h->fex, Tp * sizeof(uint4));
  e = e ? e : cudaMalloc(&h->cs, Tp * sizeof(cd));
  e = e ? e : cudaMalloc(&h->ct, Tp * sizeof(cd));
  e = e ? e : cudaMalloc(&h->acs, Tp * sizeof(double));
  e = e ? e : cudaMalloc(&h->act, Tp * sizeof(double));
  h->pslot = nullptr;
  if (!e && d->param_slot) e = cudaMalloc(&h->pslot, Tp);
  if (!e && d->start_kind == 2) e = cudaMalloc(&h->tw, Tp * sizeof(double));
  if (!e && d->start_kind == 2 && T) e = cudaMemcpy(h->tw, d->term_texp, T * sizeof(double), cudaMemcpyHostToDevice);
  if (!e) e = cudaMemcpy(h->row_off, off.data(), (n + 1) * sizeof(int), cudaMemcpyHostToDevice);
  if (!e && T) e = cudaMemcpy(h->expo, d->expo, T * sizeof(uint4), cudaMemcpyHostToDevice);
  if (!e && T) {
    // factor lists of every term (the tracker's evaluator loops over the
    // variables a term contains instead of over all n)
    std::vector<uint4> fac(T), fex(T);
    for (int k = 0; k < T; ++k) {
      unsigned long long vl = 0;
      unsigned ex[4] = {0, 0, 0, 0};
      int nf = 0;
      for (int v = 0; v < n; ++v) {
        const int a = d->expo[k * NID_MAX_VARS + v];
        if (!a) continue;
        vl |= (unsigned long long)v << (4 * nf);
        ex[nf >> 2] |= (unsigned)a << (8 * (nf & 3));
        ++nf;
      }
      fac[k] = make_uint4((unsigned)vl, (unsigned)(vl >> 32), (unsigned)nf, 0u);
      fex[k] = make_uint4(ex[0], ex[1], ex[2], ex[3]);
    }
    // w: end of the run of equal factor counts starting at k (within its row)
    for (int i = 0; i < n; ++i)
      for (int k = off[i + 1] - 1; k >= off[i]; --k)
        fac[k].w = (k + 1 < off[i + 1] && fac[k + 1].z == fac[k].z) ? fac[k + 1].w : (unsigned)(k + 1);
    // the parameter-bank table (csrc/track_ptab.cuh) when the system fits it
    if (!d->param_slot && T <= PT_MAXT) {
      PTab* pt = new PTab();
      memset(pt, 0, sizeof(PTab));
      int nr = 0, nf = 0;
      bool fits = true;
      for (int i = 0; i < n && fits; ++i) {
        pt->row_run[i] = (unsigned short)nr;
        for (int k = off[i]; k < off[i + 1] && fits;) {
          const int K = (int)fac[k].z;
          int k1 = k;
          while (k1 < off[i + 1] && (int)fac[k1].z == K && k1 - k < 255) ++k1;
          if (nr >= PT_MAXR || nf + (k1 - k) * K > PT_MAXF) {
            fits = false;
            break;
          }
          pt->run_k0[nr] = (unsigned short)k;
          pt->run_f0[nr] = (unsigned short)nf;
          pt->run_K[nr] = (unsigned char)K;
          pt->run_n[nr] = (unsigned char)(k1 - k);
          ++nr;
          for (int kk = k; kk < k1; ++kk)
            for (int v = 0; v < n; ++v) {
              const int a = d->expo[kk * NID_MAX_VARS + v];
              if (!a) continue;
              pt->foff[nf] = (unsigned)(v * rows::SLOTS * sizeof(cd));
              pt->fexp[nf] = (unsigned char)a;
              ++nf;
            }
          k = k1;
        }
      }
      pt->row_run[n] = (unsigned short)nr;
      for (int k = 0; k < T && fits; ++k) {
        pt->ct[k] = cd{d->coef_target[2 * k], d->coef_target[2 * k + 1]};
        pt->cs[k] = cd{d->coef_start[2 * k], d->coef_start[2 * k + 1]};
        pt->act[k] = act[k];
        pt->acs[k] = acs[k];
      }
      if (d->start_kind == 2) {
        pt->poly = 1;
        for (int k = 0; k < T; ++k) pt->tw[k] = d->term_texp[k];
      }
      if (fits) h->ptab = pt;
      else delete pt;
    }
    e = cudaMemcpy(h->fac, fac.data(), T * sizeof(uint4), cudaMemcpyHostToDevice);
    if (!e) e = cudaMemcpy(h->fex, fex.data(), T * sizeof(uint4), cudaMemcpyHostToDevice);
    // streamed records for the large-system tracker (csrc/track_rec.cuh): per
    // warp group, its rows in order, each row's terms grouped by factor count
    // (stable), records contiguous; every term of total degree <= 12
    bool rec_ok = n >= 8 && !h->ptab && d->start_kind != 2;  // ctl::rec_on<n>()
    for (int k = 0; k < T && rec_ok; ++k) {
      int deg = 0;
      for (int v = 0; v < n; ++v) deg += d->expo[k * NID_MAX_VARS + v];
      if (deg > 12) rec_ok = false;
    }
    if (!e && rec_ok) {
      const int G = rows::groups_for(n);
      std::vector<TermRec> recs;
      std::vector<uint4> runs;
      recs.reserve(T + 16);
      for (int gg = 0; gg <= 16; ++gg) h->grun[gg] = 0;
      for (int gg = 0; gg < G; ++gg) {
        h->grun[gg] = (int)runs.size();
        const long long grp_base = (long long)recs.size();
        for (int gi = h->goff[gg]; gi < h->goff[gg + 1]; ++gi) {
          const int i = h->grow[gi];
          // (total degree, and for degree <= rec::SDUPK the repeat pattern << 8; term):
          // a run of short terms shares one pattern, so the evaluator's body for it
          // loads every distinct variable once and folds repeats without selects
          std::vector<std::pair<int, int>> byk;
          for (int k = off[i]; k < off[i + 1]; ++k) {
            int deg = 0, pat = 0;
            for (int v = 0; v < n; ++v)
              for (int a = 0; a < d->expo[k * NID_MAX_VARS + v]; ++a) {
                if (a > 0) pat |= 1 << deg;
                ++deg;
              }
            const bool stat = deg >= 1 && deg <= rec::SDUPK && !getenv("NID_REC_NO_STATIC_DUP");
            // sort key: degree first, so a row's runs of one factor count stay adjacent
            // (the per-slot evaluator walks them as one run)
            byk.push_back({(deg << 12) | (stat ? (0x800 | pat) : 0), k});
          }
          std::stable_sort(byk.begin(), byk.end(),
                           [](const std::pair<int, int>& a, const std::pair<int, int>& b) { return a.first < b.first; });
          if (byk.empty()) runs.push_back(make_uint4((unsigned)i, 0u, (unsigned)recs.size(), 0u));
          for (size_t q = 0; q < byk.size();) {
            size_t q1 = q;
            while (q1 < byk.size() && byk[q1].first == byk[q].first) ++q1;
            const int deg_q = byk[q].first >> 12;
            const unsigned ykey = (unsigned)deg_q | ((byk[q].first & 0x800) ? (0x100u | ((unsigned)(byk[q].first & 0x7ff) << 9)) : 0u);
            // bit 30: some term of the run takes a per-path coefficient (membership
            // targets): only such runs look at the records' parameter slots
            unsigned hasp = 0u;
            if (d->param_slot)
              for (size_t z = q; z < q1; ++z)
                if (d->param_slot[byk[z].second] >= 0) hasp = 1u << 30;
            runs.push_back(make_uint4((unsigned)i, ykey | hasp, (unsigned)recs.size(), (unsigned)(q1 - q)));
            // Order the run as [one single if the run starts at an odd offset from the
            // group's first record] [pairs of terms with disjoint variables (greedy, first
            // fit within a window): the evaluator interleaves their product chains] [the
            // remaining singles]; the run descriptor carries the lead flag (y bit 28) and
            // the pair count (y bits 16..27), so the evaluator tells a pair by position.
            std::vector<int> pend;
            for (size_t z = q; z < q1; ++z) pend.push_back(byk[z].second);
            auto vmask = [&](int k) {
              unsigned mk = 0;
              for (int v = 0; v < n; ++v)
                if (d->expo[k * NID_MAX_VARS + v]) mk |= 1u << v;
              return mk;
            };
            std::vector<std::pair<int, int>> pairs;
            std::vector<int> singles;
            while (!pend.empty()) {
              const int a = pend.front();
              pend.erase(pend.begin());
              bool paired = false;
              if (deg_q > 0 && deg_q <= 6 && pairs.size() < 4095) {  // rec::PAIRK
                const unsigned ma = vmask(a);
                for (size_t z = 0; z < pend.size() && z < 64; ++z)
                  if (!(vmask(pend[z]) & ma)) {
                    pairs.push_back({a, pend[z]});
                    pend.erase(pend.begin() + z);
                    paired = true;
                    break;
                  }
              }
              if (!paired) singles.push_back(a);
            }
            const bool odd = ((recs.size() - (size_t)grp_base) & 1) != 0;
            if (odd && !pairs.empty() && singles.empty()) {  // no single to realign with: split a pair
              singles.push_back(pairs.back().first);
              singles.push_back(pairs.back().second);
              pairs.pop_back();
            }
            std::vector<std::pair<int, bool>> order;  // (term, paired with the next)
            unsigned lead = 0u;
            if (odd && !pairs.empty()) {
              order.push_back({singles.front(), false});
              singles.erase(singles.begin());
              lead = 1u;
            }
            for (auto& pr : pairs) {
              order.push_back({pr.first, true});
              order.push_back({pr.second, false});
            }
            for (int k1 : singles) order.push_back({k1, false});
            runs.back().y |= (lead << 28) | ((unsigned)pairs.size() << 16);
            for (size_t z = 0; z < order.size(); ++z) {
              const int k = order[z].first;
              TermRec r;
              memset(&r, 0, sizeof(r));
              r.ctr = d->coef_target[2 * k];
              r.cti = d->coef_target[2 * k + 1];
              r.csr = d->coef_start[2 * k];
              r.csi = d->coef_start[2 * k + 1];
              r.acs = acs[k];
              r.act = act[k];
              unsigned long long meta = 0;
              int npos = 0;
              for (int v = 0; v < n; ++v)
                for (int a = 0; a < d->expo[k * NID_MAX_VARS + v]; ++a) {
                  meta |= (unsigned long long)v << (4 * npos);
                  if (a > 0) meta |= 1ull << (52 + npos);
                  ++npos;
                }
              meta |= (unsigned long long)npos << 48;
              if (order[z].second) meta |= 1ull << 52;  // paired with the next record
              r.meta = meta;
              r.pslot = d->param_slot ? (int)d->param_slot[k] : -1;
              recs.push_back(r);
            }
            q = q1;
          }
        }
      }
      for (int gg = G; gg <= 16; ++gg) h->grun[gg] = (int)runs.size();
      for (int z = 0; z < 16; ++z) {  // the ring reads up to two chunks past a group's end
        TermRec r;
        memset(&r, 0, sizeof(r));
        recs.push_back(r);
      }
      e = cudaMalloc(&h->rec, recs.size() * sizeof(TermRec));
      if (!e) e = cudaMemcpy(h->rec, recs.data(), recs.size() * sizeof(TermRec), cudaMemcpyHostToDevice);
      if (!e) e = cudaMalloc(&h->runs, (runs.size() + 1) * sizeof(uint4));
      if (!e && !runs.empty()) e = cudaMemcpy(h->runs, runs.data(), runs.size() * sizeof(uint4), cudaMemcpyHostToDevice);
      h->hruns = runs;
      if (e || getenv("NID_NO_REC") || runs.size() > (size_t)NID_MAX_RUNS) {
        cudaFree(h->rec);
        cudaFree(h->runs);
        h->rec = nullptr;
        h->runs = nullptr;
      }
      // the column-owner stream (csrc/track_col.cuh) beside the records, which
      // stay for the per-slot evaluator; n = 8 .. 14 (ctl::lat_on<n>(): the
      // partial sums of the values use the per-slot scratch)
      if (!e && h->rec && n <= 14 && !getenv("NID_NO_COL")) {
        std::vector<uint4> pieces, cruns;
        if (colhost::build(d, n, T, off, acs, act, G, h->td != 0, pieces, cruns, h->cgrun, h->cgbase)) {
          e = cudaMalloc(&h->crec, pieces.size() * sizeof(uint4));
          if (!e) e = cudaMemcpy(h->crec, pieces.data(), pieces.size() * sizeof(uint4), cudaMemcpyHostToDevice);
          h->hcruns = cruns;
        }
      }
    }
  }
  if (!e && T) e = cudaMemcpy(h->cs, d->coef_start, T * sizeof(cd), cudaMemcpyHostToDevice);
  if (!e && T) e = cudaMemcpy(h->ct, d->coef_target, T * sizeof(cd), cudaMemcpyHostToDevice);
  if (!e && T) e = cudaMemcpy(h->acs, acs.data(), T * sizeof(double), cudaMemcpyHostToDevice);
  if (!e && T) e = cudaMemcpy(h->act, act.data(), T * sizeof(double), cudaMemcpyHostToDevice);
  if (!e && T && d->param_slot) e = cudaMemcpy(h->pslot, d->param_slot, T, cudaMemcpyHostToDevice);
  if (e) {
    g_err = std::string("homotopy upload: ") + cudaGetErrorString(e);
    nid_homotopy_destroy(h);  // frees whatever was allocated (members start null)
    return 2;
  }
  *out = h;
  return 0;
}

int nid_col_lower(const NidHomotopyDesc* d, int groups, unsigned* pieces, long long cap_pieces, long long* n_pieces,
                  unsigned* runs, long long cap_runs, long long* n_runs, int* cgrun, int* cgbase, int* eligible) {
  if (!d || !n_pieces || !n_runs || !cgrun || !cgbase || !eligible) FAIL("null argument");
  if (d->n < 1 || d->n > NID_MAX_VARS || d->nterms < 0) FAIL("bad table shape");
  if (groups < 1 || groups > 16) FAIL("groups must be in 1..16");
  const int n = d->n, T = d->nterms;
  std::vector<int> off(d->row_off, d->row_off + n + 1);
  if (off[0] != 0 || off[n] != T) FAIL("row offsets do not cover the term table");
  std::vector<double> acs(T), act(T);
  for (int k = 0; k < T; ++k) {
    acs[k] = hypot(d->coef_start[2 * k], d->coef_start[2 * k + 1]);
    act[k] = hypot(d->coef_target[2 * k], d->coef_target[2 * k + 1]);
  }
  std::vector<uint4> pc, rn;
  int gr[17], gb[17];
  const bool ok = colhost::build(d, n, T, off, acs, act, groups, d->start_kind == 1, pc, rn, gr, gb);
  *eligible = ok ? 1 : 0;
  if (!ok) return 0;
  *n_pieces = (long long)pc.size();
  *n_runs = (long long)rn.size();
  for (int w = 0; w < 17; ++w) {
    cgrun[w] = gr[w];
    cgbase[w] = gb[w];
  }
  if (pieces)
    for (long long z = 0; z < (long long)pc.size() && z < cap_pieces; ++z) memcpy(pieces + 4 * z, &pc[z], 16);
  if (runs)
    for (long long z = 0; z < (long long)rn.size() && z < cap_runs; ++z) memcpy(runs + 4 * z, &rn[z], 16);
  return 0;
}

int nid_homotopy_destroy(NidHomotopy* h) {
  if (!h) return 0;
  BIND_H(h);
  cudaFree(h->row_off);
  cudaFree(h->expo);
  delete h->ptab;
  cudaFree(h->fac);
  cudaFree(h->fex);
  if (h->rec) cudaFree(h->rec);
  if (h->runs) cudaFree(h->runs);
  if (h->crec) cudaFree(h->crec);
  cudaFree(h->cs);
  cudaFree(h->ct);
  cudaFree(h->acs);
  cudaFree(h->act);
  if (h->pslot) cudaFree(h->pslot);
  if (h->tw) cudaFree(h->tw);
  delete h;
  return 0;
}

int nid_track_groups(int n) { return (n < 1 || n > 16) ? -1 : rows::groups_for(n); }

int nid_phase_cycles(unsigned long long* out7) {
  if (!out7) FAIL("null argument");
  for (int i = 0; i < 7; ++i) out7[i] = g_phase[i];
  return 0;
}

int nid_last_counters(NidCounters* c) {
  if (!c) FAIL("null argument");
  *c = g_counters;
  return 0;
}

// slot map for the workspace cache
enum {
  W_STARTS = 0, W_PARAMS, W_XEND, W_STATUS, W_STEPS, W_TREACH, W_RESID, W_COND, W_REG,
  W_COUNT, W_SCR, W_DDSCR, W_X, W_T, W_H, W_J, W_SCALE, W_I32, W_I8, W_I8B, W_TOL, W_ROOTS, W_GSTATE, W_PTW, W_TRACE, W_TRACEN, W_CBLK, W_COFF, W_GBUF, W_GIDX
};

static int track_impl(NidHomotopy* h, const NidTrackParams* prm, int P, const double* starts, long long first_index,
                      long long index_stride, const int32_t* degrees, const double* params, int param_div,
                      const double* path_texp, NidPathOut* out, int device_io, void* stream, int trace_cap = 0,
                      double* trace = nullptr, int32_t* trace_n = nullptr);

int nid_track_batch(NidHomotopy* h, const NidTrackParams* prm, int P, const double* starts,
                    long long first_index, const int32_t* degrees, const double* params, int param_div,
                    NidPathOut* out, int device_io, void* stream) {
  return nid_track_batch_strided(h, prm, P, starts, first_index, 1, degrees, params, param_div, out, device_io,
                                 stream);
}

int nid_track_batch_strided(NidHomotopy* h, const NidTrackParams* prm, int P, const double* starts,
                            long long first_index, long long index_stride, const int32_t* degrees,
                            const double* params, int param_div, NidPathOut* out, int device_io,
                            void* stream) {
  return track_impl(h, prm, P, starts, first_index, index_stride, degrees, params, param_div, nullptr, out, device_io,
                    stream);
}

int nid_track_trace(NidHomotopy* h, const NidTrackParams* prm, int P, const double* starts, const double* params,
                    int param_div, NidPathOut* out, int trace_cap, double* trace, int32_t* trace_n) {
  if (!starts) FAIL("nid_track_trace needs explicit start points");
  if (trace_cap < 1) FAIL("trace_cap must be >= 1");
  return track_impl(h, prm, P, starts, 0, 1, nullptr, params, param_div, nullptr, out, 0, nullptr, trace_cap, trace,
                    trace_n);
}

int nid_track_cells(NidHomotopy* h, const NidTrackParams* prm, int P, const double* starts, const double* path_texp,
                    NidPathOut* out, int device_io, void* stream) {
  if (!h || !h->tw) FAIL("nid_track_cells needs a polyhedral homotopy (start_kind 2)");
  if (!starts || !path_texp) FAIL("nid_track_cells needs start points and per-path t-exponent rows");
  return track_impl(h, prm, P, starts, 0, 1, nullptr, nullptr, 1, path_texp, out, device_io, stream);
}

static int track_impl(NidHomotopy* h, const NidTrackParams* prm, int P, const double* starts, long long first_index,
                      long long index_stride, const int32_t* degrees, const double* params, int param_div,
                      const double* path_texp, NidPathOut* out, int device_io, void* stream, int trace_cap,
                      double* trace, int32_t* trace_n) {
  if (!h || !prm || !out) FAIL("null argument");
  if (prm->precision != 0 && prm->precision != 1) FAIL("precision must be 0 (double) or 1 (double_double)");
  const bool use_aux = prm->precision == 1 || trace_cap > 0;
  if (use_aux && (h->tw || path_texp))
    FAIL("double-double tracking and step traces are not available for per-cell polyhedral homotopies");
  if (trace_cap > 0 && (!trace || !trace_n)) FAIL("trace buffers missing");
  if (trace_cap > 0 && device_io) FAIL("step traces are returned to host buffers only");
  BIND_H(h);
  if (index_stride < 1) FAIL("index_stride must be >= 1");
  if (P < 0) FAIL("negative path count");
  const int n = h->n;
  cudaStream_t s = (cudaStream_t)stream;
  memset(&g_counters, 0, sizeof(g_counters));
  if (P == 0) return 0;
  if (!starts && !degrees) FAIL("need explicit starts or total-degree degrees");
  if (trace_cap > 0 && (size_t)P * trace_cap * 3 * sizeof(double) > ((size_t)1 << 31))
    FAIL("step trace: P * trace_cap too large (trace small batches)");
  if (h->tw && h->rec) FAIL("polyhedral homotopy: the streamed-record tracker does not evaluate t-weighted coefficients");
  if (h->tw && !starts) FAIL("polyhedral homotopy: explicit (binomial) start points are required");
  if (h->nparam > 0 && !params) FAIL("homotopy has per-path parameters but none were given");
  if (param_div < 1) param_div = 1;

  const cd* d_starts = nullptr;
  const cd* d_params = nullptr;
  cd* d_x;
  int8_t *d_st, *d_reg;
  int* d_steps;
  double *d_tr, *d_res, *d_cond;
  if (device_io) {
    // complex arrays are read/written as 128-bit words
    if (((uintptr_t)starts | (uintptr_t)params | (uintptr_t)out->x_end) & 15)
      FAIL("device_io: starts, params and x_end must be 16-byte aligned");
    d_starts = (const cd*)starts;
    d_params = (const cd*)params;
    d_x = (cd*)out->x_end;
    d_st = out->status;
    d_steps = out->steps;
    d_tr = out->t_reached;
    d_res = out->residual;
    d_cond = out->condition;
    d_reg = out->regular;
  } else {
    if (starts) {
      cd* p = ws<cd>(W_STARTS, (size_t)P * n);
      if (!p) FAIL("out of device memory (starts)");
      CK(cudaMemcpyAsync(p, starts, (size_t)P * n * sizeof(cd), cudaMemcpyHostToDevice, s));
      d_starts = p;
    }
    if (params && h->nparam > 0) {
      size_t np = ((size_t)(P - 1) / param_div + 1) * h->nparam;
      cd* p = ws<cd>(W_PARAMS, np);
      if (!p) FAIL("out of device memory (params)");
      CK(cudaMemcpyAsync(p, params, np * sizeof(cd), cudaMemcpyHostToDevice, s));
      d_params = p;
    }
    d_x = ws<cd>(W_XEND, (size_t)P * n);
    d_st = ws<int8_t>(W_STATUS, P);
    d_steps = ws<int>(W_STEPS, P);
    d_tr = ws<double>(W_TREACH, P);
    d_res = ws<double>(W_RESID, P);
    d_cond = ws<double>(W_COND, P);
    d_reg = ws<int8_t>(W_REG, P);
    if (!d_x || !d_st || !d_steps || !d_tr || !d_res || !d_cond || !d_reg) FAIL("out of device memory (outputs)");
  }
  const double* d_ptw = nullptr;
  if (path_texp) {
    if (device_io) {
      d_ptw = path_texp;
    } else {
      double* p = ws<double>(W_PTW, (size_t)P * (h->nterms > 0 ? h->nterms : 1));
      if (!p) FAIL("out of device memory (t-exponent rows)");
      CK(cudaMemcpyAsync(p, path_texp, (size_t)P * h->nterms * sizeof(double), cudaMemcpyHostToDevice, s));
      d_ptw = p;
    }
  }
  unsigned long long* d_cnt = ws<unsigned long long>(W_COUNT, 16);
  if (!d_cnt) FAIL("out of device memory (counters)");
  CK(cudaMemsetAsync(d_cnt, 0, 16 * sizeof(unsigned long long), s));

  TrackArgs a;
  memset(&a, 0, sizeof(a));
  a.H = h->dev();
  a.prm = *prm;
  a.P = P;
  a.first_index = first_index;
  a.index_stride = index_stride;
  a.starts = d_starts;
  for (int v = 0; v < NID_MAX_VARS; ++v) a.deg[v] = (degrees && v < n) ? degrees[v] : 1;
  if (!starts) {
    // roots of unity exp(2 pi i k/d) = cos/sin(pi * (2k/d)), the formula of
    // systems.total_degree_starts on the host side
    std::vector<cd> roots;
    for (int v = 0; v < n; ++v) {
      if (a.deg[v] < 1) FAIL("total-degree start degrees must be >= 1");
      a.root_off[v] = (int)roots.size();
      for (int k = 0; k < a.deg[v]; ++k) {
        double ang = 3.141592653589793 * (2.0 * (double)k / (double)a.deg[v]);
        roots.push_back(cd{cos(ang), sin(ang)});
      }
    }
    cd* dr = ws<cd>(W_ROOTS, roots.size());
    if (!dr) FAIL("out of device memory (roots)");
    CK(cudaMemcpyAsync(dr, roots.data(), roots.size() * sizeof(cd), cudaMemcpyHostToDevice, s));
    CK(cudaStreamSynchronize(s));
    a.roots = dr;
  }
  a.params = d_params;
  a.param_div = param_div;
  a.ptw = d_ptw;
  a.next = d_cnt + 7;
  a.x_end = d_x;
  a.status = d_st;
  a.steps = d_steps;
  a.t_reached = d_tr;
  a.resid = d_res;
  a.counters = d_cnt;
  // lstsq scratch for every resident thread (one path per thread)
  const int max_blocks = sm_count() * 8;
  a.scratch = ws<cd>(W_SCR, (size_t)max_blocks * k_tthreads[n]() * (3 * n * n + 2 * n));
  if (!a.scratch) FAIL("out of device memory (scratch)");
  a.gstate = ws<cd>(W_GSTATE, (size_t)max_blocks * 3 * n * rows::SLOTS);
  // per-slot evaluation (streamed-record tracker, n >= 8) when a block has at
  // most lat_slots evaluating slots: the drain of a launch and launches smaller
  // than the machine, where a level lasts as long as its slowest paths
  // (the column-owner stream's descriptors when the table has one: track_col.cuh)
  const std::vector<uint4>& lruns = h->crec ? h->hcruns : h->hruns;
  for (size_t u = 0; u < lruns.size() && u < (size_t)NID_MAX_RUNS; ++u) a.runs_c[u] = lruns[u];
  a.lat_slots = 4;  // (8 until the column-owner block pass: profiles/lat_slots_sweep_r02.log)
  if (getenv("NID_LAT_SLOTS")) a.lat_slots = atoi(getenv("NID_LAT_SLOTS"));
  if (!a.gstate) FAIL("out of device memory (slot state)");

  double* d_trace = nullptr;
  int* d_trace_n = nullptr;
  if (trace_cap > 0) {
    d_trace = ws<double>(W_TRACE, (size_t)P * trace_cap * 3);
    d_trace_n = ws<int>(W_TRACEN, P);
    if (!d_trace || !d_trace_n) FAIL("out of device memory (step trace)");
    CK(cudaMemsetAsync(d_trace_n, 0, (size_t)P * sizeof(int), s));
    a.trace = d_trace;
    a.trace_n = d_trace_n;
    a.trace_cap = trace_cap;
  }
  a.H.dd = prm->precision == 1;

  Events ev;
  CK(cudaEventCreate(&ev.e[0]));
  CK(cudaEventCreate(&ev.e[1]));
  CK(cudaEventCreate(&ev.e[2]));
  cudaEvent_t e0 = ev.e[0], e1 = ev.e[1], e2 = ev.e[2];
  CK(cudaEventRecord(e0, s));
  if (use_aux) {
    k_track_aux[n](a, max_blocks, s);
  } else if (h->ptab && !getenv("NID_NO_PTAB")) {
    TrackArgsPT* pa = new TrackArgsPT;  // ~22 KB: off the stack
    pa->a = a;
    pa->t = *h->ptab;
    k_track_pt[n](*pa, max_blocks, s);
    delete pa;
  } else {
    k_track[n](a, max_blocks, s);
  }
  CK(cudaGetLastError());
  CK(cudaEventRecord(e1, s));

  EndpointArgs E;
  memset(&E, 0, sizeof(E));
  E.H = h->dev();
  E.P = P;
  E.dd_steps = prm->dd_refine_singular > 0 ? (prm->dd_refine_singular > 14 ? prm->dd_refine_singular : 14) : 0;
  E.dd_mode = prm->precision == 1;
  if (E.dd_mode) E.dd_steps = prm->dd_refine_singular > 3 ? prm->dd_refine_singular : 3;  // tracker.py:489
  E.params = d_params;
  E.param_div = param_div;
  E.x_end = d_x;
  E.status = d_st;
  E.resid = d_res;
  E.cond = d_cond;
  E.regular = d_reg;
  E.counters = d_cnt + 4;
  int eblocks = grid_for(P, n, 4);
  E.ddscratch = ws<cdd>(W_DDSCR, (size_t)groups_of(eblocks, n) * (2 * n * n + 4 * n));
  E.cscratch = ws<cd>(W_TOL, (size_t)groups_of(eblocks, n) * (2 * n * n));
  if (!E.ddscratch || !E.cscratch) FAIL("out of device memory (endpoint scratch)");
  k_endpoint[n](E, eblocks, s);
  CK(cudaGetLastError());
  CK(cudaEventRecord(e2, s));

  if (!device_io) {
    CK(cudaMemcpyAsync(out->x_end, d_x, (size_t)P * n * sizeof(cd), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(out->status, d_st, P, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(out->steps, d_steps, P * sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(out->t_reached, d_tr, P * sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(out->residual, d_res, P * sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(out->condition, d_cond, P * sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(out->regular, d_reg, P, cudaMemcpyDeviceToHost, s));
  }
  if (trace_cap > 0) {
    CK(cudaMemcpyAsync(trace, d_trace, (size_t)P * trace_cap * 3 * sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(trace_n, d_trace_n, (size_t)P * sizeof(int), cudaMemcpyDeviceToHost, s));
  }
  unsigned long long hc[16];
  CK(cudaMemcpyAsync(hc, d_cnt, sizeof(hc), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  for (int i = 0; i < 7; ++i) g_phase[i] = hc[8 + i];
  float ms1 = 0.f, ms2 = 0.f;
  cudaEventElapsedTime(&ms1, e0, e1);
  cudaEventElapsedTime(&ms2, e1, e2);
  g_counters.evals = (long long)hc[0];
  g_counters.jacs = (long long)hc[1];
  g_counters.scales = (long long)hc[2];
  g_counters.lstsq_fallbacks = (long long)hc[3];
  g_counters.dd_polished = (long long)hc[4];
  g_counters.paths = P;
  g_counters.kernel_ms_track = ms1;
  g_counters.kernel_ms_endpoint = ms2;
  return 0;
}

int nid_eval_batch(NidHomotopy* h, int P, const double* x, const double* t, const double* params, int param_div,
                   double* H, double* J, double* scale) {
  if (!h || !x || !t || !H || !J || !scale) FAIL("null argument");
  BIND_H(h);
  if (P <= 0) return 0;
  const int n = h->n;
  if (param_div < 1) param_div = 1;
  cd* dx = ws<cd>(W_X, (size_t)P * n);
  double* dt = ws<double>(W_T, P);
  cd* dH = ws<cd>(W_H, (size_t)P * n);
  cd* dJ = ws<cd>(W_J, (size_t)P * n * n);
  double* ds = ws<double>(W_SCALE, P);
  if (!dx || !dt || !dH || !dJ || !ds) FAIL("out of device memory");
  cd* dp = nullptr;
  if (h->nparam > 0) {
    if (!params) FAIL("homotopy has per-path parameters but none were given");
    size_t np = ((size_t)(P - 1) / param_div + 1) * h->nparam;
    dp = ws<cd>(W_PARAMS, np);
    CK(cudaMemcpy(dp, params, np * sizeof(cd), cudaMemcpyHostToDevice));
  }
  CK(cudaMemcpy(dx, x, (size_t)P * n * sizeof(cd), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dt, t, P * sizeof(double), cudaMemcpyHostToDevice));
  EvalArgs E;
  E.H = h->dev();
  E.P = P;
  E.x = dx;
  E.t = dt;
  E.params = dp;
  E.param_div = param_div;
  E.Hout = dH;
  E.Jout = dJ;
  E.scale = ds;
  k_eval[n](E, grid_for(P, n, 8), 0);
  CK(cudaGetLastError());
  CK(cudaMemcpy(H, dH, (size_t)P * n * sizeof(cd), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(J, dJ, (size_t)P * n * n * sizeof(cd), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(scale, ds, P * sizeof(double), cudaMemcpyDeviceToHost));
  return 0;
}

int nid_newton_step_batch(int n, int P, const double* J, const double* r, double* dx) {
  if (!J || !r || !dx) FAIL("null argument");
  BIND();
  if (n < 1 || n > 16) FAIL("n must be in 1..16");
  if (P <= 0) return 0;
  cd* dJ = ws<cd>(W_J, (size_t)P * n * n);
  cd* dr = ws<cd>(W_H, (size_t)P * n);
  cd* dd_ = ws<cd>(W_X, (size_t)P * n);
  int blocks = grid_for(P, n, 8);
  cd* sc = ws<cd>(W_SCR, (size_t)groups_of(blocks, n) * (3 * n * n + 2 * n));
  if (!dJ || !dr || !dd_ || !sc) FAIL("out of device memory");
  CK(cudaMemcpy(dJ, J, (size_t)P * n * n * sizeof(cd), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dr, r, (size_t)P * n * sizeof(cd), cudaMemcpyHostToDevice));
  NewtonArgs A;
  A.P = P;
  A.J = dJ;
  A.r = dr;
  A.dx = dd_;
  A.cscratch = sc;
  k_newton[n](A, blocks, 0);
  CK(cudaGetLastError());
  CK(cudaMemcpy(dx, dd_, (size_t)P * n * sizeof(cd), cudaMemcpyDeviceToHost));
  return 0;
}

int nid_svd_batch(int m, int n, int P, const double* A, double* sv) {
  if (!A || !sv) FAIL("null argument");
  BIND();
  if (n < 1 || n > 16 || m < n || m > 32) FAIL("need 1 <= n <= 16 and n <= m <= 32");
  if (P <= 0) return 0;
  cd* dA = ws<cd>(W_J, (size_t)P * m * n);
  cd* sc = ws<cd>(W_SCR, (size_t)P * m * n);
  double* ds = ws<double>(W_SCALE, (size_t)P * n);
  if (!dA || !sc || !ds) FAIL("out of device memory");
  CK(cudaMemcpy(dA, A, (size_t)P * m * n * sizeof(cd), cudaMemcpyHostToDevice));
  svd_kernel<<<(P + 127) / 128, 128>>>(m, n, P, dA, sc, ds);
  CK(cudaGetLastError());
  CK(cudaMemcpy(sv, ds, (size_t)P * n * sizeof(double), cudaMemcpyDeviceToHost));
  return 0;
}

int nid_refine_batch(NidHomotopy* h, int P, double* x, double tol, int iters, int n_original,
                     double infinity_threshold, double* residual, double* condition, int8_t* regular,
                     int32_t* rank, int8_t* slack_class) {
  if (!h || !x || !residual || !condition || !regular || !rank || !slack_class) FAIL("null argument");
  BIND_H(h);
  if (h->nparam > 0) FAIL("refine does not take per-path parameters");
  if (P <= 0) return 0;
  const int n = h->n;
  int blocks = grid_for(P, n, 4);
  cd* dx = ws<cd>(W_X, (size_t)P * n);
  double* dres = ws<double>(W_RESID, P);
  double* dcond = ws<double>(W_COND, P);
  int8_t* dreg = ws<int8_t>(W_REG, P);
  int* drank = ws<int>(W_I32, P);
  int8_t* dcls = ws<int8_t>(W_I8, P);
  cd* sc = ws<cd>(W_SCR, (size_t)groups_of(blocks, n) * (3 * n * n + 2 * n));
  if (!dx || !dres || !dcond || !dreg || !drank || !dcls || !sc) FAIL("out of device memory");
  CK(cudaMemcpy(dx, x, (size_t)P * n * sizeof(cd), cudaMemcpyHostToDevice));
  RefineArgs R;
  R.H = h->dev();
  R.P = P;
  R.tol = tol;
  R.iters = iters;
  R.n_original = n_original;
  R.inf_thr = infinity_threshold;
  R.x = dx;
  R.resid = dres;
  R.cond = dcond;
  R.regular = dreg;
  R.rank = drank;
  R.slack = dcls;
  R.cscratch = sc;
  k_refine[n](R, blocks, 0);
  CK(cudaGetLastError());
  CK(cudaMemcpy(x, dx, (size_t)P * n * sizeof(cd), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(residual, dres, P * sizeof(double), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(condition, dcond, P * sizeof(double), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(regular, dreg, P, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(rank, drank, P * sizeof(int), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(slack_class, dcls, P, cudaMemcpyDeviceToHost));
  return 0;
}

int nid_dd_refine_batch(NidHomotopy* h, int P, double* x, int steps, int8_t* ok) {
  if (!h || !x || !ok) FAIL("null argument");
  BIND_H(h);
  if (h->nparam > 0) FAIL("dd refine does not take per-path parameters");
  if (P <= 0) return 0;
  const int n = h->n;
  int blocks = grid_for(P, n, 4);
  cd* dx = ws<cd>(W_X, (size_t)P * n);
  int8_t* dok = ws<int8_t>(W_I8B, P);
  cdd* sc = ws<cdd>(W_DDSCR, (size_t)groups_of(blocks, n) * (2 * n * n + 4 * n));
  if (!dx || !dok || !sc) FAIL("out of device memory");
  CK(cudaMemcpy(dx, x, (size_t)P * n * sizeof(cd), cudaMemcpyHostToDevice));
  DDRefineArgs D;
  D.H = h->dev();
  D.P = P;
  D.steps = steps;
  D.x = dx;
  D.ok = dok;
  D.ddscratch = sc;
  k_ddrefine[n](D, blocks, 0);
  CK(cudaGetLastError());
  CK(cudaMemcpy(x, dx, (size_t)P * n * sizeof(cd), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(ok, dok, P, cudaMemcpyDeviceToHost));
  return 0;
}

int nid_match_pairs(int n, int ncmp, int P, const double* X, int32_t* pairs, long long max_pairs,
                    long long* npairs) {
  if (!X || !npairs) FAIL("null argument");
  BIND();
  if (ncmp < 1 || ncmp > n) FAIL("need 1 <= ncmp <= n");
  *npairs = 0;
  if (P <= 1) return 0;
  cd* dX = ws<cd>(W_X, (size_t)P * n);
  double* tol = ws<double>(W_T, P);
  int* dp = ws<int>(W_I32, (size_t)2 * (max_pairs > 0 ? max_pairs : 1));
  unsigned long long* cnt = ws<unsigned long long>(W_COUNT, 8);
  if (!dX || !tol || !dp || !cnt) FAIL("out of device memory");
  CK(cudaMemcpy(dX, X, (size_t)P * n * sizeof(cd), cudaMemcpyHostToDevice));
  CK(cudaMemset(cnt, 0, sizeof(unsigned long long)));
  match_tol_kernel<<<(P + 255) / 256, 256>>>(n, ncmp, P, dX, tol);
  match_pairs_kernel<<<(P + 127) / 128, 128>>>(n, ncmp, P, dX, tol, dp, max_pairs, cnt);
  CK(cudaGetLastError());
  unsigned long long c = 0;
  CK(cudaMemcpy(&c, cnt, sizeof(c), cudaMemcpyDeviceToHost));
  *npairs = (long long)c;
  long long k = (long long)c < max_pairs ? (long long)c : max_pairs;
  if (k > 0 && pairs) CK(cudaMemcpy(pairs, dp, (size_t)k * 2 * sizeof(int), cudaMemcpyDeviceToHost));
  return 0;
}

// K7 pre-pass on the current device: succeeded endpoints of one shard,
// compacted in path order (device pointers in and out)
static int compact_finite(int n, long long P, const cd* x, const int8_t* status, long long first_index,
                          long long index_stride, cd* out, long long* index_out, long long capacity, long long* count,
                          cudaStream_t s) {
  *count = 0;
  if (P <= 0) return 0;
  const int nb = (int)((P + 255) / 256);
  int* d_cnt = ws<int>(W_CBLK, nb);
  long long* d_off = ws<long long>(W_COFF, nb);
  if (!d_cnt || !d_off) FAIL("out of device memory (compaction)");
  finite_count_kernel<<<nb, 256, 0, s>>>(P, status, d_cnt);
  CK(cudaGetLastError());
  std::vector<int> hc(nb);
  CK(cudaMemcpyAsync(hc.data(), d_cnt, nb * sizeof(int), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  std::vector<long long> ho(nb);
  long long tot = 0;
  for (int b = 0; b < nb; ++b) {
    ho[b] = tot;
    tot += hc[b];
  }
  *count = tot;
  if (tot > capacity) FAIL("compaction: output capacity too small");
  if (tot == 0) return 0;
  CK(cudaMemcpyAsync(d_off, ho.data(), nb * sizeof(long long), cudaMemcpyHostToDevice, s));
  finite_compact_kernel<<<nb, 256, 0, s>>>(P, n, x, status, d_off, first_index, index_stride, out, index_out);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(s));
  return 0;
}

int nid_compact_finite(int n, long long P, const double* x_end, const int8_t* status, long long first_index,
                       long long index_stride, double* x_out, long long* index_out, long long capacity,
                       long long* count, void* stream) {
  if (n < 1 || n > NID_MAX_VARS || !x_end || !status || !x_out || !count) FAIL("bad argument");
  BIND();
  return compact_finite(n, P, (const cd*)x_end, status, first_index, index_stride, (cd*)x_out, index_out, capacity,
                        count, (cudaStream_t)stream);
}

int nid_gather_endpoints(int nparts, const int* part_device, const double* const* x_end, const int8_t* const* status,
                         const long long* counts, const long long* first_index, const long long* index_stride, int n,
                         int root_device, double* x_out, long long* index_out, long long capacity, long long* total) {
  if (g_ndev == 0) FAIL("nid_gather_endpoints: call nid_init_devices first");
  if (nparts < 1 || !part_device || !x_end || !status || !counts || !x_out || !total) FAIL("bad argument");
  if (n < 1 || n > NID_MAX_VARS) FAIL("n must be in 1..16");
  if (root_device < 0 || root_device >= g_ndev) FAIL("root device index out of range");
  const int saved = t_device;
  const int root = g_devs[root_device];
  long long off = 0;
  int rc = 0;
  for (int p = 0; p < nparts && rc == 0; ++p) {
    if (part_device[p] < 0 || part_device[p] >= g_ndev) {
      g_err = "part device index out of range";
      rc = 1;
      break;
    }
    const int dev = g_devs[part_device[p]];
    t_device = dev;
    cudaError_t e = cudaSetDevice(dev);
    if (e != cudaSuccess) {
      g_err = std::string("cudaSetDevice: ") + cudaGetErrorString(e);
      rc = 2;
      break;
    }
    const long long P = counts[p];
    cd* buf = ws<cd>(W_GBUF, (size_t)(P > 0 ? P : 1) * n);
    long long* ibuf = index_out ? ws<long long>(W_GIDX, (size_t)(P > 0 ? P : 1)) : nullptr;
    if (!buf || (index_out && !ibuf)) {
      g_err = "out of device memory (gather staging)";
      rc = 1;
      break;
    }
    long long cnt = 0;
    rc = compact_finite(n, P, (const cd*)x_end[p], status[p], first_index ? first_index[p] : 0,
                        index_stride ? index_stride[p] : 1, buf, ibuf, P, &cnt, 0);
    if (rc) break;
    if (off + cnt > capacity) {
      g_err = "nid_gather_endpoints: output capacity too small";
      rc = 1;
      break;
    }
    if (cnt > 0) {
      // device-to-device over NVLink when the part lives on another GPU
      e = cudaMemcpyPeer((cd*)x_out + off * n, root, buf, dev, (size_t)cnt * n * sizeof(cd));
      if (e == cudaSuccess && index_out)
        e = cudaMemcpyPeer(index_out + off, root, ibuf, dev, (size_t)cnt * sizeof(long long));
      if (e != cudaSuccess) {
        g_err = std::string("cudaMemcpyPeer: ") + cudaGetErrorString(e);
        rc = 2;
        break;
      }
    }
    off += cnt;
  }
  *total = off;
  t_device = saved;
  if (cur_device() >= 0) cudaSetDevice(cur_device());
  return rc;
}

}  // extern "C"
