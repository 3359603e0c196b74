// solver.h -- internal host-side types shared by the C ABI (mg_api.cu) and
// the multi-GPU slab solver (dist2.cu).  Not part of the public ABI.
#pragma once
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <algorithm>
#include <string>
#include <vector>

#include "../../include/mg.h"
#include "kernels.h"

using namespace mg;

namespace {

constexpr int kHistCap = 4096;

int log2_exact(int64_t v) {
  if (v < 1) return -1;
  int k = 0;
  while ((int64_t(1) << k) < v) k++;
  return ((int64_t(1) << k) == v) ? k : -1;
}

int64_t round_up(int64_t v, int64_t m) { return (v + m - 1) / m * m; }

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (dev >= 0) {
      cudaGetDevice(&prev);
      if (prev != dev) cudaSetDevice(dev);
      else prev = -1;
    }
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

}  // namespace

// Slab plan (2D y-slabs): the first octave whose levels are agglomerated:
// fewer than `ag` interior nodes on A(s), or fewer than 4 rows per rank.
static inline int slab_agglom_octave(int64_t n, int k, int P, int64_t ag, int dim = 2) {
  for (int o = 1; o < k; o++) {
    int64_t M = (n - 1) >> o, m = M - 1;
    int64_t pts = dim == 2 ? m * m : m * m * m;
    if (pts < ag || M / P < 4) return o;
  }
  return k - 1;
}

// Ghost bands of the communication-avoiding 2D slab schedule (Dist2CA,
// DESIGN.md 8), in fine rows, for oa distributed octaves: WD / WA the descent
// bands of r_D(s) / r_A(s) (octave o), waD / waA the ascent bands of v_D(s) /
// v_A(s); returns Gu, the rows of u a rank needs from each neighbour per cycle.
// Bands are whole rows of their level (D(s): 2s fine rows; A(s): pairs of
// rows, the A-level tiles start on even rows).
static inline int slab_bands_2d(int oa, std::vector<int> &WD, std::vector<int> &WA, std::vector<int> &waD,
                                std::vector<int> &waA) {
  auto up = [](int v, int m) { return (v + m - 1) / m * m; };
  WD.assign(oa, 0);
  WA.assign(oa + 1, 0);
  waD.assign(oa, 0);
  waA.assign(oa + 1, 0);
  std::vector<int> rDneed(oa, 0), rAneed(oa + 1, 0);
  int reqD = 2;   // the finest ascent (A(1), own rows) reads v_D(1) within 2 rows
  for (int o = 0; o < oa; o++) {
    const int s_ = 1 << o;
    waD[o] = up(reqD, 2 * s_);               // D(s) band w: v_A(2s) on w + 2s, r_D(s) on w + s
    rDneed[o] = waD[o] + s_;
    const int reqA = waD[o] + 2 * s_;
    if (o + 1 < oa) {
      waA[o + 1] = up(reqA, 4 * s_);         // A(2s) band w: v_D(2s) on w + 4s, r_A(2s) on w + 2s
      rAneed[o + 1] = waA[o + 1] + 2 * s_;
      reqD = waA[o + 1] + 4 * s_;
    }
  }
  WA[oa] = 0;   // the agglomeration level: own rows (all-gathered)
  for (int o = oa - 1; o >= 0; o--) {
    const int s_ = 1 << o;
    WD[o] = up(std::max(rDneed[o], WA[o + 1] + s_), 2 * s_);     // + the next restriction's reach
    if (o >= 1) WA[o] = up(std::max(rAneed[o], WD[o] + s_), 2 * s_);
  }
  return up(WD[0] + 2, 2);   // the finest descent reads u within 2 rows of its band
}

// ---------------------------------------------------------------- profiler
// Step markers: in profile mode every step of the cycle is preceded by a CUDA
// event on the solver's stream; otherwise the markers cost nothing.
struct StepInfo {
  std::string name;
  int level, launches;
  double bytes;
};
struct Prof {
  cudaStream_t st = nullptr;
  bool first = true;
  std::vector<StepInfo> steps;
  std::vector<cudaEvent_t> evs;   // (nsteps + 1) per cycle
  bool debug = getenv("MG_DEBUG_SYNC") != nullptr;
  std::string last;
  void step(const char *name, int level, int launches, double bytes) {
    if (debug) {
      cudaError_t e = cudaStreamSynchronize(st);
      if (e != cudaSuccess) fprintf(stderr, "[mg debug] error after step '%s': %s\n", last.c_str(), cudaGetErrorString(e));
      last = name;
    }
    if (first) steps.push_back(StepInfo{name, level, launches, bytes});
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, st);
    evs.push_back(e);
  }
  void end_cycle() {
    if (debug) {
      cudaError_t er = cudaStreamSynchronize(st);
      if (er != cudaSuccess) fprintf(stderr, "[mg debug] error after step '%s': %s\n", last.c_str(), cudaGetErrorString(er));
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, st);
    evs.push_back(e);
    first = false;
  }
  ~Prof() {
    for (auto e : evs) cudaEventDestroy(e);
  }
};
#define STEP(name, lev, nl, bytes) \
  do {                              \
    if (prof) prof->step(name, lev, nl, bytes); \
  } while (0)

// ---------------------------------------------------------------- solver
struct mg_solver;
// the passes compute the residual norms (MG_NORM_ALWAYS=1: in every call, as round 1 did -- A/B only)
static bool hist_on(const mg_solver *s);

struct ImplBase {
  virtual ~ImplBase() {}
  virtual cudaError_t alloc() = 0;
  // One V-cycle reading u_in and writing u_out = u_in + v (u_out may equal
  // u_in only when !fast()).
  virtual void enqueue_cycle(const void *u_in, void *u_out, const void *f_eff, cudaStream_t st,
                             Prof *prof = nullptr) = 0;
  // true: the TMA tile kernels run (they update u out of place)
  virtual bool fast() const { return false; }
  // Cross-cycle fusion.  Mode bits of enqueue_cycle_mode:
  // kSkipDesc -- this cycle's finest descent already ran (fused into the
  // previous cycle's ascent, which also pushed its residual norm);
  // kFuseNext -- the finest ascent also runs the next cycle's descent.
  enum { kSkipDesc = 1, kFuseNext = 2 };
  virtual bool fuses_cycles() const { return false; }
  virtual void enqueue_cycle_mode(const void *u_in, void *u_out, const void *f_eff, cudaStream_t st, Prof *prof,
                                  int mode) {
    (void)mode;
    enqueue_cycle(u_in, u_out, f_eff, st, prof);
  }
  virtual void enqueue_final_norm(void *u, const void *f_eff, cudaStream_t st) = 0;
  // what a kSkipDesc cycle expects to have run before it (mg_profile's unprofiled descent)
  virtual void enqueue_pre_descent(void *u, const void *f_eff, cudaStream_t st) { enqueue_final_norm(u, f_eff, st); }
  // Caller-facing helpers.  u, r (residual) and f (f~) are in the caller's layout
  // (mg_solver::pitch); the extra pitch is that of the other operand: f of the
  // residual (the caller's f, or the library's f~ in the work layout), the f~
  // output, the normed array.  Multi-GPU / conventional solvers have one layout.
  virtual void enqueue_residual(const void *u, const void *f, void *r, cudaStream_t st, int64_t fpitch) = 0;
  virtual void enqueue_ftilde(const void *f, void *ft, cudaStream_t st, int64_t ftpitch) = 0;
  virtual void enqueue_norm(const void *x, unsigned long long *mx, double *ss, cudaStream_t st, int64_t xpitch) = 0;
  virtual int launches_per_cycle() const = 0;
  // ---- multi-GPU hooks (single-GPU defaults)
  // elements of one caller field (u, f, r) as this rank holds it
  virtual size_t local_elems() const { return 0; }
  // rows/planes [lo, hi) owned and ghost rows carried by the caller's arrays
  virtual bool extent(int64_t *, int64_t *, int64_t *) const { return false; }
  // loopback (virtual ranks in one process): the whole mg_vcycle; 1 = not handled
  virtual int vcycle_all(mg_solver *, void *, const void *, int, double *) { return 1; }
  // combine the per-cycle residual-norm maxima over ranks
  virtual cudaError_t reduce_hist(unsigned long long *, int, cudaStream_t) { return cudaSuccess; }   // + mg_solver::d_l2
  // sticky failure of an enqueue_* call whose transport step failed (halo
  // exchange, all-gather, all-reduce) or an asynchronous transport error:
  // returns an mg_status (MG_OK when healthy) and clears it; *msg says why
  virtual int take_status(std::string *msg) {
    (void)msg;
    return 0;
  }
  std::vector<void *> bufs;
  size_t bytes = 0;
  std::vector<double> Nl;   // interior nodes per level
  cudaError_t dalloc(void **p, size_t n) {
    cudaError_t e = cudaMalloc(p, n);
    if (e != cudaSuccess) return e;
    bufs.push_back(*p);
    bytes += n;
    return cudaMemset(*p, 0, n);
  }
  // A pitched level array of `rows` rows of `width` elements (zeroed).  With
  // MG_POISON=1 (a bounds check of our own: compute-sanitizer is not available
  // on the B200 pool) the array gets one guard row above and below and its
  // pitch padding [width, pitch), all filled with 0xFF bytes (a NaN in fp32 and
  // fp64): a read outside the level's extent turns the iterate into NaN (the
  // oracle comparisons fail), a write there is found by check_guards().
  struct Guard {
    char *base;
    size_t rowb, wb;
    int64_t rows;
  };
  std::vector<Guard> guards;
  static bool poison() {
    static const bool p = env_flag("MG_POISON");
    return p;
  }
  cudaError_t dalloc2d(void **p, size_t esz, int64_t width, int64_t pitch, int64_t rows) {
    if (!poison()) return dalloc(p, esz * pitch * rows);
    void *base;
    const size_t rowb = esz * pitch, wb = esz * width;
    cudaError_t e = dalloc(&base, rowb * (rows + 2));
    if (e) return e;
    char *b = (char *)base;
    if ((e = cudaMemset(b, 0xFF, rowb)) || (e = cudaMemset(b + rowb * (rows + 1), 0xFF, rowb))) return e;
    if (rowb > wb && (e = cudaMemset2D(b + rowb + wb, rowb, 0xFF, rowb - wb, rows))) return e;
    guards.push_back(Guard{b, rowb, wb, rows});
    if (guards.size() == 1 && env_flag("MG_POISON_SELFTEST") && (e = cudaMemset(b + rowb + wb, 0, 1)))
      return e;   // tests/test_gpu_paths.py: a planted stray write must be reported
    *p = b + rowb;
    return cudaSuccess;
  }
  // number of poisoned arrays whose guard bytes were overwritten (synchronises)
  int check_guards() {
    int bad = 0;
    for (const Guard &g : guards) {
      std::vector<unsigned char> h(g.rowb * (g.rows + 2));
      if (cudaMemcpy(h.data(), g.base, h.size(), cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
      bool ok = true;
      for (size_t i = 0; i < g.rowb && ok; i++) ok = h[i] == 0xFF && h[g.rowb * (g.rows + 1) + i] == 0xFF;
      for (int64_t r = 1; r <= g.rows && ok; r++)
        for (size_t i = g.wb; i < g.rowb && ok; i++) ok = h[g.rowb * r + i] == 0xFF;
      bad += !ok;
    }
    return bad;
  }
  void free_all() {
    for (void *p : bufs) cudaFree(p);
    bufs.clear();
  }
};

struct mg_solver {
  mg_config cfg{};
  int k = 0, L = 0, esz = 8;
  int64_t pitch = 0;    // row pitch of the caller's arrays (elements)
  int64_t wpitch = 0;   // row pitch of the work layout the cycle kernels read: = pitch when that is
                        // 16-byte aligned, else n rounded up to 128 bytes (the caller's arrays are
                        // then staged through d_u_stage / d_f_stage, one 2D copy per array and call)
  int device = 0;
  cudaStream_t user = nullptr, st = nullptr;
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  std::unique_ptr<ImplBase> impl;
  unsigned long long *d_hist = nullptr;   // kHistCap slots
  int *d_counter = nullptr;
  unsigned long long *d_mx = nullptr;
  double *d_ss = nullptr;
  void *d_ft = nullptr;                    // order-4 f~ (work layout)
  void *d_u_stage = nullptr, *d_f_stage = nullptr;   // work-layout staging of u, f (host calls, unaligned layouts)
  // mg_solve_host_batch: a second staging pair and the copy streams, so that one problem's
  // upload and another's download overlap the current problem's cycles
  void *d_u_stage2 = nullptr, *d_f_stage2 = nullptr;
  cudaStream_t st_h2d = nullptr, st_d2h = nullptr;
  cudaEvent_t ev_h2d[2] = {}, ev_comp[2] = {}, ev_d2h[2] = {};
  struct GraphEntry {
    cudaGraphExec_t exec;
    const void *uin, *uout, *f;
    int mode, count;   // count cycles per graph, u alternating uin <-> uout when they differ
    bool l2, hist;
  };
  std::vector<GraphEntry> graphs;   // captured cycles keyed by pointers
  void *d_ualt = nullptr;            // out-of-place partner of the caller's u
  void *d_zero = nullptr;            // zero right-hand side (mg_convergence_factor)
  unsigned long long *h_hist = nullptr;    // pinned
  double *d_l2 = nullptr, *h_l2 = nullptr;  // per-cycle sums of r^2 (kHistCap slots; host copy pinned)
  double *l2_out = nullptr;                // the current call's L2 history destination (mg_vcycle_norms) or null
  bool want_hist = false;                  // the current call asked for a residual history: the passes
                                           // compute the norms only then (the finest passes are instruction-bound)
  bool sum_l2 = false;                     // the current call's passes accumulate sum r^2 (only when asked:
                                           // it costs the issue-bound fp32 fused pass ~7 %)
  std::string err;
  size_t field_elems() const {   // one caller field (u, f, r), elements
    size_t le = impl ? impl->local_elems() : 0;
    return le ? le : (size_t)((cfg.dim == 2) ? cfg.n * pitch : cfg.n * cfg.n * pitch);
  }
  size_t rows() const { return field_elems() / (size_t)pitch; }   // rows of one field (n, n^2, or the slab's)
  size_t work_elems() const { return rows() * (size_t)wpitch; }
};

// conv.cu: the paper's "usual" V(0,1) multigrid (MG_FLAG_CONVENTIONAL, NEXT-3)
namespace mg {
ImplBase *make_conv(const mg_solver *s);
}

static int fail(mg_solver *s, int code, const std::string &msg) {
  if (s) s->err = msg;
  return code;
}

#define CKS(s, call)                                                                          \
  do {                                                                                        \
    cudaError_t e_ = (call);                                                                  \
    if (e_ != cudaSuccess)                                                                    \
      return fail((s), e_ == cudaErrorMemoryAllocation ? MG_ENOMEM : MG_ECUDA,                \
                  std::string(#call) + ": " + cudaGetErrorString(e_));                        \
  } while (0)

// The residual histories of a call's ncycles + 1 slots, to the host: res_hist
// (L-inf, bit patterns of max |r|) and, when the call asked for it, s->l2_out
// (||r||_{2,h} = (h^d sum r^2)^(1/2)).  Synchronises.
static int read_hist(mg_solver *s, int ncycles, double *res_hist, cudaStream_t st) {
  const int nslots = ncycles + 1;
  CKS(s, cudaMemcpyAsync(s->h_hist, s->d_hist, sizeof(unsigned long long) * nslots, cudaMemcpyDeviceToHost, st));
  if (s->l2_out) CKS(s, cudaMemcpyAsync(s->h_l2, s->d_l2, sizeof(double) * nslots, cudaMemcpyDeviceToHost, st));
  CKS(s, cudaStreamSynchronize(st));
  const double hd = std::pow(1.0 / (double)(s->cfg.n - 1), s->cfg.dim);
  bool finite = true;
  for (int i = 0; i <= ncycles; i++) {
    double v;
    unsigned long long b = s->h_hist[i];
    std::memcpy(&v, &b, sizeof v);
    res_hist[i] = v;
    if (!std::isfinite(v)) finite = false;
    if (s->l2_out) {
      s->l2_out[i] = std::sqrt(hd * s->h_l2[i]);
      if (!std::isfinite(s->l2_out[i])) finite = false;
    }
  }
  if (!finite) return fail(s, MG_EDIVERGED, "non-finite residual norm");
  return MG_OK;
}
static cudaError_t clear_hist(mg_solver *s, int nslots, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(s->d_hist, 0, sizeof(unsigned long long) * nslots, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(s->d_l2, 0, sizeof(double) * nslots, st);
  return e;
}

static bool hist_on(const mg_solver *s) {
  static const bool always = env_flag("MG_NORM_ALWAYS");
  return s->want_hist || always;
}
