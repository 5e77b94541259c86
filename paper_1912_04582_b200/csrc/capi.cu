// Host runtime of the TT-DVM CUDA library: context, arenas, static summand
// lists and the explicit-step driver behind the C ABI (include/ttdvm_cuda.h).
//
// Data layout in HBM: every tensor family (state,
// f_S, J, face fluxes, residuals) is a TensorSet = per-tensor (r1, r2) and
// offset into a bump-allocated FP64 arena holding the packed cores of the
// C ABI (first | middle slices | last, col-major).  Rounding kernels
// allocate their outputs with one atomicAdd per tensor; an overflowing
// launch sets a flag, the host grows that arena and repeats the launch.
// The state is double-buffered across steps.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <chrono>
#include <mutex>
#include <vector>
#include <string>
#include <array>
#include <unordered_map>
#include <vector>

#include "../../include/ttdvm_cuda.h"
#include "ttdvm_device.cuh"

namespace ttdvm {
cudaError_t launch_round(const RoundArgs& a, cudaStream_t st);
cudaError_t launch_round_bins(const RoundArgs& a, int* counts, int* bmax, int* lists,
                              cudaStream_t st);
// exact-Gram rounding kernels, 128-thread (round.cu) and 256-thread
// (round256.cu) CTAs; same source, same plan
#define TTDVM_GRAM_API                                                                        \
  size_t round_gram_smem_bytes(int n1, int n3, int RM1, int RM2, int MSMAX, int JB, bool spill); \
  long long round_gram_spill_doubles(int n1, int n3, int RM1, int RM2);                        \
  cudaError_t round_gram_resident(const RoundArgs& a, int* resident);                          \
  int round_gram_tiny_d();                                                                     \
  int round_gram_tiny_minb();                                                                  \
  cudaError_t launch_round_gram(const RoundArgs& a, int nblocks, cudaStream_t st);
namespace g128 {
TTDVM_GRAM_API
}
namespace g256 {
TTDVM_GRAM_API
}
namespace g512 {
TTDVM_GRAM_API
}
namespace g32 {
TTDVM_GRAM_API
// the bulk rank bins as a pipeline of six phase kernels (round_pipe.cuh)
bool round_pipe_eligible(const RoundArgs& p);
long long round_pipe_record_doubles(const RoundArgs& p);
cudaError_t launch_round_pipe(const RoundArgs& p, int first, int count, double* rec,
                              cudaStream_t st);
}
#undef TTDVM_GRAM_API
using g128::round_gram_smem_bytes;  // the plan does not depend on the CTA width
using g128::round_gram_spill_doubles;
size_t round_smem_bytes(int n1, int n2, int n3, int RM1, int RM2, int HMAX, int MSMAX);
struct MacroArgs {
  TSet set;
  int count, n;
  const double* nodes;
  const double* weights;
  double gas[6];
  double* macro;
  double* nu;
  int* status;
};
cudaError_t launch_macro(const MacroArgs& a, int rmax, cudaStream_t st);
cudaError_t launch_shakhov_raw(const double* macro, int count, int n, const double* nodes,
                               double R, double prandtl, double* out, cudaStream_t st);
cudaError_t launch_lusgs_diag(const double* nu, const double* geom, double inv_dt, int count,
                              const int* pos_f, const int* pos_b, double* diag, double* inv_f,
                              double* inv_b, cudaStream_t st);
cudaError_t launch_gather(const TSet& s, int count, const long long* dst_off, int n1, int n2,
                          int n3, double* dst, cudaStream_t st);
struct FaceFactorArgs {
  int n;
  const double* nodes;
  int count;
  const double* normals;
  int cap;
  int mode;
  int* ranks;
  double* cores;
  long long stride;
  double* diag;
  int* status;
};
cudaError_t launch_face_factor(const FaceFactorArgs& a, cudaStream_t st);
cudaError_t launch_xin(const double* normals, int count, int n, const double* nodes,
                       double* cores, long long stride, int* ranks, cudaStream_t st);
struct WallArgs {
  int n;
  int count;
  const double* weights;
  const int* face_of;
  const int* pr;
  const double* pcore;
  const int* nrk;
  const double* ncore;
  long long fstride;
  TSet state;
  const int* cell;
  const double* maxw;
  double* denom;
  double* nw;
  int compute_denom;
  int* status;
};
cudaError_t launch_wall(const WallArgs& a, cudaStream_t st);
cudaError_t launch_dfma_probe(double* out, int blocks, int threads, int iters, cudaStream_t st);
cudaError_t launch_place(const TSet& s, const int* src_ids, int count, int n1, int n2, int n3,
                         int* dst_ranks, long long* dst_off, const int* dst_ids,
                         const long long* new_off, double* dst_base, cudaStream_t st);
cudaError_t launch_gather_ids(const TSet& s, const int* src_ids, int count,
                              const long long* dst_off, int n1, int n2, int n3, double* dst,
                              cudaStream_t st);
}  // namespace ttdvm

using namespace ttdvm;

namespace {

struct Fail {
  int code;
  std::string msg;
};

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e_ = (x);                                                            \
    if (e_ != cudaSuccess)                                                           \
      throw Fail{TTDVM_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_)};      \
  } while (0)

// Deferred device frees.  cudaFree synchronises the device and, measured on
// the box with ~10-50 GB allocated, costs 0.2-0.5 s whatever the block size;
// arenas regrown inside a step therefore park their old block here
// (DevBuf::retire) instead of freeing it.  Parked blocks are freed when an
// allocation fails (then retried once) and when a context is destroyed.  The
// parked total stays below the live arenas' own size (each regrowth at least
// doubles).  TTDVM_DEFER_FREE=0 restores immediate frees (A/B).
// Blocks above kParkMaxBytes are freed at once and regrown without headroom:
// the memory-tight configurations (config 5's blocked step runs within a few
// GB of the 180 GB) must not carry parked or headroom copies of their large
// arenas into the out-of-memory fallback.
constexpr size_t kParkMaxBytes = 4ull << 30;
std::mutex g_park_mu;
std::vector<void*> g_parked;
bool defer_free_on() {
  static const bool on = [] {
    const char* e = getenv("TTDVM_DEFER_FREE");
    return !(e && *e == '0');
  }();
  return on;
}
bool flush_parked() {
  std::vector<void*> v;
  {
    std::lock_guard<std::mutex> lk(g_park_mu);
    v.swap(g_parked);
  }
  if (v.empty()) return false;
  cudaDeviceSynchronize();
  for (void* q : v) cudaFree(q);
  return true;
}

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  // A regrowth (a block already held) parks the old block and takes 1.5x
  // headroom, so buffers that creep up step by step (spill scratch, bin
  // lists) neither cudaFree inside a step nor regrow every step.
  void alloc(size_t count) {
    if (count <= n && p) return;
    const bool regrow = p != nullptr;
    retire();
    if (count == 0) return;
    const size_t want = regrow && count * sizeof(T) <= kParkMaxBytes ? count + count / 2 : count;
    cudaError_t e = cudaMalloc(&p, want * sizeof(T));
    if (e != cudaSuccess) {
      cudaGetLastError();
      flush_parked();
      e = cudaMalloc(&p, count * sizeof(T));
      if (e == cudaSuccess) n = count;
    } else {
      n = want;
    }
    if (e != cudaSuccess) {
      cudaGetLastError();
      p = nullptr;
      n = 0;
      throw Fail{TTDVM_ENOMEM, "cudaMalloc of " + std::to_string(count * sizeof(T)) + " bytes"};
    }
  }
  void free() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  // free without a device synchronisation inside a step (see g_parked); the
  // caller guarantees no pending work still reads the block's content
  // beyond the stream order (parked blocks are only freed after a device sync)
  void retire() {
    if (p && defer_free_on() && n * sizeof(T) <= kParkMaxBytes) {
      std::lock_guard<std::mutex> lk(g_park_mu);
      g_parked.push_back(p);
      p = nullptr;
      n = 0;
      return;
    }
    free();
  }
};

// A family of tensors in one arena.
struct TensorSet {
  int count = 0;
  DevBuf<int> ranks;
  DevBuf<long long> off;
  DevBuf<double> arena;
  long long used = 0;  // doubles in use (host copy after the last launch)
  int maxr1 = 0, maxr2 = 0;
  const double* tscale = nullptr;
  double uscale = 1.0;

  void resize(int c) {
    count = c;
    ranks.alloc(std::max(1, 2 * c));
    off.alloc(std::max(1, c));
  }
  TSet view() const {
    TSet s;
    s.ranks = ranks.p;
    s.off = off.p;
    s.base = arena.p;
    s.tscale = tscale;
    s.uscale = uscale;
    return s;
  }
  void free() {
    ranks.free();
    off.free();
    arena.free();
  }
};

long long tt_size(int n1, int n2, int n3, int r1, int r2) {
  return (long long)n1 * r1 + (long long)n2 * r1 * r2 + (long long)r2 * n3;
}

enum SetId {
  S_STATE = 0,
  S_FSRAW = 1,
  S_FS = 2,
  S_JR = 3,
  S_PHI = 4,
  S_RES = 5,
  S_FREE = 6,
  S_IN = 7,
  S_XIN = 8,   // exact rank-2 xi_n per oblique normal
  S_EABS = 9,  // |xi_n| estimate per oblique normal
  S_DSTAR = 10,  // LU-SGS forward increments (brackets B*, per-tensor scale 1/d), sweep order
  S_DELTA = 11,  // LU-SGS backward increments (brackets B, per-tensor scale 1/d), sweep order
};

struct TermList {
  std::vector<long long> off;  // CSR
  std::vector<Term> terms;
  DevBuf<long long> d_off;
  DevBuf<Term> d_terms;
  int maxk = 0;
  void upload() {
    d_off.alloc(off.size());
    d_terms.alloc(std::max<size_t>(1, terms.size()));
    if (!off.empty()) CK(cudaMemcpy(d_off.p, off.data(), off.size() * 8, cudaMemcpyHostToDevice));
    if (!terms.empty())
      CK(cudaMemcpy(d_terms.p, terms.data(), terms.size() * sizeof(Term), cudaMemcpyHostToDevice));
    maxk = 0;
    for (size_t o = 0; o + 1 < off.size(); ++o) maxk = std::max<int>(maxk, (int)(off[o + 1] - off[o]));
  }
  int nout() const { return off.empty() ? 0 : (int)off.size() - 1; }
  void free() {
    d_off.free();
    d_terms.free();
  }
};

}  // namespace

constexpr int kNPhase = 9;

// One peer of the halo plan: the owned local cells it needs from this rank
// and the ghost local cells it fills here, both in the order the two sides
// agreed on (ascending global id, partition.build_part).
struct HaloPeer {
  int rank = -1;
  std::vector<int> send_ids, recv_ids;
  DevBuf<int> d_send_ids;
  DevBuf<int> d_send_rk, d_recv_rk;   // (r1, r2) pairs
  std::vector<int> h_send_rk;
  int* h_recv_rk = nullptr;           // pinned
  DevBuf<long long> d_send_off;
  std::vector<long long> h_send_off, h_recv_off;
  DevBuf<double> send_buf, recv_buf;
  long long send_doubles = 0, recv_doubles = 0;
};

struct ttdvm_ctx {
  int device = 0;
  cudaStream_t st = nullptr;
  std::string err;
  int n = 0;
  double bound = 0.0;
  std::vector<double> nodes;
  DevBuf<double> d_nodes, d_weights;
  double gas[6] = {1.0, 0.5, 2.0 / 3.0, 1.0, 1.0, 0.5};
  // mesh
  int ncell = 0, nface = 0;
  int nowned = -1;  // cells [0, nowned) are stepped; the rest are halo ghosts
  std::vector<int> left, right, group;
  std::vector<double> area, normal, volume;
  std::vector<long long> cfo;
  std::vector<int> cfid;
  std::vector<signed char> cfs;
  std::vector<ttdvm_bc> bcs;
  bool terms_dirty = true;
  // face factors: [nfac][3n]
  std::vector<double> factors;
  DevBuf<double> d_factors;
  TermList t_fs, t_col, t_flux, t_res, t_upd, t_batch;
  // LU-SGS (N4): per-face factor ids kept from build_step_terms, the level
  // schedules of the two sweeps and their summand lists
  std::vector<int> facp, facm, nid;
  bool lusgs_built = false;
  std::vector<int> lev_off_f, lev_off_b;   // outputs of level l: [lev_off[l], lev_off[l+1])
  std::vector<int> pos_f, pos_b;           // cell -> position in the sweep order
  TermList t_lf, t_lb, t_lu;
  TensorSet dstar, delta;
  DevBuf<int> d_pos_f, d_pos_b;
  DevBuf<double> d_lgeom, d_ldiag, d_linv_f, d_linv_b;
  const double* dscale_override = nullptr;  // RoundArgs::dscale of the LU-SGS launches
  // blocked step (bounded memory): owned cells in nblocks contiguous ranges,
  // each with its own flux (faces it touches), residual and update lists
  int nblocks = 1;           // blocks in use
  bool auto_blocks = true;   // grow nblocks when the step runs out of memory
  int built_blocks = 0;      // nblocks the per-block lists were built for
  std::vector<int> blk_c0;   // [nblocks + 1] cell ranges
  std::vector<TermList> bt_flux, bt_res, bt_upd;
  unsigned long long h_base_used = 0;
  // tensor sets
  TensorSet state[2];
  int cur = 0;
  TensorSet fsraw, fs, jr, phi, res, freestream, in, result;
  // oblique-normal face factors: per distinct
  // normal, xi_n (exact rank 2) and the |xi_n| estimate E (rank <= cap_rank)
  TensorSet xin, eabs;
  std::vector<double> obl_normals;  // [3 * n_oblique]
  int n_oblique = 0;
  int noise_floor = 0;
  double ff_ms = 0.0;
  // diffuse walls (T19): per wall face the xi_n^{+/-} factors, the unit
  // Maxwellian M(1, T_w, 0), the setup denominator and the per-step n_w
  int nwall = 0;
  long long wstride = 0;
  DevBuf<int> d_wface, d_wcell, d_wpr, d_wnr;
  DevBuf<double> d_wpos, d_wneg, d_wmaxw, d_wden, d_nw;
  DevBuf<double> d_macro, d_nu;
  DevBuf<int> d_status;
  int* h_status = nullptr;  // pinned, kStWords + 2 longs
  DevBuf<double> d_margins;
  DevBuf<int> d_bins, d_olist;  // rank bins of the current rounding launch
  DevBuf<double> d_gscratch;     // per-CTA slices of spill-plan rounding launches
  DevBuf<double> d_pipe;         // per-output records of the phase-pipeline launches
  long long pipe_budget = 0;     // bytes of records per pipelined bin (fixed at the first sizing)
  DevBuf<long long> d_tmp_off;
  DevBuf<double> d_tmp;
  bool profiling = false;
  // phases: 0 moments, 1 f_S build, 2-6 roundings (f_S, collision, flux,
  // residual, update), 7 bookkeeping, 8 wall densities
  double phase_ms[kNPhase] = {0};
  double phase_flops[kNPhase] = {0}, phase_bytes[kNPhase] = {0};
  int phase_launches[kNPhase] = {0};
  DevBuf<double> d_acc;
  DevBuf<unsigned long long> d_prof;  // per-phase cycles of the rounding kernel
  bool round_prof = false;
  int cur_phase = 7;
  long long launches = 0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  // multi-GPU halo exchange inside the library: the
  // NCCL communicator (created here from a unique id, or adopted), the halo
  // plan per peer and preallocated device / pinned buffers
  void* comm = nullptr;  // ncclComm_t
  bool own_comm = false;
  int nranks = 1, rank = 0;
  std::vector<HaloPeer> peers;
  cudaStream_t comm_st = nullptr;
  cudaEvent_t halo_ready = nullptr, halo_done = nullptr;
  bool halo_pending = false;
  int* h_rk_all = nullptr;  // pinned, 2 * ncell
  size_t h_rk_all_n = 0;
  DevBuf<int> d_flag;
  int* h_flag = nullptr;  // pinned
  double halo_ms = 0.0;
  long long halo_bytes_sent = 0, halo_bytes_recv = 0, halo_exchanges = 0;
  // auxiliary streams for concurrent rank bins (run_round), created lazily
  cudaStream_t aux[3] = {nullptr, nullptr, nullptr};
  cudaEvent_t fork_ev = nullptr, join_ev[3] = {nullptr, nullptr, nullptr};
};

namespace {

void set_err(ttdvm_ctx* c, const std::string& m) {
  if (c) c->err = m;
}

template <class F>
int guard(ttdvm_ctx* c, F&& f) {
  if (!c) return TTDVM_EINVAL;
  try {
    f();
    c->err.clear();
    return TTDVM_OK;
  } catch (const Fail& e) {
    set_err(c, e.msg);
    return e.code;
  } catch (const std::exception& e) {
    set_err(c, e.what());
    return TTDVM_EINVAL;
  }
}

void require(bool ok, const std::string& m) {
  if (!ok) throw Fail{TTDVM_EINVAL, m};
}

struct Timer {
  ttdvm_ctx* c;
  int phase;
  explicit Timer(ttdvm_ctx* c_, int p) : c(c_), phase(p) {
    static const char* const kNames[kNPhase] = {
        "ttdvm:moments",        "ttdvm:shakhov_build", "ttdvm:round_fs",
        "ttdvm:round_collision", "ttdvm:round_flux",    "ttdvm:round_residual",
        "ttdvm:round_update",   "ttdvm:bookkeeping",   "ttdvm:wall_densities"};
    c->cur_phase = p;
    nvtxRangePushA(kNames[p]);  // NVTX range per step phase (no-op without a tool attached)
    if (c->profiling) CK(cudaEventRecord(c->ev0, c->st));
  }
  ~Timer() {
    nvtxRangePop();
    if (c->profiling) {
      cudaEventRecord(c->ev1, c->st);
      cudaEventSynchronize(c->ev1);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, c->ev0, c->ev1);
      c->phase_ms[phase] += ms;
    }
  }
};

void reset_counters(ttdvm_ctx* c) {
  for (int i = 0; i < kNPhase; ++i) {
    c->phase_ms[i] = 0.0;
    c->phase_flops[i] = 0.0;
    c->phase_bytes[i] = 0.0;
    c->phase_launches[i] = 0;
  }
  c->launches = 0;
}

void upload_batch(ttdvm_ctx* c, const ttdvm_tt_batch* b, TensorSet& s) {
  require(b && b->count >= 0, "null batch");
  require(b->n1 == c->n && b->n2 == c->n && b->n3 == c->n,
          "batch mode sizes must equal the velocity grid size");
  s.resize(b->count);
  int m1 = 0, m2 = 0;
  for (int t = 0; t < b->count; ++t) {
    const int r1 = b->ranks[2 * t], r2 = b->ranks[2 * t + 1];
    require(r1 >= 1 && r2 >= 1, "ranks must be >= 1");
    require(b->offsets[t + 1] - b->offsets[t] == tt_size(b->n1, b->n2, b->n3, r1, r2),
            "offsets do not match ranks");
    m1 = std::max(m1, r1);
    m2 = std::max(m2, r2);
  }
  const long long total = b->count ? b->offsets[b->count] : 0;
  s.arena.alloc(std::max<long long>(1, total));
  if (b->count) {
    CK(cudaMemcpyAsync(s.ranks.p, b->ranks, 8LL * b->count, cudaMemcpyHostToDevice, c->st));
    CK(cudaMemcpyAsync(s.off.p, b->offsets, 8LL * b->count, cudaMemcpyHostToDevice, c->st));
    CK(cudaMemcpyAsync(s.arena.p, b->cores, 8LL * total, cudaMemcpyHostToDevice, c->st));
  }
  s.used = total;
  s.maxr1 = m1;
  s.maxr2 = m2;
  CK(cudaStreamSynchronize(c->st));
}

void ensure_static(ttdvm_ctx* c) {
  if (c->d_status.p == nullptr) {
    c->d_acc.alloc(2 * kAccSlots);
    c->d_status.alloc(kStWords + 4);
    CK(cudaMallocHost(&c->h_status, 64 * sizeof(int)));
  }
}

// TTDVM_ARENA_LOG=1: report arena regrowth and overflow-repeat events (phase,
// sizes, host time of the reallocation) on stderr.
bool diag_log_on() {
  static const bool on = [] {
    const char* e = getenv("TTDVM_ARENA_LOG");
    return e && *e && *e != '0';
  }();
  return on;
}
void arena_log(ttdvm_ctx* c, const char* what, size_t from, size_t to,
               std::chrono::steady_clock::time_point t0) {
  if (!diag_log_on()) return;
  const double ms =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  fprintf(stderr, "[ttdvm arena] phase %d %s: %.2f -> %.2f GB (%.1f ms)\n", c->cur_phase, what,
          from * 8e-9, to * 8e-9, ms);
}

// Arena size for a regrowth: `want` doubles when the device has room for
// it (keeping 4 GB for the step's other buffers), else as much as fits but
// at least `need` -- headroom must never turn a fitting step into an
// out-of-memory failure (config 5 runs within a few GB of the 180 GB).
size_t fit_free(size_t want, size_t need) {
  size_t fr = 0, tot = 0;
  if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) {
    cudaGetLastError();
    return want;
  }
  const size_t keep = 4ull << 30;
  size_t room = fr > keep ? (fr - keep) / sizeof(double) : 0;
  // parked blocks (DevBuf::retire) are not counted free by cudaMemGetInfo:
  // release them before clamping a regrowth below its wish
  if (want > room && flush_parked() && cudaMemGetInfo(&fr, &tot) == cudaSuccess)
    room = fr > keep ? (fr - keep) / sizeof(double) : 0;
  if (want <= room) return want;
  return std::max(need, room);
}

// Run one rounding launch: sets bound into RoundArgs, output into `out`.
// Repeats the launch with a larger arena if it overflowed.
void grow_preserve(ttdvm_ctx* c, TensorSet& s, long long keep, long long need);

// Round the sums of `tl` into `out`.  obase >= 0 selects append mode (the
// blocked step): output o becomes entry obase + o of `out` (sized by the
// caller) and is placed after the `out.used` doubles already in its arena.
void run_round(ttdvm_ctx* c, const TermList& tl, TensorSet* const sets[kMaxSets], TensorSet& out,
               double eps, int cap, double* margins_dev, long long obase = -1, int first = 0,
               int count = -1) {
  // (first, count): round only outputs [first, first + count) of the list
  const int nout = count >= 0 ? count : tl.nout();
  const bool append = obase >= 0;
  if (!append) out.resize(nout);
  if (nout == 0) return;
  require(tl.maxk <= kMaxTerms, "too many summands per rounded output");
  ensure_static(c);
  const int n = c->n;
  RoundArgs a;
  memset(&a, 0, sizeof(a));
  for (int s = 0; s < kMaxSets; ++s)
    if (sets[s]) a.sets[s] = sets[s]->view();
  a.term_off = tl.d_off.p + first;
  a.terms = tl.d_terms.p;
  a.factors = c->d_factors.p;
  a.dscale = c->dscale_override ? c->dscale_override : c->d_nw.p;
  a.n1 = a.n2 = a.n3 = n;
  a.nout = nout;
  a.eps = eps;
  a.cap = cap;
  a.status = c->d_status.p;
  a.margins = margins_dev;
  a.acc = c->d_acc.p;
  a.prof = c->round_prof ? c->d_prof.p : nullptr;
  static const bool no_dmma = [] {  // A/B: TTDVM_DMMA=0 keeps every slice product on DFMA
    const char* e = getenv("TTDVM_DMMA");
    return e && *e == '0';
  }();
  a.no_dmma = no_dmma ? 1 : 0;
  // rank bins: per-bin shared-memory plans (one tiny kernel + readback)
  constexpr int kBinAll = kRankBins * (1 + kBinWords);
  c->d_bins.alloc((size_t)kBinAll);
  c->d_olist.alloc((size_t)kRankBins * nout);
  CK(cudaMemsetAsync(c->d_bins.p, 0, kBinAll * sizeof(int), c->st));
  CK(launch_round_bins(a, c->d_bins.p, c->d_bins.p + kRankBins, c->d_olist.p, c->st));
  c->launches += 1;
  int hb[kBinAll];
  CK(cudaMemcpyAsync(hb, c->d_bins.p, sizeof(hb), cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  const int* bcount = hb;
  const int* bmax = hb + kRankBins;
  int RM1 = 1, RM2 = 1, MSMAX = 1;
  for (int b = 0; b < kRankBins; ++b) {
    if (!bcount[b]) continue;
    RM1 = std::max(RM1, bmax[kBinWords * b]);
    RM2 = std::max(RM2, bmax[kBinWords * b + 1]);
    MSMAX = std::max(MSMAX, bmax[kBinWords * b + 2]);
  }
  const int mx = n;
  // exact-Gram route by default; TTDVM_ROUND=tsqr selects the Householder
  // TSQR route (kept for A/B comparison; one launch, global bounds, n <= 48)
  static const bool use_tsqr = [] {
    const char* e = getenv("TTDVM_ROUND");
    return e && std::string(e) == "tsqr";
  }();
  int HMAX = mx;
  if (use_tsqr) {
    if (mx > 48) throw Fail{TTDVM_EINVAL, "the TSQR route supports at most 48 nodes per axis"};
    HMAX = mx <= 32 ? mx : 48;
    if (round_smem_bytes(n, n, n, RM1, RM2, HMAX, MSMAX) > 227 * 1024)
      throw Fail{TTDVM_ENOMEM, "rounding working set exceeds shared memory"};
  }
  constexpr size_t kSmemMax = 227 * 1024;
  struct Launch {
    int bin, count, rm1, rm2, ms, jb;
    bool spill, wide, narrow;
    int oc = 0;  // doubles of the operand cache (TMA bulk copies of whole operands), 0 = off
    bool xwide = false;       // 512-thread CTAs (round512.cu): high-rank, one-CTA-per-SM bins
    bool pipe = false;        // six phase kernels, one warp per output (round_pipe.cuh)
    size_t pipe_off = 0;      // this launch's records in d_pipe (doubles)
    long long pipe_stride = 0;
    int pipe_chunk = 0;       // outputs per pass through the six kernels
  };
  // 256-thread CTAs from Gram dimension TTDVM_WIDE_D (default 16) up: the
  // measured crossover between the short-phase small tiles (128 threads, four
  // CTAs per SM) and the slice-product-heavy larger ones
  static const int wide_d = [] {
    const char* e = getenv("TTDVM_WIDE_D");
    return e ? atoi(e) : 16;
  }();
  // one-warp CTAs (round32.cu) up to Gram dimension TTDVM_NARROW_D (default
  // 4).  Measured on config 4 (same box, half scale): the rank-<=4 bins --
  // all f_S roundings, most collision and update sums -- run 30-45 % faster
  // than on 128-thread CTAs; the (4, 8] bins lose a little on the updates,
  // and (8, 12] (the face fluxes) run 2.4x slower.
  static const int narrow_d = [] {
    const char* e = getenv("TTDVM_NARROW_D");
    return e ? atoi(e) : 4;
  }();
  auto gram_d = [&](int rm1, int rm2) { return std::max(std::min(n, rm1), std::min(n, rm2)); };
  // CTAs per SM the kernel variant is built for (its launch bounds)
  auto blocks_per_sm = [&](int rm1, int rm2) {
    const int d = gram_d(rm1, rm2);
    const int ne = d * (d + 1) / 2;
    if (d >= wide_d) return ne <= 3 * 256 ? 2 : 1;
    if (d <= narrow_d) return 12;  // one-warp CTAs: many outputs per SM
    if (d <= g128::round_gram_tiny_d()) return g128::round_gram_tiny_minb();  // its launch bounds
    return ne <= 3 * 128 ? 4 : (ne <= 10 * 128 ? 3 : 1);
  };
  // slices per barrier phase: about a quarter of the slices (measured best
  // on config 4: fewer phases pay for a lower CTA count), shrunk while the
  // plan would leave fewer CTAs per SM than the variant's launch bounds --
  // or than the JB = 1 plan itself fits (then the spare shared memory goes
  // to larger slice batches: config 3, +6 %)
  // (oc: bytes of the operand cache the plan must also hold; *ctas returns
  // the CTAs per SM the chosen plan fits)
  auto pick_jb = [&](const Launch& l, size_t oc = 0, int* ctas = nullptr) {
    const size_t base = round_gram_smem_bytes(n, n, l.rm1, l.rm2, l.ms, 1, false) + oc;
    const int fit1 = std::max(1, (int)(228 * 1024 / (base + 1024)));
    const int k = std::min(blocks_per_sm(l.rm1, l.rm2), fit1);
    const size_t budget =
        std::max(base, std::min(kSmemMax, (size_t)(228 * 1024 / k) - 2048));
    int jb = (n + 3) / 4;
    while (jb > 1 && round_gram_smem_bytes(n, n, l.rm1, l.rm2, l.ms, jb, false) + oc > budget) --jb;
    if (ctas) *ctas = k;
    return jb;
  };
  // Operand cache (round.cu): every distinct operand tensor of an output is
  // fetched whole into shared memory by one cp.async.bulk (TMA).  Taken when
  // the bin's largest operand set fits without costing a CTA per SM or a
  // slice of the batch.  Measured (config 4, half scale, same box,
  // scripts/gpu_r2_oc.sh): where the cache halves the slice batch -- the D = 12
  // face-flux bin, JB 10 -> 5 -- the phase slows by 20 % (the L1 prefetch at
  // set-up already hides the operands' latency; the barrier phases saved by
  // larger slice batches matter more); where the batch is kept (the D = 16
  // residual bin) it is neutral to -3 %.  TTDVM_OPCACHE=0 turns it off, =2
  // forces it wherever it fits at all (A/B).
  static const int opcache_mode = [] {
    const char* e = getenv("TTDVM_OPCACHE");
    return e ? atoi(e) : 1;
  }();
  std::vector<Launch> plan;
  for (int b = kRankBins - 1; b >= 0; --b) {  // large ranks first (long CTAs start early)
    if (!bcount[b]) continue;
    const int* bm = bmax + kBinWords * b;
    Launch l{b, bcount[b], std::max(1, bm[0]), std::max(1, bm[1]), std::max(1, bm[2]), 1, false,
             false, false};
    l.wide = gram_d(l.rm1, l.rm2) >= wide_d;
    // 512-thread CTAs from Gram dimension TTDVM_XWIDE_D up (default 32: the
    // bins whose plan leaves one CTA per SM); 0 = never.  Measured same-box:
    // config 3 (D = 32) 101k -> 112k tensors/s, config-4 flux phase -7 %,
    // config-5 residuals -9 %; from D = 24 it is 25 % slower on config 4.
    static const int xwide_d = [] {
      const char* e = getenv("TTDVM_XWIDE_D");
      return e ? atoi(e) : 32;
    }();
    l.xwide = xwide_d > 0 && gram_d(l.rm1, l.rm2) >= xwide_d;
    l.narrow = !l.wide && gram_d(l.rm1, l.rm2) <= narrow_d;
    // working sets above the shared-memory budget (n = 64, summed ranks of
    // ~100 and more) take the spill plan: F, last^T, XP and the Gram region
    // in a per-CTA global scratch slice, persistent CTAs
    l.spill = !use_tsqr &&
              round_gram_smem_bytes(n, n, l.rm1, l.rm2, l.ms, 1, false) > kSmemMax;
    // TTDVM_SPILL_D=d (experiment): bins with Gram dimension >= d take the
    // spill plan although they fit shared memory -- their CTAs then need
    // ~80 KB instead of ~200 KB and can share an SM with the pipeline's
    static const int spill_d = [] {
      const char* e = getenv("TTDVM_SPILL_D");
      return e ? atoi(e) : 0;
    }();
    if (spill_d > 0 && !use_tsqr && gram_d(l.rm1, l.rm2) >= spill_d) l.spill = true;
    if (l.spill) l.narrow = false;
    if (!use_tsqr && !l.spill) {
      int k0 = 1, k1 = 1;
      l.jb = pick_jb(l, 0, &k0);
      const size_t ocb = 8 * (size_t)((std::max(0, bm[4]) + 1) & ~1);
      if (opcache_mode > 0 && bm[4] > 0 &&
          round_gram_smem_bytes(n, n, l.rm1, l.rm2, l.ms, 1, false) + ocb <= kSmemMax) {
        const int jb1 = pick_jb(l, ocb, &k1);
        if (opcache_mode >= 2 || (k1 >= k0 && jb1 >= l.jb)) {
          l.oc = bm[4];
          l.jb = jb1;
        }
      }
    }
    static const int force_jb = [] {  // diagnostics: TTDVM_JB=k forces k slices per phase
      const char* e = getenv("TTDVM_JB");
      return e ? atoi(e) : 0;
    }();
    if (force_jb > 0 && !use_tsqr && !l.spill) {
      l.jb = std::min(n, force_jb);
      while (l.jb > 1 && round_gram_smem_bytes(n, n, l.rm1, l.rm2, l.ms, l.jb, false) +
                                 8 * (size_t)((l.oc + 1) & ~1) > kSmemMax)
        --l.jb;
    }
    // Bulk bins (the LEAN condition) take the phase pipeline: TTDVM_PIPE=0
    // keeps the one-kernel path (A/B), TTDVM_PIPE_MIN = fewest outputs worth
    // six launches per chunk.
    static const int pipe_mode = [] {
      const char* e = getenv("TTDVM_PIPE");
      return e ? atoi(e) : 1;
    }();
    static const int pipe_min = [] {
      const char* e = getenv("TTDVM_PIPE_MIN");
      return e ? atoi(e) : 2048;
    }();
    if (pipe_mode > 0 && !use_tsqr && !l.spill && l.count >= pipe_min) {
      RoundArgs ra = a;
      ra.RM1 = l.rm1;
      ra.RM2 = l.rm2;
      ra.MSMAX = l.ms;
      if (g32::round_pipe_eligible(ra)) {
        l.pipe = true;
        l.pipe_stride = g32::round_pipe_record_doubles(ra);
        l.oc = 0;
      }
    }
    if (l.spill && round_gram_smem_bytes(n, n, l.rm1, l.rm2, l.ms, 1, true) > kSmemMax)
      throw Fail{TTDVM_ENOMEM, "rounding working set exceeds shared memory (n=" +
                                   std::to_string(n) + ", summed ranks " +
                                   std::to_string(l.rm1) + "x" + std::to_string(l.rm2) + ")"};
    plan.push_back(l);
  }
  a.HMAX = HMAX;
  // arena: a modest first estimate; an overflowing launch reports the exact
  // total (the bump counter keeps counting), so one retry always suffices
  const long long base_used = append ? out.used : 0;
  if (append) {
    const int re = std::min(n, 4);
    grow_preserve(c, out, base_used, base_used + (long long)nout * tt_size(n, n, n, re, re) + 1024);
  } else if (out.arena.n == 0) {
    const int re = std::min(n, 4);
    out.arena.alloc((size_t)nout * tt_size(n, n, n, re, re) + 1024);
  } else {
    // headroom: ranks drift upward from step to step; an arena that held
    // this set's previous result with less than 25 % to spare is regrown
    // (its content is dead) to twice it, so neither the overflow-and-repeat
    // path below nor the regrowth itself (a multi-GB cudaFree + cudaMalloc,
    // up to hundreds of ms) recurs step after step as the ranks creep up
    if ((double)out.arena.n < (double)out.used * 1.25 + 1024) {
      const auto t0 = std::chrono::steady_clock::now();
      const size_t was = out.arena.n;
      out.arena.retire();
      const auto t1 = std::chrono::steady_clock::now();
      arena_log(c, "headroom regrow: release", was, 0, t0);
      out.arena.alloc(fit_free((size_t)((double)out.used * 2.0) + 1024,
                               std::max(was, (size_t)out.used + 1024)));
      arena_log(c, "headroom regrow: cudaMalloc", was, out.arena.n, t1);
    }
  }
  for (int attempt = 0; attempt < 4; ++attempt) {
    // (the output arena may have moved; a sweep reads the set it appends to)
    for (int s = 0; s < kMaxSets; ++s)
      if (sets[s]) a.sets[s] = sets[s]->view();
    a.out.ranks = out.ranks.p + (append ? 2 * obase : 0);
    a.out.off = out.off.p + (append ? obase : 0);
    a.out.base = out.arena.p;
    a.out.used = reinterpret_cast<unsigned long long*>(c->d_status.p + kStWords);
    a.out.capacity = (long long)out.arena.n;
    CK(cudaMemsetAsync(c->d_status.p, 0, (kStWords + 4) * sizeof(int), c->st));
    if (append) {  // the bump counter starts after the entries already placed
      c->h_base_used = (unsigned long long)base_used;
      CK(cudaMemcpyAsync(a.out.used, &c->h_base_used, sizeof(unsigned long long),
                         cudaMemcpyHostToDevice, c->st));
    }
    CK(cudaMemsetAsync(c->d_acc.p, 0, 2 * kAccSlots * sizeof(double), c->st));
    if (use_tsqr) {
      a.RM1 = RM1;
      a.RM2 = RM2;
      a.MSMAX = MSMAX;
      a.olist = nullptr;
      CK(launch_round(a, c->st));
      c->launches += 1;
    } else {
      // Rank bins are independent launches (disjoint outputs; the arena bump
      // counter, status words and FLOP accumulators are atomics).  The bin
      // with the most outputs runs on the context stream; the other bins --
      // a few hundred high-rank outputs each, whose single-CTA latency
      // (2-10 ms) would otherwise leave most SMs idle -- run concurrently on
      // auxiliary streams (spill bins serialised on aux[0]: they share the
      // spill scratch).  TTDVM_BIN_STREAMS=0 serialises everything (A/B).
      static const bool bin_streams = [] {
        const char* e = getenv("TTDVM_BIN_STREAMS");
        return !(e && *e == '0');
      }();
      const bool dlog = diag_log_on();
      const bool fork = bin_streams && !dlog && plan.size() > 1;
      // Spill bins share one scratch buffer (d_gscratch), so they all run on
      // one stream: the context stream when the biggest bin spills, aux[0]
      // otherwise.  The scratch is sized once for the largest spill launch
      // before any launch is issued (a regrowth between launches would free
      // a block a queued launch still uses).
      size_t big = 0;
      for (size_t i = 1; i < plan.size(); ++i)
        if (plan[i].count > plan[big].count) big = i;
      const bool big_spills = !plan.empty() && plan[big].spill;
      size_t scratch_need = 0;
      for (const Launch& l : plan) {
        if (!l.spill) continue;
        int resident = 0;
        RoundArgs ra = a;
        ra.RM1 = l.rm1;
        ra.RM2 = l.rm2;
        ra.MSMAX = l.ms;
        ra.JB = l.jb;
        CK(l.xwide  ? g512::round_gram_resident(ra, &resident)
           : l.wide ? g256::round_gram_resident(ra, &resident)
                    : g128::round_gram_resident(ra, &resident));
        if (resident <= 0) throw Fail{TTDVM_ENOMEM, "spill rounding plan does not fit an SM"};
        const size_t g = (size_t)std::min(l.count, resident);
        scratch_need = std::max(scratch_need, g * (size_t)round_gram_spill_doubles(n, n, l.rm1, l.rm2));
      }
      if (scratch_need) c->d_gscratch.alloc(scratch_need);
      // records of the pipelined bins: one region per bin (bins run
      // concurrently), each a chunk of at most kPipeChunk outputs
      // (at most 65,536 outputs and about 2 GB of records)
      size_t pipe_need = 0;
      long long pipe_budget = 2LL << 30;  // bytes of records per pipelined bin
      {
        bool any = false;
        for (const Launch& l : plan) any = any || l.pipe;
        if (any && c->pipe_budget == 0) {  // first sizing: leave memory-tight runs their arenas
          size_t fr = 0, tot = 0;
          if (cudaMemGetInfo(&fr, &tot) == cudaSuccess)
            pipe_budget = std::min<long long>(pipe_budget, std::max<long long>(256LL << 20, (long long)(fr / 16)));
          c->pipe_budget = pipe_budget;
        }
        if (c->pipe_budget) pipe_budget = c->pipe_budget;
      }
      for (Launch& l : plan) {
        if (!l.pipe) continue;
        const long long fit = pipe_budget / (8 * std::max<long long>(1, l.pipe_stride));
        l.pipe_chunk = (int)std::min<long long>(std::min(l.count, 65536), std::max<long long>(8192, fit));
        l.pipe_off = pipe_need;
        pipe_need += (size_t)l.pipe_chunk * (size_t)l.pipe_stride;
      }
      // 30 % headroom on growth: the bins' record strides creep up with the
      // ranks, and regrowing a multi-GB block by a few MB every step costs a
      // cudaFree + cudaMalloc (tens of ms) each time
      if (pipe_need > c->d_pipe.n) {
        try {
          c->d_pipe.alloc(pipe_need + pipe_need * 3 / 10);
        } catch (const Fail& e) {
          // no room for the records: these bins take the one-kernel path
          if (e.code != TTDVM_ENOMEM) throw;
          for (Launch& l : plan) l.pipe = false;
        }
      }
      bool used_aux[3] = {false, false, false};
      if (fork) {
        if (!c->fork_ev) {
          CK(cudaEventCreateWithFlags(&c->fork_ev, cudaEventDisableTiming));
          for (int k = 0; k < 3; ++k) {
            CK(cudaStreamCreateWithFlags(&c->aux[k], cudaStreamNonBlocking));
            CK(cudaEventCreateWithFlags(&c->join_ev[k], cudaEventDisableTiming));
          }
        }
        CK(cudaEventRecord(c->fork_ev, c->st));
      }
      int rr = 0;
      for (size_t li = 0; li < plan.size(); ++li) {
        const Launch& l = plan[li];
        cudaStream_t lst = c->st;
        if (fork && li != big && !(l.spill && big_spills)) {
          const int k = l.spill ? 0 : 1 + (rr++ & 1);
          if (!used_aux[k]) {
            CK(cudaStreamWaitEvent(c->aux[k], c->fork_ev, 0));
            used_aux[k] = true;
          }
          lst = c->aux[k];
        }
        a.RM1 = l.rm1;
        a.RM2 = l.rm2;
        a.MSMAX = l.ms;
        a.JB = l.jb;
        a.OC = l.spill ? 0 : l.oc;
        a.olist = c->d_olist.p + (size_t)l.bin * nout;
        a.gscratch = nullptr;
        a.gstride = 0;
        a.nblk = l.count;
        int grid = l.count;
        if (l.spill) {
          int resident = 0;
          CK(l.xwide  ? g512::round_gram_resident(a, &resident)
             : l.wide ? g256::round_gram_resident(a, &resident)
                      : g128::round_gram_resident(a, &resident));
          if (resident <= 0) throw Fail{TTDVM_ENOMEM, "spill rounding plan does not fit an SM"};
          grid = std::min(l.count, resident);
          a.gstride = round_gram_spill_doubles(n, n, l.rm1, l.rm2);
          if ((size_t)grid * (size_t)a.gstride > c->d_gscratch.n)
            throw Fail{TTDVM_ENOMEM, "spill scratch smaller than planned"};
          a.gscratch = c->d_gscratch.p;
        }
        cudaEvent_t d0 = nullptr, d1 = nullptr;
        if (dlog) {
          CK(cudaEventCreate(&d0));
          CK(cudaEventCreate(&d1));
          CK(cudaEventRecord(d0, c->st));
        }
        if (l.pipe) {
          for (int f0 = 0; f0 < l.count; f0 += l.pipe_chunk) {
            const int cnt = std::min(l.pipe_chunk, l.count - f0);
            CK(g32::launch_round_pipe(a, f0, cnt, c->d_pipe.p + l.pipe_off, lst));
            c->launches += 6;
          }
        } else {
          CK(l.xwide    ? g512::launch_round_gram(a, grid, lst)
             : l.wide   ? g256::launch_round_gram(a, grid, lst)
             : l.narrow ? g32::launch_round_gram(a, grid, lst)
                        : g128::launch_round_gram(a, grid, lst));
          c->launches += 1;
        }
        if (dlog) {  // diagnostics only: per-bin device time (serialises the launches)
          CK(cudaEventRecord(d1, c->st));
          CK(cudaEventSynchronize(d1));
          float ms = 0.f;
          cudaEventElapsedTime(&ms, d0, d1);
          cudaEventDestroy(d0);
          cudaEventDestroy(d1);
          fprintf(stderr,
                  "[ttdvm bin] phase %d bin %d outputs %d summed ranks %dx%d D %d jb %d oc %d %s%s grid %d:"
                  " %.2f ms\n",
                  c->cur_phase, l.bin, l.count, l.rm1, l.rm2, gram_d(l.rm1, l.rm2), l.jb, l.oc,
                  l.pipe ? "pipe" : (l.xwide ? "g512" : (l.wide ? "g256" : (l.narrow ? "g32" : "g128"))),
                  l.spill ? " spill" : "", grid, ms);
        }
      }
      for (int k = 0; k < 3; ++k)
        if (used_aux[k]) {
          CK(cudaEventRecord(c->join_ev[k], c->aux[k]));
          CK(cudaStreamWaitEvent(c->st, c->join_ev[k], 0));
        }
    }
    CK(cudaMemcpyAsync(c->h_status, c->d_status.p, (kStWords + 4) * sizeof(int),
                       cudaMemcpyDeviceToHost, c->st));
    double accs[2 * kAccSlots];
    CK(cudaMemcpyAsync(accs, c->d_acc.p, sizeof(accs), cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    double acc[2] = {0.0, 0.0};
    for (int k = 0; k < kAccSlots; ++k) {
      acc[0] += accs[2 * k];
      acc[1] += accs[2 * k + 1];
    }
    if (!c->h_status[kStOverflow]) {
      c->phase_flops[c->cur_phase] += acc[0];
      c->phase_bytes[c->cur_phase] += acc[1];
      c->phase_launches[c->cur_phase] += use_tsqr ? 1 : (int)plan.size();
    }
    const unsigned long long used =
        *reinterpret_cast<unsigned long long*>(c->h_status + kStWords);
    if (c->h_status[kStOverflow]) {
      const size_t want = fit_free(std::max<size_t>(out.arena.n + 1024, (size_t)(used * 1.5) + 1024),
                                   std::max<size_t>(out.arena.n + 1024, (size_t)used + 1024));
      arena_log(c, "overflow, launch repeated", out.arena.n, want,
                std::chrono::steady_clock::now());
      if (append) {
        grow_preserve(c, out, base_used, (long long)want);
      } else {
        out.arena.retire();
        out.arena.alloc(want);
      }
      continue;
    }
    out.used = (long long)used;
    const int m1 = c->h_status[kStMaxR1] > 0 ? c->h_status[kStMaxR1] : 1;
    const int m2 = c->h_status[kStMaxR2] > 0 ? c->h_status[kStMaxR2] : 1;
    out.maxr1 = append ? std::max(out.maxr1, m1) : m1;
    out.maxr2 = append ? std::max(out.maxr2, m2) : m2;
    if (c->h_status[kStError])
      throw Fail{TTDVM_EDOMAIN, "rounding: non-finite input in output " +
                                    std::to_string(c->h_status[kStErrIdx])};
    return;
  }
  throw Fail{TTDVM_ENOMEM, "rounding arena could not be grown"};
}

void run_macro(ttdvm_ctx* c, TensorSet& s, double* macro, double* nu, int count = -1) {
  ensure_static(c);
  MacroArgs a;
  a.set = s.view();
  a.count = count < 0 ? s.count : count;
  a.n = c->n;
  a.nodes = c->d_nodes.p;
  a.weights = c->d_weights.p;
  for (int i = 0; i < 6; ++i) a.gas[i] = c->gas[i];
  a.macro = macro;
  a.nu = nu;
  a.status = c->d_status.p;
  CK(cudaMemsetAsync(c->d_status.p, 0, (kStWords + 4) * sizeof(int), c->st));
  CK(launch_macro(a, std::max(s.maxr1, s.maxr2), c->st));
  c->launches += 1;
  CK(cudaMemcpyAsync(c->h_status, c->d_status.p, (kStWords + 4) * sizeof(int),
                     cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  if (c->h_status[kStError] == kErrDensity)
    throw Fail{TTDVM_EDOMAIN,
               "compute_macro: nonpositive density in cell " + std::to_string(c->h_status[kStErrIdx])};
  if (c->h_status[kStError] == kErrTemperature)
    throw Fail{TTDVM_EDOMAIN, "compute_macro: nonpositive temperature in cell " +
                                  std::to_string(c->h_status[kStErrIdx])};
}

// collision of `s` (set 0): f_S raw -> round -> (f_S - f) round; J_r in c->jr
void run_collision(ttdvm_ctx* c, TensorSet& s, double eps, int count_ = -1) {
  const int count = count_ < 0 ? s.count : count_;
  const int n = c->n;
  c->d_macro.alloc(std::max(1, 11 * count));
  c->d_nu.alloc(std::max(1, count));
  {
    Timer t(c, 0);
    run_macro(c, s, c->d_macro.p, c->d_nu.p, count);
    // algorithmic work: 16 convolutions of
    // 2 (n r1 + n r1 r2 + r2 n) flops; the cores are read in two passes
    const double doubles = (double)s.used * (s.count ? (double)count / s.count : 0.0);
    c->phase_flops[0] += 32.0 * doubles;
    c->phase_bytes[0] += 16.0 * doubles + 96.0 * count;
    c->phase_launches[0] += 1;
  }
  {
    Timer t(c, 1);
    // exact rank-4 f_S: 24 n doubles written per cell from 11 moments;
    // ~6 flops per entry plus 3 n exponentials (~20 flops each)
    c->phase_flops[1] += (double)count * n * (24.0 * 6.0 + 60.0);
    c->phase_bytes[1] += (double)count * (24.0 * n + 11.0) * 8.0;
    c->phase_launches[1] += 1;
    c->fsraw.resize(count);
    c->fsraw.arena.alloc(std::max<size_t>(1, (size_t)count * 24 * n));
    std::vector<int> rk(2 * (size_t)count, 4);
    std::vector<long long> of(count);
    for (int i = 0; i < count; ++i) of[i] = (long long)i * 24 * n;
    if (count) {
      CK(cudaMemcpyAsync(c->fsraw.ranks.p, rk.data(), 8LL * count, cudaMemcpyHostToDevice, c->st));
      CK(cudaMemcpyAsync(c->fsraw.off.p, of.data(), 8LL * count, cudaMemcpyHostToDevice, c->st));
    }
    c->fsraw.maxr1 = c->fsraw.maxr2 = 4;
    CK(launch_shakhov_raw(c->d_macro.p, count, n, c->d_nodes.p, c->gas[1], c->gas[2],
                          c->fsraw.arena.p, c->st));
    c->launches += 1;
  }
  // one-summand lists (identity) for f_S; (f_S, -f) for J
  if ((int)c->t_fs.off.size() != count + 1) {
    c->t_fs.off.resize(count + 1);
    c->t_fs.terms.resize(count);
    c->t_col.off.resize(count + 1);
    c->t_col.terms.resize(2 * (size_t)count);
    for (int i = 0; i <= count; ++i) {
      c->t_fs.off[i] = i;
      c->t_col.off[i] = 2LL * i;
    }
    for (int i = 0; i < count; ++i) {
      c->t_fs.terms[i] = Term{S_FSRAW, i, 1.0, -1, 0};
      c->t_col.terms[2 * i] = Term{S_FS, i, 1.0, -1, 0};
      c->t_col.terms[2 * i + 1] = Term{S_STATE, i, -1.0, -1, 0};
    }
    c->t_fs.upload();
    c->t_col.upload();
  }
  TensorSet* sets[kMaxSets] = {&s,         &c->fsraw,      &c->fs, &c->jr,  &c->phi,
                                &c->res,    &c->freestream, &c->in, &c->xin, &c->eabs};
  {
    Timer t(c, 2);
    run_round(c, c->t_fs, sets, c->fs, eps, 0, nullptr);
  }
  {
    Timer t(c, 3);
    run_round(c, c->t_col, sets, c->jr, eps, 0, nullptr);
  }
}

// Exactly axis-aligned unit normal -> axis (0..2) and sign, else -1.
int axis_of(const double* nv, double* sgn) {
  int axis = -1;
  for (int a = 0; a < 3; ++a) {
    if (nv[a] != 0.0) {
      if (axis >= 0) return -1;
      axis = a;
    }
  }
  if (axis >= 0 && sgn) *sgn = nv[axis];
  return axis;
}

// Unit Maxwellian maxwell_tt(n, T, u) cores (proj/src/physics.cpp:69-87),
// rank 1: [first n | middle n | last n], density folded into the first.
void maxwell_cores(const ttdvm_ctx* c, double nd, double t, const double u[3], double* out) {
  const int n = c->n;
  const double two_rt = 2.0 * c->gas[1] * t;
  const double norm1d = 1.0 / std::sqrt(M_PI * two_rt);
  for (int a = 0; a < 3; ++a)
    for (int i = 0; i < n; ++i) {
      const double v = c->nodes[i] - u[a];
      double val = norm1d * std::exp(-v * v / two_rt);
      if (a == 0) val *= nd;
      out[a * n + i] = val;
    }
}

double elapsed_ms(cudaEvent_t a, cudaEvent_t b) {
  float f = 0.f;
  cudaEventElapsedTime(&f, a, b);
  return f;
}

// Face factors of the distinct oblique normals on the device: xi_n (exact
// rank 2) and abs_xi_estimate(normal, 4) (velocity_grid.cpp:61-136).
void build_oblique_factors(ttdvm_ctx* c) {
  const int n = c->n, no = c->n_oblique;
  ensure_static(c);
  DevBuf<double> dn;
  dn.alloc(std::max(1, 3 * no));
  if (no) CK(cudaMemcpy(dn.p, c->obl_normals.data(), 24LL * no, cudaMemcpyHostToDevice));
  const long long sx = 8LL * n;
  c->xin.resize(no);
  c->xin.arena.alloc(std::max<long long>(1, sx * no));
  const int cap = 4;  // abs_flux_rank_cap, abs_xi_estimate(normal, 4)
  const long long se = (long long)n * cap + (long long)n * cap * cap + (long long)cap * n;
  c->eabs.resize(no);
  c->eabs.arena.alloc(std::max<long long>(1, se * no));
  std::vector<long long> of(std::max(1, no));
  for (int i = 0; i < no; ++i) of[i] = i * sx;
  if (no) CK(cudaMemcpy(c->xin.off.p, of.data(), 8LL * no, cudaMemcpyHostToDevice));
  for (int i = 0; i < no; ++i) of[i] = i * se;
  if (no) CK(cudaMemcpy(c->eabs.off.p, of.data(), 8LL * no, cudaMemcpyHostToDevice));
  CK(cudaMemsetAsync(c->d_status.p, 0, (kStWords + 4) * sizeof(int), c->st));
  CK(cudaEventRecord(c->ev0, c->st));
  CK(launch_xin(dn.p, no, n, c->d_nodes.p, c->xin.arena.p, sx, c->xin.ranks.p, c->st));
  FaceFactorArgs a;
  a.n = n;
  a.nodes = c->d_nodes.p;
  a.count = no;
  a.normals = dn.p;
  a.cap = cap;
  a.mode = 0;
  a.ranks = c->eabs.ranks.p;
  a.cores = c->eabs.arena.p;
  a.stride = se;
  a.diag = nullptr;
  a.status = c->d_status.p;
  CK(launch_face_factor(a, c->st));
  CK(cudaEventRecord(c->ev1, c->st));
  c->launches += 2;
  CK(cudaMemcpyAsync(c->h_status, c->d_status.p, kStWords * sizeof(int), cudaMemcpyDeviceToHost,
                     c->st));
  CK(cudaStreamSynchronize(c->st));
  c->ff_ms = elapsed_ms(c->ev0, c->ev1);
  if (c->h_status[kStError])
    throw Fail{TTDVM_EDOMAIN, "abs_xi_estimate: degenerate operand for oblique normal " +
                                  std::to_string(c->h_status[kStErrIdx])};
  c->noise_floor = c->h_status[kStAux];
  c->xin.used = sx * no;
  c->xin.maxr1 = c->xin.maxr2 = 2;
  c->eabs.used = se * no;
  c->eabs.maxr1 = c->eabs.maxr2 = cap;
  dn.free();
}

// Diffuse-wall faces: xi_n^{+/-} = from_full(max/min(xi_n, 0), 1e-12, cap + 2)
// (velocity_grid.cpp:127-128; analytic rank 1 for axis-aligned normals,
// where the reference's SVD gives the same rank-1 tensor), the unit wall
// Maxwellian and the state-independent denominator of n_w.
void build_walls(ttdvm_ctx* c, const std::vector<int>& wall_faces) {
  const int n = c->n, nw = (int)wall_faces.size();
  c->nwall = nw;
  if (nw == 0) return;
  const int cap = 6;  // cap_rank + 2 (wall_ghost(..., 4), boundary.cpp:86-87)
  const long long st = (long long)n * cap + (long long)n * cap * cap + (long long)cap * n;
  c->wstride = st;
  c->d_wpos.alloc(st * nw);
  c->d_wneg.alloc(st * nw);
  c->d_wpr.alloc(2 * nw);
  c->d_wnr.alloc(2 * nw);
  c->d_wface.alloc(nw);
  c->d_wcell.alloc(nw);
  c->d_wmaxw.alloc(3LL * n * nw);
  c->d_wden.alloc(nw);
  c->d_nw.alloc(nw);
  std::vector<double> obl, mw(3LL * n * nw);
  std::vector<int> obl_w, cells(nw);
  for (int w = 0; w < nw; ++w) {
    const int f = wall_faces[w];
    cells[w] = c->left[f];
    const ttdvm_bc& b = c->bcs[c->group[f]];
    const double u0[3] = {0.0, 0.0, 0.0};
    maxwell_cores(c, 1.0, b.wall_temperature, u0, &mw[3LL * n * w]);
    const double* nv = &c->normal[3 * f];
    double sgn = 0.0;
    const int axis = axis_of(nv, &sgn);
    if (axis < 0) {
      obl.insert(obl.end(), nv, nv + 3);
      obl_w.push_back(w);
      continue;
    }
    for (int pm = 0; pm < 2; ++pm) {
      std::vector<double> core(3 * n, 1.0);
      for (int i = 0; i < n; ++i) {
        const double v = sgn * c->nodes[i];
        core[axis * n + i] = pm == 0 ? (v > 0.0 ? v : 0.0) : (v < 0.0 ? v : 0.0);
      }
      const int rk[2] = {1, 1};
      CK(cudaMemcpy((pm == 0 ? c->d_wpos.p : c->d_wneg.p) + st * w, core.data(), 24LL * n,
                    cudaMemcpyHostToDevice));
      CK(cudaMemcpy((pm == 0 ? c->d_wpr.p : c->d_wnr.p) + 2 * w, rk, 8, cudaMemcpyHostToDevice));
    }
  }
  CK(cudaMemcpy(c->d_wface.p, wall_faces.data(), 4LL * nw, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(c->d_wcell.p, cells.data(), 4LL * nw, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(c->d_wmaxw.p, mw.data(), 8LL * mw.size(), cudaMemcpyHostToDevice));
  const int no = (int)obl_w.size();
  if (no) {
    DevBuf<double> dn, tp, tn;
    DevBuf<int> rp, rn;
    dn.alloc(3 * no);
    tp.alloc(st * no);
    tn.alloc(st * no);
    rp.alloc(2 * no);
    rn.alloc(2 * no);
    CK(cudaMemcpy(dn.p, obl.data(), 24LL * no, cudaMemcpyHostToDevice));
    CK(cudaMemsetAsync(c->d_status.p, 0, (kStWords + 4) * sizeof(int), c->st));
    for (int pm = 0; pm < 2; ++pm) {
      FaceFactorArgs a;
      a.n = n;
      a.nodes = c->d_nodes.p;
      a.count = no;
      a.normals = dn.p;
      a.cap = cap;
      a.mode = 1 + pm;
      a.ranks = pm == 0 ? rp.p : rn.p;
      a.cores = pm == 0 ? tp.p : tn.p;
      a.stride = st;
      a.diag = nullptr;
      a.status = c->d_status.p;
      CK(launch_face_factor(a, c->st));
      c->launches += 1;
    }
    for (int i = 0; i < no; ++i) {
      const int w = obl_w[i];
      CK(cudaMemcpyAsync(c->d_wpos.p + st * w, tp.p + st * i, 8LL * st, cudaMemcpyDeviceToDevice, c->st));
      CK(cudaMemcpyAsync(c->d_wneg.p + st * w, tn.p + st * i, 8LL * st, cudaMemcpyDeviceToDevice, c->st));
      CK(cudaMemcpyAsync(c->d_wpr.p + 2 * w, rp.p + 2 * i, 8, cudaMemcpyDeviceToDevice, c->st));
      CK(cudaMemcpyAsync(c->d_wnr.p + 2 * w, rn.p + 2 * i, 8, cudaMemcpyDeviceToDevice, c->st));
    }
    CK(cudaMemcpyAsync(c->h_status, c->d_status.p, kStWords * sizeof(int), cudaMemcpyDeviceToHost,
                       c->st));
    CK(cudaStreamSynchronize(c->st));
    if (c->h_status[kStError])
      throw Fail{TTDVM_EDOMAIN, "xi_normal_positive/negative: degenerate wall normal"};
    dn.free();
    tp.free();
    tn.free();
    rp.free();
    rn.free();
  }
}

WallArgs wall_args(ttdvm_ctx* c, const TensorSet& s, int compute_denom) {
  WallArgs a;
  a.n = c->n;
  a.count = c->nwall;
  a.weights = c->d_weights.p;
  a.face_of = c->d_wface.p;
  a.pr = c->d_wpr.p;
  a.pcore = c->d_wpos.p;
  a.nrk = c->d_wnr.p;
  a.ncore = c->d_wneg.p;
  a.fstride = c->wstride;
  a.state = s.view();
  a.cell = c->d_wcell.p;
  a.maxw = c->d_wmaxw.p;
  a.denom = c->d_wden.p;
  a.nw = c->d_nw.p;
  a.compute_denom = compute_denom;
  a.status = c->d_status.p;
  return a;
}

// n_w per wall face from the current state (wall_ghost, boundary.cpp:84-101).
void run_walls(ttdvm_ctx* c, const TensorSet& s, int compute_denom) {
  if (c->nwall == 0) return;
  ensure_static(c);
  CK(cudaMemsetAsync(c->d_status.p, 0, (kStWords + 4) * sizeof(int), c->st));
  CK(launch_wall(wall_args(c, s, compute_denom), c->st));
  c->launches += 1;
  CK(cudaMemcpyAsync(c->h_status, c->d_status.p, kStWords * sizeof(int), cudaMemcpyDeviceToHost,
                     c->st));
  CK(cudaStreamSynchronize(c->st));
  if (c->h_status[kStError] == kErrWallDegenerate)
    throw Fail{TTDVM_EDOMAIN, "wall_ghost: degenerate wall Maxwellian flux (face " +
                                  std::to_string(c->h_status[kStErrIdx]) + ")"};
  if (c->h_status[kStError] == kErrWallDensity)
    throw Fail{TTDVM_EDOMAIN,
               "wall_ghost: impermeability balance gave nonpositive density (face " +
                   std::to_string(c->h_status[kStErrIdx]) + ")"};
}

// Static summand lists of the step (rebuilt when mesh / BCs / grid change).
void build_step_terms(ttdvm_ctx* c) {
  if (!c->terms_dirty) return;
  require(c->n > 0, "set_grid first");
  require(c->ncell > 0, "set_mesh first");
  const int n = c->n;
  const int ng = (int)c->bcs.size();
  // ---- face factors ----
  // axis-aligned normals: (xi.n)^{+/-} = ((xi_n +- |xi_n|)/2) on one axis and
  // ones on the others, exactly the reference's (its rank-1 E is exact for
  // axis normals, proj/tests/test_velocity_grid.cpp:98-115); oblique
  // normals: xi_n and E per distinct normal, computed on the device.
  c->factors.clear();
  std::vector<int>&facp = c->facp, &facm = c->facm, &nid = c->nid;
  facp.assign(c->nface, -1);
  facm.assign(c->nface, -1);
  nid.assign(c->nface, -1);
  c->lusgs_built = false;
  int pair_id[6];
  for (int k = 0; k < 6; ++k) pair_id[k] = -1;
  struct KeyHash {
    size_t operator()(const std::array<long long, 3>& k) const {
      return std::hash<long long>()(k[0] * 1000003LL ^ k[1] * 7919LL ^ k[2]);
    }
  };
  std::unordered_map<std::array<long long, 3>, int, KeyHash> key_of;
  c->obl_normals.clear();
  for (int f = 0; f < c->nface; ++f) {
    const double* nv = &c->normal[3 * f];
    const double nn = std::sqrt(nv[0] * nv[0] + nv[1] * nv[1] + nv[2] * nv[2]);
    require(std::fabs(nn - 1.0) <= 1e-12, "xi_normal: normal must be a unit vector (face " +
                                              std::to_string(f) + ")");
    double sgn = 0.0;
    const int axis = axis_of(nv, &sgn);
    if (axis < 0) {
      // VelocityGrid::cached key: normal quantised to 1e-12 (velocity_grid.cpp:66-69)
      const std::array<long long, 3> key = {std::llround(nv[0] / 1e-12),
                                            std::llround(nv[1] / 1e-12),
                                            std::llround(nv[2] / 1e-12)};
      auto it = key_of.find(key);
      if (it == key_of.end()) {
        const int id = (int)(c->obl_normals.size() / 3);
        key_of.emplace(key, id);
        c->obl_normals.insert(c->obl_normals.end(), nv, nv + 3);
        nid[f] = id;
      } else {
        nid[f] = it->second;
      }
      continue;
    }
    const int key = axis * 2 + (sgn > 0 ? 1 : 0);
    if (pair_id[key] < 0) {
      pair_id[key] = (int)(c->factors.size() / (3 * n));
      for (int pm = 0; pm < 2; ++pm) {
        std::vector<double> fac(3 * n, 1.0);
        for (int i = 0; i < n; ++i) {
          const double xn = sgn * c->nodes[i];
          const double ab = std::fabs(c->nodes[i]);
          fac[axis * n + i] = pm == 0 ? (xn + ab) * 0.5 : (xn - ab) * 0.5;
        }
        c->factors.insert(c->factors.end(), fac.begin(), fac.end());
      }
    }
    facp[f] = pair_id[key];
    facm[f] = pair_id[key] + 1;
  }
  c->n_oblique = (int)(c->obl_normals.size() / 3);
  if (c->n_oblique > 0)
    require(n <= 48, "oblique face normals need a velocity grid of at most 48 nodes per axis");
  c->d_factors.alloc(std::max<size_t>(1, c->factors.size()));
  if (!c->factors.empty())
    CK(cudaMemcpy(c->d_factors.p, c->factors.data(), c->factors.size() * 8, cudaMemcpyHostToDevice));
  build_oblique_factors(c);

  // ---- free-stream Maxwellians per group (maxwell_tt, physics.cpp:69-87);
  // wall groups hold the unit wall Maxwellian M(1, T_w, 0) ----
  {
    std::vector<int> rk(2 * std::max(1, ng), 1);
    std::vector<long long> of(std::max(1, ng));
    std::vector<double> cores((size_t)std::max(1, ng) * 3 * n, 0.0);
    for (int g = 0; g < ng; ++g) {
      of[g] = (long long)g * 3 * n;
      const ttdvm_bc& b = c->bcs[g];
      if (b.kind == 4 || b.kind == 5) {
        require(b.free_n > 0.0 && b.free_t > 0.0, "maxwell_tt: state must have n > 0, T > 0");
        maxwell_cores(c, b.free_n, b.free_t, b.free_u, &cores[(size_t)g * 3 * n]);
      } else if (b.kind == 0) {
        const double u0[3] = {0.0, 0.0, 0.0};
        maxwell_cores(c, 1.0, b.wall_temperature, u0, &cores[(size_t)g * 3 * n]);
      }
    }
    c->freestream.resize(std::max(1, ng));
    c->freestream.arena.alloc(cores.size());
    CK(cudaMemcpy(c->freestream.ranks.p, rk.data(), rk.size() * 4, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(c->freestream.off.p, of.data(), of.size() * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(c->freestream.arena.p, cores.data(), cores.size() * 8, cudaMemcpyHostToDevice));
    c->freestream.maxr1 = c->freestream.maxr2 = 1;
  }

  // ---- walls ----
  std::vector<int> wall_faces, wall_of(c->nface, -1);
  for (int f = 0; f < c->nface; ++f) {
    if (c->right[f] >= 0) continue;
    const int g = c->group[f];
    require(g >= 0 && g < ng, "boundary face " + std::to_string(f) + " has no boundary condition");
    if (c->bcs[g].kind == 0) {
      wall_of[f] = (int)wall_faces.size();
      wall_faces.push_back(f);
    }
  }
  build_walls(c, wall_faces);
  run_walls(c, c->state[c->cur], 1);  // state-independent denominators

  // ---- flux: Phi_f = round(xp o f_L + xm o f_R) ----
  // oblique normals: xp = (xi_n + E)/2, xm = (xi_n - E)/2 enter as the four
  // Hadamard terms 0.5 xi_n o f_L, 0.5 E o f_L, 0.5 xi_n o f_R, -0.5 E o f_R
  // (the reference rounds xp, xm at 1e-14 first -- the same tensors to 1e-14)
  TermList& fl = c->t_flux;
  fl.off.assign(1, 0);
  fl.terms.clear();
  fl.terms.reserve((size_t)c->nface * 4);
  for (int f = 0; f < c->nface; ++f) {
    Term L{S_STATE, c->left[f], 1.0}, R{S_STATE, 0, 1.0};
    const int r = c->right[f];
    if (r >= 0) {
      R.idx = r;
    } else {
      const int g = c->group[f];
      const int kind = c->bcs[g].kind;
      if (kind >= 1 && kind <= 3) {
        R.idx = c->left[f];  // symmetry_ghost: mode reflection (boundary.cpp:103-107)
        R.refl = kind;
      } else if (kind == 4 || kind == 5) {
        R.set = S_FREE;      // freestream_ghost (boundary.hpp:51-53)
        R.idx = g;
      } else {
        R.set = S_FREE;      // wall_ghost = n_w M(1, T_w, 0) (boundary.cpp:84-101)
        R.idx = g;
        R.dsi = wall_of[f];
      }
    }
    if (nid[f] < 0) {
      L.fac = facp[f];
      R.fac = facm[f];
      fl.terms.push_back(L);
      fl.terms.push_back(R);
    } else {
      for (int side = 0; side < 2; ++side) {
        Term t = side == 0 ? L : R;
        t.fidx = nid[f];
        t.fset = S_XIN;
        t.scale = 0.5;
        fl.terms.push_back(t);
        t.fset = S_EABS;
        t.scale = side == 0 ? 0.5 : -0.5;
        fl.terms.push_back(t);
      }
    }
    fl.off.push_back((long long)fl.terms.size());
  }
  fl.upload();
  // residual: R_i = round(J_i + sum_j Phi_j * (-s A_j / V_i))
  const int nown = c->nowned < 0 ? c->ncell : c->nowned;
  TermList& rl = c->t_res;
  rl.off.assign(1, 0);
  rl.terms.clear();
  for (int i = 0; i < nown; ++i) {
    rl.terms.push_back(Term{S_JR, i, 1.0, -1, 0});
    for (long long e = c->cfo[i]; e < c->cfo[i + 1]; ++e) {
      const int fid = c->cfid[e];
      const int s = c->cfs[e];
      const double sc = -s * c->area[fid] / c->volume[i];
      rl.terms.push_back(Term{S_PHI, fid, sc, -1, 0});
    }
    rl.off.push_back((long long)rl.terms.size());
  }
  rl.upload();
  // update: f_i' = round(f_i + R_i * dt)   (dt is the uniform scale of R)
  TermList& ul = c->t_upd;
  ul.off.resize(nown + 1);
  ul.terms.resize(2 * (size_t)nown);
  for (int i = 0; i <= nown; ++i) ul.off[i] = 2LL * i;
  for (int i = 0; i < nown; ++i) {
    ul.terms[2 * i] = Term{S_STATE, i, 1.0, -1, 0};
    ul.terms[2 * i + 1] = Term{S_RES, i, 1.0, -1, 0};
  }
  ul.upload();
  c->terms_dirty = false;
  c->built_blocks = 0;  // per-block lists follow the global ones
}

// Grow an arena to hold `need` doubles, preserving its first `keep` doubles.
void grow_preserve(ttdvm_ctx* c, TensorSet& s, long long keep, long long need) {
  if ((long long)s.arena.n >= need) return;
  DevBuf<double> nb;
  // The old arena is still held during the copy, so large arenas (config 5's
  // blocked step runs within a few GB of the 180 GB) grow exactly; small ones
  // take 1.5x headroom, clamped to the free device memory.
  const size_t exact = (size_t)need;
  const size_t want = exact * sizeof(double) > kParkMaxBytes
                          ? exact
                          : fit_free(std::max(exact, s.arena.n * 3 / 2), exact);
  nb.alloc(want);
  if (keep > 0) CK(cudaMemcpyAsync(nb.p, s.arena.p, 8LL * keep, cudaMemcpyDeviceToDevice, c->st));
  CK(cudaStreamSynchronize(c->st));
  s.arena.retire();
  s.arena = nb;
  nb.p = nullptr;
  nb.n = 0;
}

// Append tensors (src set, src_ids on device or null = 0..count-1) to the
// arena of dst as entries dst_ids (host); ranks_host gives their ranks.
void append_tensors(ttdvm_ctx* c, const TSet& src, const int* src_ids_dev, int count,
                    const int* ranks_host, const int* dst_ids_host, TensorSet& dst) {
  if (count == 0) return;
  std::vector<long long> off(count);
  long long at = dst.used;
  int m1 = dst.maxr1, m2 = dst.maxr2;
  for (int i = 0; i < count; ++i) {
    off[i] = at;
    at += tt_size(c->n, c->n, c->n, ranks_host[2 * i], ranks_host[2 * i + 1]);
    m1 = std::max(m1, ranks_host[2 * i]);
    m2 = std::max(m2, ranks_host[2 * i + 1]);
  }
  grow_preserve(c, dst, dst.used, at);
  c->d_tmp_off.alloc(count);
  CK(cudaMemcpy(c->d_tmp_off.p, off.data(), 8LL * count, cudaMemcpyHostToDevice));
  DevBuf<int> ids;
  ids.alloc(count);
  CK(cudaMemcpy(ids.p, dst_ids_host, 4LL * count, cudaMemcpyHostToDevice));
  CK(launch_place(src, src_ids_dev, count, c->n, c->n, c->n, dst.ranks.p, dst.off.p, ids.p,
                  c->d_tmp_off.p, dst.arena.p, c->st));
  c->launches += 1;
  CK(cudaStreamSynchronize(c->st));
  ids.free();
  dst.used = at;
  dst.maxr1 = m1;
  dst.maxr2 = m2;
}

// Per-block summand lists of the blocked step, derived from the global
// ones (same summands, same order, so every output is the same sum): block b
// owns cells [blk_c0[b], blk_c0[b+1]); its flux list holds the faces those
// cells touch (cut faces are rounded in both adjacent blocks), its residual
// list points into that local flux set, its update list into the local
// residual set.
void build_block_terms(ttdvm_ctx* c) {
  const int nb = c->nblocks;
  if (c->built_blocks == nb) return;
  const int nown = c->nowned < 0 ? c->ncell : c->nowned;
  for (auto* v : {&c->bt_flux, &c->bt_res, &c->bt_upd})
    for (TermList& t : *v) t.free();
  c->bt_flux.assign(nb, TermList());
  c->bt_res.assign(nb, TermList());
  c->bt_upd.assign(nb, TermList());
  c->blk_c0.assign(nb + 1, 0);
  for (int b = 0; b <= nb; ++b) c->blk_c0[b] = (int)((long long)nown * b / nb);
  std::vector<int> pos(c->nface, -1);
  for (int b = 0; b < nb; ++b) {
    const int c0 = c->blk_c0[b], c1 = c->blk_c0[b + 1];
    TermList& fl = c->bt_flux[b];
    TermList& rl = c->bt_res[b];
    TermList& ul = c->bt_upd[b];
    fl.off.assign(1, 0);
    rl.off.assign(1, 0);
    ul.off.assign(1, 0);
    std::vector<int> faces;
    for (int i = c0; i < c1; ++i)
      for (long long e = c->cfo[i]; e < c->cfo[i + 1]; ++e) {
        const int fid = c->cfid[e];
        if (pos[fid] >= 0) continue;
        pos[fid] = (int)faces.size();
        faces.push_back(fid);
        for (long long k = c->t_flux.off[fid]; k < c->t_flux.off[fid + 1]; ++k)
          fl.terms.push_back(c->t_flux.terms[k]);
        fl.off.push_back((long long)fl.terms.size());
      }
    for (int i = c0; i < c1; ++i) {
      for (long long k = c->t_res.off[i]; k < c->t_res.off[i + 1]; ++k) {
        Term t = c->t_res.terms[k];
        if (t.set == S_PHI) t.idx = pos[t.idx];
        rl.terms.push_back(t);
      }
      rl.off.push_back((long long)rl.terms.size());
      for (long long k = c->t_upd.off[i]; k < c->t_upd.off[i + 1]; ++k) {
        Term t = c->t_upd.terms[k];
        if (t.set == S_RES) t.idx -= c0;
        ul.terms.push_back(t);
      }
      ul.off.push_back((long long)ul.terms.size());
    }
    for (int fid : faces) pos[fid] = -1;
    fl.upload();
    rl.upload();
    ul.upload();
  }
  c->built_blocks = nb;
}

// Pieces (1), (2) and the time update of one step, blocked when nblocks > 1.
void step_fluxes_updates(ttdvm_ctx* c, TensorSet& s, TensorSet& nxt, double dt, double eps,
                         int cap) {
  TensorSet* sets[kMaxSets] = {&s,         &c->fsraw,      &c->fs, &c->jr,  &c->phi,
                                &c->res,    &c->freestream, &c->in, &c->xin, &c->eabs};
  if (c->nwall) {
    Timer t(c, 8);
    run_walls(c, s, 0);
    // n_w = <xi_n^+ o f> / -<xi_n^- o M>: two TT inner products per wall
    // face against the cell's cores (ranks ~ maxr) and the face's factors
    const double fsz = (double)c->n * (s.maxr1 + (double)s.maxr1 * s.maxr2 + s.maxr2);
    c->phase_flops[8] += (double)c->nwall * 2.0 * 6.0 * fsz;
    c->phase_bytes[8] += (double)c->nwall * 8.0 * (fsz + (double)c->wstride);
    c->phase_launches[8] += 1;
  }
  if (c->nblocks <= 1) {
    {
      Timer t(c, 4);
      run_round(c, c->t_flux, sets, c->phi, eps, cap, nullptr);
    }
    c->res.uscale = 1.0;
    {
      Timer t(c, 5);
      run_round(c, c->t_res, sets, c->res, eps, cap, nullptr);
    }
    c->res.uscale = dt;
    nxt.resize(c->ncell);
    {
      Timer t(c, 6);
      run_round(c, c->t_upd, sets, nxt, eps, cap, nullptr);
    }
    c->res.uscale = 1.0;
    return;
  }
  build_block_terms(c);
  nxt.resize(c->ncell);
  nxt.used = 0;
  nxt.maxr1 = nxt.maxr2 = 1;
  for (int b = 0; b < c->nblocks; ++b) {
    {
      Timer t(c, 4);
      run_round(c, c->bt_flux[b], sets, c->phi, eps, cap, nullptr);
    }
    c->res.uscale = 1.0;
    {
      Timer t(c, 5);
      run_round(c, c->bt_res[b], sets, c->res, eps, cap, nullptr);
    }
    c->res.uscale = dt;
    {
      Timer t(c, 6);
      run_round(c, c->bt_upd[b], sets, nxt, eps, cap, nullptr, c->blk_c0[b]);
    }
    c->res.uscale = 1.0;
  }
}


// ---------------------------------------------------------------------------
// Multi-GPU: halo exchange of TT cores over NCCL inside the library
// (the reference is single-process, PAPER.md:478 lists
// multi-GPU as future work).  libnccl is bound at run time (dlopen), so a
// single-GPU build or host has no NCCL dependency.
struct ncclUniqueIdBytes {  // ncclUniqueId (nccl.h): 128 opaque bytes, passed by value
  char internal[128];
};
struct NcclApi {
  void* lib = nullptr;
  int (*GetUniqueId)(void*) = nullptr;
  int (*CommInitRank)(void**, int, ncclUniqueIdBytes, int) = nullptr;
  int (*CommDestroy)(void*) = nullptr;
  int (*Send)(const void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*Recv)(void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*AllReduce)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*GroupStart)() = nullptr;
  int (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
};
// nccl.h constants (stable across NCCL 2.x): ncclInt32 = 2, ncclFloat64 = 8, ncclMax = 2
constexpr int kNcclInt32 = 2, kNcclFloat64 = 8, kNcclMax = 2;

NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    const char* names[] = {getenv("TTDVM_NCCL_LIB"), "libnccl.so.2", "libnccl.so"};
    for (const char* nm : names) {
      if (!nm || !*nm) continue;
      a.lib = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
      if (a.lib) break;
    }
    if (!a.lib) return a;
    auto sym = [&](const char* n) { return dlsym(a.lib, n); };
    a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(sym("ncclGetUniqueId"));
    a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(sym("ncclCommInitRank"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(sym("ncclCommDestroy"));
    a.Send = reinterpret_cast<decltype(a.Send)>(sym("ncclSend"));
    a.Recv = reinterpret_cast<decltype(a.Recv)>(sym("ncclRecv"));
    a.AllReduce = reinterpret_cast<decltype(a.AllReduce)>(sym("ncclAllReduce"));
    a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(sym("ncclGroupStart"));
    a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(sym("ncclGroupEnd"));
    a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(sym("ncclGetErrorString"));
    return a;
  }();
  return api;
}

void require_nccl() {
  NcclApi& a = nccl();
  if (!a.lib || !a.GetUniqueId || !a.CommInitRank || !a.Send || !a.Recv || !a.AllReduce ||
      !a.GroupStart || !a.GroupEnd)
    throw Fail{TTDVM_ENCCL, "libnccl.so.2 could not be loaded (set TTDVM_NCCL_LIB or LD_LIBRARY_PATH)"};
}

#define NK(x)                                                                          \
  do {                                                                                 \
    const int r_ = (x);                                                                \
    if (r_ != 0)                                                                       \
      throw Fail{TTDVM_ENCCL, std::string(#x) + ": " +                                 \
                                  (nccl().GetErrorString ? nccl().GetErrorString(r_) : "NCCL error")}; \
  } while (0)

void ensure_comm_stream(ttdvm_ctx* c) {
  if (c->comm_st) return;
  CK(cudaStreamCreateWithFlags(&c->comm_st, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&c->halo_ready, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&c->halo_done, cudaEventDisableTiming));
  c->d_flag.alloc(2);
  CK(cudaMallocHost(&c->h_flag, 2 * sizeof(int)));
}

void free_peers(ttdvm_ctx* c) {
  for (HaloPeer& p : c->peers) {
    p.d_send_ids.free();
    p.d_send_rk.free();
    p.d_recv_rk.free();
    p.d_send_off.free();
    p.send_buf.free();
    p.recv_buf.free();
    if (p.h_recv_rk) cudaFreeHost(p.h_recv_rk);
  }
  c->peers.clear();
}

// Start the exchange of the ghost cells of `s` (the state the step starts
// from): (1) the (r1, r2) pairs of the cells every peer needs, one grouped
// ncclSend/ncclRecv, read back so both sides know the packed sizes; (2) the
// send cells' cores are gathered into per-peer buffers on the compute stream
// and go out in one grouped ncclSend/ncclRecv on the communication stream.
// Returns with phase (2) in flight: the moments, f_S and collision roundings
// of the owned cells -- which read no ghost -- overlap it.  The state arena
// is grown for the incoming ghosts here, before those kernels are queued.
void halo_begin(ttdvm_ctx* c, TensorSet& s) {
  if (!c->comm || c->peers.empty()) return;
  nvtxRangePushA("ttdvm:halo_begin");
  struct Pop {
    ~Pop() { nvtxRangePop(); }
  } pop_;
  NcclApi& a = nccl();
  const int n = c->n;
  ensure_comm_stream(c);
  const auto t0 = std::chrono::steady_clock::now();
  if (c->h_rk_all_n < 2 * (size_t)s.count) {
    if (c->h_rk_all) cudaFreeHost(c->h_rk_all);
    CK(cudaMallocHost(&c->h_rk_all, 2 * (size_t)s.count * sizeof(int)));
    c->h_rk_all_n = 2 * (size_t)s.count;
  }
  CK(cudaMemcpyAsync(c->h_rk_all, s.ranks.p, 8LL * s.count, cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  for (HaloPeer& p : c->peers) {
    const int ns = (int)p.send_ids.size();
    p.h_send_rk.resize(2 * (size_t)ns);
    p.h_send_off.resize((size_t)ns + 1);
    long long o = 0;
    for (int i = 0; i < ns; ++i) {
      const int r1 = c->h_rk_all[2 * p.send_ids[i]], r2 = c->h_rk_all[2 * p.send_ids[i] + 1];
      p.h_send_rk[2 * i] = r1;
      p.h_send_rk[2 * i + 1] = r2;
      p.h_send_off[i] = o;
      o += tt_size(n, n, n, r1, r2);
    }
    p.h_send_off[ns] = o;
    p.send_doubles = o;
    if (ns) {
      CK(cudaMemcpyAsync(p.d_send_rk.p, p.h_send_rk.data(), 8LL * ns, cudaMemcpyHostToDevice, c->st));
      CK(cudaMemcpyAsync(p.d_send_off.p, p.h_send_off.data(), 8LL * ns, cudaMemcpyHostToDevice, c->st));
    }
  }
  // phase 1: ranks
  CK(cudaEventRecord(c->halo_ready, c->st));
  CK(cudaStreamWaitEvent(c->comm_st, c->halo_ready, 0));
  NK(a.GroupStart());
  for (HaloPeer& p : c->peers) {
    if (!p.send_ids.empty())
      NK(a.Send(p.d_send_rk.p, 2 * p.send_ids.size(), kNcclInt32, p.rank, c->comm, c->comm_st));
    if (!p.recv_ids.empty())
      NK(a.Recv(p.d_recv_rk.p, 2 * p.recv_ids.size(), kNcclInt32, p.rank, c->comm, c->comm_st));
  }
  NK(a.GroupEnd());
  for (HaloPeer& p : c->peers)
    if (!p.recv_ids.empty())
      CK(cudaMemcpyAsync(p.h_recv_rk, p.d_recv_rk.p, 8LL * p.recv_ids.size(), cudaMemcpyDeviceToHost,
                         c->comm_st));
  CK(cudaStreamSynchronize(c->comm_st));
  long long incoming = 0;
  for (HaloPeer& p : c->peers) {
    const int nr = (int)p.recv_ids.size();
    p.h_recv_off.resize((size_t)nr + 1);
    long long o = 0;
    for (int i = 0; i < nr; ++i) {
      const int r1 = p.h_recv_rk[2 * i], r2 = p.h_recv_rk[2 * i + 1];
      if (r1 < 1 || r2 < 1 || r1 > 4 * n || r2 > 4 * n)
        throw Fail{TTDVM_ENCCL, "halo exchange: implausible ranks received from rank " +
                                    std::to_string(p.rank)};
      p.h_recv_off[i] = o;
      o += tt_size(n, n, n, r1, r2);
    }
    p.h_recv_off[nr] = o;
    p.recv_doubles = o;
    incoming += o;
    p.send_buf.alloc(std::max<size_t>(1, (size_t)p.send_doubles));
    p.recv_buf.alloc(std::max<size_t>(1, (size_t)p.recv_doubles));
    c->halo_bytes_sent += 8 * p.send_doubles + 8LL * (long long)p.send_ids.size();
    c->halo_bytes_recv += 8 * p.recv_doubles + 8LL * nr;
  }
  // room for the incoming ghosts now: no arena regrowth while the collision
  // kernels read the owned cells
  grow_preserve(c, s, s.used, s.used + incoming);
  // phase 2: cores
  for (HaloPeer& p : c->peers) {
    if (p.send_ids.empty()) continue;
    CK(launch_gather_ids(s.view(), p.d_send_ids.p, (int)p.send_ids.size(), p.d_send_off.p, n, n, n,
                         p.send_buf.p, c->st));
    c->launches += 1;
  }
  CK(cudaEventRecord(c->halo_ready, c->st));
  CK(cudaStreamWaitEvent(c->comm_st, c->halo_ready, 0));
  NK(a.GroupStart());
  for (HaloPeer& p : c->peers) {
    if (p.send_doubles)
      NK(a.Send(p.send_buf.p, (size_t)p.send_doubles, kNcclFloat64, p.rank, c->comm, c->comm_st));
    if (p.recv_doubles)
      NK(a.Recv(p.recv_buf.p, (size_t)p.recv_doubles, kNcclFloat64, p.rank, c->comm, c->comm_st));
  }
  NK(a.GroupEnd());
  CK(cudaEventRecord(c->halo_done, c->comm_st));
  c->halo_pending = true;
  c->halo_exchanges += 1;
  c->halo_ms +=
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

// Wait for the cores and place them as the ghost entries of `s`.
void halo_end(ttdvm_ctx* c, TensorSet& s) {
  if (!c->halo_pending) return;
  c->halo_pending = false;
  const auto t0 = std::chrono::steady_clock::now();
  CK(cudaStreamWaitEvent(c->st, c->halo_done, 0));
  for (HaloPeer& p : c->peers) {
    if (p.recv_ids.empty()) continue;
    TSet src;
    src.ranks = p.d_recv_rk.p;
    src.off = nullptr;
    src.base = p.recv_buf.p;
    src.tscale = nullptr;
    src.uscale = 1.0;
    DevBuf<long long> of;  // source offsets on the device
    of.alloc(p.recv_ids.size());
    CK(cudaMemcpy(of.p, p.h_recv_off.data(), 8LL * p.recv_ids.size(), cudaMemcpyHostToDevice));
    src.off = of.p;
    append_tensors(c, src, nullptr, (int)p.recv_ids.size(), p.h_recv_rk, p.recv_ids.data(), s);
    of.retire();
  }
  c->halo_ms +=
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

// max over ranks of a status code: a rank that failed inside its step skips
// to this point, its peers finish theirs, and every rank then reports the
// failure together instead of waiting for a halo that never comes.
int allreduce_status(ttdvm_ctx* c, int local) {
  if (!c->comm) return local;
  NcclApi& a = nccl();
  ensure_comm_stream(c);
  c->h_flag[0] = local;
  CK(cudaMemcpyAsync(c->d_flag.p, c->h_flag, sizeof(int), cudaMemcpyHostToDevice, c->comm_st));
  NK(a.AllReduce(c->d_flag.p, c->d_flag.p + 1, 1, kNcclInt32, kNcclMax, c->comm, c->comm_st));
  CK(cudaMemcpyAsync(c->h_flag + 1, c->d_flag.p + 1, sizeof(int), cudaMemcpyDeviceToHost, c->comm_st));
  CK(cudaStreamSynchronize(c->comm_st));
  return c->h_flag[1];
}

void step_once(ttdvm_ctx* c, double dt, double eps, int cap) {
  TensorSet& s = c->state[c->cur];
  TensorSet& nxt = c->state[1 - c->cur];
  const int nown = c->nowned < 0 ? c->ncell : c->nowned;
  // pieces (3) + (4): moments, f_S, J_r = round(f_S - f) over the owned
  // cells; nu applied as J's per-tensor scale (TtTensor::scaled after
  // rounding, physics.cpp:118)
  halo_begin(c, s);  // ghosts of t^n in flight while the owned cells' collision terms run
  run_collision(c, s, eps, nown);
  c->jr.tscale = c->d_nu.p;
  halo_end(c, s);
  for (;;) {
    try {
      step_fluxes_updates(c, s, nxt, dt, eps, cap);
      break;
    } catch (const Fail& e) {
      // out of device memory: release the flux / residual / next-state
      // arenas and redo pieces (1), (2) and the update in 4x more cell
      // blocks (the state and J_r are untouched, so the step is unchanged)
      if (e.code != TTDVM_ENOMEM || !c->auto_blocks || c->nblocks >= 256 || nown < 8 * c->nblocks)
        throw;
      c->phi.free();
      c->res.free();
      nxt.arena.free();
      nxt.used = 0;
      c->nblocks *= 4;
    }
  }
  c->res.uscale = 1.0;
  nxt.count = c->ncell;
  if (nown < c->ncell) {
    // ghosts carry over unchanged until a halo exchange replaces them
    const int ng = c->ncell - nown;
    std::vector<int> rk(2 * (size_t)ng), ids(ng);
    CK(cudaMemcpy(rk.data(), s.ranks.p + 2LL * nown, 8LL * ng, cudaMemcpyDeviceToHost));
    for (int i = 0; i < ng; ++i) ids[i] = nown + i;
    DevBuf<int> sid;
    sid.alloc(ng);
    CK(cudaMemcpy(sid.p, ids.data(), 4LL * ng, cudaMemcpyHostToDevice));
    append_tensors(c, s.view(), sid.p, ng, rk.data(), ids.data(), nxt);
    sid.free();
  }
  c->cur = 1 - c->cur;
}


// ---------------------------------------------------------------------------
// LU-SGS implicit iteration (the
// rank-1 divisor of TtTensor::divided_by_rank_one, tt_tensor.cpp:247-261).
// The reference's sweeps run over the cells in index order; here a cell's
// LEVEL is the length of its longest chain of lower-indexed (forward) or
// higher-indexed (backward) neighbours, and each level is one batched
// rounding launch: every cell sees exactly the neighbour increments the
// sequential sweep would give it and sums them in the same (face) order, so
// the result is that of the natural-order sweep.
void build_lusgs_terms(ttdvm_ctx* c) {
  if (c->lusgs_built) return;
  const int nc = c->ncell;
  auto neighbour = [&](int i, int fid) {
    const int l = c->left[fid], r = c->right[fid];
    return r < 0 ? -1 : (l == i ? r : l);
  };
  // level schedules
  std::vector<int> lev(nc, 0);
  auto schedule = [&](bool forward, std::vector<int>& lev_off, std::vector<int>& pos) {
    std::fill(lev.begin(), lev.end(), 0);
    int nlev = 0;
    for (int q = 0; q < nc; ++q) {
      const int i = forward ? q : nc - 1 - q;
      int l = 0;
      for (long long e = c->cfo[i]; e < c->cfo[i + 1]; ++e) {
        const int k = neighbour(i, c->cfid[e]);
        if (k >= 0 && (forward ? k < i : k > i)) l = std::max(l, lev[k] + 1);
      }
      lev[i] = l;
      nlev = std::max(nlev, l + 1);
    }
    lev_off.assign(nlev + 1, 0);
    for (int i = 0; i < nc; ++i) lev_off[lev[i] + 1] += 1;
    for (int l = 0; l < nlev; ++l) lev_off[l + 1] += lev_off[l];
    std::vector<int> fill(lev_off.begin(), lev_off.end() - 1);
    pos.assign(nc, 0);
    for (int i = 0; i < nc; ++i) pos[i] = fill[lev[i]]++;  // ascending cell id inside a level
  };
  schedule(true, c->lev_off_f, c->pos_f);
  schedule(false, c->lev_off_b, c->pos_b);
  std::vector<int> order_f(nc), order_b(nc);
  for (int i = 0; i < nc; ++i) {
    order_f[c->pos_f[i]] = i;
    order_b[c->pos_b[i]] = i;
  }
  // -c_ik o d_k: i left of the face: -(A/V) xm o d_k; i right: +(A/V) xp o d_k
  auto push_offdiag = [&](TermList& tl, int i, int fid, int set, int kpos) {
    const bool is_left = c->left[fid] == i;
    const double w = c->area[fid] / c->volume[i];
    const double sc = is_left ? -w : w;
    Term t{set, kpos, sc};
    if (c->nid[fid] < 0) {
      t.fac = is_left ? c->facm[fid] : c->facp[fid];
      tl.terms.push_back(t);
    } else {
      t.fidx = c->nid[fid];
      t.fset = S_XIN;
      t.scale = 0.5 * sc;
      tl.terms.push_back(t);
      t.fset = S_EABS;
      t.scale = (is_left ? -0.5 : 0.5) * sc;  // xm = (xi_n - E)/2, xp = (xi_n + E)/2
      tl.terms.push_back(t);
    }
  };
  TermList &lf = c->t_lf, &lb = c->t_lb, &lu = c->t_lu;
  lf.off.assign(1, 0);
  lf.terms.clear();
  lb.off.assign(1, 0);
  lb.terms.clear();
  for (int o = 0; o < nc; ++o) {
    const int i = order_f[o];
    lf.terms.push_back(Term{S_RES, i, 1.0});
    for (long long e = c->cfo[i]; e < c->cfo[i + 1]; ++e) {
      const int k = neighbour(i, c->cfid[e]);
      if (k >= 0 && k < i) push_offdiag(lf, i, c->cfid[e], S_DSTAR, c->pos_f[k]);
    }
    lf.off.push_back((long long)lf.terms.size());
  }
  for (int o = 0; o < nc; ++o) {
    const int i = order_b[o];
    Term bs{S_DSTAR, c->pos_f[i], 1.0};
    bs.dsi = i;  // x d_i: the undivided forward bracket B*_i
    lb.terms.push_back(bs);
    for (long long e = c->cfo[i]; e < c->cfo[i + 1]; ++e) {
      const int k = neighbour(i, c->cfid[e]);
      if (k >= 0 && k > i) push_offdiag(lb, i, c->cfid[e], S_DELTA, c->pos_b[k]);
    }
    lb.off.push_back((long long)lb.terms.size());
  }
  lu.off.resize(nc + 1);
  lu.terms.resize(2 * (size_t)nc);
  for (int i = 0; i <= nc; ++i) lu.off[i] = 2LL * i;
  for (int i = 0; i < nc; ++i) {
    lu.terms[2 * i] = Term{S_STATE, i, 1.0};
    lu.terms[2 * i + 1] = Term{S_DELTA, c->pos_b[i], 1.0};
  }
  lf.upload();
  lb.upload();
  lu.upload();
  require(std::max(lf.maxk, lb.maxk) <= kMaxTerms, "LU-SGS: too many faces per cell");
  // geometric part of the diagonal
  std::vector<double> geom(nc);
  const double xi_abs_max = std::sqrt(3.0) * c->bound;
  for (int i = 0; i < nc; ++i) {
    double sa = 0.0;
    for (long long e = c->cfo[i]; e < c->cfo[i + 1]; ++e) sa += c->area[c->cfid[e]];
    geom[i] = 0.5 * sa * xi_abs_max / c->volume[i];
  }
  c->d_lgeom.alloc(nc);
  c->d_ldiag.alloc(nc);
  c->d_linv_f.alloc(nc);
  c->d_linv_b.alloc(nc);
  c->d_pos_f.alloc(nc);
  c->d_pos_b.alloc(nc);
  CK(cudaMemcpy(c->d_lgeom.p, geom.data(), 8LL * nc, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(c->d_pos_f.p, c->pos_f.data(), 4LL * nc, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(c->d_pos_b.p, c->pos_b.data(), 4LL * nc, cudaMemcpyHostToDevice));
  c->lusgs_built = true;
}

void lusgs_once(ttdvm_ctx* c, double dt, double eps, int cap) {
  require(c->nowned < 0 || c->nowned == c->ncell, "LU-SGS runs on an unpartitioned mesh");
  TensorSet& s = c->state[c->cur];
  TensorSet& nxt = c->state[1 - c->cur];
  const int nc = c->ncell;
  build_lusgs_terms(c);
  run_collision(c, s, eps, nc);
  c->jr.tscale = c->d_nu.p;
  TensorSet* sets[kMaxSets] = {&s,      &c->fsraw,      &c->fs, &c->jr,  &c->phi,  &c->res,
                                &c->freestream, &c->in, &c->xin, &c->eabs, &c->dstar, &c->delta};
  if (c->nwall) {
    Timer t(c, 8);
    run_walls(c, s, 0);
  }
  {
    Timer t(c, 4);
    run_round(c, c->t_flux, sets, c->phi, eps, cap, nullptr);
  }
  c->res.uscale = 1.0;
  {
    Timer t(c, 5);
    run_round(c, c->t_res, sets, c->res, eps, cap, nullptr);
  }
  CK(launch_lusgs_diag(c->d_nu.p, c->d_lgeom.p, 1.0 / dt, nc, c->d_pos_f.p, c->d_pos_b.p,
                       c->d_ldiag.p, c->d_linv_f.p, c->d_linv_b.p, c->st));
  c->launches += 1;
  c->dscale_override = c->d_ldiag.p;
  try {
    Timer t(c, 6);
    for (int pass = 0; pass < 2; ++pass) {
      TensorSet& out = pass == 0 ? c->dstar : c->delta;
      const TermList& tl = pass == 0 ? c->t_lf : c->t_lb;
      const std::vector<int>& lo = pass == 0 ? c->lev_off_f : c->lev_off_b;
      out.resize(nc);
      out.used = 0;
      out.maxr1 = out.maxr2 = 1;
      out.tscale = pass == 0 ? c->d_linv_f.p : c->d_linv_b.p;
      for (size_t l = 0; l + 1 < lo.size(); ++l)
        run_round(c, tl, sets, out, eps, cap, nullptr, lo[l], lo[l], lo[l + 1] - lo[l]);
    }
    nxt.resize(nc);
    run_round(c, c->t_lu, sets, nxt, eps, cap, nullptr);
  } catch (...) {
    c->dscale_override = nullptr;
    throw;
  }
  c->dscale_override = nullptr;
  nxt.count = nc;
  c->cur = 1 - c->cur;
}

// One step; with a communicator, every rank learns of a failure on any rank
// (ncclAllReduce max of the status code) and fails with it.
void step_synced(ttdvm_ctx* c, double dt, double eps, int cap) {
  if (!c->comm) {
    step_once(c, dt, eps, cap);
    return;
  }
  Fail local{TTDVM_OK, ""};
  try {
    step_once(c, dt, eps, cap);
  } catch (const Fail& e) {
    local = e;
    if (c->halo_pending) {  // drain the exchange this rank started
      cudaStreamSynchronize(c->comm_st);
      c->halo_pending = false;
    }
  }
  const int global = allreduce_status(c, local.code);
  if (local.code != TTDVM_OK) throw local;
  if (global != TTDVM_OK)
    throw Fail{global, "explicit_step failed on another rank of the partition (status " +
                           std::to_string(global) + ")"};
}

void layout_of(ttdvm_ctx* c, const TensorSet& s, int32_t* ranks, int64_t* offsets) {
  std::vector<int> rk(2 * (size_t)s.count);
  if (s.count)
    CK(cudaMemcpy(rk.data(), s.ranks.p, rk.size() * 4, cudaMemcpyDeviceToHost));
  long long o = 0;
  for (int t = 0; t < s.count; ++t) {
    if (ranks) {
      ranks[2 * t] = rk[2 * t];
      ranks[2 * t + 1] = rk[2 * t + 1];
    }
    if (offsets) offsets[t] = o;
    o += tt_size(c->n, c->n, c->n, rk[2 * t], rk[2 * t + 1]);
  }
  if (offsets) offsets[s.count] = o;
}

void download_set(ttdvm_ctx* c, const TensorSet& s, double* cores, int64_t capacity) {
  std::vector<int64_t> offs(s.count + 1);
  layout_of(c, s, nullptr, offs.data());
  const long long total = offs[s.count];
  require(capacity >= total, "download capacity too small: need " + std::to_string(total));
  if (s.count == 0) return;
  // gathered in chunks of at most `chunk` doubles (2 GB), so a download never
  // needs a staging copy of the whole set next to the step's arenas (config
  // 5's state is ~19 GB with the device nearly full); one chunk for config 4
  long long chunk = 256LL << 20;
  if (const char* e = getenv("TTDVM_DOWNLOAD_CHUNK")) {  // tests: force many chunks
    const long long v = atoll(e);
    if (v > 0) chunk = v;
  }
  c->d_tmp_off.alloc(s.count);
  long long maxsz = 1;
  for (int t = 0; t < s.count; ++t) maxsz = std::max<long long>(maxsz, offs[t + 1] - offs[t]);
  long long lim = std::max(maxsz, std::min(total, chunk));
  // Memory-tight runs (config 5 holds the device within a few GB): when the
  // staging buffer does not fit, release the rounding scratch (dead between
  // calls) and then halve the chunk down to the largest tensor.
  for (;;) {
    try {
      c->d_tmp.alloc((size_t)lim);
      break;
    } catch (const Fail& e) {
      if (e.code != TTDVM_ENOMEM) throw;
      if (c->d_pipe.p || c->d_gscratch.p) {
        CK(cudaStreamSynchronize(c->st));
        c->d_pipe.free();
        c->d_gscratch.free();
        continue;
      }
      if (lim <= maxsz) throw;
      lim = std::max(maxsz, lim / 2);
    }
  }
  int t0 = 0;
  while (t0 < s.count) {
    // chunks are bounded by the requested chunk size, not by the staging
    // buffer (which never shrinks and may hold a whole earlier download)
    int t1 = t0 + 1;  // one tensor per chunk at least
    while (t1 < s.count && offs[t1 + 1] - offs[t0] <= lim) ++t1;
    const long long base = offs[t0], len = offs[t1] - offs[t0];
    std::vector<long long> rel(t1 - t0);
    for (int t = t0; t < t1; ++t) rel[t - t0] = offs[t] - base;
    CK(cudaMemcpy(c->d_tmp_off.p, rel.data(), 8LL * (t1 - t0), cudaMemcpyHostToDevice));
    TSet v = s.view();
    v.ranks += 2LL * t0;
    v.off += t0;
    if (v.tscale) v.tscale += t0;
    CK(launch_gather(v, t1 - t0, c->d_tmp_off.p, c->n, c->n, c->n, c->d_tmp.p, c->st));
    c->launches += 1;
    CK(cudaStreamSynchronize(c->st));
    CK(cudaMemcpy(cores + base, c->d_tmp.p, 8LL * len, cudaMemcpyDeviceToHost));
    t0 = t1;
  }
}

}  // namespace

extern "C" {

int ttdvm_cuda_create(int device, ttdvm_ctx** out) {
  if (!out) return TTDVM_EINVAL;
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return TTDVM_ECUDA;
  }
  if (device < 0 || device >= ndev) return TTDVM_EINVAL;
  if (cudaSetDevice(device) != cudaSuccess) return TTDVM_ECUDA;
  ttdvm_ctx* c = new ttdvm_ctx();
  c->device = device;
  if (cudaStreamCreateWithFlags(&c->st, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreate(&c->ev0) != cudaSuccess || cudaEventCreate(&c->ev1) != cudaSuccess) {
    delete c;
    return TTDVM_ECUDA;
  }
  *out = c;
  return TTDVM_OK;
}

int ttdvm_cuda_destroy(ttdvm_ctx* c) {
  if (!c) return TTDVM_EINVAL;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->st);
  flush_parked();
  for (TensorSet* s : {&c->state[0], &c->state[1], &c->fsraw, &c->fs, &c->jr, &c->phi, &c->res,
                       &c->freestream, &c->in, &c->result, &c->xin, &c->eabs})
    s->free();
  for (TermList* t : {&c->t_fs, &c->t_col, &c->t_flux, &c->t_res, &c->t_upd, &c->t_batch, &c->t_lf,
                      &c->t_lb, &c->t_lu})
    t->free();
  c->dstar.free();
  c->delta.free();
  c->d_pos_f.free();
  c->d_pos_b.free();
  for (DevBuf<double>* b : {&c->d_lgeom, &c->d_ldiag, &c->d_linv_f, &c->d_linv_b}) b->free();
  for (auto* v : {&c->bt_flux, &c->bt_res, &c->bt_upd})
    for (TermList& t : *v) t.free();
  c->d_gscratch.free();
  c->d_pipe.free();
  c->d_nodes.free();
  c->d_weights.free();
  c->d_factors.free();
  for (DevBuf<int>* b : {&c->d_wface, &c->d_wcell, &c->d_wpr, &c->d_wnr}) b->free();
  for (DevBuf<double>* b : {&c->d_wpos, &c->d_wneg, &c->d_wmaxw, &c->d_wden, &c->d_nw}) b->free();
  c->d_macro.free();
  c->d_nu.free();
  c->d_status.free();
  c->d_acc.free();
  c->d_prof.free();
  c->d_margins.free();
  c->d_bins.free();
  c->d_olist.free();
  c->d_tmp.free();
  c->d_tmp_off.free();
  if (c->h_status) cudaFreeHost(c->h_status);
  free_peers(c);
  if (c->comm_st) {
    cudaStreamSynchronize(c->comm_st);
    cudaStreamDestroy(c->comm_st);
    cudaEventDestroy(c->halo_ready);
    cudaEventDestroy(c->halo_done);
    cudaFreeHost(c->h_flag);
  }
  c->d_flag.free();
  if (c->h_rk_all) cudaFreeHost(c->h_rk_all);
  if (c->comm && c->own_comm && nccl().CommDestroy) nccl().CommDestroy(c->comm);
  cudaEventDestroy(c->ev0);
  cudaEventDestroy(c->ev1);
  if (c->fork_ev) {
    for (int k = 0; k < 3; ++k) {
      cudaStreamSynchronize(c->aux[k]);
      cudaStreamDestroy(c->aux[k]);
      cudaEventDestroy(c->join_ev[k]);
    }
    cudaEventDestroy(c->fork_ev);
  }
  cudaStreamDestroy(c->st);
  delete c;
  return TTDVM_OK;
}

const char* ttdvm_cuda_last_error(const ttdvm_ctx* c) { return c ? c->err.c_str() : "null context"; }

int ttdvm_cuda_set_grid(ttdvm_ctx* c, int n, double bound) {
  return guard(c, [&] {
    // VelocityGrid(n, bound), proj/src/velocity_grid.cpp:11-19
    require(n >= 2, "VelocityGrid: need at least 2 nodes");
    require(bound > 0.0, "VelocityGrid: bound must be positive");
    require(n <= 64, "velocity grids above 64 nodes per axis are not supported");
    cudaSetDevice(c->device);
    c->n = n;
    c->bound = bound;
    const double dxi = 2.0 * bound / (n - 1);
    c->nodes.resize(n);
    for (int i = 0; i < n; ++i) c->nodes[i] = -bound + i * dxi;
    std::vector<double> w(n, dxi);
    c->d_nodes.alloc(n);
    c->d_weights.alloc(n);
    CK(cudaMemcpy(c->d_nodes.p, c->nodes.data(), 8 * n, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(c->d_weights.p, w.data(), 8 * n, cudaMemcpyHostToDevice));
    c->terms_dirty = true;
  });
}

int ttdvm_cuda_set_gas(ttdvm_ctx* c, const double gas[6]) {
  return guard(c, [&] {
    require(gas != nullptr, "null gas");
    for (int i = 0; i < 6; ++i) c->gas[i] = gas[i];
    c->terms_dirty = true;
  });
}

int ttdvm_cuda_set_mesh(ttdvm_ctx* c, int32_t ncell, int32_t nface, const int32_t* left,
                        const int32_t* right, const int32_t* group, const double* area,
                        const double* normal, const double* volume, const int64_t* cfo,
                        const int32_t* cfid, const int8_t* cfs) {
  return guard(c, [&] {
    require(ncell > 0 && nface >= 0, "empty mesh");
    c->ncell = ncell;
    c->nface = nface;
    c->left.assign(left, left + nface);
    c->right.assign(right, right + nface);
    c->group.assign(group, group + nface);
    c->area.assign(area, area + nface);
    c->normal.assign(normal, normal + 3 * (size_t)nface);
    c->volume.assign(volume, volume + ncell);
    c->cfo.assign(cfo, cfo + ncell + 1);
    c->cfid.assign(cfid, cfid + cfo[ncell]);
    c->cfs.assign(cfs, cfs + cfo[ncell]);
    for (int f = 0; f < nface; ++f) {
      require(left[f] >= 0 && left[f] < ncell, "face left cell out of range");
      require(right[f] >= -1 && right[f] < ncell, "face right cell out of range");
    }
    for (int i = 0; i < ncell; ++i) {
      require(cfo[i + 1] - cfo[i] + 1 <= kMaxTerms, "too many faces per cell");
      require(volume[i] > 0.0, "nonpositive cell volume");
    }
    c->terms_dirty = true;
  });
}

int ttdvm_cuda_set_bcs(ttdvm_ctx* c, int32_t ngroup, const ttdvm_bc* bcs) {
  return guard(c, [&] {
    require(ngroup >= 0 && (ngroup == 0 || bcs), "null bcs");
    for (int g = 0; g < ngroup; ++g) {
      require(bcs[g].kind >= 0 && bcs[g].kind <= 5, "unknown boundary condition kind");
      if (bcs[g].kind == 0)
        require(bcs[g].wall_temperature > 0.0, "wall boundary requires positive temperature");
    }
    c->bcs.assign(bcs, bcs + ngroup);
    c->terms_dirty = true;
  });
}

int ttdvm_cuda_upload_state(ttdvm_ctx* c, const ttdvm_tt_batch* f) {
  return guard(c, [&] {
    require(c->n > 0, "set_grid first");
    cudaSetDevice(c->device);
    c->cur = 0;
    upload_batch(c, f, c->state[0]);
  });
}

int ttdvm_cuda_state_layout(ttdvm_ctx* c, int32_t* ranks, int64_t* offsets) {
  return guard(c, [&] { layout_of(c, c->state[c->cur], ranks, offsets); });
}

int ttdvm_cuda_download_state(ttdvm_ctx* c, double* cores, int64_t capacity) {
  return guard(c, [&] { download_set(c, c->state[c->cur], cores, capacity); });
}

int ttdvm_cuda_step(ttdvm_ctx* c, double dt, double eps, int32_t cap, int32_t nsteps) {
  return guard(c, [&] {
    require(eps > 0.0, "rounded: eps must be > 0");
    require(c->state[c->cur].count == c->ncell, "state count must equal the mesh cell count");
    cudaSetDevice(c->device);
    build_step_terms(c);
    reset_counters(c);
    for (int k = 0; k < nsteps; ++k) step_synced(c, dt, eps, cap);
  });
}

int ttdvm_cuda_lusgs_step(ttdvm_ctx* c, double dt, double eps, int32_t cap, int32_t niter) {
  return guard(c, [&] {
    require(eps > 0.0, "rounded: eps must be > 0");
    require(dt > 0.0, "lusgs_step: dt must be > 0");
    require(c->state[c->cur].count == c->ncell, "state count must equal the mesh cell count");
    require(c->comm == nullptr, "LU-SGS runs on an unpartitioned mesh");
    cudaSetDevice(c->device);
    build_step_terms(c);
    reset_counters(c);
    for (int k = 0; k < niter; ++k) lusgs_once(c, dt, eps, cap);
  });
}

int ttdvm_cuda_lusgs_levels(ttdvm_ctx* c, int32_t* forward_levels, int32_t* backward_levels) {
  return guard(c, [&] {
    build_step_terms(c);
    build_lusgs_terms(c);
    if (forward_levels) *forward_levels = (int)c->lev_off_f.size() - 1;
    if (backward_levels) *backward_levels = (int)c->lev_off_b.size() - 1;
  });
}

int ttdvm_cuda_macros(ttdvm_ctx* c, double* out) {
  return guard(c, [&] {
    require(c->d_macro.p != nullptr, "no step has run");
    const int nown = c->nowned < 0 ? c->ncell : c->nowned;
    CK(cudaMemcpy(out, c->d_macro.p, 8LL * 11 * nown, cudaMemcpyDeviceToHost));
  });
}

static TensorSet* stage_set(ttdvm_ctx* c, int set) {
  switch (set) {
    case 0: return &c->phi;
    case 1: return &c->jr;
    case 2: return &c->res;
    case 3: return &c->fs;
    default: throw Fail{TTDVM_EINVAL, "unknown stage set"};
  }
}

int ttdvm_cuda_stage_layout(ttdvm_ctx* c, int32_t set, int32_t* count, int32_t* ranks,
                            int64_t* offsets) {
  return guard(c, [&] {
    TensorSet* s = stage_set(c, set);
    if (count) *count = s->count;
    if (ranks || offsets) layout_of(c, *s, ranks, offsets);
  });
}

int ttdvm_cuda_stage_download(ttdvm_ctx* c, int32_t set, double* cores, int64_t capacity) {
  return guard(c, [&] { download_set(c, *stage_set(c, set), cores, capacity); });
}

int ttdvm_cuda_round_batch(ttdvm_ctx* c, const ttdvm_tt_batch* in, int32_t nout,
                           const int64_t* group_off, const double* scale, double eps, int32_t cap,
                           double* margins) {
  return guard(c, [&] {
    require(eps > 0.0, "rounded: eps must be > 0");
    require(c->n > 0, "set_grid first");
    cudaSetDevice(c->device);
    upload_batch(c, in, c->in);
    TermList& tl = c->t_batch;
    require(nout >= 0, "rounded: negative output count");
    tl.off.resize(nout + 1);
    tl.terms.clear();
    for (int o = 0; o <= nout; ++o) {
      tl.off[o] = group_off ? group_off[o] : o;
      require(o == 0 ? tl.off[0] == 0 : tl.off[o] > tl.off[o - 1],
              "group offsets must start at 0 and increase (every sum has a summand)");
    }
    require(tl.off[nout] == in->count, "group offsets must cover the input batch");
    for (int t = 0; t < in->count; ++t)
      tl.terms.push_back(Term{S_IN, t, scale ? scale[t] : 1.0, -1, 0});
    tl.upload();
    TensorSet* sets[kMaxSets] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, &c->in};
    double* dm = nullptr;
    if (margins) {
      c->d_margins.alloc(std::max(1, 2 * nout));
      dm = c->d_margins.p;
    }
    reset_counters(c);
    {
      Timer t(c, 2);
      run_round(c, tl, sets, c->result, eps, cap, dm);
    }
    if (margins && nout)
      CK(cudaMemcpy(margins, dm, 16LL * nout, cudaMemcpyDeviceToHost));
  });
}

int ttdvm_cuda_round_resident(ttdvm_ctx* c, double eps, int32_t cap, int32_t repeats,
                              double* ms) {
  return guard(c, [&] {
    require(eps > 0.0, "rounded: eps must be > 0");
    require(c->t_batch.nout() > 0, "ttdvm_cuda_round_batch first");
    require(repeats >= 1, "repeats must be >= 1");
    cudaSetDevice(c->device);
    TensorSet* sets[kMaxSets] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, &c->in};
    reset_counters(c);
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    CK(cudaStreamSynchronize(c->st));
    CK(cudaEventRecord(a, c->st));
    for (int k = 0; k < repeats; ++k) {
      Timer t(c, 2);
      run_round(c, c->t_batch, sets, c->result, eps, cap, nullptr);
    }
    CK(cudaEventRecord(b, c->st));
    CK(cudaEventSynchronize(b));
    float f = 0.f;
    CK(cudaEventElapsedTime(&f, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    if (ms) *ms = f;
  });
}

int ttdvm_cuda_result_layout(ttdvm_ctx* c, int32_t* ranks, int64_t* offsets) {
  return guard(c, [&] { layout_of(c, c->result, ranks, offsets); });
}

int ttdvm_cuda_result_download(ttdvm_ctx* c, double* cores, int64_t capacity) {
  return guard(c, [&] { download_set(c, c->result, cores, capacity); });
}

int ttdvm_cuda_macro_batch(ttdvm_ctx* c, const ttdvm_tt_batch* in, double* out) {
  return guard(c, [&] {
    require(c->n > 0, "set_grid first");
    cudaSetDevice(c->device);
    upload_batch(c, in, c->in);
    c->d_macro.alloc(std::max(1, 11 * in->count));
    c->launches = 0;
    run_macro(c, c->in, c->d_macro.p, nullptr);
    if (in->count)
      CK(cudaMemcpy(out, c->d_macro.p, 88LL * in->count, cudaMemcpyDeviceToHost));
  });
}

int ttdvm_cuda_collision_batch(ttdvm_ctx* c, const ttdvm_tt_batch* in, double eps,
                               double* macros) {
  return guard(c, [&] {
    require(eps > 0.0, "rounded: eps must be > 0");
    require(c->n > 0, "set_grid first");
    cudaSetDevice(c->device);
    upload_batch(c, in, c->in);
    c->t_fs.off.clear();  // force rebuild of the per-count lists
    c->launches = 0;
    run_collision(c, c->in, eps);
    // result = J_r, the rounded f_S - f before the nu scale; nu is
    // macros[11*i + 10] (compute_collision applies scaled(nu) last).
    c->result.free();
    c->result.resize(c->jr.count);
    c->result.arena.alloc(std::max<long long>(1, c->jr.used));
    CK(cudaMemcpy(c->result.arena.p, c->jr.arena.p, 8LL * std::max<long long>(1, c->jr.used),
                  cudaMemcpyDeviceToDevice));
    if (c->jr.count) {
      CK(cudaMemcpy(c->result.ranks.p, c->jr.ranks.p, 8LL * c->jr.count, cudaMemcpyDeviceToDevice));
      CK(cudaMemcpy(c->result.off.p, c->jr.off.p, 8LL * c->jr.count, cudaMemcpyDeviceToDevice));
    }
    c->result.maxr1 = c->jr.maxr1;
    c->result.maxr2 = c->jr.maxr2;
    c->t_fs.off.clear();
    if (macros && c->in.count)
      CK(cudaMemcpy(macros, c->d_macro.p, 88LL * c->in.count, cudaMemcpyDeviceToHost));
  });
}

int ttdvm_cuda_face_factors(ttdvm_ctx* c, int32_t count, const double* normals, int32_t cap,
                            int32_t mode, double* diag) {
  return guard(c, [&] {
    require(c->n > 0, "set_grid first");
    require(c->n <= 48, "face factors need a velocity grid of at most 48 nodes per axis");
    require(count >= 0 && (count == 0 || normals), "null normals");
    require(cap >= 1 && cap <= 8, "normal tensors: cap_rank >= 1");
    require(mode >= 0 && mode <= 2, "unknown face factor mode");
    for (int i = 0; i < count; ++i) {
      const double* nv = normals + 3 * i;
      require(std::fabs(std::sqrt(nv[0] * nv[0] + nv[1] * nv[1] + nv[2] * nv[2]) - 1.0) <= 1e-12,
              "normal tensors: normal must be a unit vector");
    }
    cudaSetDevice(c->device);
    ensure_static(c);
    const int n = c->n;
    const long long st = (long long)n * cap + (long long)n * cap * cap + (long long)cap * n;
    DevBuf<double> dn, dd;
    dn.alloc(std::max(1, 3 * count));
    if (count) CK(cudaMemcpy(dn.p, normals, 24LL * count, cudaMemcpyHostToDevice));
    if (diag) dd.alloc(std::max(1, 4 * count));
    c->result.free();
    c->result.resize(count);
    c->result.arena.alloc(std::max<long long>(1, st * count));
    std::vector<long long> of(std::max(1, count));
    for (int i = 0; i < count; ++i) of[i] = i * st;
    if (count) CK(cudaMemcpy(c->result.off.p, of.data(), 8LL * count, cudaMemcpyHostToDevice));
    CK(cudaMemsetAsync(c->d_status.p, 0, (kStWords + 4) * sizeof(int), c->st));
    FaceFactorArgs a;
    a.n = n;
    a.nodes = c->d_nodes.p;
    a.count = count;
    a.normals = dn.p;
    a.cap = cap;
    a.mode = mode;
    a.ranks = c->result.ranks.p;
    a.cores = c->result.arena.p;
    a.stride = st;
    a.diag = diag ? dd.p : nullptr;
    a.status = c->d_status.p;
    c->launches = 0;
    CK(launch_face_factor(a, c->st));
    c->launches += 1;
    CK(cudaMemcpyAsync(c->h_status, c->d_status.p, kStWords * sizeof(int), cudaMemcpyDeviceToHost,
                       c->st));
    CK(cudaStreamSynchronize(c->st));
    if (c->h_status[kStError])
      throw Fail{TTDVM_EDOMAIN, "normal tensors: degenerate operand for normal " +
                                    std::to_string(c->h_status[kStErrIdx])};
    c->noise_floor = c->h_status[kStAux];
    c->result.used = st * count;
    c->result.maxr1 = c->result.maxr2 = cap;
    if (diag && count) CK(cudaMemcpy(diag, dd.p, 32LL * count, cudaMemcpyDeviceToHost));
    dn.free();
    dd.free();
  });
}

int ttdvm_cuda_wall_densities(ttdvm_ctx* c, double* out) {
  return guard(c, [&] {
    if (c->nwall) CK(cudaMemcpy(out, c->d_nw.p, 8LL * c->nwall, cudaMemcpyDeviceToHost));
  });
}

int ttdvm_cuda_setup_info(ttdvm_ctx* c, int64_t* info5) {
  return guard(c, [&] {
    info5[0] = c->n_oblique;
    info5[1] = c->noise_floor;
    info5[2] = c->nwall;
    info5[3] = (int64_t)(c->ff_ms * 1000.0);
    info5[4] = c->nblocks;
  });
}

int ttdvm_cuda_phase_times(ttdvm_ctx* c, double* ms8) {
  return guard(c, [&] {
    for (int i = 0; i < 8; ++i) ms8[i] = c->phase_ms[i];
  });
}

int ttdvm_cuda_set_blocks(ttdvm_ctx* c, int32_t nblocks) {
  return guard(c, [&] {
    require(nblocks >= 0, "set_blocks: nblocks must be >= 0");
    c->auto_blocks = nblocks == 0;
    c->nblocks = std::max(1, (int)nblocks);
  });
}

int ttdvm_cuda_nccl_unique_id(char* id128) {
  try {
    require_nccl();
    if (!id128) return TTDVM_EINVAL;
    ncclUniqueIdBytes id;
    if (nccl().GetUniqueId(&id) != 0) return TTDVM_ENCCL;
    memcpy(id128, id.internal, 128);
    return TTDVM_OK;
  } catch (const Fail& e) {
    return e.code;
  }
}

int ttdvm_cuda_comm_init(ttdvm_ctx* c, int32_t nranks, int32_t rank, const char* id128) {
  return guard(c, [&] {
    require(id128 && nranks >= 1 && rank >= 0 && rank < nranks, "comm_init: bad rank / id");
    require_nccl();
    cudaSetDevice(c->device);
    if (c->comm && c->own_comm) nccl().CommDestroy(c->comm);
    c->comm = nullptr;
    ncclUniqueIdBytes id;
    memcpy(id.internal, id128, 128);
    void* comm = nullptr;
    NK(nccl().CommInitRank(&comm, nranks, id, rank));
    c->comm = comm;
    c->own_comm = true;
    c->nranks = nranks;
    c->rank = rank;
    ensure_comm_stream(c);
  });
}

int ttdvm_cuda_set_comm(ttdvm_ctx* c, void* nccl_comm, int32_t nranks, int32_t rank) {
  return guard(c, [&] {
    require(nranks >= 1 && rank >= 0 && rank < nranks, "set_comm: bad rank");
    if (nccl_comm) require_nccl();
    cudaSetDevice(c->device);
    if (c->comm && c->own_comm) nccl().CommDestroy(c->comm);
    c->comm = nccl_comm;
    c->own_comm = false;
    c->nranks = nranks;
    c->rank = rank;
    if (nccl_comm) ensure_comm_stream(c);
  });
}

int ttdvm_cuda_set_partition(ttdvm_ctx* c, int32_t nowned, int32_t npeers, const int32_t* peer_rank,
                             const int64_t* send_off, const int32_t* send_ids,
                             const int64_t* recv_off, const int32_t* recv_ids) {
  return guard(c, [&] {
    require(nowned >= 1 && nowned <= c->ncell, "owned cell count out of range");
    require(npeers >= 0 && (npeers == 0 || (peer_rank && send_off && recv_off)),
            "set_partition: null halo plan");
    cudaSetDevice(c->device);
    free_peers(c);
    c->nowned = nowned;
    c->terms_dirty = true;
    c->peers.resize(npeers);
    for (int q = 0; q < npeers; ++q) {
      HaloPeer& p = c->peers[q];
      p.rank = peer_rank[q];
      require(p.rank >= 0 && p.rank < std::max(1, c->nranks), "set_partition: peer rank out of range");
      p.send_ids.assign(send_ids + send_off[q], send_ids + send_off[q + 1]);
      p.recv_ids.assign(recv_ids + recv_off[q], recv_ids + recv_off[q + 1]);
      for (int id : p.send_ids) require(id >= 0 && id < nowned, "set_partition: send id is not an owned cell");
      for (int id : p.recv_ids)
        require(id >= nowned && id < c->ncell, "set_partition: recv id is not a ghost cell");
      const size_t ns = p.send_ids.size(), nr = p.recv_ids.size();
      p.d_send_ids.alloc(std::max<size_t>(1, ns));
      p.d_send_rk.alloc(std::max<size_t>(1, 2 * ns));
      p.d_recv_rk.alloc(std::max<size_t>(1, 2 * nr));
      p.d_send_off.alloc(std::max<size_t>(1, ns));
      if (ns) CK(cudaMemcpy(p.d_send_ids.p, p.send_ids.data(), 4 * ns, cudaMemcpyHostToDevice));
      CK(cudaMallocHost(&p.h_recv_rk, std::max<size_t>(1, 2 * nr) * sizeof(int)));
    }
  });
}

int ttdvm_cuda_halo_stats(ttdvm_ctx* c, double* out4) {
  return guard(c, [&] {
    require(out4 != nullptr, "halo_stats: null output");
    out4[0] = (double)c->halo_exchanges;
    out4[1] = (double)c->halo_bytes_sent;
    out4[2] = (double)c->halo_bytes_recv;
    out4[3] = c->halo_ms;
  });
}

int ttdvm_cuda_set_owned(ttdvm_ctx* c, int32_t nowned) {
  return guard(c, [&] {
    require(nowned >= 1 && nowned <= c->ncell, "owned cell count out of range");
    c->nowned = nowned;
    c->terms_dirty = true;
  });
}

int ttdvm_cuda_halo_pack(ttdvm_ctx* c, int32_t count, const int32_t* ids, int32_t* ranks_out,
                         int64_t* offsets_out, double* dev_dst, int64_t capacity) {
  return guard(c, [&] {
    TensorSet& s = c->state[c->cur];
    std::vector<int> all(2 * (size_t)s.count);
    if (s.count) CK(cudaMemcpy(all.data(), s.ranks.p, all.size() * 4, cudaMemcpyDeviceToHost));
    long long o = 0;
    std::vector<long long> off(std::max(1, count));
    for (int i = 0; i < count; ++i) {
      require(ids[i] >= 0 && ids[i] < s.count, "halo id out of range");
      ranks_out[2 * i] = all[2 * ids[i]];
      ranks_out[2 * i + 1] = all[2 * ids[i] + 1];
      off[i] = o;
      offsets_out[i] = o;
      o += tt_size(c->n, c->n, c->n, ranks_out[2 * i], ranks_out[2 * i + 1]);
    }
    offsets_out[count] = o;
    if (o > capacity)
      throw Fail{TTDVM_ENOMEM, "halo buffer too small: need " + std::to_string(o) + " doubles"};
    if (count == 0) return;
    DevBuf<int> did;
    did.alloc(count);
    CK(cudaMemcpy(did.p, ids, 4LL * count, cudaMemcpyHostToDevice));
    c->d_tmp_off.alloc(count);
    CK(cudaMemcpy(c->d_tmp_off.p, off.data(), 8LL * count, cudaMemcpyHostToDevice));
    CK(launch_gather_ids(s.view(), did.p, count, c->d_tmp_off.p, c->n, c->n, c->n, dev_dst, c->st));
    c->launches += 1;
    CK(cudaStreamSynchronize(c->st));
    did.free();
  });
}

int ttdvm_cuda_halo_unpack(ttdvm_ctx* c, int32_t count, const int32_t* ids, const int32_t* ranks,
                           const int64_t* offsets, const double* dev_src) {
  return guard(c, [&] {
    TensorSet& s = c->state[c->cur];
    if (count == 0) return;
    for (int i = 0; i < count; ++i)
      require(ids[i] >= 0 && ids[i] < s.count, "halo id out of range");
    DevBuf<int> rk;
    DevBuf<long long> of;
    rk.alloc(2 * (size_t)count);
    of.alloc(count);
    CK(cudaMemcpy(rk.p, ranks, 8LL * count, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(of.p, offsets, 8LL * count, cudaMemcpyHostToDevice));
    TSet src;
    src.ranks = rk.p;
    src.off = of.p;
    src.base = dev_src;
    src.tscale = nullptr;
    src.uscale = 1.0;
    append_tensors(c, src, nullptr, count, ranks, ids, s);
    rk.free();
    of.free();
  });
}

int ttdvm_cuda_phase_work(ttdvm_ctx* c, double* flops8, double* bytes8, int32_t* launches8) {
  return guard(c, [&] {
    for (int i = 0; i < 8; ++i) {
      if (flops8) flops8[i] = c->phase_flops[i];
      if (bytes8) bytes8[i] = c->phase_bytes[i];
      if (launches8) launches8[i] = c->phase_launches[i];
    }
  });
}

int ttdvm_cuda_phase_report(ttdvm_ctx* c, int32_t nphase, double* ms, double* flops,
                            double* bytes, int32_t* launches) {
  return guard(c, [&] {
    require(nphase >= 0 && nphase <= kNPhase, "phase_report: at most 9 phases");
    for (int i = 0; i < nphase; ++i) {
      if (ms) ms[i] = c->phase_ms[i];
      if (flops) flops[i] = c->phase_flops[i];
      if (bytes) bytes[i] = c->phase_bytes[i];
      if (launches) launches[i] = c->phase_launches[i];
    }
  });
}

int ttdvm_cuda_timed_step(ttdvm_ctx* c, double dt, double eps, int32_t cap, int32_t nsteps,
                          double* ms) {
  return guard(c, [&] {
    require(eps > 0.0, "rounded: eps must be > 0");
    require(c->state[c->cur].count == c->ncell, "state count must equal the mesh cell count");
    cudaSetDevice(c->device);
    build_step_terms(c);
    reset_counters(c);
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    CK(cudaStreamSynchronize(c->st));
    CK(cudaEventRecord(a, c->st));
    for (int k = 0; k < nsteps; ++k) step_synced(c, dt, eps, cap);
    CK(cudaEventRecord(b, c->st));
    CK(cudaEventSynchronize(b));
    float f = 0.f;
    CK(cudaEventElapsedTime(&f, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    if (ms) *ms = f;
  });
}

int ttdvm_cuda_round_profile(ttdvm_ctx* c, int on, uint64_t* cycles16) {
  return guard(c, [&] {
    c->d_prof.alloc(16);
    if (cycles16) CK(cudaMemcpy(cycles16, c->d_prof.p, 16 * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemset(c->d_prof.p, 0, 16 * 8));
    c->round_prof = on != 0;
  });
}

int ttdvm_cuda_fp64_peak(ttdvm_ctx* c, double* tflops) {
  return guard(c, [&] {
    cudaSetDevice(c->device);
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device));
    const int threads = 512, blocks = sms * 4, iters = 4000;
    DevBuf<double> out;
    out.alloc(blocks);
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    CK(launch_dfma_probe(out.p, blocks, threads, 100, c->st));  // warm-up
    CK(cudaEventRecord(a, c->st));
    CK(launch_dfma_probe(out.p, blocks, threads, iters, c->st));
    CK(cudaEventRecord(b, c->st));
    CK(cudaEventSynchronize(b));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, a, b));
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    out.free();
    const double flops = 2.0 * 8 * 16 * (double)iters * threads * blocks;
    *tflops = flops / (ms * 1e-3) / 1e12;
  });
}

int64_t ttdvm_cuda_launch_count(const ttdvm_ctx* c) { return c ? c->launches : -1; }

int ttdvm_cuda_set_profiling(ttdvm_ctx* c, int on) {
  return guard(c, [&] { c->profiling = on != 0; });
}

}  // extern "C"
