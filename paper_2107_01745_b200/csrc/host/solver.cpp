// SPDX-License-Identifier: MIT
//
// Solver layer over the device kernels: the forward-backward step, the FBE
// gradient, the line-search certificate, L-BFGS, the power iteration, and the
// MINFBE / NAMA / GPAD loops with the reference's exact control flow
// (solvers.hpp:89-720, fbe.hpp, lbfgs.hpp). All vector work runs on the
// device (sweep.cu, dualops.cu); the host only sequences kernels and reads a
// few scalars at the decision points the reference's loops branch on.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <atomic>
#include <cstring>
#include <limits>
#include <random>
#include <string>
#include <mutex>
#include <vector>

#include "capi_internal.hpp"

using namespace scn;

// ------------------------------------------------------------------ workspace
struct scenopt_dev::Work {
  int D = 0, nblk = 0;
  double* S = nullptr;
  int* I = nullptr;
  double* part = nullptr;
  unsigned* bar = nullptr;
  double* hS = nullptr;  // pinned mirrors
  int* hI = nullptr;
  // mapped pinned flagged words of S / I written by k_publish or a fused FB
  // finish (dual.hpp kPubWords); seq is the number of the last publish issued
  unsigned long long* pLL = nullptr;
  unsigned long long* dpLL = nullptr;
  unsigned seq = 0;
  cudaEvent_t pubEv = nullptr;
  // pinned staging words of asynchronous scalar writes; a word is reused only
  // after a stream synchronisation has retired every copy that read it
  static constexpr int kRing = 256;
  double* hRing = nullptr;
  int ring_next = 0;
  int* hIRing = nullptr;  // the same for int-block writes (kRing words)
  int iring_next = 0;
  // two FbStates (ping-pong)
  double *y[2] = {}, *Hx[2] = {}, *z[2] = {}, *R[2] = {}, *T[2] = {}, *x[2] = {}, *u[2] = {};
  double *Hx0 = nullptr, *x0 = nullptr, *u0 = nullptr;
  double *grad = nullptr, *prev_y = nullptr, *prev_g = nullptr, *dir = nullptr, *Hd = nullptr,
         *HR = nullptr, *v = nullptr, *Hv = nullptr, *w = nullptr, *yp = nullptr, *weight = nullptr,
         *tmp = nullptr, *tmp2 = nullptr;
  double *Sb = nullptr, *Qb = nullptr;
  double* Mb = nullptr;  // compact L-BFGS: S'Y and Y'Y of the stored pairs (2 x 64 x 64)
  double* small = nullptr;  // 64 doubles of API scratch
  double *xs = nullptr, *xr = nullptr;  // sharded: per-phase totals of this rank / of all ranks
  int lb_slots = 0;
  bool fhat0_ready = false;
  DualCtx ctx(const DevState& d) const {
    DualCtx c{};
    c.D = D;
    c.nblk = nblk;
    c.g = RowG{d.row_kind, d.row_lo, d.row_hi, d.row_wg};
    c.S = S;
    c.I = I;
    c.part = part;
    c.bar = bar;
    if (d.sharded()) {  // reductions over this rank's rows, combined across ranks (DualCtx)
      c.cnt = d.row_counted;
      c.xc = d.comm.get();
      c.world = d.world;
      c.xs = xs;
      c.xr = xr;
    }
    return c;
  }
};

namespace {
void prewarm_results(const Layout& L);
}

scenopt_dev::scenopt_dev() = default;
scenopt_dev::~scenopt_dev() {
  if (w) {
    if (w->hS) cudaFreeHost(w->hS);
    if (w->hI) cudaFreeHost(w->hI);
    if (w->hRing) cudaFreeHost(w->hRing);
    if (w->hIRing) cudaFreeHost(w->hIRing);
    if (w->pLL) cudaFreeHost(w->pLL);
    if (w->pubEv) cudaEventDestroy(w->pubEv);
  }
}

void scenopt_dev::init_solver_buffers() {
  DevState& ds = *d;
  SCN_CUDA(cudaSetDevice(ds.device));
  w = std::make_unique<Work>();
  Work& k = *w;
  const Layout& L = ds.lay;
  k.D = std::max(L.dual_dim, 1);
  k.nblk = std::min(ds.sm_count, dual_max_blocks());  // grid of the dual-space kernels: one co-resident block per SM
  k.S = ds.alloc<double>(sl::kScalars);
  k.I = ds.alloc<int>(il::kInts);
  k.part = ds.alloc<double>(static_cast<size_t>(2) * 64 * k.nblk);
  k.bar = ds.alloc<unsigned>(4);
  SCN_CUDA(cudaMemset(k.S, 0, sl::kScalars * sizeof(double)));
  SCN_CUDA(cudaMemset(k.I, 0, il::kInts * sizeof(int)));
  SCN_CUDA(cudaMemset(k.bar, 0, 4 * sizeof(unsigned)));
  SCN_CUDA(cudaMallocHost(&k.hS, sl::kScalars * sizeof(double)));
  SCN_CUDA(cudaMallocHost(&k.hI, il::kInts * sizeof(int)));
  SCN_CUDA(cudaMallocHost(&k.hRing, scenopt_dev::Work::kRing * sizeof(double)));
  SCN_CUDA(cudaMallocHost(&k.hIRing, scenopt_dev::Work::kRing * sizeof(int)));
  SCN_CUDA(cudaHostAlloc(&k.pLL, kPubWords * sizeof(unsigned long long), cudaHostAllocMapped));
  std::memset(k.pLL, 0, kPubWords * sizeof(unsigned long long));  // flag 0: no publish yet
  SCN_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&k.dpLL), k.pLL, 0));
  SCN_CUDA(cudaEventCreateWithFlags(&k.pubEv, cudaEventDisableTiming));
  const size_t D = static_cast<size_t>(k.D), nxn = static_cast<size_t>(L.nx) * L.n,
               nuf = static_cast<size_t>(L.nu) * std::max(L.first_leaf, 1);
  for (int s = 0; s < 2; ++s) {
    k.y[s] = ds.alloc<double>(D);
    k.Hx[s] = ds.alloc<double>(D);
    k.z[s] = ds.alloc<double>(D);
    k.R[s] = ds.alloc<double>(D);
    k.T[s] = ds.alloc<double>(D);
    k.x[s] = ds.alloc<double>(nxn);
    k.u[s] = ds.alloc<double>(nuf);
  }
  k.small = ds.alloc<double>(64);
  if (ds.sharded()) {
    k.xs = ds.alloc<double>(kXMax);
    k.xr = ds.alloc<double>(static_cast<size_t>(kXMax) * ds.world);
  }
  k.Hx0 = ds.alloc<double>(D);
  k.x0 = ds.alloc<double>(nxn);
  k.u0 = ds.alloc<double>(nuf);
  for (double** p : {&k.grad, &k.prev_y, &k.prev_g, &k.dir, &k.Hd, &k.HR, &k.v, &k.Hv, &k.w, &k.yp,
                     &k.weight, &k.tmp, &k.tmp2})
    *p = ds.alloc<double>(D);
  if (ds.has_factor) prewarm_results(L);
}

namespace {

double now_ms() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

// Result arrays of a report (x, u, y, z): page-locked host memory from a
// process-wide pool, so the final download runs at full PCIe rate (a fresh
// pageable 10.5 MB vector costs ~2.7 ms of page faults and zero-fill at C3,
// and pageable D2H copies are staged at a fraction of the pinned rate; both
// sit inside wall_ms). Destroyed reports return their arrays to the pool
// (at most 16 arrays and 1 GB; a request takes the smallest array that
// fits, and only one at most twice its size; 1 GB holds the results of two
// C4-sized solves, whose fresh page-locked allocation would cost more than
// the faster copy saves). Falls back to pageable memory when page-locked
// memory is unavailable.
class ResultArray {
 public:
  ResultArray() = default;
  ResultArray(const ResultArray&) = delete;
  ResultArray& operator=(const ResultArray&) = delete;
  ResultArray(ResultArray&& o) noexcept { swap(o); }
  ResultArray& operator=(ResultArray&& o) noexcept {
    swap(o);
    return *this;
  }
  ~ResultArray() { give(); }
  void take(size_t n);  // n elements, contents unspecified (overwritten by the download)
  void give();          // back to the pool
  void assign(size_t n, double v) {
    take(n);
    std::fill(p_, p_ + n_, v);
  }
  size_t size() const { return n_; }
  bool empty() const { return n_ == 0; }
  double* data() { return p_; }
  const double* data() const { return p_; }
  double& operator[](size_t i) { return p_[i]; }
  double operator[](size_t i) const { return p_[i]; }
  double* begin() { return p_; }
  double* end() { return p_ + n_; }

 private:
  void swap(ResultArray& o) noexcept {
    std::swap(p_, o.p_);
    std::swap(n_, o.n_);
    std::swap(cap_, o.cap_);
    std::swap(pinned_, o.pinned_);
  }
  double* p_ = nullptr;
  size_t n_ = 0, cap_ = 0;
  bool pinned_ = false;
};

namespace {
struct PoolBlock {
  double* p;
  size_t cap;
  bool pinned;
};
std::mutex g_arrays_mu;
std::vector<PoolBlock> g_arrays;
size_t g_arrays_bytes = 0;
constexpr size_t kArraysKept = 16, kArraysMaxBytes = size_t(1) << 30;
void free_block(const PoolBlock& b) {
  if (b.pinned)
    cudaFreeHost(b.p);
  else
    std::free(b.p);
}
}  // namespace

void ResultArray::take(size_t n) {
  give();
  if (n == 0) return;
  {
    std::lock_guard<std::mutex> lk(g_arrays_mu);
    size_t best = g_arrays.size();
    for (size_t i = 0; i < g_arrays.size(); ++i)  // the smallest that fits, at most 2n
      if (g_arrays[i].cap >= n && g_arrays[i].cap <= 2 * n &&
          (best == g_arrays.size() || g_arrays[i].cap < g_arrays[best].cap))
        best = i;
    if (best < g_arrays.size()) {
      const PoolBlock b = g_arrays[best];
      g_arrays_bytes -= b.cap * sizeof(double);
      g_arrays.erase(g_arrays.begin() + static_cast<std::ptrdiff_t>(best));
      p_ = b.p;
      cap_ = b.cap;
      pinned_ = b.pinned;
      n_ = n;
      return;
    }
  }
  void* q = nullptr;
  if (cudaMallocHost(&q, n * sizeof(double)) == cudaSuccess) {
    pinned_ = true;
  } else {
    cudaGetLastError();
    q = std::malloc(n * sizeof(double));
    if (!q) throw std::bad_alloc();
    pinned_ = false;
  }
  p_ = static_cast<double*>(q);
  cap_ = n_ = n;
}

void ResultArray::give() {
  if (!p_) return;
  const PoolBlock b{p_, cap_, pinned_};
  p_ = nullptr;
  n_ = cap_ = 0;
  {
    std::lock_guard<std::mutex> lk(g_arrays_mu);
    if (g_arrays.size() < kArraysKept && g_arrays_bytes + b.cap * sizeof(double) <= kArraysMaxBytes) {
      g_arrays_bytes += b.cap * sizeof(double);
      g_arrays.push_back(b);
      return;
    }
  }
  free_block(b);
}

// Page-locked result arrays for two live reports of this shape go into the
// pool at handle creation, so the first solves' downloads do not pay for
// the allocation inside wall_ms.
void prewarm_results(const Layout& L) {
  const size_t sizes[4] = {static_cast<size_t>(L.nx) * L.n, static_cast<size_t>(L.nu) * L.first_leaf,
                           static_cast<size_t>(L.dual_dim), static_cast<size_t>(L.dual_dim)};
  ResultArray a[8];
  for (int r = 0; r < 2; ++r)
    for (int q = 0; q < 4; ++q) a[4 * r + q].take(sizes[q]);
}  // ~ResultArray returns them to the pool

struct Report {  // SolverReport, solvers.hpp:66-84
  int status = 1, iterations = 0;
  Stats stats;
  uint64_t lipschitz_calls = 0;
  double lipschitz_estimate = 0.0, lambda_final = 0.0, eps = 0.0,
         residual_inf = std::numeric_limits<double>::infinity(), wall_ms = 0.0;
  bool verified = false;
  double verify_residual_inf = std::numeric_limits<double>::infinity();
  double verify_subdiff_dist = std::numeric_limits<double>::infinity();
  std::vector<double> residual_trace, fbe_trace;
  ResultArray x, u, y, z;
};

// solvers.hpp:48-60
void validate_config(const scenopt_solver_config& c) {
  if (c.lambda0 < 0.0) fail(SCENOPT_E_INVALID_PARAMS, "lambda0 must be >= 0");
  if (!(c.eps > 0.0)) fail(SCENOPT_E_INVALID_PARAMS, "eps must be > 0");
  if (!(c.eps_curv > 0.0)) fail(SCENOPT_E_INVALID_PARAMS, "eps_curv must be > 0");
  if (!(c.eps_bt > 0.0 && c.eps_bt < 0.5)) fail(SCENOPT_E_INVALID_PARAMS, "eps_bt must lie in (0, 1/2)");
  if (c.beta_bt < 0.0 || c.beta_bt >= 1.0) fail(SCENOPT_E_INVALID_PARAMS, "beta_bt must lie in [0, 1)");
  if (c.memory < 1) fail(SCENOPT_E_INVALID_PARAMS, "memory must be >= 1");
  if (c.memory > 48) fail(SCENOPT_E_INVALID_PARAMS, "memory must be <= 48 on the device");
  if (c.max_iters < 1) fail(SCENOPT_E_INVALID_PARAMS, "max_iters must be >= 1");
  if (c.warm_start_iters < 0) fail(SCENOPT_E_INVALID_PARAMS, "warm_start_iters must be >= 0");
  if (c.backtracking_rule < 0 || c.backtracking_rule > 2)
    fail(SCENOPT_E_INVALID_PARAMS, "unknown backtracking rule");
}

// a sharded handle runs the compact L-BFGS form only (one reduction per direction)
void validate_for(const scenopt_solver_config& c, const DevState& d) {
  validate_config(c);
  if (d.sharded() && c.memory > kLbfgsCompactMaxMem)
    fail(SCENOPT_E_INVALID_PARAMS, "memory must be <= 6 on a sharded handle");
}

// solvers.hpp:122-127
double halve_lambda(double lambda) {
  const double next = 0.5 * lambda;
  if (next < 1e-14) fail(SCENOPT_E_STEP_UNDERFLOW, "backtracking drove lambda below 1e-14");
  return next;
}

}  // namespace

namespace scn {
void check_solver_config(const scenopt_solver_config& c) { validate_config(c); }  // experiment.cpp
}  // namespace scn

// Engine: the per-handle solver operations (device resident).
struct Engine {
  scenopt_dev& h;
  DevState& d;
  scenopt_dev::Work& k;
  cudaStream_t st;
  Engine(scenopt_dev& hh) : h(hh), d(*hh.d), k(*hh.w), st(hh.d->stream) { SCN_CUDA(cudaSetDevice(d.device)); }
  DualCtx ctx() const { return k.ctx(d); }
  size_t D() const { return static_cast<size_t>(d.lay.dual_dim); }

  // Stream-ordered scalar write, no host synchronisation.
  void set_scalar(int slot, double v) {
    if (k.ring_next == scenopt_dev::Work::kRing) {  // every staging word may still be in flight
      SCN_CUDA(cudaStreamSynchronize(st));
      k.ring_next = 0;
    }
    double* w = k.hRing + k.ring_next++;
    *w = v;
    k.hS[slot] = v;  // host mirror
    SCN_CUDA(cudaMemcpyAsync(k.S + slot, w, sizeof(double), cudaMemcpyHostToDevice, st));
  }
  // Stream-ordered write of n ints at I[slot..] from pinned staging words
  // (ordered with every kernel of the handle's stream, no host synchronisation).
  void set_ints(int slot, const int* v, int n) {
    if (k.iring_next + n > scenopt_dev::Work::kRing) {  // every staging word may still be in flight
      SCN_CUDA(cudaStreamSynchronize(st));
      k.iring_next = 0;
    }
    int* w = k.hIRing + k.iring_next;
    k.iring_next += n;
    std::memcpy(w, v, n * sizeof(int));
    std::memcpy(k.hI + slot, v, n * sizeof(int));  // host mirror
    SCN_CUDA(cudaMemcpyAsync(k.I + slot, w, n * sizeof(int), cudaMemcpyHostToDevice, st));
  }
  // Host reads of the scalar block. publish() enqueues its copy into mapped
  // host memory and marks it with an event; wait_published() waits for that
  // event only, so work enqueued after publish() keeps the GPU busy while the
  // host decides (speculation). read_scalars() = publish + full stream sync.
  cudaEvent_t pub_pre = nullptr;
  void publish() {
    if (timer.on) {
      cudaEventCreate(&pub_pre);
      cudaEventRecord(pub_pre, st);
    }
    SCN_CUDA(k_publish(k.S, k.I, k.dpLL, ++k.seq, st));
    mark("read.copy");
  }
  // Spin on the mapped flagged words (no driver call, no sleep / wake-up):
  // word by word until each carries this publish's flag, then decode them
  // into the host mirrors. Every 4096 polls the stream is queried so a device
  // fault cannot hang it.
  void wait_published(bool full) {
    const double h0 = timer.on ? now_ms() : 0.0;
    const volatile unsigned long long* w = k.pLL;
    const unsigned long long want = k.seq;
    unsigned spins = 0;
    double drained_at = -1.0;  // the stream has finished while words were missing
    for (int i = 0; i < kPubWords;) {
      if ((w[i] >> 32) == want) {
        ++i;
        continue;
      }
      if ((++spins & 4095u) == 0) {
        if (drained_at < 0.0) {
          const cudaError_t q = cudaStreamQuery(st);
          if (q != cudaSuccess && q != cudaErrorNotReady) SCN_CUDA(q);
          if (q == cudaSuccess) drained_at = now_ms();
        } else if (now_ms() - drained_at > 100.0) {
          // a finished kernel's posted writes land within microseconds: after
          // the grace period the words are not coming
          if (full || static_cast<int>(static_cast<unsigned>(w[i] >> 32) - static_cast<unsigned>(want)) > 0)
            fail(SCENOPT_E_ERROR, "scalar publish " + std::to_string(want) + " never arrived (word " +
                                      std::to_string(i) + " carries " + std::to_string(w[i] >> 32) + ")");
          break;  // no publish was enqueued: the mirrors keep what the words hold
        }
      }
    }
    std::atomic_thread_fence(std::memory_order_acquire);
    if (full) k.ring_next = k.iring_next = 0;  // publish ran after every earlier copy: all staging words consumed
    if (timer.on) timer.host_sync_ms += now_ms() - h0;
    for (int t = 0; t < sl::kScalars; ++t) {
      const unsigned long long b = (w[2 * t] & 0xffffffffull) | ((w[2 * t + 1] & 0xffffffffull) << 32);
      std::memcpy(&k.hS[t], &b, sizeof(double));
    }
    for (int t = 0; t < il::kInts; ++t) k.hI[t] = static_cast<int>(static_cast<unsigned>(w[2 * sl::kScalars + t]));
    if (timer.on) {  // GPU-side cost of this host round trip: copy + wake-up + re-enqueue
      cudaEvent_t post;
      cudaEventCreate(&post);
      cudaEventRecord(post, st);
      timer.sync_ev.emplace_back(pub_pre, post);
    }
  }
  void read_scalars() {
    publish();
    wait_published(true);
  }
  void mark(const char* tag) {
    if (!timer.marks) return;
    cudaEvent_t ev;
    cudaEventCreate(&ev);
    cudaEventRecord(ev, st);
    timer.mk.emplace_back(tag, ev);
  }
  double S(int slot) const { return k.hS[slot]; }
  int I(int slot) const { return k.hI[slot]; }
  void copy(double* dst, const double* src, size_t n) {
    SCN_CUDA(cudaMemcpyAsync(dst, src, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
  }
  // SCN_SOLVE_TIMING=1: CUDA-event time of every sweep, summed to stderr at exit (diagnostics)
  struct SweepTimer {
    bool on = std::getenv("SCN_SOLVE_TIMING") != nullptr;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;
    std::vector<double> seq_ms;
    std::vector<int> kind;  // per sweep: 0 homogeneous, 1 affine, 2 affine + fused FB finish, 3 two RHS
    ~SweepTimer() {
      report_marks();
      if (!on || ev.empty()) return;
      cudaDeviceSynchronize();
      double tot = 0.0, by_kind[4] = {0, 0, 0, 0};
      int n_kind[4] = {0, 0, 0, 0};
      for (size_t i = 0; i < ev.size(); ++i) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ev[i].first, ev[i].second);
        seq_ms.push_back(ms);
        tot += ms;
        by_kind[kind[i]] += ms;
        ++n_kind[kind[i]];
        cudaEventDestroy(ev[i].first);
        cudaEventDestroy(ev[i].second);
      }
      std::fprintf(stderr, "[scn] %zu sweeps, %.3f ms GPU (%.1f us each)\n", ev.size(), tot, 1e3 * tot / ev.size());
      if (std::atoi(std::getenv("SCN_SOLVE_TIMING")) == 3) {  // every sweep in order: kind:us
        std::fprintf(stderr, "[scn]   seq");
        for (size_t i = 0; i < ev.size(); ++i) std::fprintf(stderr, " %d:%.0f", kind[i], 1e3 * seq_ms[i]);
        std::fprintf(stderr, "\n");
      }
      static const char* const names[4] = {"homogeneous", "affine", "affine+fb", "2-rhs"};
      for (int q = 0; q < 4; ++q)
        if (n_kind[q])
          std::fprintf(stderr, "[scn]   %-12s %3d x %.1f us\n", names[q], n_kind[q], 1e3 * by_kind[q] / n_kind[q]);
      double st = 0.0;
      for (auto& p : sync_ev) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, p.first, p.second);
        st += ms;
      }
      if (!sync_ev.empty())
        std::fprintf(stderr, "[scn] %zu host round trips, %.3f ms (%.1f us each)\n", sync_ev.size(), st,
                     1e3 * st / sync_ev.size());
      for (auto& p : sync_ev) {
        cudaEventDestroy(p.first);
        cudaEventDestroy(p.second);
      }
      std::fprintf(stderr, "[scn] host: %.3f ms enqueuing sweeps (%.1f us each), %.3f ms blocked in reads\n",
                   host_launch_ms, 1e3 * host_launch_ms / ev.size(), host_sync_ms);
    }
    double host_launch_ms = 0.0, host_sync_ms = 0.0;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> sync_ev;
    // SCN_SOLVE_TIMING=2: an event after every stream op of the loops; the
    // time between consecutive marks (op + any idle before it) averaged per tag
    bool marks = on && std::atoi(std::getenv("SCN_SOLVE_TIMING")) >= 2;
    std::vector<std::pair<const char*, cudaEvent_t>> mk;
    void report_marks() {
      if (mk.size() < 2) return;
      cudaDeviceSynchronize();
      std::vector<std::pair<std::string, std::pair<double, int>>> agg;
      for (size_t i = 1; i < mk.size(); ++i) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, mk[i - 1].second, mk[i].second);
        size_t t = 0;
        while (t < agg.size() && agg[t].first != mk[i].first) ++t;
        if (t == agg.size()) agg.push_back({mk[i].first, {0.0, 0}});
        agg[t].second.first += ms;
        ++agg[t].second.second;
      }
      for (auto& a : agg)
        std::fprintf(stderr, "[scn]   %-14s %4d x %8.1f us = %8.3f ms\n", a.first.c_str(), a.second.second,
                     1e3 * a.second.first / a.second.second, a.second.first);
      for (auto& m : mk) cudaEventDestroy(m.second);
      mk.clear();
    }
  } timer;
  template <class F>
  void timed(F&& f, int kind = 0) {
    if (!timer.on) return f();
    timer.kind.push_back(kind);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, st);
    const double h0 = now_ms();
    f();
    timer.host_launch_ms += now_ms() - h0;  // host cost of enqueuing the sweep
    cudaEventRecord(b, st);
    timer.ev.emplace_back(a, b);
  }
  void sweep1(bool affine, const double* y, double* x, double* u, double* Hx) {
    timed([&] { dev_sweep(d, 1, affine, &y, x ? &x : nullptr, u ? &u : nullptr, &Hx); },
          affine ? (d.fb_next ? 2 : 1) : 0);
  }
  // H x0(r) launched only if the last fb_finish missed the stop tolerance
  // (I[CONV], see k_fb_finish): a speculative sweep costs a launch at convergence
  struct SkipScope {  // sweeps launched in scope return at once when I[CONV] != 0
    DevState& d;
    SkipScope(DevState& dd, const int* w) : d(dd) { d.sweep_skip = w; }
    ~SkipScope() { d.sweep_skip = nullptr; }
  };
  void sweep1_unless_converged(const double* r, double* Hr) {
    SkipScope g(d, k.I + il::CONV);
    sweep1(false, r, nullptr, nullptr, Hr);
  }
  // the GATE_RULE code of fb_finish's skip word for solver kind (0 MINFBE, 1 NAMA)
  void set_gate(const scenopt_solver_config& cfg, int kind) {
    set_scalar(sl::EPS_STOP, cfg.eps);
    set_scalar(sl::GATE_RULE, cfg.backtracking_rule == 1 && kind == 1 ? 3 : cfg.backtracking_rule);
    set_scalar(sl::BETA_BT, cfg.beta_bt);
    set_scalar(sl::EPS_BT, cfg.eps_bt);
  }
  void sweep2(const double* a, const double* b, double* Ha, double* Hb) {
    const double* ys[2] = {a, b};
    double* hs[2] = {Ha, Hb};
    timed([&] { dev_sweep(d, 2, false, ys, nullptr, nullptr, hs); }, 3);
  }

  // f_hat(0) and H x(0), once per handle (fhat identity)
  void ensure_fhat0() {
    if (k.fhat0_ready) return;
    SCN_CUDA(cudaMemsetAsync(k.tmp, 0, D() * sizeof(double), st));
    sweep1(true, k.tmp, k.x0, k.u0, k.Hx0);
    SCN_CUDA(k_eval_f(ctx(), d.cost, k.x0, k.u0, 1e-8, st));  // sharded: own nodes, summed over ranks
    read_scalars();
    const double f0 = S(sl::EVALF);
    if (S(sl::EVALF_INF) != 0.0 || !std::isfinite(f0))
      fail(SCENOPT_E_ERROR, "fhat(0): the oracle's minimiser violated the dynamics");
    set_scalar(sl::FHAT0, -f0);
    k.fhat0_ready = true;
  }

  // fb_step (fbe.hpp:55-67) into state s: dual_grad sweep + fused finish
  // publish_after: fb_finish also publishes the scalar block (= publish() right after it)
  void fb_step(int s, const double* ydev, double lambda, const double* weight, Stats& stats,
               bool publish_after = false) {
    if (!(lambda > 0.0)) fail(SCENOPT_E_INVALID_PARAMS, "fb_step: lambda must be > 0");
    ensure_fhat0();
    if (ydev != k.y[s]) copy(k.y[s], ydev, D());
    set_scalar(s * sl::kStateStride + sl::LAM, lambda);
    if (publish_after && timer.on) {
      cudaEventCreate(&pub_pre);
      cudaEventRecord(pub_pre, st);
    }
    if (!d.sharded() && d.fb_part) {
      // finish_fb_fields fused into the sweep: its last CTA writes the step's
      // scalars (and publishes them) once every CTA has finished its rows
      DevState::FbFuse f;
      f.S = k.S;
      f.I = k.I;
      f.state = s;
      f.Hx0 = k.Hx0;
      f.weight = weight;
      f.z = k.z[s];
      f.R = k.R[s];
      f.T = k.T[s];
      if (publish_after) {
        f.pub = k.dpLL;
        f.seq = ++k.seq;
      }
      struct Reset {
        DevState& d;
        ~Reset() { d.fb_next = nullptr; }
      } reset{d};
      d.fb_next = &f;
      sweep1(true, k.y[s], k.x[s], k.u[s], k.Hx[s]);
    } else {
      sweep1(true, k.y[s], k.x[s], k.u[s], k.Hx[s]);
      DualCtx c = ctx();
      if (publish_after) {
        c.pub = k.dpLL;
        c.seq = ++k.seq;
      }
      SCN_CUDA(k_fb_finish(c, s, 0, k.y[s], k.Hx[s], k.Hx0, weight, k.z[s], k.R[s], k.T[s], st));
    }
    ++stats.dual_grad_calls;
    ++stats.prox_calls;
    ++stats.conj_calls;
  }
  // rescale_state (fbe.hpp:72-77): no sweep
  void rescale(int s, double lambda, const double* weight, Stats& stats) {
    if (!(lambda > 0.0)) fail(SCENOPT_E_INVALID_PARAMS, "rescale_state: lambda must be > 0");
    set_scalar(s * sl::kStateStride + sl::LAM, lambda);
    SCN_CUDA(k_fb_finish(ctx(), s, 1, k.y[s], k.Hx[s], k.Hx0, weight, k.z[s], k.R[s], k.T[s], st));
    ++stats.prox_calls;
    ++stats.conj_calls;
  }
  void lbfgs_reset(int mem) {
    if (k.lb_slots < mem + 1) {
      k.Sb = d.alloc<double>(static_cast<size_t>(mem + 1) * D());
      k.Qb = d.alloc<double>(static_cast<size_t>(mem + 1) * D());
      if (!k.Mb) k.Mb = d.alloc<double>(2 * 64 * 64);
      k.lb_slots = mem + 1;
    }
    int ints[il::LB_ORDER + 64] = {};
    for (int j = 0; j <= mem; ++j) ints[il::LB_ORDER + j] = j;
    set_ints(il::LB_COUNT, ints + il::LB_COUNT, 2);                   // count, pushed
    set_ints(il::LB_ORDER, ints + il::LB_ORDER, mem + 1);
    set_scalar(sl::GAMMA0, 1.0);
  }
  void lbfgs_clear() {  // lbfgs.hpp:64-67
    const int zero = 0;
    set_ints(il::LB_COUNT, &zero, 1);
    set_scalar(sl::GAMMA0, 1.0);
  }

  // estimate_dual_lipschitz (solvers.hpp:89-113)
  double lipschitz(uint64_t* calls, double rel_tol = 1e-6, int max_rounds = 100) {
    if (max_rounds <= 0) return 1e-12;  // no round: the Rayleigh quotient stays 0 (solvers.hpp:99-112)
    const int n = d.lay.dual_dim;
    std::vector<double> v(static_cast<size_t>(n));
    std::mt19937_64 gen(0x5eed5eed5eed5eedULL);
    for (int i = 0; i < n; ++i) v[i] = 2.0 * ((gen() >> 11) * 0x1.0p-53) - 1.0;
    double nn = 0.0;
    for (double a : v) nn += a * a;
    nn = std::sqrt(nn);
    for (double& a : v) a /= nn;
    // pageable source: the copy is stream-ordered and v is staged before the call returns
    SCN_CUDA(cudaMemcpyAsync(k.v, v.data(), v.size() * sizeof(double), cudaMemcpyHostToDevice, st));
    set_scalar(sl::RAYLEIGH, 0.0);
    // Rounds are enqueued kBatch at a time and read once per batch: the power
    // kernel sets a sticky stop flag at the reference's stopping round (settled,
    // zero image or max_rounds), after which the remaining launches of the
    // batch, sweeps included, return at once. Same rounds, same estimate.
    const int init[3] = {0, 0, max_rounds};
    set_ints(il::PDONE, init, 3);
    struct SkipGuard {
      DevState& d;
      ~SkipGuard() { d.sweep_skip = nullptr; }
    } guard{d};
    d.sweep_skip = k.I + il::PDONE;
    constexpr int kBatch = 8;
    for (int round = 0; round < max_rounds; round += kBatch) {
      for (int b = 0; b < kBatch && round + b < max_rounds; ++b) {
        sweep1(false, k.v, nullptr, nullptr, k.Hv);
        SCN_CUDA(k_power(ctx(), k.v, k.Hv, rel_tol, st));
      }
      read_scalars();
      if (I(il::PDONE)) break;
    }
    if (calls) *calls += static_cast<uint64_t>(I(il::PROUNDS));
    if (I(il::PZERO)) return 1e-12;
    return std::max(S(sl::PNEXT), 1e-12);
  }
};

namespace {

// Trace bookkeeping shared by the loops (solvers.hpp:151-169).
struct Loop {
  Engine& e;
  Report& rep;
  const double* weight;
  double t0;
  void push_trace(int s) {
    rep.residual_trace.push_back(e.S(s * sl::kStateStride + sl::RESID));
    rep.fbe_trace.push_back(e.S(s * sl::kStateStride + sl::VALUE));
  }
  void refresh_tail(int s) {
    e.read_scalars();
    rep.residual_trace.back() = e.S(s * sl::kStateStride + sl::RESID);
    rep.fbe_trace.back() = e.S(s * sl::kStateStride + sl::VALUE);
  }
  void finish(int status, int s, double residual, double lambda) {
    rep.status = status;
    rep.residual_inf = residual;
    rep.lambda_final = lambda;
    const Layout& L = e.d.lay;
    rep.x.take(static_cast<size_t>(L.nx) * L.n);
    rep.u.take(static_cast<size_t>(L.nu) * L.first_leaf);
    rep.y.take(static_cast<size_t>(L.dual_dim));
    rep.z.take(static_cast<size_t>(L.dual_dim));
    auto dl = [&](ResultArray& dst, const double* src) {
      if (!dst.empty())
        SCN_CUDA(cudaMemcpyAsync(dst.data(), src, dst.size() * sizeof(double), cudaMemcpyDeviceToHost, e.st));
    };
    const double f0 = now_ms();
    // sharded: assemble the full point (the gathers read the states, never write them)
    const auto xu = dev_gather_primal(e.d, e.k.x[s], e.k.u[s]);
    dl(rep.x, xu.first);
    dl(rep.u, xu.second);
    dl(rep.y, dev_gather_dual(e.d, e.k.y[s]));
    dl(rep.z, dev_gather_dual(e.d, e.k.z[s]));
    SCN_CUDA(cudaStreamSynchronize(e.st));
    rep.wall_ms = now_ms() - t0;
    if (e.timer.on) std::fprintf(stderr, "[scn] finish: %.3f ms (result copies)\n", now_ms() - f0);
  }
};

double resolve_lambda0(Engine& e, const scenopt_solver_config& cfg, int kind, Report& rep) {
  // solvers.hpp:129-138
  if (cfg.lambda0 > 0.0) return cfg.lambda0;
  rep.lipschitz_estimate = e.lipschitz(&rep.lipschitz_calls);
  const bool fixed = kind == 2 || cfg.backtracking_rule == 2;
  return (fixed ? 0.95 : 0.9) / rep.lipschitz_estimate;
}

// Speculative next-iteration sweeps in MINFBE / NAMA (SCENOPT_SPEC_HR=0 disables)
bool spec_on() {
  static const bool on = [] {
    const char* v = std::getenv("SCENOPT_SPEC_HR");
    return !(v && v[0] == '0');
  }();
  return on;
}

// solve_minfbe, solvers.hpp:234-356
Report solve_minfbe(Engine& e, const scenopt_solver_config& cfg, const double* y0dev, const double* weight) {
  validate_config(cfg);
  Report rep;
  Loop lp{e, rep, weight, now_ms()};
  rep.eps = cfg.eps;
  double lambda = resolve_lambda0(e, cfg, 0, rep);
  e.lbfgs_reset(cfg.memory);
  auto& k = e.k;
  int cur = 0;
  e.fb_step(cur, y0dev, lambda, weight, rep.stats);
  bool grad_valid = false, have_pair = false, fresh = true;
  int iter = 0;
  // The previous iterate and gradient of the L-BFGS pair are not copied: the
  // previous iterate is the other state's y (overwritten only by the next
  // certificate, after the L-BFGS kernel read it) and the gradient buffers
  // swap roles on every accepted step.
  double *grad = k.grad, *prev_g = k.prev_g, *prev_y = k.prev_y;
  // Speculative FBE-gradient sweep: after an FB step at the certified point
  // the next iteration's H x0(R) is enqueued before the host has read the
  // step's results (skipped on the device when the step converged), so the
  // host decides while it runs. A rejected step (lambda halving) discards it.
  e.set_gate(cfg, 0);
  bool scalars_fresh = false, hr_ready = false;
  for (;;) {
    if (!scalars_fresh) e.read_scalars();
    scalars_fresh = false;
    const double residual = e.S(cur * sl::kStateStride + sl::RESID);
    if (fresh) {
      lp.push_trace(cur);
      fresh = false;
    }
    if (residual <= cfg.eps) {
      rep.iterations = iter;
      lp.finish(0, cur, residual, lambda);
      return rep;
    }
    if (iter >= cfg.max_iters) {
      rep.iterations = iter;
      lp.finish(1, cur, residual, lambda);
      return rep;
    }
    // fbe_grad (fbe.hpp:89-94): its elementwise part and norms run inside the
    // compact L-BFGS kernel below when that kernel is used (memory <= 6)
    const bool fuse_grad = !grad_valid && cfg.memory <= kLbfgsCompactMaxMem;
    if (!grad_valid) {
      e.mark("idle>grad");
      if (!hr_ready) e.sweep1(false, k.R[cur], nullptr, nullptr, k.HR);
      hr_ready = false;
      e.mark("sweep.HR");
      ++rep.stats.hessian_vec_calls;
      if (!fuse_grad) SCN_CUDA(k_fbe_grad(e.ctx(), cur, k.R[cur], k.HR, grad, e.st));
      e.mark("fbe_grad");
      grad_valid = true;
    }
    // The L-BFGS direction, its image, the certificate and the FB step at the
    // certified point are all enqueued before the simple rule's test
    // (solvers.hpp:279-302) and the certificate's results are read; the host
    // waits only for the published scalars while the FB step runs. When the
    // rule fires, the reference clears the buffer and rebuilds the state
    // before any of that work counts: the speculative results are discarded
    // (a push made by them is undone by the clear; state nxt is rebuilt).
    SCN_CUDA(k_lbfgs(e.ctx(), cfg.memory, cfg.eps_curv, -1.0, have_pair ? 1 : 0, k.y[cur], prev_y, grad, prev_g,
                     grad, k.dir, k.Sb, k.Qb, e.st, k.Mb, fuse_grad ? k.R[cur] : nullptr, k.HR, cur, grad));
    e.mark("lbfgs");
    e.sweep1(false, k.dir, nullptr, nullptr, k.Hd);
    e.mark("sweep.Hd");
    const int nxt = cur ^ 1;
    SCN_CUDA(k_cert_search(e.ctx(), cur, 0, 1, k.y[cur], k.R[cur], k.Hx[cur], k.HR, k.dir, k.Hd, k.y[nxt],
                           e.st));
    e.mark("cert");
    Stats spec;
    const bool spec_hr = spec_on() && iter + 1 < cfg.max_iters;
    if (!spec_hr) e.publish();
    e.fb_step(nxt, k.y[nxt], lambda, weight, spec, spec_hr);  // spec: fb_finish publishes
    e.mark("fb_step");
    if (spec_hr) {  // certificate and FB-step scalars published; the host reads them while HR runs
      e.sweep1_unless_converged(k.R[nxt], k.HR);
      e.wait_published(true);
    } else {
      e.wait_published(false);
    }
    if (cfg.backtracking_rule == 1) {  // simple rule (solvers.hpp:279-302)
      bool halved = false;
      for (;;) {
        const bool trigger = lambda * std::sqrt(e.S(sl::IMG2)) > cfg.eps_bt * std::sqrt(e.S(sl::R2));
        if (!trigger) break;
        lambda = halve_lambda(lambda);
        e.lbfgs_clear();
        have_pair = false;
        e.rescale(cur, lambda, weight, rep.stats);
        e.sweep1(false, k.R[cur], nullptr, nullptr, k.HR);
        ++rep.stats.hessian_vec_calls;
        SCN_CUDA(k_fbe_grad(e.ctx(), cur, k.R[cur], k.HR, grad, e.st));
        e.read_scalars();
        halved = true;
      }
      if (halved) {
        lp.refresh_tail(cur);
        continue;
      }
    }
    have_pair = false;
    ++rep.stats.hessian_vec_calls;
    if (e.S(sl::STALL) != 0.0) {
      rep.stats.prox_calls += 61;
      rep.stats.conj_calls += 61;
      fail(SCENOPT_E_LINE_SEARCH_STALLED, "no step in {2^-nu, nu <= 60} decreases the envelope");
    }
    const uint64_t trials = static_cast<uint64_t>(e.S(sl::KSTAR)) + 1;
    rep.stats.prox_calls += trials;
    rep.stats.conj_calls += trials;
    rep.stats.dual_grad_calls += spec.dual_grad_calls;  // the FB step at the certified point now counts
    rep.stats.prox_calls += spec.prox_calls;
    rep.stats.conj_calls += spec.conj_calls;
    if (cfg.backtracking_rule == 0) {  // original rule (solvers.hpp:329-346)
      if (!spec_hr) e.read_scalars();
      // f_hat(T(w)) > f_hat(w) + lam <Hx(w), R(w)> + (1 - beta)/2 lam |R(w)|^2, evaluated
      // once, by fb_finish on the device (I[REJECT]); the host never re-rounds it
      if (e.I(il::REJECT)) {
        lambda = halve_lambda(lambda);
        e.lbfgs_clear();
        have_pair = false;
        e.rescale(cur, lambda, weight, rep.stats);
        lp.refresh_tail(cur);
        grad_valid = false;
        continue;
      }
    }
    prev_y = k.y[cur];
    std::swap(grad, prev_g);
    grad_valid = false;
    have_pair = true;
    cur = nxt;
    ++iter;
    fresh = true;
    hr_ready = spec_hr && e.I(il::CONV) == 0;  // H x0(R) of the new iterate is in flight
    scalars_fresh = spec_hr;   // and its scalars were read after its FB step
  }
}

// solve_nama, solvers.hpp:362-492
Report solve_nama(Engine& e, const scenopt_solver_config& cfg, const double* y0dev, const double* weight) {
  validate_config(cfg);
  Report rep;
  Loop lp{e, rep, weight, now_ms()};
  rep.eps = cfg.eps;
  double lambda = resolve_lambda0(e, cfg, 1, rep);
  e.lbfgs_reset(cfg.memory);
  auto& k = e.k;
  int cur = 0;
  e.fb_step(cur, y0dev, lambda, weight, rep.stats);
  bool have_pair = false, fresh = true;
  int iter = 0;
  // previous iterate / residual of the L-BFGS pair: the other state's y and R
  // (intact until the next certificate and FB step, which follow the L-BFGS kernel)
  double *prev_y = k.prev_y, *prev_res = k.prev_g;
  // As in MINFBE: after the FB step at the certified point, the next
  // iteration's L-BFGS direction and its two homogeneous images are enqueued
  // before the host reads the step, gated by fb_finish's skip word; a rejected
  // step clears the L-BFGS buffer, which undoes the speculative push.
  e.set_gate(cfg, 1);
  bool scalars_fresh = false, next_ready = false;
  for (;;) {
    if (!scalars_fresh) e.read_scalars();
    scalars_fresh = false;
    const double residual = e.S(cur * sl::kStateStride + sl::RESID);
    if (fresh) {
      lp.push_trace(cur);
      fresh = false;
    }
    if (residual <= cfg.eps) {
      rep.iterations = iter;
      lp.finish(0, cur, residual, lambda);
      return rep;
    }
    if (iter >= cfg.max_iters) {
      rep.iterations = iter;
      lp.finish(1, cur, residual, lambda);
      return rep;
    }
    // the L-BFGS direction, then the two homogeneous images x0(r), x0(d): one
    // 2-RHS sweep when the parallel line search is on (p-NAMA), two sweeps
    // otherwise; the arithmetic is identical either way (solvers.hpp:410-422)
    auto direction_and_images = [&](DualCtx c, int s, int push, const double* py, const double* pr) {
      SCN_CUDA(k_lbfgs(c, cfg.memory, cfg.eps_curv, -1.0, push, k.y[s], py, k.R[s], pr, k.R[s], k.dir, k.Sb,
                       k.Qb, e.st, k.Mb));
      if (cfg.nama_parallel_linesearch)
        e.sweep2(k.R[s], k.dir, k.HR, k.Hd);
      else {
        e.sweep1(false, k.R[s], nullptr, nullptr, k.HR);
        e.sweep1(false, k.dir, nullptr, nullptr, k.Hd);
      }
    };
    if (!next_ready) direction_and_images(e.ctx(), cur, have_pair ? 1 : 0, prev_y, prev_res);
    next_ready = false;
    have_pair = false;
    rep.stats.hessian_vec_calls += 2;
    const int nxt = cur ^ 1;
    SCN_CUDA(k_cert_search(e.ctx(), cur, 1, cfg.nama_update_tlambda ? 1 : 0, k.y[cur], k.R[cur], k.Hx[cur],
                           k.HR, k.dir, k.Hd, k.y[nxt], e.st));
    // the FB step at the certified point runs while the host reads the
    // certificate (discarded when the simple rule halves lambda)
    const bool spec_next = spec_on() && iter + 1 < cfg.max_iters;
    if (!spec_next) e.publish();
    Stats spec;
    e.fb_step(nxt, k.y[nxt], lambda, weight, spec, spec_next);  // spec: fb_finish publishes
    if (spec_next) {
      DualCtx cs = e.ctx();
      cs.skip = k.I + il::CONV;
      Engine::SkipScope g(e.d, k.I + il::CONV);
      direction_and_images(cs, nxt, 1, k.y[cur], k.R[cur]);
      e.wait_published(true);
    } else {
      e.wait_published(false);
    }
    if (cfg.backtracking_rule == 1) {  // simple rule (solvers.hpp:424-438)
      const bool trigger = lambda * std::sqrt(e.S(sl::HR2)) > cfg.eps_bt * std::sqrt(e.S(sl::RR2));
      if (trigger) {
        lambda = halve_lambda(lambda);
        e.lbfgs_clear();
        have_pair = false;
        e.rescale(cur, lambda, weight, rep.stats);
        lp.refresh_tail(cur);
        continue;
      }
    }
    rep.stats.prox_calls += 1;  // shifted anchor (fbe.hpp:192-197)
    rep.stats.conj_calls += 1;
    if (e.S(sl::STALL) != 0.0) {
      rep.stats.prox_calls += 61;
      rep.stats.conj_calls += 61;
      fail(SCENOPT_E_LINE_SEARCH_STALLED, "no step in {2^-nu, nu <= 60} decreases the envelope");
    }
    const uint64_t trials = static_cast<uint64_t>(e.S(sl::KSTAR)) + 1;
    rep.stats.prox_calls += trials;
    rep.stats.conj_calls += trials;
    rep.stats.dual_grad_calls += spec.dual_grad_calls;
    rep.stats.prox_calls += spec.prox_calls;
    rep.stats.conj_calls += spec.conj_calls;
    if (cfg.backtracking_rule == 0) {  // original rule (solvers.hpp:467-483), decided on the device
      if (!spec_next) e.read_scalars();
      if (e.I(il::REJECT)) {
        lambda = halve_lambda(lambda);
        e.lbfgs_clear();
        have_pair = false;
        e.rescale(cur, lambda, weight, rep.stats);
        lp.refresh_tail(cur);
        continue;
      }
    }
    prev_y = k.y[cur];
    prev_res = k.R[cur];
    have_pair = true;
    cur = nxt;
    ++iter;
    fresh = true;
    next_ready = spec_next && e.I(il::CONV) == 0;  // direction and images of the new iterate in flight
    scalars_fresh = spec_next;
  }
}

// solve_gpad, solvers.hpp:498-540
Report solve_gpad(Engine& e, const scenopt_solver_config& cfg, const double* y0dev, const double* weight) {
  validate_config(cfg);
  Report rep;
  Loop lp{e, rep, weight, now_ms()};
  rep.eps = cfg.eps;
  const double lambda = resolve_lambda0(e, cfg, 2, rep);
  auto& k = e.k;
  const size_t D = e.D();
  e.copy(k.yp, y0dev, D);
  double t = 1.0;
  int cur = 0;
  e.fb_step(cur, y0dev, lambda, weight, rep.stats);
  int iter = 0;
  // The next extrapolation and FB step are enqueued before the host reads the
  // current residual (the GPU keeps working during the read); they are
  // discarded when the loop stops, and counted only when it continues.
  for (;;) {
    e.publish();
    const double t_next = 0.5 * (1.0 + std::sqrt(1.0 + 4.0 * t * t));
    const int nxt = cur ^ 1;
    Stats spec;
    const bool more = iter < cfg.max_iters;
    if (more) {
      SCN_CUDA(k_extrapolate(e.ctx(), k.T[cur], k.yp, k.w, (t - 1.0) / t_next, e.st));
      e.fb_step(nxt, k.w, lambda, weight, spec);
    }
    e.wait_published(false);
    const double residual = e.S(cur * sl::kStateStride + sl::RESID);
    lp.push_trace(cur);
    if (residual <= cfg.eps) {
      rep.iterations = iter;
      lp.finish(0, cur, residual, lambda);
      return rep;
    }
    if (!more) {
      rep.iterations = iter;
      lp.finish(1, cur, residual, lambda);
      return rep;
    }
    rep.stats.dual_grad_calls += spec.dual_grad_calls;
    rep.stats.prox_calls += spec.prox_calls;
    rep.stats.conj_calls += spec.conj_calls;
    t = t_next;
    cur = nxt;
    ++iter;
  }
}

// warm_start, solvers.hpp:545-564: GPAD iterations from zero; result in k.tmp2
void warm_start(Engine& e, const scenopt_solver_config& cfg, double lambda, Stats& stats) {
  auto& k = e.k;
  const size_t D = e.D();
  SCN_CUDA(cudaMemsetAsync(k.tmp2, 0, D * sizeof(double), e.st));
  if (cfg.warm_start_iters <= 0) return;
  if (!(lambda > 0.0)) fail(SCENOPT_E_INVALID_PARAMS, "warm_start: lambda must be > 0");
  SCN_CUDA(cudaMemsetAsync(k.w, 0, D * sizeof(double), e.st));
  double t = 1.0;
  for (int it = 0; it < cfg.warm_start_iters; ++it) {
    e.fb_step(0, k.w, lambda, nullptr, stats);
    const double t_next = 0.5 * (1.0 + std::sqrt(1.0 + 4.0 * t * t));
    // w = T + mom (T - y); y = T
    SCN_CUDA(k_extrapolate(e.ctx(), k.T[0], k.tmp2, k.w, (t - 1.0) / t_next, e.st));
    t = t_next;
  }
  SCN_CUDA(cudaStreamSynchronize(e.st));
}

Report dispatch(Engine& e, const scenopt_solver_config& cfg, int kind, const double* y0dev,
                const double* weight) {
  switch (kind) {
    case 0:
      return solve_minfbe(e, cfg, y0dev, weight);
    case 1:
      return solve_nama(e, cfg, y0dev, weight);
    case 2:
      return solve_gpad(e, cfg, y0dev, weight);
  }
  fail(SCENOPT_E_INVALID_PARAMS, "unknown solver kind");
}

// verify_report, solvers.hpp:630-639, on a handle of the problem to verify
void verify(scenopt_dev& h, Report& rep) {
  Engine e(h);
  auto& k = e.k;
  const Layout& L = e.d.lay;
  const size_t D = static_cast<size_t>(L.dual_dim);
  SCN_CUDA(cudaMemcpyAsync(k.x[0], rep.x.data(), rep.x.size() * sizeof(double), cudaMemcpyHostToDevice, e.st));
  if (!rep.u.empty())
    SCN_CUDA(cudaMemcpyAsync(k.u[0], rep.u.data(), rep.u.size() * sizeof(double), cudaMemcpyHostToDevice, e.st));
  SCN_CUDA(cudaMemcpyAsync(k.y[0], rep.y.data(), D * sizeof(double), cudaMemcpyHostToDevice, e.st));
  SCN_CUDA(cudaMemcpyAsync(k.z[0], rep.z.data(), D * sizeof(double), cudaMemcpyHostToDevice, e.st));
  SCN_CUDA(k_apply_H(e.d.hrows, k.x[0], k.u[0], k.Hx[0], e.st));
  SCN_CUDA(k_max_abs_diff(e.ctx(), k.z[0], k.Hx[0], e.st));
  e.read_scalars();
  rep.verify_residual_inf = e.S(sl::RED0);
  SCN_CUDA(k_dist_subdiff(e.ctx(), k.y[0], k.z[0], e.st));
  e.read_scalars();
  rep.verify_subdiff_dist = e.S(sl::RED0);
  const double slop = 1.0 + 1e-9;
  rep.verified = rep.status == 0 && rep.verify_residual_inf <= rep.eps * slop &&
                 rep.verify_subdiff_dist <= rep.lambda_final * rep.eps * slop;
}

}  // namespace

struct scenopt_report {
  Report r;
};
static const Problem* scenopt_problem_ptr(const scenopt_problem* p) { return &p->p; }
static const Factor* scenopt_factor_ptr(const scenopt_factor* f) { return &f->f; }
struct scenopt_lbfgs {
  scenopt_dev* h;                   // owning solver handle, or NULL (standalone buffer)
  std::unique_ptr<DevState> own;    // standalone: bare device context (device 0)
  DevState* dev;
  int n, mem;
  double eps_curv;
  DualCtx c;
  double *Sb, *Qb, *g, *out, *a, *b, *cc, *dd;
  double* Mb;
};

// ------------------------------------------------------------------ C-ABI
extern "C" {

int scenopt_dev_refactor_device(scenopt_dev* h) {
  SCN_GUARD({
    dev_factor_device(*h->d);
    h->w->fhat0_ready = false;  // f_hat(0) and H x(0) depend on the factor
  });
}

int scenopt_dev_refactor_affine(scenopt_dev* h, const scenopt_problem* p) {
  SCN_GUARD({
    dev_refactor_affine(*h->d, p->p);
    h->w->fhat0_ready = false;
  });
}

int scenopt_fhat_value(scenopt_dev* h, const double* y, double* out, int flags) {
  SCN_GUARD({
    Engine e(*h);
    const double* yd = h->in_dual(y, flags, 0);
    e.sweep1(true, yd, e.k.x[1], e.k.u[1], e.k.Hx[1]);
    ++h->stats.dual_grad_calls;
    SCN_CUDA(k_eval_f(e.ctx(), h->d->cost, e.k.x[1], e.k.u[1], 1e-8, e.st));
    SCN_CUDA(k_dot(e.ctx(), e.k.Hx[1], yd, e.st));
    e.read_scalars();
    const double f = e.S(sl::EVALF_INF) != 0.0 ? std::numeric_limits<double>::infinity() : e.S(sl::EVALF);
    *out = -e.S(sl::RED0) - f;  // tree_oracles.hpp:125-129
  });
}

int scenopt_apply_H(scenopt_dev* h, const double* x, const double* u, double* z, int flags) {
  SCN_GUARD({
    Engine e(*h);
    const Layout& L = h->d->lay;
    const double *xd = x, *ud = u;
    if (flags & SCENOPT_HOST_IO) {
      SCN_CUDA(cudaMemcpyAsync(e.k.x[1], x, sizeof(double) * L.nx * L.n, cudaMemcpyHostToDevice, e.st));
      if (L.first_leaf > 0)
        SCN_CUDA(cudaMemcpyAsync(e.k.u[1], u, sizeof(double) * L.nu * L.first_leaf, cudaMemcpyHostToDevice, e.st));
      xd = e.k.x[1];
      ud = e.k.u[1];
    }
    double* zd = (flags & SCENOPT_HOST_IO) ? e.k.tmp : z;
    SCN_CUDA(k_apply_H(h->d->hrows, xd, ud, zd, e.st));
    h->out_copy(z, zd, static_cast<size_t>(L.dual_dim), flags);
    h->sync();
  });
}

int scenopt_prox_g(scenopt_dev* h, const double* v, double gamma_prox, double* out, int flags) {
  SCN_GUARD({
    if (!(gamma_prox > 0.0)) fail(SCENOPT_E_INVALID_PARAMS, "prox_g: gamma_prox must be > 0");
    Engine e(*h);
    const double* vd = h->in_dual(v, flags, 0);
    double* od = (flags & SCENOPT_HOST_IO) ? e.k.tmp : out;
    SCN_CUDA(k_prox(e.ctx(), vd, gamma_prox, od, e.st));
    h->out_copy(out, od, e.D(), flags);
    h->sync();
  });
}

int scenopt_conj_value_g(scenopt_dev* h, const double* w, double* out, int flags) {
  SCN_GUARD({
    Engine e(*h);
    SCN_CUDA(k_conj(e.ctx(), h->in_dual(w, flags, 0), e.st));
    e.read_scalars();
    *out = e.S(sl::RED0);
  });
}

int scenopt_dist_subdiff_inf(scenopt_dev* h, const double* y, const double* z, double* out, int flags) {
  SCN_GUARD({
    Engine e(*h);
    const double* yd = h->in_dual(y, flags, 0);
    const double* zd = h->in_dual(z, flags, 1);
    SCN_CUDA(k_dist_subdiff(e.ctx(), yd, zd, e.st));
    e.read_scalars();
    *out = e.S(sl::RED0);
  });
}

int scenopt_fb_step(scenopt_dev* h, const double* y, double lambda, double* x, double* u, double* Hx,
                    double* z, double* R, double* T, double* scalars, int flags) {
  SCN_GUARD({
    Engine e(*h);
    auto& k = e.k;
    e.fb_step(0, h->in_dual(y, flags, 0), lambda, nullptr, h->stats);
    const Layout& L = h->d->lay;
    DevState& d = *h->d;  // sharded: outputs assembled over the ranks
    const auto xu = dev_gather_primal(d, x ? k.x[0] : nullptr, u ? k.u[0] : nullptr);
    h->out_copy(x, xu.first, static_cast<size_t>(L.nx) * L.n, flags);
    h->out_copy(u, xu.second, static_cast<size_t>(L.nu) * L.first_leaf, flags);
    for (auto [dst, src] : {std::pair<double*, double*>{Hx, k.Hx[0]}, {z, k.z[0]}, {R, k.R[0]}, {T, k.T[0]}})
      if (dst) {
        h->out_copy(dst, dev_gather_dual(d, src), e.D(), flags);
        if (d.sharded()) SCN_CUDA(cudaStreamSynchronize(e.st));  // the gather scratch is reused next
      }
    e.read_scalars();
    if (scalars) {
      scalars[0] = e.S(sl::FHAT);
      scalars[1] = e.S(sl::CONJ);
      scalars[2] = e.S(sl::ZN2);
      scalars[3] = e.S(sl::VALUE);
    }
  });
}

int scenopt_fbe_grad(scenopt_dev* h, const double* R, double lambda, double* grad, int flags) {
  SCN_GUARD({
    Engine e(*h);
    auto& k = e.k;
    const double* Rd = h->in_dual(R, flags, 0);
    e.set_scalar(sl::LAM, lambda);
    e.sweep1(false, Rd, nullptr, nullptr, k.HR);
    ++h->stats.hessian_vec_calls;
    SCN_CUDA(k_fbe_grad(e.ctx(), 0, Rd, k.HR, k.grad, e.st));
    h->out_copy(grad, dev_gather_dual(*h->d, k.grad), e.D(), flags);
    h->sync();
  });
}

int scenopt_linesearch_cert(scenopt_dev* h, const double* y, const double* Hx, double lambda,
                            const double* ss, const double* shift, const double* dir, int ntau,
                            const double* taus, double* deltas, double* cs, double* cfh, double* w,
                            double* Hx_w, double* z, double* R, double* T, int flags) {
  SCN_GUARD({
    if (!(lambda > 0.0)) fail(SCENOPT_E_INVALID_PARAMS, "linesearch_cert: lambda must be > 0");
    if (ntau < 1 || ntau > 16) fail(SCENOPT_E_INVALID_PARAMS, "linesearch_cert: 1..16 taus");
    if (h->d->sharded()) fail(SCENOPT_E_INVALID_PARAMS, "linesearch_cert: explicit trials need an unsharded handle");
    Engine e(*h);
    auto& k = e.k;
    const size_t D = e.D();
    const bool host = (flags & SCENOPT_HOST_IO) != 0;
    auto in = [&](const double* src, double* dst) {
      SCN_CUDA(cudaMemcpyAsync(dst, src, D * sizeof(double), host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice,
                               e.st));
    };
    in(y, k.y[0]);
    in(Hx, k.Hx[0]);
    in(dir, k.dir);
    e.set_scalar(sl::LAM, lambda);
    e.set_scalar(sl::FHAT, ss[0]);
    e.set_scalar(sl::CONJ, ss[1]);
    e.set_scalar(sl::ZN2, ss[2]);
    e.set_scalar(sl::VALUE, ss[3]);
    e.sweep1(false, k.dir, nullptr, nullptr, k.Hd);
    if (shift) {  // the kernel's shift is -lambda R: pass R = -shift / lambda
      in(shift, k.tmp);
      SCN_CUDA(k_scale(e.ctx(), static_cast<int>(D), -1.0 / lambda, k.tmp, 0.0, nullptr, k.R[0], e.st));
      e.sweep1(false, k.R[0], nullptr, nullptr, k.HR);
    }
    double* dev_deltas = k.small;
    double* dev_cfh = k.small + 16;
    SCN_CUDA(k_cert_eval(e.ctx(), 0, shift ? 1 : 0, k.y[0], k.R[0], k.Hx[0], k.HR, k.dir, k.Hd, ntau, taus,
                         dev_deltas, dev_cfh, k.z[1], k.Hx[1], k.T[1], k.R[1], k.grad, e.st));
    SCN_CUDA(cudaStreamSynchronize(e.st));
    std::vector<double> hd(static_cast<size_t>(ntau)), hc(static_cast<size_t>(ntau));
    SCN_CUDA(cudaMemcpy(hd.data(), dev_deltas, ntau * sizeof(double), cudaMemcpyDeviceToHost));
    SCN_CUDA(cudaMemcpy(hc.data(), dev_cfh, ntau * sizeof(double), cudaMemcpyDeviceToHost));
    std::copy(hd.begin(), hd.end(), deltas);
    if (cfh) std::copy(hc.begin(), hc.end(), cfh);
    e.read_scalars();
    if (cs) {
      cs[0] = e.S(sl::ALPHA1);
      cs[1] = e.S(sl::ALPHA2);
      cs[2] = e.S(sl::CONJ_A);
      cs[3] = e.S(sl::ZN2_A);
      cs[4] = e.S(sl::VALUE_A);
      cs[5] = e.S(sl::FHAT_A);
    }
    h->out_copy(w, k.z[1], D, flags);
    h->out_copy(Hx_w, k.Hx[1], D, flags);
    h->out_copy(z, k.T[1], D, flags);
    h->out_copy(R, k.R[1], D, flags);
    h->out_copy(T, k.grad, D, flags);
    h->sync();
  });
}

int scenopt_estimate_lipschitz(scenopt_dev* h, uint64_t* calls, double* out) {
  SCN_GUARD({
    Engine e(*h);
    *out = e.lipschitz(calls);
  });
}

int scenopt_estimate_lipschitz_ex(scenopt_dev* h, double rel_tol, int max_rounds, uint64_t* calls, double* out) {
  SCN_GUARD({
    Engine e(*h);
    *out = e.lipschitz(calls, rel_tol, max_rounds);
  });
}

int scenopt_dev_solve(scenopt_dev* h, const scenopt_solver_config* cfg, int kind, const double* y0,
                      const double* weight, scenopt_report** out) {
  SCN_GUARD({
    validate_for(*cfg, *h->d);
    Engine e(*h);
    const size_t D = e.D();
    if (y0)
      SCN_CUDA(cudaMemcpyAsync(e.k.tmp2, y0, D * sizeof(double), cudaMemcpyHostToDevice, e.st));
    else
      SCN_CUDA(cudaMemsetAsync(e.k.tmp2, 0, D * sizeof(double), e.st));
    const double* wd = nullptr;
    if (weight) {
      SCN_CUDA(cudaMemcpyAsync(e.k.weight, weight, D * sizeof(double), cudaMemcpyHostToDevice, e.st));
      wd = e.k.weight;
    }
    auto r = std::make_unique<scenopt_report>();
    r->r = dispatch(e, *cfg, kind, e.k.tmp2, wd);
    *out = r.release();
  });
}

int scenopt_warm_start(scenopt_dev* h, const scenopt_solver_config* cfg, double lambda, double* y_out,
                       uint64_t* dual_grad_calls) {
  SCN_GUARD({
    Engine e(*h);
    Stats st;
    warm_start(e, *cfg, lambda, st);
    // stream-ordered: warm_start may return with its zero fill still queued (no iterations)
    SCN_CUDA(cudaMemcpyAsync(y_out, e.k.tmp2, e.D() * sizeof(double), cudaMemcpyDeviceToHost, e.st));
    SCN_CUDA(cudaStreamSynchronize(e.st));
    if (dual_grad_calls) *dual_grad_calls = st.dual_grad_calls;
  });
}

int scenopt_report_summary_get(const scenopt_report* rr, scenopt_report_summary* s) {
  SCN_GUARD({
    const Report& r = rr->r;
    s->status = r.status;
    s->iterations = r.iterations;
    s->verified = r.verified ? 1 : 0;
    s->trace_len = static_cast<int32_t>(r.residual_trace.size());
    s->dual_grad_calls = r.stats.dual_grad_calls;
    s->hessian_vec_calls = r.stats.hessian_vec_calls;
    s->prox_calls = r.stats.prox_calls;
    s->conj_calls = r.stats.conj_calls;
    s->lipschitz_calls = r.lipschitz_calls;
    s->lipschitz_estimate = r.lipschitz_estimate;
    s->lambda_final = r.lambda_final;
    s->eps = r.eps;
    s->residual_inf = r.residual_inf;
    s->wall_ms = r.wall_ms;
    s->verify_residual_inf = r.verify_residual_inf;
    s->verify_subdiff_dist = r.verify_subdiff_dist;
  });
}

int scenopt_report_arrays(const scenopt_report* rr, double* x, double* u, double* y, double* z, double* rt,
                          double* ft) {
  SCN_GUARD({
    const Report& r = rr->r;
    auto cp = [](const auto& v, double* dst) {
      if (dst && !v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(double));
    };
    cp(r.x, x);
    cp(r.u, u);
    cp(r.y, y);
    cp(r.z, z);
    cp(r.residual_trace, rt);
    cp(r.fbe_trace, ft);
  });
}

void scenopt_report_destroy(scenopt_report* r) { delete r; }  // result arrays go back to the pool

// ------------------------------------------------------------------ L-BFGS handle (lbfgs.hpp)
int scenopt_lbfgs_create(scenopt_dev* h, int memory, double eps_curv, scenopt_lbfgs** out) {
  SCN_GUARD({
    if (memory < 1) fail(SCENOPT_E_INVALID_PARAMS, "LbfgsBuffer: memory must be >= 1");
    if (memory > 48) fail(SCENOPT_E_INVALID_PARAMS, "LbfgsBuffer: memory must be <= 48 on the device");
    if (!(eps_curv > 0.0)) fail(SCENOPT_E_INVALID_PARAMS, "LbfgsBuffer: eps_curv must be > 0");
    auto b = std::make_unique<scenopt_lbfgs>();
    b->h = h;
    b->n = 0;
    b->mem = memory;
    b->eps_curv = eps_curv;
    if (h) {
      b->dev = h->d.get();
    } else {  // LbfgsBuffer(memory, eps_curv) has no problem attached: own a bare context
      b->own = dev_create_bare(0);
      b->dev = b->own.get();
    }
    DevState& d = *b->dev;
    SCN_CUDA(cudaSetDevice(d.device));
    if (h) {
      b->c = h->w->ctx(d);
    } else {
      b->c = DualCtx{};
      b->c.nblk = std::min(d.sm_count, dual_max_blocks());
    }
    b->c.S = d.alloc<double>(sl::kScalars);
    b->c.I = d.alloc<int>(il::kInts);
    b->c.part = d.alloc<double>(static_cast<size_t>(2) * 64 * b->c.nblk);
    b->c.bar = d.alloc<unsigned>(4);
    SCN_CUDA(cudaMemset(b->c.S, 0, sl::kScalars * sizeof(double)));
    SCN_CUDA(cudaMemset(b->c.bar, 0, 4 * sizeof(unsigned)));
    std::vector<int> ints(il::kInts, 0);
    for (int j = 0; j <= memory; ++j) ints[il::LB_ORDER + j] = j;
    SCN_CUDA(cudaMemcpy(b->c.I, ints.data(), ints.size() * sizeof(int), cudaMemcpyHostToDevice));
    const double one = 1.0;
    SCN_CUDA(cudaMemcpy(b->c.S + sl::GAMMA0, &one, sizeof(double), cudaMemcpyHostToDevice));
    b->Sb = b->Qb = b->g = b->out = b->a = b->b = b->cc = b->dd = b->Mb = nullptr;
    *out = b.release();
  });
}

namespace {
void lb_ensure(scenopt_lbfgs* b, int n) {
  if (b->n == n) return;
  if (b->n != 0) fail(SCENOPT_E_DIMENSION_MISMATCH, "LbfgsBuffer: vector length changed");
  DevState& d = *b->dev;
  b->n = n;
  b->c.D = n;
  b->Sb = d.alloc<double>(static_cast<size_t>(b->mem + 1) * n);
  b->Qb = d.alloc<double>(static_cast<size_t>(b->mem + 1) * n);
  b->Mb = d.alloc<double>(2 * 64 * 64);
  for (double** p : {&b->g, &b->out, &b->a, &b->b, &b->cc, &b->dd}) *p = d.alloc<double>(n);
  SCN_CUDA(cudaMemset(b->b, 0, n * sizeof(double)));
  SCN_CUDA(cudaMemset(b->dd, 0, n * sizeof(double)));
}
}  // namespace

int scenopt_lbfgs_push(scenopt_lbfgs* b, int n, const double* step, const double* change, double scale_ref) {
  try {
    SCN_CUDA(cudaSetDevice(b->dev->device));
    lb_ensure(b, n);
    cudaStream_t st = b->dev->stream;
    // push(step, change, scale_ref) (lbfgs.hpp:33-44): s = step - 0,
    // q = change - 0 with an explicit scale_ref for the curvature gate.
    SCN_CUDA(cudaMemcpyAsync(b->a, step, n * sizeof(double), cudaMemcpyHostToDevice, st));
    SCN_CUDA(cudaMemcpyAsync(b->cc, change, n * sizeof(double), cudaMemcpyHostToDevice, st));
    SCN_CUDA(k_lbfgs(b->c, b->mem, b->eps_curv, scale_ref, 1, b->a, b->b, b->cc, b->dd, b->a, b->out, b->Sb,
                     b->Qb, st, b->Mb));
    int pushed = 0;
    SCN_CUDA(cudaMemcpyAsync(&pushed, b->c.I + il::LB_PUSHED, sizeof(int), cudaMemcpyDeviceToHost, st));
    SCN_CUDA(cudaStreamSynchronize(st));
    return pushed;
  } catch (const Error& e) {
    g_last_error = e.what();
    return e.code;
  }
}

int scenopt_lbfgs_apply(scenopt_lbfgs* b, int n, const double* grad, double* out) {
  SCN_GUARD({
    SCN_CUDA(cudaSetDevice(b->dev->device));
    lb_ensure(b, n);
    cudaStream_t st = b->dev->stream;
    SCN_CUDA(cudaMemcpyAsync(b->g, grad, n * sizeof(double), cudaMemcpyHostToDevice, st));
    SCN_CUDA(k_lbfgs(b->c, b->mem, b->eps_curv, -1.0, 0, nullptr, nullptr, nullptr, nullptr, b->g, b->out, b->Sb, b->Qb, st, b->Mb));
    SCN_CUDA(cudaMemcpyAsync(out, b->out, n * sizeof(double), cudaMemcpyDeviceToHost, st));
    SCN_CUDA(cudaStreamSynchronize(st));
  });
}

int scenopt_lbfgs_clear(scenopt_lbfgs* b) {
  SCN_GUARD({
    const int zero = 0;
    const double one = 1.0;
    SCN_CUDA(cudaSetDevice(b->dev->device));
    cudaStream_t st = b->dev->stream;  // ordered with the buffer's kernels
    SCN_CUDA(cudaMemcpyAsync(b->c.I + il::LB_COUNT, &zero, sizeof(int), cudaMemcpyHostToDevice, st));
    SCN_CUDA(cudaMemcpyAsync(b->c.S + sl::GAMMA0, &one, sizeof(double), cudaMemcpyHostToDevice, st));
    SCN_CUDA(cudaStreamSynchronize(st));  // the sources are on this frame
  });
}

int scenopt_lbfgs_size(const scenopt_lbfgs* b) {
  int c = 0;
  if (cudaSetDevice(b->dev->device) != cudaSuccess) return -20;
  if (cudaMemcpy(&c, b->c.I + il::LB_COUNT, sizeof(int), cudaMemcpyDeviceToHost) != cudaSuccess) return -20;
  return c;
}

double scenopt_lbfgs_gamma0(const scenopt_lbfgs* b) {
  double g = 0.0;
  cudaSetDevice(b->dev->device);
  cudaMemcpy(&g, b->c.S + sl::GAMMA0, sizeof(double), cudaMemcpyDeviceToHost);
  return g;
}

void scenopt_lbfgs_destroy(scenopt_lbfgs* b) { delete b; }

// ------------------------------------------------------------------ solve() driver
int scenopt_solve(const scenopt_problem* p, const scenopt_solver_config* cfg, int kind,
                  const scenopt_factor* shared, int device, scenopt_report** out) {
  SCN_GUARD({
    validate_config(*cfg);
    if (kind < 0 || kind > 2) fail(SCENOPT_E_INVALID_PARAMS, "unknown solver kind");
    const double t0 = now_ms();
    const Problem& prob = *scenopt_problem_ptr(p);
    auto run = [&](scenopt_dev& h, const double* wdev) {
      Engine e(h);
      double lhat = 0.0;
      uint64_t lhat_calls = 0;
      scenopt_solver_config run_cfg = *cfg;
      if (!(cfg->lambda0 > 0.0)) {  // solvers.hpp:673-679
        lhat = e.lipschitz(&lhat_calls);
        const bool fixed = kind == 2 || cfg->backtracking_rule == 2;
        run_cfg.lambda0 = (fixed ? 0.95 : 0.9) / lhat;
      }
      Stats warm;
      SCN_CUDA(cudaMemsetAsync(e.k.tmp2, 0, e.D() * sizeof(double), e.st));
      if (cfg->warm_start) {
        const double lam_ws = cfg->lambda0 > 0.0 ? cfg->lambda0 : 0.95 / lhat;
        warm_start(e, *cfg, lam_ws, warm);
      }
      Report r = dispatch(e, run_cfg, kind, e.k.tmp2, wdev);
      r.stats.dual_grad_calls += warm.dual_grad_calls;
      r.stats.hessian_vec_calls += warm.hessian_vec_calls;
      r.stats.prox_calls += warm.prox_calls;
      r.stats.conj_calls += warm.conj_calls;
      r.lipschitz_estimate = lhat;
      r.lipschitz_calls = lhat_calls;
      return r;
    };
    auto rep = std::make_unique<scenopt_report>();
    // Without a shared factor the instance is factored on the device (K9,
    // DESIGN.md §3.3) straight into the sweep layout: at C3 0.4 s for the
    // handle against 0.75 s of host factor plus 0.6-0.8 s of packing and
    // upload, all inside wall_ms as in the reference (solvers.hpp:646-717).
    if (!cfg->precondition) {
      const Factor* f = shared ? scenopt_factor_ptr(shared) : nullptr;
      scenopt_dev h;
      h.d = f ? dev_create(prob, f, device) : dev_create_device_factor(prob, device);
      h.init_solver_buffers();
      const double t1 = now_ms();
      rep->r = run(h, nullptr);
      const double t2 = now_ms();
      verify(h, rep->r);
      if (std::getenv("SCN_SOLVE_TIMING"))
        std::fprintf(stderr, "[scn] solve(): handle %.1f ms, lipschitz + warm start + solver %.1f ms, verify %.1f ms\n",
                     t1 - t0, t2 - t1, now_ms() - t2);
    } else {
      const Problem scaled = precondition(prob);
      const std::vector<double> roots = probability_roots(prob);
      std::vector<double> weight(roots.size());
      for (size_t i = 0; i < roots.size(); ++i) weight[i] = 1.0 / roots[i];
      {
        scenopt_dev h;
        h.d = dev_create_device_factor(scaled, device);
        h.init_solver_buffers();
        SCN_CUDA(cudaMemcpy(h.w->weight, weight.data(), weight.size() * sizeof(double), cudaMemcpyHostToDevice));
        rep->r = run(h, h.w->weight);
      }
      for (size_t i = 0; i < rep->r.y.size(); ++i) rep->r.y[i] = rep->r.y[i] * roots[i];
      for (size_t i = 0; i < rep->r.z.size(); ++i) rep->r.z[i] = rep->r.z[i] * weight[i];
      scenopt_dev ho;  // factor-less handle of the original problem for verification
      ho.d = dev_create(prob, nullptr, device);
      ho.init_solver_buffers();
      verify(ho, rep->r);
    }
    rep->r.wall_ms = now_ms() - t0;
    *out = rep.release();
  });
}

int scenopt_verify_report(const scenopt_problem* p, scenopt_report* r, const double* z_override, int device) {
  SCN_GUARD({
    const Problem& prob = *scenopt_problem_ptr(p);
    if (z_override) std::copy(z_override, z_override + prob.dual_dim, r->r.z.begin());
    scenopt_dev h;
    h.d = dev_create(prob, nullptr, device);
    h.init_solver_buffers();
    verify(h, r->r);
  });
}

}  // extern "C"
