// SPDX-License-Identifier: MIT
// Host/device I/O helpers of the scenopt_dev handle.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "capi_internal.hpp"

using namespace scn;

void scenopt_dev::sync() { SCN_CUDA(cudaStreamSynchronize(d->stream)); }

const double* scenopt_dev::in_dual(const double* src, int flags, int slot) {
  if (!(flags & SCENOPT_HOST_IO)) return src;
  if (!src) fail(SCENOPT_E_INVALID_PARAMS, "null input vector");
  double* dst = d->ys[slot];
  SCN_CUDA(cudaMemcpyAsync(dst, src, sizeof(double) * static_cast<size_t>(d->lay.dual_dim),
                           cudaMemcpyHostToDevice, d->stream));
  return dst;
}

void scenopt_dev::out_copy(double* dst, const double* dev_src, size_t count, int flags) {
  if (!dst || dst == dev_src) return;
  SCN_CUDA(cudaMemcpyAsync(dst, dev_src, sizeof(double) * count,
                           (flags & SCENOPT_HOST_IO) ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice,
                           d->stream));
}

static int env_kb(const char* name, int dflt);

void scenopt_dev::sweep(int nrhs, bool affine, const double* const* y, double* const* x,
                        double* const* u, double* const* Hx, int flags, bool sync_after) {
  SCN_CUDA(cudaSetDevice(d->device));
  if (nrhs < 1 || nrhs > kMaxRhs) fail(SCENOPT_E_INVALID_PARAMS, "sweep: nrhs must be 1 or 2");
  const Layout& L = d->lay;
  const double* yd[kMaxRhs] = {nullptr, nullptr};
  double* xd[kMaxRhs] = {nullptr, nullptr};
  double* ud[kMaxRhs] = {nullptr, nullptr};
  double* hd[kMaxRhs] = {nullptr, nullptr};
  const bool host = (flags & SCENOPT_HOST_IO) != 0;
  static const bool mapped_y_on = [] {
    const char* v = std::getenv("SCENOPT_MAPPED_Y");
    return !(v && std::string(v) == "0");
  }();
  const bool mapped_y = host && (x || u) && mapped_y_on && !d->sharded() && zero_copy_ok(nrhs, x, u);
  for (int r = 0; r < nrhs; ++r) {
    // a pinned dual input can be read in place by the backward's staging copies
    double* m = mapped_y && y[r] ? mapped(const_cast<double*>(y[r])) : nullptr;
    yd[r] = m ? m : in_dual(y[r], flags, r);
    if (!host) {
      xd[r] = x ? x[r] : nullptr;
      ud[r] = u ? u[r] : nullptr;
      hd[r] = Hx ? Hx[r] : nullptr;
    }
  }
  const bool want_primal = (x != nullptr) || (u != nullptr);
  if (host && want_primal && overlap_ready()) {
    // Host copies of x / u overlap the sweep: the forward pass retires its
    // stages in order and counts the finished nodes per stage on the device;
    // a copy stream waits on each stage's counter and moves that stage's
    // contiguous x / u rows while later stages are still being computed.
    DevState::Overlap& o = d->overlap;
    for (int t = 0; t <= L.N; ++t) o.expected[t] += d->stage_ctas[t];
    const bool dbg = std::getenv("SCN_OVERLAP_DEBUG") != nullptr;
    std::vector<cudaEvent_t> evs;
    auto mark = [&](cudaStream_t st) {
      if (!dbg) return;
      cudaEvent_t e;
      cudaEventCreate(&e);
      cudaEventRecord(e, st);
      evs.push_back(e);
    };
    mark(d->stream);
    dev_sweep(*d, nrhs, affine, yd, xd, ud, hd, false, o.stage_done);
    mark(d->stream);
    // stages are copied in groups of >= SCENOPT_OVERLAP_KB (default 1536 KB):
    // one wait (on the group's last stage) and one contiguous copy per array
    const size_t group_bytes = static_cast<size_t>(std::max(1, env_kb("SCENOPT_OVERLAP_KB", 1536))) * 1024;
    int t0 = 0;
    size_t acc = 0;
    for (int t = 0; t <= L.N; ++t) {
      acc += sizeof(double) * nrhs * static_cast<size_t>(L.stage_offsets[t + 1] - L.stage_offsets[t]) * (L.nx + L.nu);
      if (acc < group_bytes && t < L.N) continue;
      for (int s = t0; s <= t; ++s) o.wait(o.copy_stream, o.stage_done + s, o.expected[s]);
      mark(o.copy_stream);
      const int lo = L.stage_offsets[t0], cnt = L.stage_offsets[t + 1] - lo;
      const int ucnt = std::min(L.stage_offsets[t + 1], L.first_leaf) - lo;  // leaves carry no input
      for (int r = 0; r < nrhs; ++r) {
        if (x && x[r])
          SCN_CUDA(cudaMemcpyAsync(x[r] + static_cast<size_t>(lo) * L.nx, d->xs[r] + static_cast<size_t>(lo) * L.nx,
                                   sizeof(double) * cnt * L.nx, cudaMemcpyDeviceToHost, o.copy_stream));
        if (u && u[r] && ucnt > 0)
          SCN_CUDA(cudaMemcpyAsync(u[r] + static_cast<size_t>(lo) * L.nu, d->us[r] + static_cast<size_t>(lo) * L.nu,
                                   sizeof(double) * ucnt * L.nu, cudaMemcpyDeviceToHost, o.copy_stream));
      }
      t0 = t + 1;
      acc = 0;
    }
    for (int r = 0; r < nrhs; ++r)
      if (Hx && Hx[r]) out_copy(Hx[r], d->hs[r], static_cast<size_t>(L.dual_dim), flags);
    mark(o.copy_stream);
    SCN_CUDA(cudaStreamSynchronize(o.copy_stream));
    sync();
    if (dbg) {
      std::string line = "[overlap] us from sweep start: kernel end";
      for (size_t i = 1; i < evs.size(); ++i) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, evs[0], evs[i]);
        line += (i == 1 ? " " : (i + 1 == evs.size() ? " | copies done " : " | wait ")) + std::to_string(ms * 1e3);
      }
      std::fprintf(stderr, "%s\n", line.c_str());
      for (auto e : evs) cudaEventDestroy(e);
    }
    return;
  }
  // Mapped (pinned) host outputs: the forward pass writes x / u to the
  // caller's buffers over PCIe as it computes them, overlapping the transfer
  // with the sweep; pageable buffers take the copy after the sweep.
  if (host && want_primal && zero_copy_ok(nrhs, x, u)) {
    struct Reset {
      DevState& d;
      ~Reset() {
        for (int r = 0; r < kMaxRhs; ++r) d.out_hx[r] = d.out_hu[r] = nullptr;
      }
    } reset{*d};
    for (int r = 0; r < nrhs; ++r) {
      d->out_hx[r] = (x && x[r]) ? mapped(x[r]) : nullptr;
      d->out_hu[r] = (u && u[r]) ? mapped(u[r]) : nullptr;
    }
    dev_sweep(*d, nrhs, affine, yd, xd, ud, hd, true);
    for (int r = 0; r < nrhs; ++r)
      if (Hx && Hx[r]) out_copy(Hx[r], d->hs[r], static_cast<size_t>(L.dual_dim), flags);
    sync();
    return;
  }
  dev_sweep(*d, nrhs, affine, yd, xd, ud, hd, want_primal);
  if (host) {
    for (int r = 0; r < nrhs; ++r) {
      if (x && x[r]) out_copy(x[r], d->xs[r], static_cast<size_t>(L.nx) * L.n, flags);
      if (u && u[r]) out_copy(u[r], d->us[r], static_cast<size_t>(L.nu) * L.first_leaf, flags);
      if (Hx && Hx[r]) out_copy(Hx[r], d->hs[r], static_cast<size_t>(L.dual_dim), flags);
    }
  }
  if (sync_after || host) sync();
}

static int env_kb(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v && *v ? std::atoi(v) : dflt;
}

// Device-visible address of a pinned host buffer (UVA: registered and
// cudaHostAlloc memory is mapped), or nullptr for pageable memory.
double* scenopt_dev::mapped(double* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return a.type == cudaMemoryTypeHost ? static_cast<double*>(a.devicePointer) : nullptr;
}

bool scenopt_dev::zero_copy_ok(int nrhs, double* const* x, double* const* u) {
  static const bool off = [] {
    const char* v = std::getenv("SCENOPT_ZERO_COPY");
    return v && std::string(v) == "0";
  }();
  if (off || d->sharded()) return false;
  for (int r = 0; r < nrhs; ++r) {
    if (x && x[r] && !mapped(x[r])) return false;
    if (u && u[r] && !mapped(u[r])) return false;
  }
  return true;
}

bool scenopt_dev::overlap_ready() {
  DevState::Overlap& o = d->overlap;
  if (o.state == 0) {
    o.state = -1;
    // opt-in (SCENOPT_OVERLAP=1): measured on B200 at C3, the stage-grouped
    // copies move ~30 GB/s against ~53 GB/s for one copy after the sweep, so
    // the overlap does not pay at these sizes (446 vs 447 us per call)
    const char* on = std::getenv("SCENOPT_OVERLAP");
    if (d->sharded() || !on || std::string(on) == "0" || std::getenv("SCENOPT_NO_OVERLAP")) return false;
    if (!o.init(*d)) return false;
    o.state = 1;
  }
  return o.state == 1;
}
