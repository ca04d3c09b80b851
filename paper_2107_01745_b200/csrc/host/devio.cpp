// SPDX-License-Identifier: MIT
// Host/device I/O helpers of the scenopt_dev handle.
#include <algorithm>
#include <cstdint>

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
  // device addresses of pinned host outputs, resolved once per call (nullptr:
  // pageable); zero copy needs every requested output pinned and 16-byte
  // aligned (the forward pass writes whole rows with 16-byte stores)
  double* mx[kMaxRhs] = {nullptr, nullptr};
  double* mu[kMaxRhs] = {nullptr, nullptr};
  auto usable = [](double* m) { return m != nullptr && (reinterpret_cast<uintptr_t>(m) & 15u) == 0; };
  bool zero_copy = host && (x || u) && !d->sharded();
  for (int r = 0; zero_copy && r < nrhs; ++r) {
    if (x && x[r]) zero_copy = usable(mx[r] = mapped(x[r]));
    if (zero_copy && u && u[r]) zero_copy = usable(mu[r] = mapped(u[r]));
  }
  const bool mapped_y = zero_copy;
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
  // Mapped (pinned) host outputs: the forward pass writes x / u to the
  // caller's buffers over PCIe as it computes them, overlapping the transfer
  // with the sweep; pageable buffers take the copy after the sweep.
  if (zero_copy) {
    struct Reset {
      DevState& d;
      ~Reset() {
        for (int r = 0; r < kMaxRhs; ++r) d.out_hx[r] = d.out_hu[r] = nullptr;
      }
    } reset{*d};
    for (int r = 0; r < nrhs; ++r) {
      d->out_hx[r] = mx[r];
      d->out_hu[r] = mu[r];
    }
    dev_sweep(*d, nrhs, affine, yd, xd, ud, hd);
    for (int r = 0; r < nrhs; ++r)
      if (Hx && Hx[r]) out_copy(Hx[r], d->hs[r], static_cast<size_t>(L.dual_dim), flags);
    sync();
    return;
  }
  dev_sweep(*d, nrhs, affine, yd, xd, ud, hd);
  if (host) {
    // sharded: host outputs are assembled over the ranks (device outputs stay rank-local)
    for (int r = 0; r < nrhs; ++r) {
      const auto xu = dev_gather_primal(*d, (x && x[r]) ? d->xs[r] : nullptr, (u && u[r]) ? d->us[r] : nullptr);
      if (x && x[r]) out_copy(x[r], xu.first, static_cast<size_t>(L.nx) * L.n, flags);
      if (u && u[r]) out_copy(u[r], xu.second, static_cast<size_t>(L.nu) * L.first_leaf, flags);
      if (Hx && Hx[r]) out_copy(Hx[r], dev_gather_dual(*d, d->hs[r]), static_cast<size_t>(L.dual_dim), flags);
      if (d->sharded()) sync();  // the gather scratch is reused by the next right-hand side
    }
  }
  if (sync_after || host) sync();
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
