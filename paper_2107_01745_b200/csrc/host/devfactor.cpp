// SPDX-License-Identifier: MIT
// Device factorization (K9, cuda/factor.cu) of a handle's own problem data,
// written into its packed sweep layout; and the device factor exported in
// the FactorCache layout (riccati.hpp:38-63) for parity checks.
#include <algorithm>
#include <string>

#include "device.hpp"
#include "../cuda/factor.hpp"

namespace scn {



namespace {
template <class T>
T* up(DevState& d, const std::vector<T>& h) {
  T* p = d.alloc<T>(std::max<size_t>(h.size(), 1));
  if (!h.empty()) SCN_CUDA(cudaMemcpy(p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
  return p;
}
}  // namespace

std::unique_ptr<DevState> dev_create_device_factor(const Problem& p, int device, const ShardSpec* shard) {
  const Factor shape = factor_shape(p, true);  // layout only: the GPU writes the factor blocks
  auto d = dev_create(p, &shape, device, shard);
  dev_factor_device(*d);
  return d;
}

namespace {
// launch parameters with the index arrays on the device (built once per handle)
FactorParams& params(DevState& d) {
  if (d.fp_ready) return d.fp;
  const Layout& L = d.lay;
  const int nx = L.nx, nu = L.nu, n = L.n;
  FactorParams& F = d.fp;
  F = FactorParams{};
  F.nx = nx;
  F.nu = nu;
  F.n = n;
  F.first_leaf = L.first_leaf;
  F.nxp = d.nxp;
  F.child_begin = up(d, L.child_begin);
  F.child_count = up(d, L.child_count);
  F.dual_offset = up(d, L.dual_offset);
  F.stage_rows = up(d, L.stage_rows);
  F.ancestor = up(d, L.ancestor);
  F.flat_off = d.flat_top ? up(d, d.h_flat_off) : nullptr;
  F.aff_fw = d.aff_fw;
  F.aff_fwh = d.aff_fwh;
  F.mmax = d.max_m;
  F.root_state = d.root_state;
  F.prob = d.cost.prob;
  F.cost_node = d.cost.node;
  F.cost_leaf = d.cost.leaf;
  F.cost_slot = d.cost.slot;
  F.leaf_slot = d.cost.lslot;
  F.hcoef = d.hrows.coef;
  F.bw_off = up(d, d.h_bw_off);
  F.bw_j = up(d, d.h_bw_j);
  F.k_off = up(d, d.h_k_off);
  F.bw_blk = d.bw_blk;
  F.fw_blk = d.fw_blk;
  F.aff_bw = d.aff_bw;
  if (!d.vq) d.vq = d.alloc<double>(static_cast<size_t>(n) * nx * nx);
  F.vq = d.vq;
  F.lchol = d.alloc<double>(static_cast<size_t>(std::max(L.first_leaf, 1)) * nu * nu);
  F.bad = d.alloc<int>(1);
  d.fp_ready = true;
  return F;
}
// the nodes of stage t this handle holds: all, or a sharded rank's own range
// below the shard stage (the replicated top above it)
std::pair<int, int> held_range(const DevState& d, int t) {
  if (d.sharded()) return d.own_range[t];
  return {d.lay.stage_offsets[t], d.lay.stage_offsets[t + 1]};
}
// flattened forward top (device.cpp, kFlatTop): stages 1 .. cut-1 in order,
// each reads its parents' maps
void run_flat(DevState& d, FactorParams& F, int consts_only) {
  if (!d.flat_top) return;
  F.flat_consts_only = consts_only;
  for (int t = 1; t < d.cut_stage; ++t) {
    const auto r = held_range(d, t);
    F.stage_first = r.first;
    F.stage_count = r.second - r.first;
    if (F.stage_count > 0) SCN_CUDA(factor_run_flat(F, std::min(d.sm_count * 2, F.stage_count), d.stream));
  }
}
}  // namespace

void dev_factor_device(DevState& d) {
  if (!d.has_factor) fail(SCENOPT_E_CACHE_MISMATCH, "device factor: handle has no sweep layout");
  if (d.sharded() && d.world > 1 && !d.comm)
    fail(SCENOPT_E_INVALID_PARAMS, "device factor: a sharded handle needs its communicator");
  const Layout& L = d.lay;
  const int nx = L.nx, nu = L.nu, n = L.n;
  SCN_CUDA(cudaSetDevice(d.device));
  FactorParams& F = params(d);
  int max_rows = 1;
  for (int c = 1; c < n; ++c) max_rows = std::max(max_rows, L.stage_rows[c]);
  const int64_t ws = factor_workspace_doubles(nx, nu, max_rows);
  F.ws_doubles = ws;
  const int grid_max = d.sm_count * 2;
  const size_t smem_bytes = static_cast<size_t>(ws) * sizeof(double);
  cudaDeviceProp prop{};
  SCN_CUDA(cudaGetDeviceProperties(&prop, d.device));
  size_t smem = 0;
  if (smem_bytes <= static_cast<size_t>(prop.sharedMemPerBlockOptin)) {
    smem = smem_bytes;
    F.ws_global = nullptr;
  } else if (!F.ws_global) {
    F.ws_global = d.alloc<double>(static_cast<size_t>(grid_max) * ws);
  }
  SCN_CUDA(cudaMemsetAsync(F.bad, 0, sizeof(int), d.stream));
  auto check_bad = [&](double others) {
    int bad = 0;
    SCN_CUDA(cudaMemcpyAsync(&bad, F.bad, sizeof(int), cudaMemcpyDeviceToHost, d.stream));
    SCN_CUDA(cudaStreamSynchronize(d.stream));
    if (bad)
      fail(SCENOPT_E_NOT_STRONGLY_CONVEX, "factor: eliminated input Hessian at node " + std::to_string(bad - 1) +
                                              " has min eigenvalue below 1e-10");
    if (others > 0.0)
      fail(SCENOPT_E_NOT_STRONGLY_CONVEX, "factor: an eliminated input Hessian of another rank's subtrees has "
                                          "min eigenvalue below 1e-10");
  };
  // riccati.hpp:106-113: leaves; then stages N-1 .. 0 (each needs the stage below).
  // A sharded rank factors its own subtrees up to the shard stage, then every
  // rank factors the replicated top from the shard-stage nodes' value
  // matrices, exchanged in one sum-allreduce (owners write their rows).
  F.affine_only = 0;
  const int s = d.sharded() ? d.shard_stage : -1;
  const auto leaves = held_range(d, L.N);
  F.stage_first = leaves.first;
  F.stage_count = leaves.second - leaves.first;
  if (F.stage_count > 0) SCN_CUDA(factor_run_leaves(F, std::min(grid_max, F.stage_count), d.stream));
  for (int t = L.N - 1; t >= 0; --t) {
    if (t == s - 1) {  // the shard-stage exchange
      const int ns = d.sstage_hi - d.sstage_lo;
      const size_t xx = static_cast<size_t>(nx) * nx;
      if (!d.vx) d.vx = d.alloc<double>(static_cast<size_t>(ns) * xx + 1);
      SCN_CUDA(cudaMemsetAsync(d.vx, 0, sizeof(double) * (ns * xx + 1), d.stream));
      if (d.shard_hi > d.shard_lo)
        SCN_CUDA(cudaMemcpyAsync(d.vx + (d.shard_lo - d.sstage_lo) * xx, d.vq + static_cast<size_t>(d.shard_lo) * xx,
                                 sizeof(double) * (d.shard_hi - d.shard_lo) * xx, cudaMemcpyDeviceToDevice, d.stream));
      int bad = 0;  // this rank's verdict travels with the exchange, so every rank stops together
      SCN_CUDA(cudaMemcpyAsync(&bad, F.bad, sizeof(int), cudaMemcpyDeviceToHost, d.stream));
      SCN_CUDA(cudaStreamSynchronize(d.stream));
      const double flag = bad ? 1.0 : 0.0;
      SCN_CUDA(cudaMemcpyAsync(d.vx + ns * xx, &flag, sizeof(double), cudaMemcpyHostToDevice, d.stream));
      dev_allreduce(d, d.vx, ns * xx + 1);
      SCN_CUDA(cudaMemcpyAsync(d.vq + static_cast<size_t>(d.sstage_lo) * xx, d.vx, sizeof(double) * ns * xx,
                               cudaMemcpyDeviceToDevice, d.stream));
      double all = 0.0;
      SCN_CUDA(cudaMemcpyAsync(&all, d.vx + ns * xx, sizeof(double), cudaMemcpyDeviceToHost, d.stream));
      SCN_CUDA(cudaStreamSynchronize(d.stream));
      check_bad(all - flag);
    }
    const auto r = held_range(d, t);
    F.stage_first = r.first;
    F.stage_count = r.second - r.first;
    if (F.stage_count > 0) SCN_CUDA(factor_run_stage(F, std::min(grid_max, F.stage_count), smem, d.stream));
  }
  run_flat(d, F, 0);
  check_bad(0.0);
  d.device_factor = true;
}

void dev_refactor_affine(DevState& d, const Problem& p) {
  const Layout& L = d.lay;
  if (p.n != L.n || p.nx != L.nx || p.nu != L.nu || p.dual_dim != L.dual_dim || p.first_leaf != L.first_leaf)
    fail(SCENOPT_E_SHAPE_CHANGED, "refactor_affine: problem shape changed since factor()");
  if (!d.device_factor)
    fail(SCENOPT_E_INVALID_PARAMS, "refactor_affine on the device needs a device-factored handle");
  if (d.sharded()) fail(SCENOPT_E_INVALID_PARAMS, "refactor_affine: not available on sharded handles");
  const int nx = L.nx, nu = L.nu, n = L.n;
  const size_t dbl = sizeof(double);
  const size_t xx = static_cast<size_t>(nx) * nx, xu = static_cast<size_t>(nx) * nu, uu = static_cast<size_t>(nu) * nu;
  const size_t csz = 2 * xx + 2 * xu + uu + 2 * static_cast<size_t>(nx) + nu, lsz = xx + nx;
  SCN_CUDA(cudaSetDevice(d.device));
  FactorParams& F = params(d);
  double* node = const_cast<double*>(d.cost.node);
  // linear terms into the eval_f cost blocks (pitched: one row per non-root node)
  if (n > 1) {
    SCN_CUDA(cudaMemcpy2DAsync(node + xx + xu, csz * dbl, p.c.data() + nx, nx * dbl, nx * dbl, n - 1,
                               cudaMemcpyHostToDevice, d.stream));
    SCN_CUDA(cudaMemcpy2DAsync(node + 2 * xx + 2 * xu + uu + nx, csz * dbl, p.q.data() + nx, nx * dbl, nx * dbl,
                               n - 1, cudaMemcpyHostToDevice, d.stream));
    SCN_CUDA(cudaMemcpy2DAsync(node + 2 * xx + 2 * xu + uu + 2 * nx, csz * dbl, p.r.data() + nu, nu * dbl,
                               nu * dbl, n - 1, cudaMemcpyHostToDevice, d.stream));
  }
  if (p.L > 0)
    SCN_CUDA(cudaMemcpy2DAsync(const_cast<double*>(d.cost.leaf) + xx, lsz * dbl, p.p.data(), nx * dbl, nx * dbl,
                               p.L, cudaMemcpyHostToDevice, d.stream));
  // forward affine terms c (aff_fw) and the root state
  SCN_CUDA(cudaMemcpyAsync(d.aff_fw, p.c.data(), static_cast<size_t>(n) * nx * dbl, cudaMemcpyHostToDevice, d.stream));
  SCN_CUDA(cudaMemcpyAsync(d.root_state, p.root_state.data(), nx * dbl, cudaMemcpyHostToDevice, d.stream));
  if (d.cost.root_state != d.root_state)
    SCN_CUDA(cudaMemcpyAsync(const_cast<double*>(d.cost.root_state), p.root_state.data(), nx * dbl,
                             cudaMemcpyHostToDevice, d.stream));
  d.lay.root_state = p.root_state;
  const int grid = d.sm_count * 4;
  F.affine_only = 1;
  F.stage_first = L.first_leaf;
  F.stage_count = L.n - L.first_leaf;
  SCN_CUDA(factor_run_leaves(F, std::min(grid, std::max(1, F.stage_count)), d.stream));
  SCN_CUDA(factor_run_affine(F, std::min(grid, std::max(1, L.first_leaf)), d.stream));
  run_flat(d, F, 1);
  SCN_CUDA(cudaStreamSynchronize(d.stream));
}

Factor dev_factor_export(DevState& d, const Problem& p) {
  if (!d.device_factor || !d.vq) fail(SCENOPT_E_INVALID_PARAMS, "factor export: handle has no device factor");
  if (d.sharded()) fail(SCENOPT_E_INVALID_PARAMS, "factor export: not available on sharded handles");
  Factor f = factor_shape(p);
  const int nx = p.nx, nu = p.nu, n = p.n, W = nx + nu, nxp = d.nxp;
  std::vector<double> bw(static_cast<size_t>(d.bw_doubles)), fw(static_cast<size_t>(d.fw_doubles)),
      aff(static_cast<size_t>(n) * W);
  SCN_CUDA(cudaSetDevice(d.device));
  SCN_CUDA(cudaStreamSynchronize(d.stream));
  SCN_CUDA(cudaMemcpy(bw.data(), d.bw_blk, bw.size() * sizeof(double), cudaMemcpyDeviceToHost));
  SCN_CUDA(cudaMemcpy(fw.data(), d.fw_blk, fw.size() * sizeof(double), cudaMemcpyDeviceToHost));
  SCN_CUDA(cudaMemcpy(aff.data(), d.aff_bw, aff.size() * sizeof(double), cudaMemcpyDeviceToHost));
  SCN_CUDA(cudaMemcpy(f.value_quad.data(), d.vq, f.value_quad.size() * sizeof(double), cudaMemcpyDeviceToHost));
  for (int c = 0; c < n; ++c) {
    const bool leaf = c >= p.first_leaf;
    if (!leaf) {  // E_c -> dual_to_input / dual_to_costate; K_c -> gain; aff -> affine terms
      const int M = f.child_dual_rows[c], off = f.child_dual_offset[c];
      const double* E = bw.data() + d.h_bw_off[c];
      for (int k = 0; k < M; ++k) {
        for (int j = 0; j < nu; ++j) f.dual_to_input[static_cast<size_t>(off + k) * nu + j] = E[k + static_cast<int64_t>(j) * M];
        for (int t = 0; t < nx; ++t)
          f.dual_to_costate[static_cast<size_t>(off + k) * nx + t] = E[k + static_cast<int64_t>(nu + t) * M];
      }
      const double* K = fw.data() + d.h_k_off[c];
      for (int j = 0; j < nu; ++j)
        for (int k = 0; k < nx; ++k) f.gain[static_cast<size_t>(c) * nu * nx + j + static_cast<size_t>(k) * nu] = K[k + static_cast<int64_t>(j) * nxp];
      for (int j = 0; j < nu; ++j) f.input_affine[static_cast<size_t>(c) * nu + j] = aff[static_cast<size_t>(c) * W + j];
      for (int t = 0; t < nx; ++t) f.costate_affine[static_cast<size_t>(c) * nx + t] = aff[static_cast<size_t>(c) * W + nu + t];
    } else {
      for (int t = 0; t < nx; ++t)
        f.leaf_costate_affine[static_cast<size_t>(c - p.first_leaf) * nx + t] = aff[static_cast<size_t>(c) * W + nu + t];
    }
    if (c != 0) {  // J_c -> child_to_input / closed_loop
      const double* J = bw.data() + d.h_bw_j[c];
      for (int k = 0; k < nx; ++k) {
        for (int j = 0; j < nu; ++j)
          f.child_to_input[static_cast<size_t>(c) * nu * nx + j + static_cast<size_t>(k) * nu] = J[k + static_cast<int64_t>(j) * nxp];
        for (int t = 0; t < nx; ++t)
          f.closed_loop[static_cast<size_t>(c) * nx * nx + k + static_cast<size_t>(t) * nx] = J[k + static_cast<int64_t>(nu + t) * nxp];
      }
    }
  }
  return f;
}

}  // namespace scn
