// SPDX-License-Identifier: MIT
// Packing (ProblemInstance, FactorCache) into the stage-major device layout
// of layout.hpp, upload, launch configuration, and the sweep entry point.
#include "device.hpp"

#include <algorithm>
#include <cstdlib>
#include <cstring>

namespace scn {

DevState::~DevState() {
  if (device >= 0) cudaSetDevice(device);
  for (void* p : owned) cudaFree(p);
  if (stream) cudaStreamDestroy(stream);
}

void DevState::free_owned(void* p) {
  auto it = std::find(owned.begin(), owned.end(), p);
  if (it == owned.end()) fail(SCENOPT_E_INVALID_PARAMS, "dev_free: pointer not owned by this handle");
  cudaFree(p);
  owned.erase(it);
}

int device_count_sm100() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  int good = 0;
  for (int d = 0; d < n; ++d) {
    cudaDeviceProp prop{};
    if (cudaGetDeviceProperties(&prop, d) == cudaSuccess && prop.major == 10) ++good;
  }
  return good;
}

namespace {

int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v && *v ? std::atoi(v) : dflt;
}

inline int64_t even(int64_t x) { return (x + 1) & ~int64_t(1); }

template <class T>
T* upload(DevState& d, const std::vector<T>& h) {
  T* p = d.alloc<T>(std::max<size_t>(h.size(), 1));
  if (!h.empty()) SCN_CUDA(cudaMemcpy(p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
  return p;
}

// Runs of consecutive same-stage nodes whose blocks total <= target bytes
// (a node larger than the target forms its own item).
void build_items(const Problem& p, const std::vector<int64_t>& off, const std::vector<int64_t>& size,
                 int pass, int max_count, int64_t target_doubles, std::vector<Item>& out,
                 int& max_cnt_seen, int64_t& max_item_doubles) {
  auto stage_items = [&](int t) {
    const int first = p.stage_offsets[t], past = p.stage_offsets[t + 1];
    int i = first;
    while (i < past) {
      int cnt = 0;
      int64_t tot = 0;
      while (i + cnt < past && cnt < max_count) {
        const int64_t s = size[i + cnt];
        if (cnt > 0 && tot + s > target_doubles) break;
        tot += s;
        ++cnt;
      }
      Item it{};
      it.off = off[i];
      it.first = i;
      it.count = cnt;
      it.bytes = static_cast<int32_t>(tot * 8);
      it.pass = pass;
      out.push_back(it);
      max_cnt_seen = std::max(max_cnt_seen, cnt);
      max_item_doubles = std::max(max_item_doubles, tot);
      i += cnt;
    }
  };
  if (pass == 0)
    for (int t = p.N; t >= 0; --t) stage_items(t);
  else
    for (int t = 0; t <= p.N; ++t) stage_items(t);
}

}  // namespace

std::unique_ptr<DevState> dev_create(const Problem& p, const Factor& f, int device) {
  check_factor_shape(f, p, "dev_create");
  require_valid(p);
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    fail(SCENOPT_E_NODEVICE, "scenopt_dev_create: no CUDA device visible (the library has no CPU path)");
  }
  if (device < 0 || device >= ndev) fail(SCENOPT_E_NODEVICE, "scenopt_dev_create: device index out of range");
  cudaDeviceProp prop{};
  SCN_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10)
    fail(SCENOPT_E_NODEVICE, std::string("scenopt_dev_create: device is ") + prop.name +
                                 " (sm_" + std::to_string(prop.major * 10 + prop.minor) +
                                 "); this build targets sm_100a (B200)");
  auto d = std::make_unique<DevState>();
  d->device = device;
  SCN_CUDA(cudaSetDevice(device));
  SCN_CUDA(cudaStreamCreateWithFlags(&d->stream, cudaStreamNonBlocking));
  d->sm_count = prop.multiProcessorCount;

  const int nx = p.nx, nu = p.nu, n = p.n, W = nx + nu, V = nx + nu;
  Layout& L = d->lay;
  L.nx = nx;
  L.nu = nu;
  L.N = p.N;
  L.n = n;
  L.L = p.L;
  L.first_leaf = p.first_leaf;
  L.dual_dim = p.dual_dim;
  L.stage_total = p.stage_total;
  L.ancestor = p.ancestor;
  L.stage_offsets = p.stage_offsets;
  L.stage_rows = p.stage_rows;
  L.terminal_rows = p.terminal_rows;
  L.child_begin = p.child_begin;
  L.child_count = p.child_count;
  L.dual_offset = p.dual_offset;
  L.tdual_offset = p.tdual_offset;
  L.probability = p.probability;
  L.root_state = p.root_state;

  // ---- per-node metadata and block sizes
  std::vector<NodeMeta> meta(static_cast<size_t>(n));
  std::vector<int64_t> bws(static_cast<size_t>(n)), fws(static_cast<size_t>(n));
  for (int c = 0; c < n; ++c) {
    NodeMeta& m = meta[c];
    const bool leaf = c >= p.first_leaf;
    m.anc = p.ancestor[c];
    m.cb = p.child_begin[c];
    m.cc = p.child_count[c];
    m.M = leaf ? 0 : f.child_dual_rows[c];
    m.cdo = leaf ? 0 : f.child_dual_offset[c];
    m.doff = c == 0 ? 0 : p.dual_offset[c];
    m.m = c == 0 ? 0 : p.stage_rows[c];
    m.tdo = leaf ? p.tdual_offset[c - p.first_leaf] : 0;
    m.mN = leaf ? p.terminal_rows[c - p.first_leaf] : 0;
    m.leaf = leaf ? 1 : 0;
    d->max_m = std::max(d->max_m, m.m);
    d->max_mN = std::max(d->max_mN, m.mN);
    int64_t b = leaf ? static_cast<int64_t>(m.mN) * nx : static_cast<int64_t>(m.M) * W;
    if (c != 0) b += static_cast<int64_t>(nx) * W;
    bws[c] = even(b);
    int64_t fw = 0;
    if (c != 0) fw += static_cast<int64_t>(V) * (nx + m.m);
    fw += leaf ? static_cast<int64_t>(nx) * m.mN : static_cast<int64_t>(nx) * nu;
    fws[c] = even(fw);
  }
  std::vector<int64_t> bwo(static_cast<size_t>(n) + 1, 0), fwo(static_cast<size_t>(n) + 1, 0);
  for (int c = 0; c < n; ++c) {
    bwo[c + 1] = bwo[c] + bws[c];
    fwo[c + 1] = fwo[c] + fws[c];
  }
  d->bw_doubles = bwo[n];
  d->fw_doubles = fwo[n];

  // ---- blocks
  std::vector<double> bw(static_cast<size_t>(bwo[n]), 0.0), fw(static_cast<size_t>(fwo[n]), 0.0);
  std::vector<double> aff_bw(static_cast<size_t>(n) * W, 0.0), aff_fw(static_cast<size_t>(n) * nx, 0.0);
  parallel_for(n, 256, [&](int b, int e) {
    for (int c = b; c < e; ++c) {
      const NodeMeta& m = meta[c];
      const bool leaf = m.leaf != 0;
      double* B0 = bw.data() + bwo[c];
      int64_t jo = 0;
      if (!leaf) {
        const double* d2i = f.dual_to_input.data() + static_cast<size_t>(m.cdo) * nu;
        const double* d2c = f.dual_to_costate.data() + static_cast<size_t>(m.cdo) * nx;
        for (int k = 0; k < m.M; ++k) {
          for (int j = 0; j < nu; ++j) B0[k + static_cast<int64_t>(j) * m.M] = d2i[j + static_cast<int64_t>(k) * nu];
          for (int t = 0; t < nx; ++t)
            B0[k + static_cast<int64_t>(nu + t) * m.M] = d2c[t + static_cast<int64_t>(k) * nx];
        }
        jo = static_cast<int64_t>(m.M) * W;
        const double* ia = f.input_affine.data() + static_cast<size_t>(c) * nu;
        const double* ca = f.costate_affine.data() + static_cast<size_t>(c) * nx;
        for (int j = 0; j < nu; ++j) aff_bw[static_cast<size_t>(c) * W + j] = ia[j];
        for (int t = 0; t < nx; ++t) aff_bw[static_cast<size_t>(c) * W + nu + t] = ca[t];
      } else {
        const int l = c - p.first_leaf;
        const double* FN = p.FNl(l);
        std::copy(FN, FN + static_cast<size_t>(m.mN) * nx, B0);
        jo = static_cast<int64_t>(m.mN) * nx;
        const double* lca = f.leaf_costate_affine.data() + static_cast<size_t>(l) * nx;
        for (int t = 0; t < nx; ++t) aff_bw[static_cast<size_t>(c) * W + nu + t] = lca[t];
      }
      if (c != 0) {
        double* J = B0 + jo;
        const double* c2i = f.child_to_input.data() + static_cast<size_t>(c) * nu * nx;
        const double* cl = f.closed_loop.data() + static_cast<size_t>(c) * nx * nx;
        for (int k = 0; k < nx; ++k) {
          for (int j = 0; j < nu; ++j) J[k + static_cast<int64_t>(j) * nx] = c2i[j + static_cast<int64_t>(k) * nu];
          for (int t = 0; t < nx; ++t) J[k + static_cast<int64_t>(nu + t) * nx] = cl[k + static_cast<int64_t>(t) * nx];
        }
      }
      // forward block
      double* F0 = fw.data() + fwo[c];
      int64_t ko = 0;
      if (c != 0) {
        const double* A = p.Ai(c);
        const double* Bm = p.Bi(c);
        const double* Fm = p.Fi(c);
        const double* Gm = p.Gi(c);
        const int mm = m.m;
        for (int r = 0; r < nx; ++r) {
          double* col = F0 + static_cast<int64_t>(r) * V;
          for (int k = 0; k < nx; ++k) col[k] = A[r + static_cast<int64_t>(k) * nx];
          for (int k = 0; k < nu; ++k) col[nx + k] = Bm[r + static_cast<int64_t>(k) * nx];
        }
        for (int s = 0; s < mm; ++s) {
          double* col = F0 + static_cast<int64_t>(nx + s) * V;
          for (int k = 0; k < nx; ++k) col[k] = Fm[s + static_cast<int64_t>(k) * mm];
          for (int k = 0; k < nu; ++k) col[nx + k] = Gm[s + static_cast<int64_t>(k) * mm];
        }
        ko = static_cast<int64_t>(V) * (nx + mm);
        const double* cc = p.ci(c);
        for (int t = 0; t < nx; ++t) aff_fw[static_cast<size_t>(c) * nx + t] = cc[t];
      }
      double* K = F0 + ko;
      if (!leaf) {
        const double* gain = f.gain.data() + static_cast<size_t>(c) * nu * nx;
        for (int j = 0; j < nu; ++j)
          for (int k = 0; k < nx; ++k) K[k + static_cast<int64_t>(j) * nx] = gain[j + static_cast<int64_t>(k) * nu];
      } else {
        const double* FN = p.FNl(c - p.first_leaf);
        for (int s = 0; s < m.mN; ++s)
          for (int k = 0; k < nx; ++k) K[k + static_cast<int64_t>(s) * nx] = FN[s + static_cast<int64_t>(k) * m.mN];
      }
    }
  });

  // ---- items
  const int64_t target = env_int("SCENOPT_ITEM_KB", 24) * 1024 / 8;
  const int cap = std::max(1, env_int("SCENOPT_ITEM_MAX_NODES", 32));
  std::vector<Item> items;
  int max_cnt = 1;
  int64_t max_item = 2;
  build_items(p, bwo, bws, 0, cap, target, items, max_cnt, max_item);
  d->items_bw = static_cast<int>(items.size());
  build_items(p, fwo, fws, 1, cap, target, items, max_cnt, max_item);
  d->items_fw = static_cast<int>(items.size()) - d->items_bw;
  d->max_count = max_cnt;
  d->slot_doubles = static_cast<int>((max_item + 15) & ~int64_t(15));
  d->vec_doubles = static_cast<int>(((static_cast<int64_t>(max_cnt) * kMaxRhs * (2 * nx + nu)) + 15) & ~int64_t(15));

  // ---- launch configuration: maximise concurrent slots per SM
  const int dbl = 8;
  int best_cps = 0, best_ns = 0;
  const int force_ns = env_int("SCENOPT_NSLOT", 0), force_cps = env_int("SCENOPT_CTAS_PER_SM", 0);
  for (int ns = kMaxSlots; ns >= 2; --ns) {
    if (force_ns && ns != force_ns) continue;
    const size_t smem = (static_cast<size_t>(ns) * d->slot_doubles + d->vec_doubles) * dbl;
    if (smem > static_cast<size_t>(prop.sharedMemPerBlockOptin)) continue;
    SCN_CUDA(sweep_configure(2, smem));
    int cps = 0;
    SCN_CUDA(sweep_occupancy(&cps, smem));
    if (force_cps) cps = std::min(cps, force_cps);
    if (cps < 1) continue;
    if (cps * ns > best_cps * best_ns || (cps * ns == best_cps * best_ns && cps > best_cps)) {
      best_cps = cps;
      best_ns = ns;
    }
  }
  if (best_cps == 0) {  // a single huge node: one slot per CTA is not supported
    const size_t smem = (2 * static_cast<size_t>(d->slot_doubles) + d->vec_doubles) * dbl;
    fail(SCENOPT_E_INVALID_PARAMS, "dev_create: node blocks too large for shared memory (" +
                                       std::to_string(smem) + " bytes needed per CTA)");
  }
  d->nslot = best_ns;
  d->ctas_per_sm = best_cps;
  d->dyn_smem = (static_cast<size_t>(best_ns) * d->slot_doubles + d->vec_doubles) * dbl;
  SCN_CUDA(sweep_configure(2, d->dyn_smem));
  d->grid = d->sm_count * best_cps;
  d->G = nx >= 40 ? 16 : (nx >= 20 ? 8 : 4);
  if (const int g = env_int("SCENOPT_GROUP", 0)) d->G = g;

  // ---- upload
  d->bw_blk = upload(*d, bw);
  d->fw_blk = upload(*d, fw);
  bw.clear();
  bw.shrink_to_fit();
  fw.clear();
  fw.shrink_to_fit();
  d->aff_bw = upload(*d, aff_bw);
  d->aff_fw = upload(*d, aff_fw);
  d->root_state = upload(*d, p.root_state);
  d->items = upload(*d, items);
  d->meta = upload(*d, meta);
  bwo.pop_back();
  fwo.pop_back();
  d->bw_off = upload(*d, bwo);
  d->fw_off = upload(*d, fwo);
  d->ctrl = d->alloc<unsigned>(4);
  d->bw_flag = d->alloc<unsigned>(static_cast<size_t>(n));
  d->fw_flag = d->alloc<unsigned>(static_cast<size_t>(n));
  SCN_CUDA(cudaMemset(d->ctrl, 0, 4 * sizeof(unsigned)));
  SCN_CUDA(cudaMemset(d->bw_flag, 0, static_cast<size_t>(n) * sizeof(unsigned)));
  SCN_CUDA(cudaMemset(d->fw_flag, 0, static_cast<size_t>(n) * sizeof(unsigned)));

  // per-row nonsmooth data
  const int D = p.dual_dim;
  std::vector<int8_t> kind(static_cast<size_t>(D), 0);
  std::vector<double> lo(static_cast<size_t>(D), 0.0), hi(static_cast<size_t>(D), 0.0),
      wg(static_cast<size_t>(D), 0.0);
  for (int i = 1; i < n; ++i)
    for (int k = 0; k < p.stage_rows[i]; ++k) {
      const int row = p.dual_offset[i] + k;
      kind[row] = static_cast<int8_t>(p.g_kind[i]);
      lo[row] = p.zmin[row];
      hi[row] = p.zmax[row];
      wg[row] = p.probability[i] * p.g_gamma[i];
    }
  for (int l = 0; l < p.L; ++l)
    for (int k = 0; k < p.terminal_rows[l]; ++k) {
      const int row = p.tdual_offset[l] + k;
      kind[row] = static_cast<int8_t>(p.tg_kind[l]);
      lo[row] = p.zmin[row];
      hi[row] = p.zmax[row];
      wg[row] = p.probability[p.first_leaf + l] * p.tg_gamma[l];
    }
  d->row_kind = upload(*d, kind);
  d->row_lo = upload(*d, lo);
  d->row_hi = upload(*d, hi);
  d->row_wg = upload(*d, wg);

  for (int r = 0; r < kMaxRhs; ++r) {
    d->contrib[r] = d->alloc<double>(static_cast<size_t>(n) * W);
    d->xs[r] = d->alloc<double>(static_cast<size_t>(n) * nx);
    d->us[r] = d->alloc<double>(static_cast<size_t>(std::max(p.first_leaf, 1)) * nu);
    d->hs[r] = d->alloc<double>(static_cast<size_t>(std::max(D, 1)));
    d->ys[r] = d->alloc<double>(static_cast<size_t>(std::max(D, 1)));
  }

  // ---- algorithmic bytes per sweep (matrices once + vector traffic)
  const int64_t F = p.first_leaf;
  const int64_t vecs = 2LL * D + static_cast<int64_t>(nx) * n + 3LL * nu * F +
                       static_cast<int64_t>(n - 1) * V + 2LL * (n - 1) * W;
  const int64_t mats = d->bw_doubles + d->fw_doubles;
  d->bytes_hom = 8 * (mats + vecs);
  d->bytes_aff = d->bytes_hom + 8 * (static_cast<int64_t>(n) * W + static_cast<int64_t>(n) * nx);
  d->bytes_hom2 = 8 * (mats + 2 * vecs);
  SCN_CUDA(cudaDeviceSynchronize());
  return d;
}

void dev_sweep(DevState& d, int nrhs, bool affine, const double* const* y, double* const* x,
               double* const* u, double* const* Hx) {
  if (nrhs < 1 || nrhs > kMaxRhs) fail(SCENOPT_E_INVALID_PARAMS, "sweep: nrhs must be 1 or 2");
  const Layout& L = d.lay;
  SweepParams P{};
  P.nx = L.nx;
  P.nu = L.nu;
  P.n = L.n;
  P.first_leaf = L.first_leaf;
  P.dual_dim = L.dual_dim;
  P.items_bw = d.items_bw;
  P.items_total = d.items_bw + d.items_fw;
  P.nslot = d.nslot;
  P.slot_doubles = d.slot_doubles;
  P.vec_doubles = d.vec_doubles;
  P.nrhs = nrhs;
  P.affine = affine ? 1 : 0;
  P.max_count = d.max_count;
  P.max_mN = d.max_mN;
  P.items = d.items;
  P.meta = d.meta;
  P.bw_off = d.bw_off;
  P.fw_off = d.fw_off;
  P.bw_blk = d.bw_blk;
  P.fw_blk = d.fw_blk;
  P.aff_bw = d.aff_bw;
  P.aff_fw = d.aff_fw;
  P.root_state = d.root_state;
  P.ctrl = d.ctrl;
  P.bw_flag = d.bw_flag;
  P.fw_flag = d.fw_flag;
  for (int r = 0; r < nrhs; ++r) {
    P.y[r] = y[r];
    P.x[r] = (x && x[r]) ? x[r] : d.xs[r];
    P.u[r] = (u && u[r]) ? u[r] : d.us[r];
    P.Hx[r] = (Hx && Hx[r]) ? Hx[r] : d.hs[r];
    P.contrib[r] = d.contrib[r];
  }
  SCN_CUDA(sweep_launch(P, d.grid, d.dyn_smem, d.G, d.max_m, d.stream));
}

}  // namespace scn
