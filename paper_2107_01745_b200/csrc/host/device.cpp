// SPDX-License-Identifier: MIT
// Packing (ProblemInstance, FactorCache) into the stage-major device layout
// of layout.hpp, upload, launch configuration, and the sweep entry point.
#include "device.hpp"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>

namespace scn {

DevState::~DevState() {
  if (device >= 0) cudaSetDevice(device);
  comm.reset();
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
// padded column length == 2 (mod 4): conflict-free 16-byte shared loads
inline int pad2(int l) { return l + ((2 - l % 4) + 4) % 4; }

template <class T>
T* upload(DevState& d, const std::vector<T>& h) {
  T* p = d.alloc<T>(std::max<size_t>(h.size(), 1));
  if (!h.empty()) SCN_CUDA(cudaMemcpy(p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
  return p;
}

// Host staging array of doubles without value-initialisation (the multi-GB
// pack buffers of large trees are zeroed in parallel where padding needs it,
// or fully overwritten).
struct HostArray {
  std::unique_ptr<double[]> p;
  size_t n = 0;
  explicit HostArray(size_t count, bool zero) : p(new double[std::max<size_t>(count, 1)]), n(count) {
    if (zero)
      parallel_for(static_cast<int>((count + (1 << 20) - 1) >> 20), 1, [&](int b, int e) {
        for (int k = b; k < e; ++k) {
          const size_t lo = static_cast<size_t>(k) << 20, hi = std::min(count, lo + (size_t(1) << 20));
          std::fill(p.get() + lo, p.get() + hi, 0.0);
        }
      });
  }
  double* data() { return p.get(); }
  void release() {
    p.reset();
    n = 0;
  }
};

double* upload(DevState& d, const HostArray& h) {
  double* q = d.alloc<double>(std::max<size_t>(h.n, 1));
  if (h.n) SCN_CUDA(cudaMemcpy(q, h.p.get(), h.n * sizeof(double), cudaMemcpyHostToDevice));
  return q;
}

}  // namespace

namespace {
void pack_common(DevState& d, const Problem& p, const std::vector<char>* mine = nullptr,
                 const std::vector<char>* held = nullptr);
}

// Per-node packed block sizes (doubles) of the backward / forward pass
// arrays (layout.hpp); M_c = the children's stage rows.
void node_block_sizes(const Problem& p, std::vector<int64_t>& bws, std::vector<int64_t>& fws) {
  const int nx = p.nx, nu = p.nu, n = p.n, W = nx + nu;
  const int nxp = pad2(nx), Vp = pad2(nx + nu);
  bws.assign(static_cast<size_t>(n), 0);
  fws.assign(static_cast<size_t>(n), 0);
  for (int c = 0; c < n; ++c) {
    const bool leaf = c >= p.first_leaf;
    const int m = c == 0 ? 0 : p.stage_rows[c];
    const int mN = leaf ? p.terminal_rows[c - p.first_leaf] : 0;
    int64_t M = 0;
    if (!leaf)
      for (int k = p.child_begin[c]; k < p.child_begin[c] + p.child_count[c]; ++k) M += p.stage_rows[k];
    int64_t b = even(leaf ? static_cast<int64_t>(mN) * nx : M * W);
    if (c != 0) b += static_cast<int64_t>(nxp) * W;
    bws[c] = b;
    int64_t fw = 0;
    if (c != 0) fw += static_cast<int64_t>(Vp) * (nx + m);
    fw += leaf ? static_cast<int64_t>(nxp) * mN : static_cast<int64_t>(nxp) * nu;
    fws[c] = even(fw);
  }
}

// Contiguous split of nodes [lo, hi) into k groups balanced by subtree bytes.
std::vector<int> balanced_split(const std::vector<int64_t>& sub, int lo, int hi, int k) {
  std::vector<int> bound(static_cast<size_t>(k) + 1, hi);
  bound[0] = lo;
  int64_t total = 0, acc = 0;
  for (int r = lo; r < hi; ++r) total += sub[r];
  int g = 1;
  for (int r = lo; r < hi && g < k; ++r) {
    acc += sub[r];
    while (g < k && acc * k >= total * g) bound[g++] = r + 1;
  }
  return bound;
}

std::vector<int64_t> subtree_bytes(const Problem& p, const std::vector<int64_t>& bws, const std::vector<int64_t>& fws) {
  std::vector<int64_t> sub(static_cast<size_t>(p.n));
  for (int c = 0; c < p.n; ++c) sub[c] = bws[c] + fws[c];
  for (int c = p.n - 1; c >= 1; --c) sub[p.ancestor[c]] += sub[c];  // BFS: parents precede children
  return sub;
}

std::vector<int> shard_plan(const Problem& p, int world, int* stage) {
  int s = *stage;
  if (world < 1) fail(SCENOPT_E_INVALID_PARAMS, "shard plan: world must be >= 1");
  if (s < 0)
    for (int t = 1; t <= p.N && s < 0; ++t)
      if (p.stage_offsets[t + 1] - p.stage_offsets[t] >= world) s = t;
  if (s < 1 || s > p.N || p.stage_offsets[s + 1] - p.stage_offsets[s] < world)
    fail(SCENOPT_E_INVALID_PARAMS, "dev_create_sharded: shard stage must lie in [1, N] and hold >= world nodes");
  std::vector<int64_t> bws, fws;
  node_block_sizes(p, bws, fws);
  *stage = s;
  return balanced_split(subtree_bytes(p, bws, fws), p.stage_offsets[s], p.stage_offsets[s + 1], world);
}

std::vector<char> shard_nodes(const Problem& p, int stage, int lo, int hi, int rank) {
  std::vector<char> mine(static_cast<size_t>(p.n), 0);
  for (int c = 0; c < p.stage_offsets[stage]; ++c) mine[c] = rank == 0;
  for (int t = stage; t <= p.N; ++t) {
    for (int c = lo; c < hi; ++c) mine[c] = 1;
    if (t < p.N && lo < hi) {
      const int nlo = p.child_begin[lo], nhi = p.child_begin[hi - 1] + p.child_count[hi - 1];
      lo = nlo;
      hi = nhi;
    }
  }
  return mine;
}

std::vector<uint8_t> shard_rows(const Problem& p, const std::vector<char>& mine) {
  std::vector<uint8_t> cnt(static_cast<size_t>(p.dual_dim), 0);
  for (int c = 1; c < p.n; ++c)
    if (mine[c])
      for (int k = 0; k < p.stage_rows[c]; ++k) cnt[p.dual_offset[c] + k] = 1;
  for (int l = 0; l < p.L; ++l)
    if (mine[p.first_leaf + l])
      for (int k = 0; k < p.terminal_rows[l]; ++k) cnt[p.tdual_offset[l] + k] = 1;
  return cnt;
}

std::unique_ptr<DevState> dev_create_bare(int device) {
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    fail(SCENOPT_E_NODEVICE, "scenopt: no CUDA device visible (the library has no CPU path)");
  }
  if (device < 0 || device >= ndev) fail(SCENOPT_E_NODEVICE, "scenopt: device index out of range");
  cudaDeviceProp prop{};
  SCN_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10) fail(SCENOPT_E_NODEVICE, std::string("scenopt: device is ") + prop.name + "; this build targets sm_100a (B200)");
  auto d = std::make_unique<DevState>();
  d->device = device;
  SCN_CUDA(cudaSetDevice(device));
  SCN_CUDA(cudaStreamCreateWithFlags(&d->stream, cudaStreamNonBlocking));
  d->sm_count = prop.multiProcessorCount;
  return d;
}

namespace {
struct FlatTop {  // flattened forward top node (see dev_create)
  std::vector<double> G, L, a, h;
};

struct PhaseClock {  // SCN_SETUP_TIMING=1: phase times of dev_create on stderr
  bool on = std::getenv("SCN_SETUP_TIMING") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(const char* what) {
    if (!on) return;
    const auto n = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[dev_create] %-22s %8.1f ms\n", what, std::chrono::duration<double, std::milli>(n - t).count());
    t = n;
  }
};
}  // namespace

std::unique_ptr<DevState> dev_create(const Problem& p, const Factor* fptr, int device, const ShardSpec* shard) {
  PhaseClock clk;
  if (fptr) check_factor_shape(*fptr, p, "dev_create");
  require_valid(p);
  if (!shard) require_full(p, "dev_create");
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

  const int nx = p.nx, nu = p.nu, n = p.n, W = nx + nu;
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

  if (!fptr) {
    pack_common(*d, p);
    SCN_CUDA(cudaDeviceSynchronize());
    return d;
  }
  const Factor& f = *fptr;
  d->has_factor = true;
  const bool fz = f.gain.empty();  // layout-only factor: the device factor writes these blocks

  // ---- per-node block sizes (doubles, even => 16-byte aligned); padded
  // column lengths pad2(l) == 2 (mod 4) for conflict-free 16-byte smem loads
  const int nxp = pad2(nx), Vp = pad2(nx + nu);
  d->nxp = nxp;
  d->Vp = Vp;
  std::vector<int64_t> bws, fws;
  node_block_sizes(p, bws, fws);
  std::vector<int32_t> M(static_cast<size_t>(n), 0), cdo(static_cast<size_t>(n), 0);
  for (int c = 0; c < n; ++c) {
    const bool leaf = c >= p.first_leaf;
    if (!leaf) {
      M[c] = f.child_dual_rows[c];
      cdo[c] = f.child_dual_offset[c];
    }
    d->max_m = std::max(d->max_m, c == 0 ? 0 : p.stage_rows[c]);
    d->max_mN = std::max(d->max_mN, leaf ? p.terminal_rows[c - p.first_leaf] : 0);
  }

  clk.mark("sizes");
  // ---- schedule. The grid is one co-resident CTA per SM.
  // A region (per-stage node ranges) is scheduled as: below a cut stage with
  // >= min_sub*G nodes every CTA owns a contiguous, byte-balanced group of
  // whole subtrees (its items depend only on items of the same CTA: a
  // shared-memory retire counter, no gpu-scope publication); the region's
  // nodes above that cut are dealt round-robin as global tickets whose
  // dependencies are released through per-node flags. Each CTA's list is in
  // rank order (backward leaves->root, then forward root->leaves) and every
  // dependency has a smaller rank, so no schedule can deadlock.
  //
  // A sharded handle (rank r of W) owns the subtrees of a contiguous,
  // byte-balanced range of shard-stage nodes and replicates the stages
  // above. Its sweep is two launches: A = the local backward below the
  // shard stage; then the shard-stage contributions are sum-allreduced; then
  // B = the (redundant) top backward, top forward and local forward.
  d->grid = d->sm_count;
  int64_t packed_bytes = 0;  // node blocks of both passes
  for (int c = 0; c < p.n; ++c) packed_bytes += (bws[c] + fws[c]) * 8;
  constexpr int64_t kLatencyBoundBytes = int64_t(512) << 20;  // below: a sweep is bound by its dependency levels
  const int min_sub_cfg = env_int("SCENOPT_MIN_SUBTREES", 4);
  if (const int g = env_int("SCENOPT_GRID", 0)) {
    d->grid = std::min(g, d->grid);  // experiments only
  } else if (min_sub_cfg > 0) {  // whole-tree widths (conservative per rank)
    // A latency-bound tree (no stage reaches min_sub * SMs nodes, and little
    // data) runs on the largest grid that still gets a subtree cut: its
    // dependencies are then CTA-local instead of cross-CTA flags at every
    // level (1023-node C5 tree: 211 -> 135 us per sweep on 16 CTAs).
    int widest = 0;
    for (int t = 1; t <= p.N; ++t) widest = std::max(widest, p.stage_offsets[t + 1] - p.stage_offsets[t]);
    if (widest < min_sub_cfg * d->grid && packed_bytes < kLatencyBoundBytes) {
      const int g = widest / min_sub_cfg;
      if (g >= 8) d->grid = g;
    }
  }
  const int G = d->grid;
  const int64_t target = env_int("SCENOPT_ITEM_KB", 24) * 1024 / 8;
  const int cap = std::max(1, env_int("SCENOPT_ITEM_MAX_NODES", 32));
  const int min_sub = env_int("SCENOPT_MIN_SUBTREES", 4);  // per CTA; 0 disables ownership
  const int min_items = 8;  // independent items per stage and CTA (local dependency distance)
  struct Run { int first, count, pass, ldep, gdep, publish, flat = 0; };
  using Lists = std::vector<std::vector<Run>>;
  auto chunk = [&](int lo, int hi, int pass, int per_stage_min, std::vector<Run>& out) {
    const std::vector<int64_t>& size = pass == 0 ? bws : fws;
    const int cnt_all = hi - lo;
    const int ncap = std::max(1, std::min(cap, (cnt_all + per_stage_min - 1) / std::max(1, per_stage_min)));
    int i = lo;
    while (i < hi) {
      int cnt = 0;
      int64_t tot = 0;
      while (i + cnt < hi && cnt < ncap) {
        const int64_t sz = size[i + cnt] + static_cast<int64_t>(sizeof(NodeMeta) / 8);
        if (cnt > 0 && tot + sz > target) break;
        tot += sz;
        ++cnt;
      }
      out.push_back(Run{i, cnt, pass, -1, 0, 0});
      i += cnt;
    }
  };
  const std::vector<int64_t> sub = subtree_bytes(p, bws, fws);
  auto split = [&](int lo, int hi, int k) { return balanced_split(sub, lo, hi, k); };
  // per-stage ranges [t0, t1] of the subtrees of nodes [lo, hi) at stage t0
  auto descend = [&](int lo, int hi, int t0, int t1) {
    std::vector<std::pair<int, int>> rng(static_cast<size_t>(p.N) + 1, {0, 0});
    for (int t = t0; t <= t1; ++t) {
      rng[t] = {lo, hi};
      if (t < p.N && lo < hi) {
        const int nlo = p.child_begin[lo], nhi = p.child_begin[hi - 1] + p.child_count[hi - 1];
        lo = nlo;
        hi = nhi;
      } else {
        lo = hi = 0;
      }
    }
    return rng;
  };
  // Region [t0, t1] with per-stage ranges rng: per CTA, the backward part
  // (local backward, then region-top backward tickets) and the forward part
  // (region-top forward tickets, then local forward).
  auto region = [&](int t0, int t1, const std::vector<std::pair<int, int>>& rng, bool allow_cut, bool want_bw,
                    bool want_fw, Lists& bw_out, Lists& fw_out) {
    int cut = -1;
    if (allow_cut && min_sub > 0)
      for (int t = std::max(t0, 1); t <= t1; ++t)
        if (rng[t].second - rng[t].first >= min_sub * G) {
          cut = t;
          break;
        }
    const int top_end = cut < 0 ? t1 + 1 : cut;
    std::vector<Run> tb, tf;
    if (want_bw)
      for (int t = top_end - 1; t >= t0; --t) chunk(rng[t].first, rng[t].second, 0, 1, tb);
    if (want_fw)
      for (int t = t0; t < top_end; ++t) chunk(rng[t].first, rng[t].second, 1, 1, tf);
    bw_out.assign(static_cast<size_t>(G), {});
    fw_out.assign(static_cast<size_t>(G), {});
    Lists lfw(static_cast<size_t>(G));
    if (cut >= 0) {
      const std::vector<int> bound = split(rng[cut].first, rng[cut].second, G);
      for (int gg = 0; gg < G; ++gg) {
        const auto grp = descend(bound[gg], bound[gg + 1], cut, t1);
        if (want_bw)
          for (int t = t1; t >= cut; --t)
            if (grp[t].first < grp[t].second) chunk(grp[t].first, grp[t].second, 0, min_items, bw_out[gg]);
        if (want_fw)
          for (int t = cut; t <= t1; ++t)
            if (grp[t].first < grp[t].second) chunk(grp[t].first, grp[t].second, 1, min_items, lfw[gg]);
      }
    }
    for (size_t i = 0; i < tb.size(); ++i) bw_out[i % G].push_back(tb[i]);
    for (size_t i = 0; i < tf.size(); ++i) fw_out[i % G].push_back(tf[i]);
    for (int gg = 0; gg < G; ++gg) fw_out[gg].insert(fw_out[gg].end(), lfw[gg].begin(), lfw[gg].end());
    return cut;
  };
  // Dependencies of one launch: a dependency node produced by the same CTA
  // is a local wait (retire counter); by another CTA a flag wait (and its
  // producer publishes); by an earlier launch / the exchange, no wait.
  auto resolve = [&](Lists& L) {
    std::vector<int> bcta(static_cast<size_t>(n), -1), bpos(static_cast<size_t>(n), -1),
        fcta(static_cast<size_t>(n), -1), fpos(static_cast<size_t>(n), -1);
    for (int gg = 0; gg < G; ++gg)
      for (int k = 0; k < static_cast<int>(L[gg].size()); ++k) {
        const Run& r = L[gg][k];
        for (int c = r.first; c < r.first + r.count; ++c) {
          (r.pass == 0 ? bcta : fcta)[c] = gg;
          (r.pass == 0 ? bpos : fpos)[c] = k;
        }
      }
    for (int gg = 0; gg < G; ++gg)
      for (int k = 0; k < static_cast<int>(L[gg].size()); ++k) {
        Run& r = L[gg][k];
        const int last = r.first + r.count - 1;
        int lo = 0, hi = 0;
        const std::vector<int>*cta = &bcta, *pos = &bpos;
        if (r.pass == 0) {
          if (r.first >= p.first_leaf) continue;
          lo = p.child_begin[r.first];
          hi = p.child_begin[last] + p.child_count[last];
        } else if (r.first == 0 || r.flat) {
          lo = 0, hi = 1;  // forward root / flattened top <- backward root
        } else {
          lo = p.ancestor[r.first];
          hi = p.ancestor[last] + 1;
          cta = &fcta;
          pos = &fpos;
        }
        int ld = -1, nloc = 0, nrem = 0, next = 0;
        for (int c = lo; c < hi; ++c) {
          const int g2 = (*cta)[c];
          if (g2 < 0) {
            ++next;
          } else if (g2 == gg) {
            ++nloc;
            ld = std::max(ld, (*pos)[c]);
          } else {
            ++nrem;
          }
        }
        if (next && (nloc || nrem)) fail(SCENOPT_E_INVALID_PARAMS, "dev_create: internal schedule error (mixed dependency)");
        if (ld >= k) fail(SCENOPT_E_INVALID_PARAMS, "dev_create: internal schedule error (dependency order)");
        if (nrem) {
          r.gdep = 1;
          for (int c = lo; c < hi; ++c) {
            std::vector<Run>& owner = L[(*cta)[c]];
            owner[(*pos)[c]].publish = 1;
          }
        } else if (nloc) {
          r.ldep = ld;
        }
      }
  };

  std::vector<Lists> launch_lists;
  std::vector<std::pair<int, int>> full(static_cast<size_t>(p.N) + 1);
  for (int t = 0; t <= p.N; ++t) full[t] = {p.stage_offsets[t], p.stage_offsets[t + 1]};
  // Flattened forward top, and the owner rules (stage cut-1 items on the CTA
  // owning their first child); shared by the single-launch and sharded schedules.
  auto mark_flat = [&](Lists& fw_l, int cut) {
    for (auto& lst : fw_l) {
        std::vector<Run> out;
        for (const Run& r : lst) {
          const int st = p.node_stage[r.first];
          if (r.pass != 1 || st < 1 || st >= cut) {
            out.push_back(r);
            continue;
          }
          int a = r.first;  // split at parent boundaries: an item's nodes share their ancestors
          while (a < r.first + r.count) {
            int b2 = a + 1;
            while (b2 < r.first + r.count && p.ancestor[b2] == p.ancestor[a]) ++b2;
            Run q = r;
            q.first = a;
            q.count = b2 - a;
            q.flat = 1;
            out.push_back(q);
            a = b2;
          }
        }
        lst.swap(out);
      }
  };
  auto owner_fw = [&](Lists& fw_l, int cut) {
    // The flattened items of stage cut-1 go to the CTA that owns their first
    // child's subtree: that child's first local forward item then waits on a
    // CTA-local retire counter instead of a cross-CTA flag, and each CTA
    // computes exactly the parents its own subtrees need before starting its
    // local forward (round-robin tickets delayed CTAs holding four of them).
    if (d->flat_top) {
      std::vector<int> owner(static_cast<size_t>(n), -1);
      for (int gg = 0; gg < G; ++gg)
        for (const Run& r : fw_l[gg])
          if (r.pass == 1 && p.node_stage[r.first] == cut)
            for (int c = r.first; c < r.first + r.count; ++c) owner[c] = gg;
      std::vector<std::vector<Run>> moved(static_cast<size_t>(G));
      for (int gg = 0; gg < G; ++gg) {
        std::vector<Run> out;
        for (const Run& r : fw_l[gg]) {
          if (r.flat && p.node_stage[r.first] == cut - 1) {
            const int g2 = owner[p.child_begin[r.first]];
            moved[g2 >= 0 ? g2 : gg].push_back(r);
          } else {
            out.push_back(r);
          }
        }
        fw_l[gg].swap(out);
      }
      for (int gg = 0; gg < G; ++gg) {  // rank order: after the CTA's top tickets, before its local forward
        auto& mv = moved[gg];
        std::sort(mv.begin(), mv.end(), [](const Run& x, const Run& y) { return x.first < y.first; });
        auto& lst = fw_l[gg];
        size_t pos = 0;
        while (pos < lst.size() && p.node_stage[lst[pos].first] < cut) ++pos;
        lst.insert(lst.begin() + static_cast<std::ptrdiff_t>(pos), mv.begin(), mv.end());
      }
    }
  };
  auto owner_bw = [&](Lists& bw_l, int cut) {
    // Likewise the backward tickets of stage cut-1: a parent's children are
    // consecutive cut-stage nodes, mostly of one CTA, so the parent placed on
    // that CTA right after its local backward waits on the retire counter.
    // (Applying the rule level by level up to the root measured no faster.)
    if (cut >= 1) {
      const int lvl = cut - 1;
      std::vector<int> owner(static_cast<size_t>(n), -1);
      for (int gg = 0; gg < G; ++gg)
        for (const Run& r : bw_l[gg])
          if (r.pass == 0 && p.node_stage[r.first] == lvl + 1)
            for (int c = r.first; c < r.first + r.count; ++c) owner[c] = gg;
      std::vector<std::vector<Run>> moved(static_cast<size_t>(G));
      for (int gg = 0; gg < G; ++gg) {
        std::vector<Run> out;
        for (const Run& r : bw_l[gg]) {
          if (r.pass == 0 && p.node_stage[r.first] == lvl) {
            const int g2 = owner[p.child_begin[r.first]];
            moved[g2 >= 0 ? g2 : gg].push_back(r);
          } else {
            out.push_back(r);
          }
        }
        bw_l[gg].swap(out);
      }
      for (int gg = 0; gg < G; ++gg) {  // rank order: after the deeper backward items, before the upper tickets
        auto& mv = moved[gg];
        std::sort(mv.begin(), mv.end(), [](const Run& x, const Run& y) { return x.first < y.first; });
        auto& lst = bw_l[gg];
        size_t pos = 0;
        while (pos < lst.size() && p.node_stage[lst[pos].first] > lvl) ++pos;
        lst.insert(lst.begin() + static_cast<std::ptrdiff_t>(pos), mv.begin(), mv.end());
      }
    }
  };
  if (!shard) {
    Lists bw_l, fw_l;
    d->cut_stage = region(0, p.N, full, true, true, true, bw_l, fw_l);
    // Flattened forward top: with a host factor and a cut at
    // stage 2..4, every node above the cut computes x / u / Hx in one level
    // from its ancestors' u_off (affine maps precomputed below) as soon as the
    // backward root is done, instead of a chain of per-stage dependencies.
    const int cut = d->cut_stage;
    d->flat_top = cut >= 2 && cut <= 4 && env_int("SCENOPT_FLAT_TOP", 1) != 0;
    if (d->flat_top) {
      mark_flat(fw_l, cut);
      owner_fw(fw_l, cut);
    }
    owner_bw(bw_l, cut);
    for (int gg = 0; gg < G; ++gg) bw_l[gg].insert(bw_l[gg].end(), fw_l[gg].begin(), fw_l[gg].end());
    launch_lists.push_back(std::move(bw_l));
  } else {
    int s = shard->stage;
    const std::vector<int> bound = shard_plan(p, shard->world, &s);
    d->shard_stage = s;
    d->shard_lo = bound[shard->rank];
    d->shard_hi = bound[shard->rank + 1];
    d->sstage_lo = p.stage_offsets[s];
    d->sstage_hi = p.stage_offsets[s + 1];
    d->dual_top = p.dual_offset[p.stage_offsets[s]];
    const auto own = descend(d->shard_lo, d->shard_hi, s, p.N);
    d->own_range.assign(static_cast<size_t>(p.N) + 1, {0, 0});
    for (int t = 0; t <= p.N; ++t)
      d->own_range[t] = t < s ? std::make_pair(p.stage_offsets[t], p.stage_offsets[t + 1]) : own[t];
    {
      auto add = [](std::vector<std::pair<int64_t, int64_t>>& v, int64_t a, int64_t b) {
        if (b <= a) return;
        if (!v.empty() && v.back().second == a)
          v.back().second = b;
        else
          v.push_back({a, b});
      };
      auto rows = [&](int a, int b) {  // stage rows of nodes [a, b), and terminal rows of leaves
        if (b <= a) return;
        add(d->zero_x, static_cast<int64_t>(a) * nx, static_cast<int64_t>(b) * nx);
        if (a < p.first_leaf)
          add(d->zero_u, static_cast<int64_t>(a) * nu, static_cast<int64_t>(std::min(b, p.first_leaf)) * nu);
        add(d->zero_hx, p.dual_offset[a], p.dual_offset[b - 1] + p.stage_rows[b - 1]);
      };
      for (int t = s; t <= p.N; ++t) {
        const int lo = p.stage_offsets[t], hi = p.stage_offsets[t + 1];
        const int olo = own[t].first < own[t].second ? own[t].first : hi, ohi = own[t].first < own[t].second ? own[t].second : hi;
        rows(lo, olo);
        rows(ohi, hi);
      }
      auto trows = [&](int a, int b) {
        if (b > a)
          add(d->zero_hx, p.tdual_offset[a - p.first_leaf],
              p.tdual_offset[b - 1 - p.first_leaf] + p.terminal_rows[b - 1 - p.first_leaf]);
      };
      const int lo = p.stage_offsets[p.N], hi = p.stage_offsets[p.N + 1];
      const bool any = own[p.N].first < own[p.N].second;
      trows(lo, any ? own[p.N].first : hi);
      if (any) trows(own[p.N].second, hi);
    }
    Lists a_bw, a_fw, t_bw, t_fw, o_bw, o_fw;
    d->cut_stage = region(s, p.N, own, true, true, false, a_bw, a_fw);
    const int cut = d->cut_stage;
    owner_bw(a_bw, cut);
    launch_lists.push_back(std::move(a_bw));
    region(0, s - 1, full, false, true, true, t_bw, t_fw);
    region(s, p.N, own, true, false, true, o_bw, o_fw);
    // launch B: every flattened node waits on the (replicated) backward root
    d->flat_top = cut >= 2 && cut <= 4 && env_int("SCENOPT_FLAT_TOP", 1) != 0;
    if (d->flat_top) {
      mark_flat(t_fw, cut);
      mark_flat(o_fw, cut);
      owner_fw(o_fw, cut);
    }
    for (int gg = 0; gg < G; ++gg) {
      t_bw[gg].insert(t_bw[gg].end(), t_fw[gg].begin(), t_fw[gg].end());
      t_bw[gg].insert(t_bw[gg].end(), o_fw[gg].begin(), o_fw[gg].end());
    }
    launch_lists.push_back(std::move(t_bw));
  }
  std::vector<Run> runs;
  std::vector<std::vector<int32_t>> cta_offs;
  int nbw = 0;
  for (Lists& L : launch_lists) {
    resolve(L);
    std::vector<int32_t> off(static_cast<size_t>(G) + 1, 0);
    const int base = static_cast<int>(runs.size());
    for (int gg = 0; gg < G; ++gg) {
      off[gg] = static_cast<int32_t>(runs.size()) - base;
      for (const Run& r : L[gg]) {
        runs.push_back(r);
        nbw += r.pass == 0;
      }
    }
    off[G] = static_cast<int32_t>(runs.size()) - base;
    cta_offs.push_back(std::move(off));
  }
  d->items_bw = nbw;
  d->items_fw = static_cast<int>(runs.size()) - nbw;

  clk.mark("schedule");
  // flattened top nodes: (nx + m) columns over the ancestors' u_off (k nu,
  // padded) followed by the gain block
  if (d->flat_top)
    for (int c = 1; c < p.stage_offsets[d->cut_stage]; ++c)
      fws[c] = even(static_cast<int64_t>(nx + p.stage_rows[c]) * pad2(p.node_stage[c] * nu) +
                    static_cast<int64_t>(nxp) * nu);
  std::vector<Item> items(runs.size());
  std::vector<int64_t> item_doubles(runs.size());
  int64_t bw_total = 0, fw_total = 0, max_item = 2, max_stage = 16;
  int max_cnt = 1;
  const int hdr_per_node = static_cast<int>(sizeof(NodeMeta) / 8);
  for (size_t q = 0; q < runs.size(); ++q) {
    const Run& ru = runs[q];
    const std::vector<int64_t>& size = ru.pass == 0 ? bws : fws;
    int64_t tot = static_cast<int64_t>(ru.count) * hdr_per_node;
    for (int i = 0; i < ru.count; ++i) tot += size[ru.first + i];
    item_doubles[q] = tot;
    Item& it = items[q];
    it.bytes = static_cast<int32_t>(tot * 8);
    it.first = ru.first;
    it.count = ru.count;
    it.pass = ru.pass;
    const int last = ru.first + ru.count - 1;
    const bool leaf = ru.first >= p.first_leaf;
    it.leaf = leaf ? 1 : 0;
    it.ldep = ru.ldep;
    it.publish = ru.publish | (ru.pass == 1 ? (p.node_stage[ru.first] + 1) << 2 : 0);
    int64_t stage = 0;
    if (ru.pass == 0) {
      if (leaf) {
        it.dep_lo = it.dep_hi = 0;
        it.v0_lo = p.tdual_offset[ru.first - p.first_leaf];
        it.v0_n = p.tdual_offset[last - p.first_leaf] + p.terminal_rows[last - p.first_leaf] - it.v0_lo;
        it.v1_lo = it.v1_n = 0;
      } else {
        it.dep_lo = p.child_begin[ru.first];
        it.dep_hi = p.child_begin[last] + p.child_count[last];
        it.v0_lo = cdo[ru.first];
        it.v0_n = cdo[last] + M[last] - it.v0_lo;
        it.v1_lo = it.dep_lo;
        it.v1_n = it.dep_hi - it.dep_lo;
      }
      it.direct = it.v1_n > 2 * ru.count ? 1 : 0;  // > 2 children per node on average
      stage = kMaxRhs * (static_cast<int64_t>(it.v0_n) + (it.direct ? 0 : static_cast<int64_t>(it.v1_n) * W)) +
              static_cast<int64_t>(ru.count) * W;
    } else if (ru.flat) {  // flattened top: ancestors a_1 / a_2 in v0_lo / v0_n, the root is a_0
      const int k = p.node_stage[ru.first];
      const int par = p.ancestor[ru.first];
      it.dep_lo = 0;
      it.dep_hi = 1;
      it.v0_lo = k >= 2 ? (k == 2 ? par : p.ancestor[par]) : 0;
      it.v0_n = k >= 3 ? par : 0;
      it.v1_lo = ru.first;
      it.v1_n = ru.count;
      it.direct = kFlatTop | (k << 8);
      stage = kMaxRhs * (static_cast<int64_t>(pad2(k * nu)) + static_cast<int64_t>(ru.count) * nu) +
              static_cast<int64_t>(ru.count) * (nx + d->max_m);
    } else {
      if (ru.first == 0) {
        it.dep_lo = 0;
        it.dep_hi = 1;
        it.v0_lo = it.v0_n = 0;
      } else {
        it.dep_lo = p.ancestor[ru.first];
        it.dep_hi = p.ancestor[last] + 1;
        it.v0_lo = it.dep_lo;
        it.v0_n = it.dep_hi - it.dep_lo;
      }
      it.v1_lo = ru.first;
      it.v1_n = leaf ? 0 : ru.count;
      stage = kMaxRhs * (static_cast<int64_t>(it.v0_n) * Vp + static_cast<int64_t>(it.v1_n) * nu) +
              static_cast<int64_t>(ru.count) * nx;
    }
    if (!ru.gdep) it.dep_hi = it.dep_lo;  // dependencies inside the CTA: retire counter
    max_stage = std::max(max_stage, stage);
    max_item = std::max(max_item, tot);
    max_cnt = std::max(max_cnt, ru.count);
  }
  // Pass-array placement in "time-major" order: item k of every CTA, then
  // item k+1, ... CTAs advance through their lists at about the same rate, so
  // the blocks streamed concurrently by the grid are neighbours in HBM instead
  // of 148 far-apart streams.
  {
    size_t base = 0;
    for (const auto& off : cta_offs) {
      int longest = 0;
      for (int gg = 0; gg < G; ++gg) longest = std::max(longest, off[gg + 1] - off[gg]);
      auto place = [&](size_t q) {
        Item& it = items[q];
        int64_t& total = it.pass == 0 ? bw_total : fw_total;
        it.off = total;
        total += item_doubles[q];
      };
      for (int k = 0; k < longest; ++k)
        for (int gg = 0; gg < G; ++gg)
          if (off[gg] + k < off[gg + 1]) place(base + off[gg] + k);
      base += off[G];
    }
  }
  d->bw_doubles = bw_total;
  d->fw_doubles = fw_total;
  d->max_count = max_cnt;
  d->stage_doubles = static_cast<int>((max_stage + 15) & ~int64_t(15));
  d->vec_doubles = static_cast<int>((static_cast<int64_t>(max_cnt) * kMaxRhs * nxp + 15) & ~int64_t(15));

  clk.mark("items");
  // ---- pass arrays: [NodeMeta x count | node blocks] per item
  HostArray bw(static_cast<size_t>(bw_total), true), fw(static_cast<size_t>(fw_total), true);
  std::vector<double> aff_bw(static_cast<size_t>(n) * W, 0.0), aff_fw(static_cast<size_t>(n) * nx, 0.0);
  // flattened forward top (host factor): x_c = a'_c + sum_i G_{c,i} u_off(a_i)
  // by the recursion x_c = CL_c x_p + B_c u_off(p) + c_c (u_p = K_p x_p + u_off(p)):
  //   G_{c,i} = CL_c G_{p,i} (i < k-1), G_{c,k-1} = B_c, a'_c = CL_c a'_p + c_c, a'_0 = x_0;
  // stage rows z_c = F_c x_p + G'_c u_p = (F_c + G'_c K_p) x_p + G'_c u_off(p).
  std::vector<FlatTop> flat;
  std::vector<double> aff_fwh(static_cast<size_t>(n) * std::max(d->max_m, 1), 0.0);
  if (d->flat_top && !fz) {  // device factor: factor_flat (cuda/factor.cu) fills these after K9
    flat.resize(static_cast<size_t>(p.stage_offsets[d->cut_stage]));
    flat[0].a.assign(p.root_state.begin(), p.root_state.end());
    for (int c = 1; c < p.stage_offsets[d->cut_stage]; ++c) {
      const int k = p.node_stage[c], pr = p.ancestor[c], mm = p.stage_rows[c];
      const FlatTop& fp = flat[pr];
      FlatTop& ft = flat[c];
      const double* CL = f.closed_loop.data() + static_cast<size_t>(c) * nx * nx;
      const double* Bc = p.Bi(c);
      ft.G.assign(static_cast<size_t>(k) * nu * nx, 0.0);  // k matrices nx x nu, column-major
      for (int i = 0; i + 1 < k; ++i)
        for (int j = 0; j < nu; ++j)
          for (int r = 0; r < nx; ++r) {
            double s2 = 0.0;
            for (int z = 0; z < nx; ++z) s2 += CL[r + static_cast<size_t>(z) * nx] * fp.G[(static_cast<size_t>(i) * nu + j) * nx + z];
            ft.G[(static_cast<size_t>(i) * nu + j) * nx + r] = s2;
          }
      for (int j = 0; j < nu; ++j)
        for (int r = 0; r < nx; ++r) ft.G[(static_cast<size_t>(k - 1) * nu + j) * nx + r] = Bc[r + static_cast<size_t>(j) * nx];
      ft.a.assign(static_cast<size_t>(nx), 0.0);
      const double* cc = p.ci(c);
      for (int r = 0; r < nx; ++r) {
        double s2 = cc[r];
        for (int z = 0; z < nx; ++z) s2 += CL[r + static_cast<size_t>(z) * nx] * fp.a[z];
        ft.a[r] = s2;
      }
      // stage rows: M = F_c + G'_c K_p (m x nx)
      const double* Fm = p.Fi(c);
      const double* Gm = p.Gi(c);
      const double* Kp = f.gain.data() + static_cast<size_t>(pr) * nu * nx;
      std::vector<double> Mf(static_cast<size_t>(mm) * nx);
      for (int z = 0; z < nx; ++z)
        for (int q = 0; q < mm; ++q) {
          double s2 = Fm[q + static_cast<size_t>(z) * mm];
          for (int w = 0; w < nu; ++w) s2 += Gm[q + static_cast<size_t>(w) * mm] * Kp[w + static_cast<size_t>(z) * nu];
          Mf[q + static_cast<size_t>(z) * mm] = s2;
        }
      ft.L.assign(static_cast<size_t>(k) * nu * mm, 0.0);  // k matrices m x nu
      for (int i = 0; i + 1 < k; ++i)
        for (int j = 0; j < nu; ++j)
          for (int q = 0; q < mm; ++q) {
            double s2 = 0.0;
            for (int z = 0; z < nx; ++z) s2 += Mf[q + static_cast<size_t>(z) * mm] * fp.G[(static_cast<size_t>(i) * nu + j) * nx + z];
            ft.L[(static_cast<size_t>(i) * nu + j) * mm + q] = s2;
          }
      for (int j = 0; j < nu; ++j)
        for (int q = 0; q < mm; ++q) ft.L[(static_cast<size_t>(k - 1) * nu + j) * mm + q] = Gm[q + static_cast<size_t>(j) * mm];
      ft.h.assign(static_cast<size_t>(mm), 0.0);
      for (int q = 0; q < mm; ++q) {
        double s2 = 0.0;
        for (int z = 0; z < nx; ++z) s2 += Mf[q + static_cast<size_t>(z) * mm] * fp.a[z];
        ft.h[q] = s2;
      }
    }
  }
  // per-node block positions (the device factor writes E / J / K in place)
  d->h_bw_off.assign(static_cast<size_t>(n), -1);
  d->h_bw_j.assign(static_cast<size_t>(n), -1);
  d->h_k_off.assign(static_cast<size_t>(n), -1);
  d->h_flat_off.assign(static_cast<size_t>(n), -1);
  parallel_for(static_cast<int>(items.size()), 64, [&](int qb, int qe) {
    for (int q = qb; q < qe; ++q) {
      const Item& it = items[q];
      double* base = (it.pass == 0 ? bw.data() : fw.data()) + it.off;
      NodeMeta* hdr = reinterpret_cast<NodeMeta*>(base);
      int64_t blk = static_cast<int64_t>(it.count) * hdr_per_node;
      for (int i = 0; i < it.count; ++i) {
        const int c = it.first + i;
        const bool leaf = c >= p.first_leaf;
        const int mm = c == 0 ? 0 : p.stage_rows[c];
        const int mN = leaf ? p.terminal_rows[c - p.first_leaf] : 0;
        NodeMeta mt{};
        mt.c = c;
        mt.blk = static_cast<int32_t>(blk);
        mt.M = M[c];
        mt.m = mm;
        mt.mN = mN;
        mt.doff = c == 0 ? 0 : p.dual_offset[c];
        mt.tdo = leaf ? p.tdual_offset[c - p.first_leaf] : 0;
        if (it.pass == 0) {
          mt.yoff = leaf ? mt.tdo - it.v0_lo : cdo[c] - it.v0_lo;
          mt.kid0 = leaf ? 0 : p.child_begin[c] - it.v1_lo;
          mt.nkid = leaf ? 0 : p.child_count[c];
        } else {
          mt.par = c == 0 ? 0 : p.ancestor[c] - it.v0_lo;
        }
        hdr[i] = mt;
        double* B0 = base + blk;
        if (it.pass == 0) {
          int64_t jo = 0;
          if (!leaf && fz) {
            jo = even(static_cast<int64_t>(M[c]) * W);
          } else if (!leaf) {
            const double* d2i = f.dual_to_input.data() + static_cast<size_t>(cdo[c]) * nu;
            const double* d2c = f.dual_to_costate.data() + static_cast<size_t>(cdo[c]) * nx;
            for (int k = 0; k < M[c]; ++k) {
              for (int j = 0; j < nu; ++j) B0[k + static_cast<int64_t>(j) * M[c]] = d2i[j + static_cast<int64_t>(k) * nu];
              for (int t = 0; t < nx; ++t)
                B0[k + static_cast<int64_t>(nu + t) * M[c]] = d2c[t + static_cast<int64_t>(k) * nx];
            }
            jo = even(static_cast<int64_t>(M[c]) * W);
            const double* ia = f.input_affine.data() + static_cast<size_t>(c) * nu;
            const double* ca = f.costate_affine.data() + static_cast<size_t>(c) * nx;
            for (int j = 0; j < nu; ++j) aff_bw[static_cast<size_t>(c) * W + j] = ia[j];
            for (int t = 0; t < nx; ++t) aff_bw[static_cast<size_t>(c) * W + nu + t] = ca[t];
          } else {
            const int l = c - p.first_leaf;
            const double* FN = p.FNl(l);
            std::copy(FN, FN + static_cast<size_t>(mN) * nx, B0);
            jo = even(static_cast<int64_t>(mN) * nx);
            if (!fz) {
              const double* lca = f.leaf_costate_affine.data() + static_cast<size_t>(l) * nx;
              for (int t = 0; t < nx; ++t) aff_bw[static_cast<size_t>(c) * W + nu + t] = lca[t];
            }
          }
          d->h_bw_off[c] = it.off + blk;
          d->h_bw_j[c] = it.off + blk + jo;
          if (c != 0 && !fz) {
            double* J = B0 + jo;
            const double* c2i = f.child_to_input.data() + static_cast<size_t>(c) * nu * nx;
            const double* cl = f.closed_loop.data() + static_cast<size_t>(c) * nx * nx;
            for (int k = 0; k < nx; ++k) {
              for (int j = 0; j < nu; ++j) J[k + static_cast<int64_t>(j) * nxp] = c2i[j + static_cast<int64_t>(k) * nu];
              for (int t = 0; t < nx; ++t) J[k + static_cast<int64_t>(nu + t) * nxp] = cl[k + static_cast<int64_t>(t) * nx];
            }
          }
          blk += bws[c];
        } else if (it.direct & kFlatTop) {
          // x_c = a'_c + sum_i G_{c,i} u_off(a_i); z_c = h'_c + sum_i L_{c,i} u_off(a_i)
          const int k = p.node_stage[c];
          const int Lp = pad2(k * nu);
          d->h_flat_off[c] = it.off + blk;
          const int64_t ko = static_cast<int64_t>(Lp) * (nx + mm);
          d->h_k_off[c] = it.off + blk + ko;
          if (fz) {
            blk += fws[c];
            continue;
          }
          const FlatTop& ft = flat[c];
          for (int r = 0; r < nx + mm; ++r) {
            double* col = B0 + static_cast<int64_t>(r) * Lp;
            for (int i = 0; i < k; ++i)
              for (int j = 0; j < nu; ++j)
                col[i * nu + j] = r < nx ? ft.G[(static_cast<size_t>(i) * nu + j) * nx + r]
                                         : ft.L[(static_cast<size_t>(i) * nu + j) * mm + (r - nx)];
          }
          for (int t = 0; t < nx; ++t) aff_fw[static_cast<size_t>(c) * nx + t] = ft.a[t];
          for (int s2 = 0; s2 < mm; ++s2) aff_fwh[static_cast<size_t>(c) * d->max_m + s2] = ft.h[s2];
          double* K = B0 + ko;
          const double* gain = f.gain.data() + static_cast<size_t>(c) * nu * nx;
          for (int j = 0; j < nu; ++j)
            for (int kk = 0; kk < nx; ++kk) K[kk + static_cast<int64_t>(j) * nxp] = gain[j + static_cast<int64_t>(kk) * nu];
          blk += fws[c];
        } else {
          int64_t ko = 0;
          if (c != 0) {
            const double* A = p.Ai(c);
            const double* Bm = p.Bi(c);
            const double* Fm = p.Fi(c);
            const double* Gm = p.Gi(c);
            for (int r = 0; r < nx; ++r) {
              double* col = B0 + static_cast<int64_t>(r) * Vp;
              for (int k = 0; k < nx; ++k) col[k] = A[r + static_cast<int64_t>(k) * nx];
              for (int k = 0; k < nu; ++k) col[nx + k] = Bm[r + static_cast<int64_t>(k) * nx];
            }
            for (int s2 = 0; s2 < mm; ++s2) {
              double* col = B0 + static_cast<int64_t>(nx + s2) * Vp;
              for (int k = 0; k < nx; ++k) col[k] = Fm[s2 + static_cast<int64_t>(k) * mm];
              for (int k = 0; k < nu; ++k) col[nx + k] = Gm[s2 + static_cast<int64_t>(k) * mm];
            }
            ko = static_cast<int64_t>(Vp) * (nx + mm);
            const double* cc = p.ci(c);
            for (int t = 0; t < nx; ++t) aff_fw[static_cast<size_t>(c) * nx + t] = cc[t];
          }
          double* K = B0 + ko;
          d->h_k_off[c] = it.off + blk + ko;
          if (!leaf && fz) {
          } else if (!leaf) {
            const double* gain = f.gain.data() + static_cast<size_t>(c) * nu * nx;
            for (int j = 0; j < nu; ++j)
              for (int k = 0; k < nx; ++k) K[k + static_cast<int64_t>(j) * nxp] = gain[j + static_cast<int64_t>(k) * nu];
          } else {
            const double* FN = p.FNl(c - p.first_leaf);
            for (int s2 = 0; s2 < mN; ++s2)
              for (int k = 0; k < nx; ++k) K[k + static_cast<int64_t>(s2) * nxp] = FN[s2 + static_cast<int64_t>(k) * mN];
          }
          blk += fws[c];
        }
      }
    }
  });

  clk.mark("pack");
  // ---- launch configuration: one co-resident CTA per SM. Preference order:
  //   1. producer-staged vectors, every item's blocks in a shared-memory slot,
  //      the deepest slot ring (<= 5) that fits;
  //   2. producer-staged, 4 slots sized for the small items: larger items keep
  //      their blocks in HBM (only the node headers are copied; kGlobalBlocks);
  //   3./4. the same with consumer-staged vectors (one staging area per team
  //      instead of the producers' staging ring) for very wide states.
  // SCENOPT_NSLOT / SCENOPT_SLOT_KB / SCENOPT_STAGE=consumer force choices (tests).
  // Kernel geometry: large trees whose items carry many nodes (small states,
  // nx ~ 10) are limited by the producers' staging of many short vectors per
  // item and take six producer warps; one-node items (C3, C4) and small,
  // latency-bound trees keep four (profiles/c5_geometry_r02.md). Both
  // compute bitwise-identical results. SCENOPT_SWEEP_PRODUCERS=4|6 forces one (tests).
  const int force_geom = env_int("SCENOPT_SWEEP_PRODUCERS", 0);
  const bool many = d->max_count >= kManyNodeItems && packed_bytes >= kLatencyBoundBytes;
  const int dbl = 8;
  const int force_ns = env_int("SCENOPT_NSLOT", 0);
  const int64_t slot_cap_env = static_cast<int64_t>(env_int("SCENOPT_SLOT_KB", 0)) * 1024 / 8;
  const bool force_consumer = std::getenv("SCENOPT_STAGE") && std::string(std::getenv("SCENOPT_STAGE")) == "consumer";
  const int64_t hdr_doubles_max = static_cast<int64_t>(d->max_count) * (sizeof(NodeMeta) / 8);
  const int ns_max = std::min(kMaxSlots, 5);
  struct Fit {
    int ns = 0;  // 0: no layout
    int64_t slot = 0;
    bool consumer = false;
    size_t smem = 0;
  };
  auto smem_for = [&](const SweepImpl& sw, int ns, int64_t slot, bool consumer) {
    return (static_cast<size_t>(ns) * slot + static_cast<size_t>(consumer ? sw.teams : sw.stage_queue) * d->stage_doubles +
            static_cast<size_t>(sw.teams) * sw.scratch_bufs * d->vec_doubles) * dbl;
  };
  auto fit_for = [&](const SweepImpl& sw) {
    const size_t optin = static_cast<size_t>(prop.sharedMemPerBlockOptin) - sw.static_smem();
    auto fits = [&](int ns, int64_t sl, bool cons) {
      const size_t smem = smem_for(sw, ns, sl, cons);
      if (smem > optin) return false;
      SCN_CUDA(sw.configure(smem));
      int cps = 0;
      SCN_CUDA(sw.occupancy(&cps, smem));
      return cps >= 1;
    };
    Fit f;
    for (int pass = 0; pass < 2 && !f.ns; ++pass) {
      const bool cons = pass == 1 || force_consumer;
      if (pass == 1 && force_consumer) break;
      // all items in smem
      if (!slot_cap_env)
        for (int ns = ns_max; ns >= 2; --ns) {
          if (force_ns && ns != force_ns) continue;
          const int64_t sl = (std::max<int64_t>(max_item, 2) + 15) & ~int64_t(15);
          if (fits(ns, sl, cons)) {
            f.ns = ns, f.slot = sl, f.consumer = cons;
            break;
          }
        }
      if (f.ns) break;
      // small items in smem, large ones from HBM. What the staging areas and
      // scratch leave is computed signed: when the (producer) staging ring alone
      // exceeds shared memory this pass cannot work (pass 1 stages per team);
      // a slot must hold at least the node headers of the largest item.
      const int ns = force_ns ? force_ns : 4;
      const int64_t left = static_cast<int64_t>(optin / dbl) -
                           static_cast<int64_t>(cons ? sw.teams : sw.stage_queue) * d->stage_doubles -
                           static_cast<int64_t>(sw.teams) * sw.scratch_bufs * d->vec_doubles;
      const int64_t hdr_slot = (hdr_doubles_max + 15) & ~int64_t(15);
      int64_t sl = slot_cap_env ? slot_cap_env : (left / ns) & ~int64_t(15);
      sl = std::max<int64_t>(sl, hdr_slot);
      if (sl <= (int64_t(1) << 26) && static_cast<int64_t>(ns) * sl <= left && fits(ns, sl, cons))
        f.ns = ns, f.slot = sl, f.consumer = cons;
    }
    if (f.ns) f.smem = smem_for(sw, f.ns, f.slot, f.consumer);
    return f;
  };
  // Kernel geometry: large trees whose items carry many nodes (small states,
  // nx ~ 10) are limited by the producers' staging of many short vectors per
  // item and take six producer warps, unless their deeper staging ring would
  // cost slots; one-node items (C3, C4) and small, latency-bound trees keep
  // four (profiles/c5_geometry_r02.md). Both geometries compute
  // bitwise-identical results. SCENOPT_SWEEP_PRODUCERS=4|6 forces one (tests).
  Fit fit;
  if (force_geom == 6 || (force_geom != 4 && many)) {
    fit = fit_for(kSweepProducers6);
    d->sweep = &kSweepProducers6;
    if (force_geom != 6) {
      const Fit f4 = fit_for(kSweepProducers4);
      if (!fit.ns || fit.ns < f4.ns || fit.consumer != f4.consumer) fit = f4, d->sweep = &kSweepProducers4;
    }
  } else {
    fit = fit_for(kSweepProducers4);
    d->sweep = &kSweepProducers4;
  }
  const SweepImpl& sw = *d->sweep;
  if (fit.ns == 0)
    fail(SCENOPT_E_INVALID_PARAMS, "dev_create: the per-item staging vectors do not fit in shared memory (" +
                                       std::to_string(smem_for(sw, 2, hdr_doubles_max, true)) + " bytes)");
  const int best_ns = fit.ns;
  const int64_t slot = fit.slot;
  const bool consumer = fit.consumer;
  d->slot_doubles = static_cast<int>(slot);
  d->consumer_stage = consumer;
  int n_global = 0;
  for (Item& it : items)
    if (it.bytes > slot * dbl) {  // blocks stay in HBM; copy only the node headers
      it.direct |= kGlobalBlocks;
      it.bytes = static_cast<int32_t>(it.count * sizeof(NodeMeta));
      ++n_global;
    }
  d->items_global = n_global;
  d->nslot = best_ns;
  d->ctas_per_sm = 1;
  d->dyn_smem = fit.smem;
  SCN_CUDA(sw.configure(d->dyn_smem));
  d->G = 0;

  clk.mark("launch config");
  // ---- upload
  d->bw_blk = upload(*d, bw);
  d->fw_blk = upload(*d, fw);
  bw.release();
  fw.release();
  d->aff_bw = upload(*d, aff_bw);
  d->aff_fw = upload(*d, aff_fw);
  d->aff_fwh = upload(*d, aff_fwh);
  d->root_state = upload(*d, p.root_state);
  {
    size_t base = 0;
    for (const auto& off : cta_offs) {
      DevState::Launch ln;
      ln.count = off.back();
      ln.items = upload(*d, std::vector<Item>(items.begin() + base, items.begin() + base + ln.count));
      ln.cta_off = upload(*d, off);
      d->launches.push_back(ln);
      base += ln.count;
    }
  }
  d->ctrl = d->alloc<unsigned>(4);
  d->bw_flag = d->alloc<unsigned>(static_cast<size_t>(n));
  d->fw_flag = d->alloc<unsigned>(static_cast<size_t>(n));
  SCN_CUDA(cudaMemset(d->ctrl, 0, 4 * sizeof(unsigned)));
  SCN_CUDA(cudaMemset(d->bw_flag, 0, static_cast<size_t>(n) * sizeof(unsigned)));
  SCN_CUDA(cudaMemset(d->fw_flag, 0, static_cast<size_t>(n) * sizeof(unsigned)));

  std::vector<char> mine;
  if (d->sharded())  // nodes whose cost this rank evaluates: own subtrees, top on rank 0
    mine = shard_nodes(p, d->shard_stage, d->shard_lo, d->shard_hi, shard->rank);
  clk.mark("upload blocks");
  std::vector<char> held;  // cost blocks kept: own subtrees, the top and every shard-stage node
  if (d->sharded()) {
    held = mine;
    for (int c = 0; c < d->sstage_hi; ++c) held[c] = 1;
    if (!p.held.empty())  // a shard's instance must hold what this rank packs
      for (int c = 0; c < n; ++c)
        if (held[c] && !p.held[c])
          fail(SCENOPT_E_INVALID_PARAMS, "dev_create_sharded: the instance does not hold node " + std::to_string(c) +
                                             " of this rank's shard (generated for another rank or plan?)");
  }
  pack_common(*d, p, d->sharded() ? &mine : nullptr, d->sharded() ? &held : nullptr);
  clk.mark("pack_common");
  const int D = p.dual_dim;
  if (d->sharded()) {
    d->rank = shard->rank;
    d->world = shard->world;
    // rows / nodes this rank owns (counted in reductions and gathers): its
    // subtrees' stage and terminal rows, and the replicated top on rank 0
    std::vector<uint8_t> cnt = shard_rows(p, mine);
    if (cnt.empty()) cnt.push_back(0);
    auto add = [](std::vector<std::pair<int64_t, int64_t>>& v, int64_t a, int64_t b) {
      if (b <= a) return;
      if (!v.empty() && v.back().second == a)
        v.back().second = b;
      else
        v.push_back({a, b});
    };
    for (int i = 0; i < D; ++i)
      if (cnt[i]) add(d->keep_y, i, i + 1);
    for (int c = 0; c < n; ++c)
      if (mine[c]) {
        add(d->keep_x, static_cast<int64_t>(c) * nx, static_cast<int64_t>(c + 1) * nx);
        if (c < p.first_leaf) add(d->keep_u, static_cast<int64_t>(c) * nu, static_cast<int64_t>(c + 1) * nu);
      }
    d->row_counted = upload(*d, cnt);
    const int last = d->sstage_hi - 1;
    d->dual_s_end = p.dual_offset[last] + p.stage_rows[last];
    d->xbuf_rhs = static_cast<int64_t>(d->sstage_hi - d->sstage_lo) * W + (d->dual_s_end - d->dual_top);
    d->xbuf = d->alloc<double>(static_cast<size_t>(kMaxRhs) * d->xbuf_rhs);
    for (int r = 0; r < kMaxRhs; ++r) d->ycomp[r] = d->alloc<double>(static_cast<size_t>(std::max(D, 1)));
    d->gx = d->alloc<double>(static_cast<size_t>(n) * nx);
    d->gu = d->alloc<double>(static_cast<size_t>(std::max(p.first_leaf, 1)) * nu);
    d->gy = d->alloc<double>(static_cast<size_t>(std::max(D, 1)));
    if (shard->emu)
      d->comm = emu_comm(shard->emu, shard->rank);
    else if (shard->nccl_id)
      d->comm = nccl_comm(device, shard->rank, shard->world, shard->nccl_id);
    // else: exchange left to the caller (phase API)
  }

  // fused FB-step finish (SweepParams::fb_*): per CTA, the stage rows of the
  // nodes of its forward items and the terminal rows of its leaves (each dual
  // row once over the grid), in item order; per-CTA partials
  if (d->launches.size() == 1) {
    const std::vector<int>& off = cta_offs[0];
    std::vector<int32_t> rows, roff(static_cast<size_t>(G) + 1, 0);
    rows.reserve(static_cast<size_t>(std::max(D, 0)));
    for (int gg = 0; gg < G; ++gg) {
      for (int q = off[gg]; q < off[gg + 1]; ++q) {
        const Item& it = items[q];
        if (it.pass != 1) continue;
        for (int c = it.first; c < it.first + it.count; ++c) {
          if (c > 0)
            for (int r = 0; r < p.stage_rows[c]; ++r) rows.push_back(p.dual_offset[c] + r);
          if (c >= p.first_leaf) {
            const int l = c - p.first_leaf;
            for (int r = 0; r < p.terminal_rows[l]; ++r) rows.push_back(p.tdual_offset[l] + r);
          }
        }
      }
      roff[gg + 1] = static_cast<int32_t>(rows.size());
    }
    if (static_cast<int64_t>(rows.size()) != static_cast<int64_t>(D))
      fail(SCENOPT_E_ERROR, "dev_create: the forward items do not cover every dual row once");
    d->fb_rows = upload(*d, rows);
    d->fb_rows_off = upload(*d, roff);
    d->fb_part = d->alloc<double>(static_cast<size_t>(G) * 8);
  }
  for (int r = 0; r < kMaxRhs; ++r) {
    d->contrib[r] = d->alloc<double>(static_cast<size_t>(n) * W);
    d->uoff[r] = d->alloc<double>(static_cast<size_t>(std::max(p.first_leaf, 1)) * nu);
    d->xs[r] = d->alloc<double>(static_cast<size_t>(n) * nx);
    d->us[r] = d->alloc<double>(static_cast<size_t>(std::max(p.first_leaf, 1)) * nu);
    d->hs[r] = d->alloc<double>(static_cast<size_t>(std::max(D, 1)));
    d->ys[r] = d->alloc<double>(static_cast<size_t>(std::max(D, 1)));
  }

  // ---- algorithmic bytes per sweep, SURVEY.md §8(d) / DESIGN.md §Roofline:
  // every matrix read once, every vector touched once (fp64).
  //   B_hom = 8 [(n-1)(2nx^2 + 2nx nu) + F nu nx + 2 sum_i m_i (nx+nu)
  //              + 2 sum_l mN_l nx] + B_vec,  B_vec = 8 (4 n nx + 3 F nu + 2 m)
  //   B_aff = B_hom + 8 [F (nx+nu) + S nx + (n-1) nx]
  //   B_hom2 (two right-hand sides) = matrices once + 2 B_vec
  const int64_t F = p.first_leaf, S = p.L, m = D;
  int64_t stage_rows_total = 0, term_rows_total = 0;
  for (int c = 1; c < n; ++c) stage_rows_total += p.stage_rows[c];
  for (int l = 0; l < p.L; ++l) term_rows_total += p.terminal_rows[l];
  const int64_t mat = static_cast<int64_t>(n - 1) * (2LL * nx * nx + 2LL * nx * nu) + F * nu * nx +
                      2 * stage_rows_total * (nx + nu) + 2 * term_rows_total * nx;
  const int64_t vec = 4LL * n * nx + 3 * F * nu + 2 * m;
  d->bytes_hom = 8 * (mat + vec);
  d->bytes_aff = d->bytes_hom + 8 * (F * (nx + nu) + S * nx + static_cast<int64_t>(n - 1) * nx);
  d->bytes_hom2 = 8 * (mat + 2 * vec);
  SCN_CUDA(cudaDeviceSynchronize());
  return d;
}

namespace {
// Per-dual-row nonsmooth data, apply_H rows and eval_f cost blocks: what
// every handle needs, with or without the sweep layout.
// mine: the nodes whose cost this handle evaluates (eval_f); held: the nodes
// whose cost blocks it keeps (the device factor's inputs). Null: all nodes.
void pack_common(DevState& dd, const Problem& p, const std::vector<char>* mine, const std::vector<char>* held) {
  DevState* d = &dd;
  const int n = p.n, nx = p.nx, nu = p.nu, D = p.dual_dim, V = nx + nu;
  std::vector<int8_t> kind(static_cast<size_t>(D), 0);
  std::vector<double> lo(static_cast<size_t>(D), 0.0), hi(static_cast<size_t>(D), 0.0),
      wg(static_cast<size_t>(D), 0.0);
  std::vector<int32_t> rnode(static_cast<size_t>(D), 0);
  std::vector<int8_t> rterm(static_cast<size_t>(D), 0);
  std::vector<double> coef(static_cast<size_t>(D) * V, 0.0);
  for (int i = 1; i < n; ++i) {
    const int m = p.stage_rows[i];
    const double* F = p.Fi(i);
    const double* G = p.Gi(i);
    for (int k = 0; k < m; ++k) {
      const int row = p.dual_offset[i] + k;
      kind[row] = static_cast<int8_t>(p.g_kind[i]);
      lo[row] = p.zmin[row];
      hi[row] = p.zmax[row];
      wg[row] = p.probability[i] * p.g_gamma[i];
      rnode[row] = p.ancestor[i];
      double* cf = coef.data() + static_cast<size_t>(row) * V;
      for (int t = 0; t < nx; ++t) cf[t] = F[k + static_cast<size_t>(t) * m];
      for (int t = 0; t < nu; ++t) cf[nx + t] = G[k + static_cast<size_t>(t) * m];
    }
  }
  for (int l = 0; l < p.L; ++l) {
    const int m = p.terminal_rows[l];
    const double* FN = p.FNl(l);
    for (int k = 0; k < m; ++k) {
      const int row = p.tdual_offset[l] + k;
      kind[row] = static_cast<int8_t>(p.tg_kind[l]);
      lo[row] = p.zmin[row];
      hi[row] = p.zmax[row];
      wg[row] = p.probability[p.first_leaf + l] * p.tg_gamma[l];
      rnode[row] = p.first_leaf + l;
      rterm[row] = 1;
      double* cf = coef.data() + static_cast<size_t>(row) * V;
      for (int t = 0; t < nx; ++t) cf[t] = FN[k + static_cast<size_t>(t) * m];
    }
  }
  d->row_kind = upload(*d, kind);
  d->row_lo = upload(*d, lo);
  d->row_hi = upload(*d, hi);
  d->row_wg = upload(*d, wg);
  d->hrows.nx = nx;
  d->hrows.nu = nu;
  d->hrows.nrows = D;
  d->hrows.row_node = upload(*d, rnode);
  d->hrows.row_term = upload(*d, rterm);
  d->hrows.coef = upload(*d, coef);
  // cost blocks: [A | B | c | Q | S | R | q | r] per non-root node, [P | p] per
  // leaf. A sharded handle holds its subtrees, the replicated top and the
  // shard-stage nodes (the device factor of the top reads them), and
  // evaluates f over its subtrees (plus the top on rank 0); the partial sums
  // are reduced over the ranks.
  std::vector<int32_t> nodes, leaves, hnodes, hleaves;
  std::vector<int32_t> slot(static_cast<size_t>(n), -1), lslot(static_cast<size_t>(std::max(p.L, 1)), -1);
  for (int i = 1; i < n; ++i) {
    if (!mine || (*mine)[i]) nodes.push_back(i);
    if (!held || (*held)[i]) {
      slot[i] = static_cast<int32_t>(hnodes.size());
      hnodes.push_back(i);
    }
  }
  for (int l = 0; l < p.L; ++l) {
    if (!mine || (*mine)[p.first_leaf + l]) leaves.push_back(p.first_leaf + l);
    if (!held || (*held)[p.first_leaf + l]) {
      lslot[l] = static_cast<int32_t>(hleaves.size());
      hleaves.push_back(p.first_leaf + l);
    }
  }
  const size_t csz = 2 * p.sxx() + 2 * p.sxu() + p.suu() + 2 * static_cast<size_t>(nx) + nu;
  HostArray cn(std::max<size_t>(hnodes.size(), 1) * csz, hnodes.empty());  // every block fully written below
  parallel_for(static_cast<int>(hnodes.size()), 256, [&](int b, int e) {
    for (int t = b; t < e; ++t) {
      const int i = hnodes[t];
      double* o = cn.data() + static_cast<size_t>(t) * csz;
      o = std::copy(p.Ai(i), p.Ai(i) + p.sxx(), o);
      o = std::copy(p.Bi(i), p.Bi(i) + p.sxu(), o);
      o = std::copy(p.ci(i), p.ci(i) + nx, o);
      o = std::copy(p.Qi(i), p.Qi(i) + p.sxx(), o);
      o = std::copy(p.Si(i), p.Si(i) + p.sxu(), o);
      o = std::copy(p.Ri(i), p.Ri(i) + p.suu(), o);
      o = std::copy(p.qi(i), p.qi(i) + nx, o);
      std::copy(p.ri(i), p.ri(i) + nu, o);
    }
  });
  const size_t lsz = p.sxx() + static_cast<size_t>(nx);
  HostArray cl(std::max<size_t>(hleaves.size(), 1) * lsz, hleaves.empty());
  for (size_t t = 0; t < hleaves.size(); ++t) {
    const int l = hleaves[t] - p.first_leaf;
    double* o = cl.data() + t * lsz;
    o = std::copy(p.Pl(l), p.Pl(l) + p.sxx(), o);
    std::copy(p.pl(l), p.pl(l) + nx, o);
  }
  d->cost.nx = nx;
  d->cost.nu = nu;
  d->cost.n = n;
  d->cost.first_leaf = p.first_leaf;
  d->cost.anc = upload(*d, p.ancestor);
  d->cost.prob = upload(*d, p.probability);
  d->cost.nodes = upload(*d, nodes);
  d->cost.nnodes = static_cast<int>(nodes.size());
  d->cost.node = upload(*d, cn);
  d->cost.slot = upload(*d, slot);
  d->cost.leaves = upload(*d, leaves);
  d->cost.nleaves = static_cast<int>(leaves.size());
  d->cost.leaf = upload(*d, cl);
  d->cost.lslot = upload(*d, lslot);
  d->cost.check_root = (!mine || (*mine)[0]) ? 1 : 0;
  d->cost.root_state = upload(*d, p.root_state);
  if (!d->root_state) d->root_state = const_cast<double*>(d->cost.root_state);
  if (!d->has_factor)
    for (int r = 0; r < kMaxRhs; ++r) {
      d->xs[r] = d->alloc<double>(static_cast<size_t>(n) * nx);
      d->us[r] = d->alloc<double>(static_cast<size_t>(std::max(p.first_leaf, 1)) * nu);
      d->hs[r] = d->alloc<double>(static_cast<size_t>(std::max(D, 1)));
      d->ys[r] = d->alloc<double>(static_cast<size_t>(std::max(D, 1)));
    }
}
}  // namespace

namespace {
SweepParams sweep_params(DevState& d, int nrhs, bool affine, const double* const* y, double* const* x,
                         double* const* u, double* const* Hx) {
  if (nrhs < 1 || nrhs > kMaxRhs) fail(SCENOPT_E_INVALID_PARAMS, "sweep: nrhs must be 1 or 2");
  if (!d.has_factor) fail(SCENOPT_E_CACHE_MISMATCH, "sweep: handle was created without a factor cache");
  const Layout& L = d.lay;
  SweepParams P{};
  P.nx = L.nx;
  P.nu = L.nu;
  P.n = L.n;
  P.first_leaf = L.first_leaf;
  P.dual_dim = L.dual_dim;
  P.nslot = d.nslot;
  P.slot_doubles = d.slot_doubles;
  P.stage_doubles = d.stage_doubles;
  P.scratch_doubles = d.vec_doubles;
  P.nrhs = nrhs;
  P.affine = affine ? 1 : 0;
  P.G = d.G;
  P.max_count = d.max_count;
  P.nxp = d.nxp;
  P.Vp = d.Vp;
  P.consumer_stage = d.consumer_stage ? 1 : 0;
  P.global_blocks = d.items_global > 0 ? 1 : 0;
  P.bw_blk = d.bw_blk;
  P.fw_blk = d.fw_blk;
  P.aff_bw = d.aff_bw;
  P.aff_fw = d.aff_fw;
  P.aff_fwh = d.aff_fwh;
  P.mmax = d.max_m;
  P.root_state = d.root_state;
  P.ctrl = d.ctrl;
  P.skip = d.sweep_skip;
  P.bw_flag = d.bw_flag;
  P.fw_flag = d.fw_flag;
  if (d.fb_next) {
    if (nrhs != 1 || !affine || d.sharded() || !d.fb_part)
      fail(SCENOPT_E_INVALID_PARAMS, "sweep: the fused FB finish needs a 1-RHS affine sweep of an unsharded handle");
    const DevState::FbFuse& f = *d.fb_next;
    P.fb_S = f.S;
    P.fb_I = f.I;
    P.fb_state = f.state;
    P.fb_Hx0 = f.Hx0;
    P.fb_weight = f.weight;
    P.fb_z = f.z;
    P.fb_R = f.R;
    P.fb_T = f.T;
    P.fb_kind = d.row_kind;
    P.fb_lo = d.row_lo;
    P.fb_hi = d.row_hi;
    P.fb_wg = d.row_wg;
    P.fb_rows = d.fb_rows;
    P.fb_rows_off = d.fb_rows_off;
    P.fb_part = d.fb_part;
    P.pub = f.pub;
    P.seq = f.seq;
  }
  for (int r = 0; r < nrhs; ++r) {
    P.y[r] = y[r];
    P.x[r] = (x && x[r]) ? x[r] : d.xs[r];
    P.u[r] = (u && u[r]) ? u[r] : d.us[r];
    P.Hx[r] = (Hx && Hx[r]) ? Hx[r] : d.hs[r];
    P.hx[r] = d.out_hx[r];
    P.hu[r] = d.out_hu[r];
    P.contrib[r] = d.contrib[r];
    P.uoff[r] = d.uoff[r];
  }
  return P;
}
void launch(DevState& d, SweepParams& P, const DevState::Launch& ln) {
  P.items_base = static_cast<int>(&ln - d.launches.data()) == 0 ? 0 : d.launches[0].count;
  P.items = ln.items;
  P.cta_off = ln.cta_off;
  P.items_total = ln.count;
  SCN_CUDA(d.sweep->launch(P, d.grid, d.dyn_smem, d.max_m, d.max_mN, d.stream));
}
// The exchange buffer's geometry for this rank (dual.hpp ExchangeDims).
ExchangeDims exchange_dims(const DevState& d, const SweepParams& P) {
  const Layout& L = d.lay;
  const int W = L.nx + L.nu;
  ExchangeDims e{};
  e.ns_w = static_cast<int64_t>(d.sstage_hi - d.sstage_lo) * W;
  e.nys = d.dual_s_end - d.dual_top;
  e.xbuf_rhs = d.xbuf_rhs;
  e.contrib_off = static_cast<int64_t>(d.sstage_lo) * W;
  e.dual_top = d.dual_top;
  if (d.shard_hi > d.shard_lo) {  // else this rank has no shard-stage node: its buffer is all zeros
    e.own_c_lo = static_cast<int64_t>(d.shard_lo - d.sstage_lo) * W;
    e.own_c_hi = static_cast<int64_t>(d.shard_hi - d.sstage_lo) * W;
    e.own_y_lo = L.dual_offset[d.shard_lo];
    e.own_y_hi = L.dual_offset[d.shard_hi - 1] + L.stage_rows[d.shard_hi - 1];
  }
  e.nrhs = P.nrhs;
  for (int r = 0; r < P.nrhs; ++r) {
    e.contrib[r] = P.contrib[r];
    e.y[r] = P.y[r];
    e.ycomp[r] = d.ycomp[r];
  }
  return e;
}
// sharded phase A: local backward; then one kernel packs this rank's
// shard-stage contributions and shard-stage dual rows into the exchange
// buffer (zero elsewhere). zero_rows (phase API only) also zeroes the Hx
// rows this rank does not write.
void phase_a(DevState& d, SweepParams& P, bool zero_rows) {
  if (zero_rows)
    for (int r = 0; r < P.nrhs; ++r)
      for (const auto& q : d.zero_hx)
        SCN_CUDA(cudaMemsetAsync(P.Hx[r] + q.first, 0, sizeof(double) * (q.second - q.first), d.stream));
  launch(d, P, d.launches[0]);
  SCN_CUDA(k_exchange_pack(exchange_dims(d, P), d.xbuf, d.stream));
}
// sharded phase B: one kernel unpacks the summed buffer (contributions back;
// launch B's dual input = the top rows of y and every rank's shard-stage
// rows, ycomp); then the top backward + forward and the local forward.
// zero_rows (phase API only): the replicated top rows of Hx are kept on
// rank 0 only.
void phase_b(DevState& d, SweepParams& P, bool zero_rows) {
  SCN_CUDA(k_exchange_unpack(exchange_dims(d, P), d.xbuf, d.stream));
  for (int r = 0; r < P.nrhs; ++r) P.y[r] = d.ycomp[r];
  launch(d, P, d.launches[1]);
  if (zero_rows && d.rank != 0)
    for (int r = 0; r < P.nrhs; ++r)
      SCN_CUDA(cudaMemsetAsync(P.Hx[r], 0, d.dual_top * sizeof(double), d.stream));
}
}  // namespace

void dev_sweep(DevState& d, int nrhs, bool affine, const double* const* y, double* const* x,
               double* const* u, double* const* Hx) {
  SweepParams P = sweep_params(d, nrhs, affine, y, x, u, Hx);
  if (!d.sharded()) {
    launch(d, P, d.launches[0]);
    return;
  }
  // sharded: A (local backward) | allreduce of the shard-stage exchange | B (top + local forward).
  // x / u / Hx stay on their owners: no other collective.
  phase_a(d, P, false);
  dev_allreduce(d, d.xbuf, static_cast<size_t>(nrhs) * d.xbuf_rhs);
  phase_b(d, P, false);
}

void dev_sweep_phase(DevState& d, int phase, int nrhs, bool affine, const double* const* y, double* const* Hx) {
  if (!d.sharded()) fail(SCENOPT_E_INVALID_PARAMS, "sweep phase: handle is not sharded");
  SweepParams P = sweep_params(d, nrhs, affine, y, nullptr, nullptr, Hx);
  if (phase == 0)
    phase_a(d, P, true);
  else
    phase_b(d, P, true);
}

namespace {
// dst = src on the ranges, 0 elsewhere; then the sum over ranks
void gather_into(DevState& d, const double* src, double* dst, size_t total,
                 const std::vector<std::pair<int64_t, int64_t>>& keep) {
  SCN_CUDA(cudaMemsetAsync(dst, 0, sizeof(double) * total, d.stream));
  for (const auto& q : keep)
    SCN_CUDA(cudaMemcpyAsync(dst + q.first, src + q.first, sizeof(double) * (q.second - q.first),
                             cudaMemcpyDeviceToDevice, d.stream));
  dev_allreduce(d, dst, total);
}
}  // namespace

std::pair<const double*, const double*> dev_gather_primal(DevState& d, const double* x, const double* u) {
  if (!d.sharded()) return {x, u};
  const Layout& L = d.lay;
  if (x) gather_into(d, x, d.gx, static_cast<size_t>(L.nx) * L.n, d.keep_x);
  if (u) gather_into(d, u, d.gu, static_cast<size_t>(L.nu) * L.first_leaf, d.keep_u);
  return {x ? d.gx : nullptr, u ? d.gu : nullptr};
}

const double* dev_gather_dual(DevState& d, const double* y) {
  if (!d.sharded()) return y;
  gather_into(d, y, d.gy, static_cast<size_t>(d.lay.dual_dim), d.keep_y);
  return d.gy;
}

}  // namespace scn
