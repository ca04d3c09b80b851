// SPDX-License-Identifier: MIT
// Device-resident packed instance (the scenopt_dev handle).
#pragma once

#include <cuda_runtime.h>

#include <memory>
#include <string>
#include <vector>

#include "../cuda/dual.hpp"
#include "../cuda/factor.hpp"
#include "../cuda/layout.hpp"
#include "model.hpp"

namespace scn {

#define SCN_CUDA(expr)                                                                     \
  do {                                                                                     \
    cudaError_t _e = (expr);                                                               \
    if (_e != cudaSuccess)                                                                 \
      ::scn::fail(_e == cudaErrorMemoryAllocation ? SCENOPT_E_NOMEM : SCENOPT_E_CUDA,      \
                  std::string(#expr) + ": " + cudaGetErrorString(_e));                     \
  } while (0)

// Device buffer owned by a handle (freed in ~DevState).
template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
};

// Collectives of a sharded handle on its stream (comm.cpp): NCCL, or an
// emulated group of handles in one process (tests on one GPU).
struct Comm {
  virtual ~Comm() = default;
  virtual void allreduce_sum(double* buf, size_t n, cudaStream_t st) = 0;
  virtual void allgather(const double* send, double* recv, size_t n, cudaStream_t st) = 0;  // recv: world x n
};
struct EmuGroup;

struct Layout {  // host copy of the layout numbers the device code needs
  int nx = 0, nu = 0, N = 0, n = 0, L = 0, first_leaf = 0, dual_dim = 0, stage_total = 0;
  std::vector<int32_t> ancestor, stage_offsets, stage_rows, terminal_rows, child_begin,
      child_count, dual_offset, tdual_offset;
  std::vector<double> probability, root_state;
};

struct DevState {
  int device = 0, sm_count = 0;
  cudaStream_t stream = nullptr;
  Layout lay;
  size_t bytes_allocated = 0;
  std::vector<void*> owned;

  // packed matrices and metadata
  double *bw_blk = nullptr, *fw_blk = nullptr, *aff_bw = nullptr, *aff_fw = nullptr,
         *root_state = nullptr;
  // Sweep launches: one (unsharded), or two for a sharded handle (local
  // backward below the rank cut, then top backward + forward), each with
  // CTA-major items and per-CTA ranges [cta_off[b], cta_off[b+1]).
  struct Launch {
    Item* items = nullptr;
    int32_t* cta_off = nullptr;
    int count = 0;
  };
  std::vector<Launch> launches;
  int cut_stage = -1;  // CTA subtree-ownership cut of the main region (-1: all global tickets)
  bool consumer_stage = false;  // teams stage their own vectors (very wide states)
  bool flat_top = false;
  const SweepImpl* sweep = &kSweepProducers4;  // compiled geometry of the sweep kernel (chosen with the layout)
  const int* sweep_skip = nullptr;  // SweepParams::skip of the next launches (power iteration batches)
  // Fused FB-step finish of the next launch (SweepParams::fb_*; set by the
  // solver engine around one affine 1-RHS sweep of an unsharded handle)
  struct FbFuse {
    double* S = nullptr;
    int* I = nullptr;
    int state = 0;
    const double *Hx0 = nullptr, *weight = nullptr;
    double *z = nullptr, *R = nullptr, *T = nullptr;
    unsigned long long* pub = nullptr;  // mapped flagged words (dual.hpp kPubWords)
    unsigned seq = 0;
  };
  const FbFuse* fb_next = nullptr;
  int32_t *fb_rows = nullptr, *fb_rows_off = nullptr;  // fused FB finish: dual rows per CTA (SweepParams)
  double* fb_part = nullptr;  // [grid][8]
  double* out_hx[kMaxRhs] = {};      // SweepParams::hx / hu of the next launches (mapped host outputs)
  double* out_hu[kMaxRhs] = {};        // flattened forward top (one level after the backward root)
  double* aff_fwh = nullptr;    // [n][max_m] constant of the flattened top's stage rows
  // node block positions in the pass arrays (doubles; -1: not on this handle)
  std::vector<int64_t> h_bw_off, h_bw_j, h_k_off, h_flat_off;
  double* vq = nullptr;         // value_quad of the device factor [n][nx*nx]
  double* vx = nullptr;         // sharded device factor: shard-stage value matrices exchanged (+ a flag)
  bool device_factor = false;   // E / J / K / aff_bw computed on the device (K9)
  FactorParams fp{};            // device-factor launch parameters (index arrays on the device)
  bool fp_ready = false;
  int items_global = 0;         // items whose node blocks are read from HBM in place
  // ---- subtree sharding over ranks
  int rank = 0, world = 1, shard_stage = -1;
  std::unique_ptr<Comm> comm;   // null: exchange left to the caller (phase API)
  int shard_lo = 0, shard_hi = 0;  // this rank's shard-stage nodes
  std::vector<std::pair<int, int>> own_range;  // per stage: the nodes this rank holds (all above the shard stage)
  int sstage_lo = 0, sstage_hi = 0;  // all shard-stage nodes [stage_offsets[s], stage_offsets[s+1])
  int64_t dual_top = 0;          // dual rows of the replicated top stages (a prefix)
  int64_t dual_s_end = 0;        // end of the shard-stage nodes' dual rows ([dual_top, dual_s_end))
  // exchange buffer, per right-hand side: [shard-stage contributions ns x (nu+nx) | shard-stage y rows]
  double* xbuf = nullptr;
  int64_t xbuf_rhs = 0;          // doubles per right-hand side
  double* ycomp[kMaxRhs] = {};   // launch B's dual input: top rows + every rank's shard-stage rows
  // Row / node ownership. Rank r holds valid values on its own rows (its
  // subtrees' stage and terminal rows) and on the replicated top rows;
  // reductions count the own rows, and the top rows on rank 0 only.
  uint8_t* row_counted = nullptr;  // [dual_dim] (device)
  std::vector<std::pair<int64_t, int64_t>> keep_x, keep_u, keep_y;  // element ranges counted on this rank
  double *gx = nullptr, *gu = nullptr, *gy = nullptr;               // gather scratch
  // [begin, end) element ranges of x / u / Hx that no launch of this rank
  // writes (other ranks' subtrees), zeroed before the sweep's allreduces
  std::vector<std::pair<int64_t, int64_t>> zero_x, zero_u, zero_hx;
  bool sharded() const { return shard_stage >= 0; }
  unsigned *ctrl = nullptr, *bw_flag = nullptr, *fw_flag = nullptr;
  int64_t bw_doubles = 0, fw_doubles = 0;
  int items_bw = 0, items_fw = 0, max_count = 1, max_m = 0, max_mN = 0, nxp = 0, Vp = 0;
  // per dual row: nonsmooth kind, box bounds, l1 radius weight*gamma
  int8_t* row_kind = nullptr;
  double *row_lo = nullptr, *row_hi = nullptr, *row_wg = nullptr;
  // sweep scratch (2 RHS)
  double* contrib[kMaxRhs] = {nullptr, nullptr};
  double* uoff[kMaxRhs] = {nullptr, nullptr};  // backward input offsets
  double* xs[kMaxRhs] = {nullptr, nullptr};
  double* us[kMaxRhs] = {nullptr, nullptr};
  double* hs[kMaxRhs] = {nullptr, nullptr};
  double* ys[kMaxRhs] = {nullptr, nullptr};
  // launch configuration
  int grid = 0, ctas_per_sm = 0, nslot = 0, slot_doubles = 0, stage_doubles = 0, vec_doubles = 0,
      G = 16;
  size_t dyn_smem = 0;
  // algorithmic bytes per sweep
  int64_t bytes_hom = 0, bytes_aff = 0, bytes_hom2 = 0;
  bool has_factor = false;
  // apply_H rows and eval_f cost blocks
  HRows hrows{};
  CostPack cost{};

  ~DevState();
  template <class T>
  T* alloc(size_t count) {
    void* p = nullptr;
    SCN_CUDA(cudaMalloc(&p, count * sizeof(T) + 16));
    owned.push_back(p);
    SCN_CUDA(cudaMemset(p, 0, count * sizeof(T) + 16));  // sharded outputs rely on zero fill
    bytes_allocated += count * sizeof(T);
    return static_cast<T*>(p);
  }
  void free_owned(void* p);
};

// f == nullptr builds a factor-less handle (apply_H, eval_f, prox/conj,
// verification) without the sweep layout.
// Bare context (device, stream, SM count) for problem-free device objects.
std::unique_ptr<DevState> dev_create_bare(int device);
struct ShardSpec {
  int rank = 0, world = 1;
  int stage = -1;              // shard cut stage (-1: smallest stage with >= world nodes)
  const void* nccl_id = nullptr;  // 128-byte ncclUniqueId shared by all ranks
  std::shared_ptr<EmuGroup> emu;  // or: an emulated group (one process, one host thread per rank)
};
// Host-only shard plan: *stage (in: -1 = auto) and the world+1 bounds of the
// ranks' contiguous shard-stage node ranges, balanced by subtree bytes.
std::vector<int> shard_plan(const Problem& p, int world, int* stage);
// Host-only ownership of rank `rank` whose shard-stage nodes are [lo, hi):
// node mask (its subtrees; the top stages on rank 0) and the dual rows it
// counts in reductions (stage and terminal rows of its nodes).
std::vector<char> shard_nodes(const Problem& p, int stage, int lo, int hi, int rank);
std::vector<uint8_t> shard_rows(const Problem& p, const std::vector<char>& mine);
std::unique_ptr<DevState> dev_create(const Problem& p, const Factor* f, int device,
                                     const ShardSpec* shard = nullptr);
// Handle whose factor is computed on the device (K9, factor.cu): the host
// packs only problem data; the factor blocks are written by the GPU.
std::unique_ptr<DevState> dev_create_device_factor(const Problem& p, int device, const ShardSpec* shard = nullptr);
// (Re)compute the factor of the handle's own problem data on the device.
void dev_factor_device(DevState& d);
// The device factor in the FactorCache layout (riccati.hpp:38-63).
Factor dev_factor_export(DevState& d, const Problem& p);
// refactor_affine (riccati.hpp:187-216) on the device: upload p's linear
// terms (q, r, c, p_N, root state; same matrices) and recompute the affine
// factor terms in place. Requires a device-factored handle.
void dev_refactor_affine(DevState& d, const Problem& p);
// ncclGetUniqueId into 128 bytes
void nccl_unique_id(void* out128);
std::unique_ptr<Comm> nccl_comm(int device, int rank, int world, const void* id128);
std::shared_ptr<EmuGroup> emu_group_create(int world);
int emu_group_world(const EmuGroup& g);
std::unique_ptr<Comm> emu_comm(const std::shared_ptr<EmuGroup>& g, int rank);
// Sum-allreduce of n doubles on the handle's stream (no-op unsharded).
void dev_allreduce(DevState& d, double* buf, size_t n);
int device_count_sm100();

// One fused sweep over nrhs right-hand sides; y/x/u/Hx are device pointers
// (x/u/Hx may be null: the handle's scratch is used). Enqueued on d.stream.
// Sharded handles: y must be valid on this rank's own and top rows; x/u/Hx
// come out valid on this rank's own and top nodes / rows only (the
// dev_gather_* calls assemble full vectors).
void dev_sweep(DevState& d, int nrhs, bool affine, const double* const* y, double* const* x,
               double* const* u, double* const* Hx);
// One phase of a sharded sweep with the exchange left to the caller (phase 0:
// zero Hx, local backward, own contributions into d.xbuf; phase 1: xbuf
// (summed over ranks by the caller) back, top backward + forward, top rows
// of Hx zeroed on ranks != 0). Emulation / tests of handles without NCCL.
void dev_sweep_phase(DevState& d, int phase, int nrhs, bool affine, const double* const* y, double* const* Hx);
// Assemble a sharded primal point / dual vector in full on every rank, into
// the handle's gather scratch (returned; the inputs are not modified). An
// unsharded handle returns the inputs.
std::pair<const double*, const double*> dev_gather_primal(DevState& d, const double* x, const double* u);
const double* dev_gather_dual(DevState& d, const double* y);

// sweep kernel diagnostics (profiling build, cuda/sweep.cu); the launchers
// are reached through DevState::sweep (layout.hpp SweepImpl)
cudaError_t sweep_profile_read(unsigned long long* out, bool reset);
cudaError_t sweep_timeline(unsigned long long* dev_buf);
cudaError_t sweep_trace(long long* dev_buf);

}  // namespace scn
