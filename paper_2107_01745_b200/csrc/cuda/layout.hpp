// SPDX-License-Identifier: MIT
// Device layout shared by the packer (host) and the sweep kernel (device).
//
// Node matrices are "dot-column" blocks (every product is out[j] = <col j, v>):
//
//  BW block (backward pass, tree_oracles.hpp:44-73):
//    interior c:  E_c  = M_c x (nu+nx)   col j<nu : row j of dual_to_input_c
//                                         col nu+k : row k of dual_to_costate_c
//    leaf c:      FN_c = mN x nx          col k    : column k of F_N (F_N' y)
//    non-root c:  J_c  = nxp x (nu+nx)    col j<nu : row j of child_to_input_c
//                                         col nu+k : column k of closed_loop_c
//  FW block (forward pass, tree_oracles.hpp:75-88, fused with apply_H,
//  problem_data.hpp:144-162):
//    non-root c:  W_c  = Vp x (nx+m_c)    col r<nx : row r of [A_c B_c]
//                                             col nx+s : row s of [F_c G_c]
//    interior c:  K_c  = nxp x nu         col j : row j of gain_c
//    leaf c:      TN_c = nxp x mN         col s : row s of F_N
//  Columns of J/W/K/TN are zero-padded to nxp = pad(nx), Vp = pad(nx+nu) with
//  pad(l) == 2 (mod 4): 16-byte loads of one column per thread then hit all
//  32 shared-memory banks without conflicts. E_c and FN_c (short columns)
//  are unpadded and rounded to an even size so J_c stays 16-byte aligned.
//
// Items are runs of consecutive same-stage nodes. Each pass array stores its
// items back to back in ticket order; an item is [NodeMeta x count | node
// blocks], 16-byte aligned, so ONE cp.async.bulk moves an item's metadata and
// matrices into shared memory.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

namespace scn {

// Per-node record at the head of an item (offsets are relative to the
// item's shared-memory slot / staged-vector areas).
struct NodeMeta {
  int32_t c;       // node id
  int32_t blk;     // offset (doubles) of the node block inside the slot
  int32_t M, m;    // child dual rows; own stage rows
  int32_t mN;      // terminal rows (leaf)
  int32_t doff;    // dual offset of the node's stage rows
  int32_t tdo;     // dual offset of the terminal rows (leaf)
  int32_t yoff;    // backward: offset of y_kids / y_N in the staged y range
  int32_t kid0;    // backward: first child's row in the staged contributions
  int32_t nkid;    // backward: number of children
  int32_t par;     // forward: parent's row in the staged parent vectors
  int32_t pad;
};
static_assert(sizeof(NodeMeta) % 16 == 0, "NodeMeta must keep 16-byte alignment");

struct Item {
  int64_t off;      // offset (doubles) of the item in its pass array
  int32_t bytes;    // bulk-copy size (multiple of 16)
  int32_t first;    // first node id
  int32_t count;    // nodes
  int32_t pass;     // 0 backward, 1 forward
  int32_t leaf;     // all nodes are leaves
  int32_t dep_lo;   // dependency flags [dep_lo, dep_hi): bw -> children (bw flags),
  int32_t dep_hi;   //   fw -> parents (fw flags), fw root -> bw flag of node 0
  int32_t v0_lo;    // staged range 0: bw y rows [v0_lo, v0_lo+v0_n) ; fw parent nodes
  int32_t v0_n;
  int32_t v1_lo;    // staged range 1: bw child contribution rows ; fw u_off of the item
  int32_t v1_n;
  int32_t direct;   // flags: kDirectContrib (bw: contributions read from L2, many children),
                    //        kGlobalBlocks (node blocks stay in HBM; only the headers are copied)
  int32_t ldep;     // local index (same CTA) of the last item this one depends on, -1: none
  int32_t publish;  // bit 0: release the nodes' flags at gpu scope (consumed by other CTAs)
};
static_assert(sizeof(Item) == 64, "Item is one 64-byte record");

constexpr int kDirectContrib = 1;
constexpr int kGlobalBlocks = 2;
constexpr int kFlatTop = 4;  // forward top node computed from its ancestors' u_off; depth in bits 8..
constexpr int kMaxRhs = 2;
constexpr int kMaxSlots = 8;
constexpr int kManyNodeItems = 8;  // largest item of at least this many nodes: six-producer sweep geometry

struct SweepParams {
  int nx, nu, n, first_leaf, dual_dim;
  int items_total;
  int items_base;  // index of this launch's first item in the handle's item order (profiling)
  int nslot, slot_doubles, stage_doubles, scratch_doubles;
  int nrhs, affine, G, max_count;
  int nxp, Vp;  // padded column lengths (== 2 mod 4) of J/K/TN and W
  int consumer_stage;  // 1: teams stage their own vectors (staging area per team, not per ring entry)
  int global_blocks;   // 1: some items keep their node blocks in HBM (kGlobalBlocks)
  const Item* items;      // CTA-major: CTA b owns items [cta_off[b], cta_off[b+1])
  const int32_t* cta_off;
  const double* bw_blk;
  const double* fw_blk;
  const double* aff_bw;  // [n][nu+nx]: [input_affine; costate_affine] / [0; pi p_N]
  const double* aff_fw;  // [n][nx]: c_c (flattened top: the constant a'_c)
  const double* aff_fwh; // [n][mmax]: constant of the flattened top's stage rows
  int mmax;
  const double* root_state;
  unsigned* ctrl;     // [0] epoch, [1] done-CTA counter
  const int* skip;    // non-null and *skip != 0: the launch does nothing (batched power iteration)
  unsigned* bw_flag;  // [n]
  unsigned* fw_flag;  // [n]
  const double* y[kMaxRhs];
  double* x[kMaxRhs];
  double* u[kMaxRhs];
  // optional second destination of x / u in mapped pinned host memory: the
  // forward pass streams its results over PCIe as it computes them (host I/O)
  double* hx[kMaxRhs];
  double* hu[kMaxRhs];
  double* uoff[kMaxRhs];  // [first_leaf][nu] backward input offsets (the forward pass reads, never overwrites)
  double* Hx[kMaxRhs];
  double* contrib[kMaxRhs];  // [n][nu+nx] scratch
  // Fused finish of an FB step (fbe.hpp:38-50) on a 1-RHS affine sweep of an
  // unsharded handle (fb_S == nullptr: off). At the end of the sweep every
  // CTA finishes the dual rows its own forward items wrote (z, R, T and the
  // step's partial sums), and the last CTA to finish combines the CTAs'
  // partials in CTA order, writes the step's scalars and publishes them.
  double* fb_S;              // scalar block (dual.hpp sl::); the state's scalars at fb_S + fb_state * kStateStride
  int* fb_I;
  int fb_state;
  const double* fb_Hx0;
  const double* fb_weight;   // residual weights or null
  double* fb_z;
  double* fb_R;
  double* fb_T;
  const int8_t* fb_kind;     // per dual row: nonsmooth kind, box bounds, l1 radius
  const double* fb_lo;
  const double* fb_hi;
  const double* fb_wg;
  const int32_t* fb_rows;      // dual rows finished by each CTA: [fb_rows_off[b], fb_rows_off[b + 1])
  const int32_t* fb_rows_off;  // (the stage and terminal rows of the CTA's forward items)
  double* fb_part;           // [grid][8] per-CTA partial sums
  unsigned long long* pub;   // non-null: the last CTA also publishes S / I (mapped flagged words, dual.hpp)
  unsigned seq;
};

// One compiled geometry of the sweep kernel: cuda/sweep.cu is built once per
// geometry (producer warps and staging-ring depth differ; the consumer teams,
// and so every product's summation order, are the same, so the geometries
// give bitwise-identical results). A handle picks one when its layout is
// built (device.cpp).
struct SweepImpl {
  const char* name;
  int producers, teams, threads, stage_queue, scratch_bufs;
  size_t (*static_smem)();
  cudaError_t (*configure)(size_t dyn_smem);
  cudaError_t (*occupancy)(int* ctas_per_sm, size_t dyn_smem);
  cudaError_t (*launch)(const SweepParams& P, int grid, size_t dyn_smem, int mmax, int mNmax, cudaStream_t st);
};
extern const SweepImpl kSweepProducers4;  // four producer warps, 8-deep staging ring (default)
extern const SweepImpl kSweepProducers6;  // six producer warps, 12-deep ring (layouts of many-node items)

}  // namespace scn
