// SPDX-License-Identifier: MIT
// Device layout shared by the packer (host) and the sweep kernel (device).
//
// Every node owns two contiguous, 16-byte aligned matrix blocks, stored in
// node-id (= stage-major BFS) order so a stage is one contiguous stream:
//
//  BW block (read by the backward pass, tree_oracles.hpp:44-73), all columns
//  are "dot columns": out[j] = <col j, vec>:
//    interior node c:  E_c  = M_c x (nu+nx)   col j<nu : row j of dual_to_input_c
//                                              col nu+k : row k of dual_to_costate_c
//    leaf c:           FN_c = mN x nx          col k    : column k of F_N (F_N' y)
//    non-root c:       J_c  = nx x (nu+nx)     col j<nu : row j of child_to_input_c
//                                              col nu+k : column k of closed_loop_c
//  FW block (read by the forward pass, tree_oracles.hpp:75-88, fused with
//  apply_H, problem_data.hpp:144-162):
//    non-root c:       W_c  = (nx+nu) x (nx+m_c)  col r<nx : row r of [A_c B_c]
//                                                 col nx+s : row s of [F_c G_c]
//    interior c:       K_c  = nx x nu          col j : row j of gain_c
//    leaf c:           TN_c = nx x mN          col s : row s of F_N
//
// Items are runs of consecutive same-stage nodes; their blocks are therefore
// contiguous and one TMA bulk copy moves a whole item into shared memory.
#pragma once
#include <cstdint>

namespace scn {

struct Item {
  int64_t off;    // offset (doubles) of the first node's block in its pass array
  int32_t first;  // first node id
  int32_t count;  // nodes in the item
  int32_t bytes;  // bulk-copy size (multiple of 16)
  int32_t pass;   // 0 backward, 1 forward
};

struct NodeMeta {
  int32_t anc, cb, cc, M;   // ancestor, first child, child count, child dual rows
  int32_t cdo, doff, m, tdo;  // child dual offset, own stage-row offset/rows, terminal offset
  int32_t mN, leaf, pad0, pad1;
};

constexpr int kMaxRhs = 2;
constexpr int kMaxSlots = 4;

struct SweepParams {
  int nx, nu, n, first_leaf, dual_dim;
  int items_bw, items_total;
  int nslot, slot_doubles, vec_doubles;  // per-CTA smem carve-up
  int nrhs, affine;
  int max_count;  // max nodes per item
  int max_mN;     // max terminal rows
  const Item* items;
  const NodeMeta* meta;
  const int64_t* bw_off;  // [n] node block offsets (doubles)
  const int64_t* fw_off;
  const double* bw_blk;
  const double* fw_blk;
  const double* aff_bw;  // [n][nu+nx]: [input_affine; costate_affine] / [0; pi p_N]
  const double* aff_fw;  // [n][nx]: c_c
  const double* root_state;
  unsigned* ctrl;      // [0] epoch, [1] ticket, [2] done
  unsigned* bw_flag;   // [n]
  unsigned* fw_flag;   // [n]
  const double* y[kMaxRhs];
  double* x[kMaxRhs];
  double* u[kMaxRhs];
  double* Hx[kMaxRhs];
  double* contrib[kMaxRhs];  // [n][nu+nx] scratch
};

}  // namespace scn
