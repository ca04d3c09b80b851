// SPDX-License-Identifier: MIT
// Device factorization (K9, factor.cu): launch parameters shared with the host.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace scn {

struct FactorParams {
  int nx, nu, n, first_leaf, nxp;
  int stage_first, stage_count;   // nodes of this launch
  const int32_t* child_begin;
  const int32_t* child_count;
  const int32_t* dual_offset;     // per node (-1 root)
  const int32_t* stage_rows;      // per node
  const int32_t* ancestor;        // per node (-1 root)
  const double* prob;
  const double* cost_node;        // per non-root node i at cost_slot[i]*csz
  const double* cost_leaf;        // per leaf l at leaf_slot[l]*lsz
  const int32_t* cost_slot;       // [n] block of node i in cost_node (-1: not on this handle)
  const int32_t* leaf_slot;       // [L] block of leaf l in cost_leaf (-1: not on this handle)
  const int32_t* aff_nodes;       // factor_affine: the non-leaf nodes of this handle (null: all)
  int n_aff_nodes;
  const double* hcoef;            // per dual row: [F row | G row]
  const int64_t* bw_off;          // per node: E / leaf F_N block start in the bw pass array
  const int64_t* bw_j;            // per non-root node: J block start
  const int64_t* k_off;           // per node: K (gain) / T_N block start in the fw pass array
  double* bw_blk;
  double* fw_blk;
  double* aff_bw;                 // [n][nu+nx]
  double* vq;                     // [n][nx*nx] value_quad
  double* lchol;                  // [first_leaf][nu*nu] Cholesky factor of the input Hessian (refactor_affine)
  const double* root_unused;      // (layout padding)
  int affine_only;                // factor_leaves: update the affine terms only
  // flattened forward top (sweep.cu kFlatTop): maps written after the factor
  const int64_t* flat_off;        // per node: start of its flattened column block (fw pass array), -1: none
  double* aff_fw;                 // [n][nx] a'_c of flattened nodes
  double* aff_fwh;                // [n][mmax] stage-row constants of flattened nodes
  int mmax;
  const double* root_state;
  int flat_consts_only;           // refactor_affine: constants only (matrices unchanged)
  double* ws_global;              // per-CTA workspace when it does not fit in shared memory
  int64_t ws_doubles;
  int* bad;                       // first failing node + 1 (0: all strongly convex)
};

int64_t factor_workspace_doubles(int nx, int nu, int max_rows);
cudaError_t factor_run_leaves(const FactorParams& F, int grid, cudaStream_t st);
cudaError_t factor_run_stage(const FactorParams& F, int grid, size_t smem, cudaStream_t st);
// flattened forward top of one stage (1..cut-1): G / L column blocks and the a' / h' constants
cudaError_t factor_run_flat(const FactorParams& F, int grid, cudaStream_t st);
// refactor_affine (riccati.hpp:187-216) of every non-leaf node: new linear terms, same factor
cudaError_t factor_run_affine(const FactorParams& F, int grid, cudaStream_t st);

}  // namespace scn
