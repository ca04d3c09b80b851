// SPDX-License-Identifier: MIT
//
// K9: the Riccati factorization (riccati.hpp:82-182) on the device, written
// straight into the packed sweep layout (layout.hpp / device.cpp), so a
// handle never needs the host factor or its upload.
//
// One launch per stage, leaves -> root (a stage needs its children's value
// matrices). A persistent grid loops over the stage's nodes; one CTA owns a
// node: it accumulates the eliminated input Hessian and the linear terms over
// the children (PA = V_c A_c, PB = V_c B_c: small dense GEMMs spread over the
// CTA's threads), checks strong convexity with a Cholesky of H - 1e-10 I
// (the reference checks the smallest eigenvalue, riccati.hpp:142-150),
// factors H, solves for the gain and the affine terms, and scatters
//   E_i  (dual_to_input / dual_to_costate over the children's rows),
//   J_c  (child_to_input / closed_loop of every child c),
//   K_i  (gain) and aff_bw[i] = [input_affine; costate_affine]
// into the pass arrays, plus V_i (value_quad) for the parent's stage.
// Problem data come from the handle's eval_f cost blocks ([A|B|c|Q|S|R|q|r]
// per non-root node, [P|p] per leaf) and apply_H rows ([F|G] per dual row).
#include <cuda_runtime.h>

#include <cstdint>

#include "factor.hpp"

namespace scn {


namespace {

constexpr int kT = 256;

// C (m x n, ldc) (+)= alpha * op(A) op(B); column-major, op = T when trans
__device__ void gemm(int m, int n, int k, bool ta, const double* A, int lda, bool tb, const double* B, int ldb,
                     double* C, int ldc, bool accumulate) {
  for (int e = threadIdx.x; e < m * n; e += kT) {
    const int i = e % m, j = e / m;
    double s = 0.0;
    for (int t = 0; t < k; ++t) {
      const double a = ta ? A[t + static_cast<int64_t>(i) * lda] : A[i + static_cast<int64_t>(t) * lda];
      const double b = tb ? B[j + static_cast<int64_t>(t) * ldb] : B[t + static_cast<int64_t>(j) * ldb];
      s = fma(a, b, s);
    }
    C[i + static_cast<int64_t>(j) * ldc] = accumulate ? C[i + static_cast<int64_t>(j) * ldc] + s : s;
  }
}

// In-place lower Cholesky of an n x n SPD matrix (column-major); returns
// false (on every thread) when a pivot is <= floor.
__device__ bool cholesky(double* L, int n, double shift, double floor) {
  __shared__ double piv;
  __shared__ int ok;
  if (threadIdx.x == 0) ok = 1;
  __syncthreads();
  for (int j = 0; j < n; ++j) {
    if (threadIdx.x == 0) {
      double d = L[j + j * n] - shift;
      for (int k = 0; k < j; ++k) d -= L[j + k * n] * L[j + k * n];
      if (!(d > floor)) ok = 0;
      piv = sqrt(d > 0.0 ? d : 1.0);
      L[j + j * n] = piv;
    }
    __syncthreads();
    if (!ok) return false;
    for (int i = j + 1 + threadIdx.x; i < n; i += kT) {
      double s = L[i + j * n];
      for (int k = 0; k < j; ++k) s -= L[i + k * n] * L[j + k * n];
      L[i + j * n] = s / piv;
    }
    __syncthreads();
  }
  return true;
}

// X (n x ncol) <- scale * (L L')^{-1} X, one column per thread
__device__ void chol_solve(const double* L, int n, double* X, int ldx, int ncol, double scale) {
  for (int c = threadIdx.x; c < ncol; c += kT) {
    double* x = X + static_cast<int64_t>(c) * ldx;
    for (int i = 0; i < n; ++i) {
      double s = x[i];
      for (int k = 0; k < i; ++k) s -= L[i + k * n] * x[k];
      x[i] = s / L[i + i * n];
    }
    for (int i = n - 1; i >= 0; --i) {
      double s = x[i];
      for (int k = i + 1; k < n; ++k) s -= L[k + i * n] * x[k];
      x[i] = s / L[i + i * n];
    }
    for (int i = 0; i < n; ++i) x[i] *= scale;
  }
}

// problem data of node c / leaf l on this handle (a sharded handle holds its
// own nodes, the replicated top and the shard-stage nodes)
__device__ __forceinline__ const double* cost_of(const FactorParams& F, int c, int64_t csz) {
  return F.cost_node + static_cast<int64_t>(F.cost_slot[c]) * csz;
}

__global__ void __launch_bounds__(kT) factor_leaves(FactorParams F) {
  const int nx = F.nx, nu = F.nu, W = nx + nu;
  const int64_t lsz = static_cast<int64_t>(nx) * nx + nx;
  for (int l = blockIdx.x; l < F.stage_count; l += gridDim.x) {  // riccati.hpp:106-113
    const int c = F.stage_first + l;
    const double pi = F.prob[c];
    const double* P = F.cost_leaf + static_cast<int64_t>(F.leaf_slot[F.stage_first - F.first_leaf + l]) * lsz;
    if (!F.affine_only)
      for (int e = threadIdx.x; e < nx * nx; e += kT) F.vq[static_cast<int64_t>(c) * nx * nx + e] = pi * P[e];
    for (int e = threadIdx.x; e < W; e += kT)
      F.aff_bw[static_cast<int64_t>(c) * W + e] = e < nu ? 0.0 : pi * P[nx * nx + (e - nu)];
  }
}

__global__ void __launch_bounds__(kT) factor_stage(FactorParams F) {
  extern __shared__ __align__(16) double smem[];
  const int nx = F.nx, nu = F.nu, W = nx + nu, nxp = F.nxp;
  const int64_t xx = static_cast<int64_t>(nx) * nx, xu = static_cast<int64_t>(nx) * nu,
                uu = static_cast<int64_t>(nu) * nu;
  const int64_t csz = 2 * xx + 2 * xu + uu + 2 * nx + nu;
  double* ws = F.ws_global ? F.ws_global + blockIdx.x * F.ws_doubles : smem;
  double *V = ws, *A = V + xx, *B = A + xx, *PA = B + xu, *PB = PA + xx, *huu = PB + xu, *hux = huu + uu,
         *hxx = hux + xu, *su = hxx + xx, *sx = su + nu, *pc2 = sx + nx, *L = pc2 + nx, *K = L + uu,
         *T = K + xu;  // T: scratch for the children blocks, max(nu, nx) x max child rows
  for (int q = blockIdx.x; q < F.stage_count; q += gridDim.x) {
    const int i = F.stage_first + q;
    const int cb = F.child_begin[i], cc = F.child_count[i];
    for (int e = threadIdx.x; e < uu; e += kT) huu[e] = 0.0;
    for (int e = threadIdx.x; e < xu; e += kT) hux[e] = 0.0;
    for (int e = threadIdx.x; e < xx; e += kT) hxx[e] = 0.0;
    for (int e = threadIdx.x; e < nu; e += kT) su[e] = 0.0;
    for (int e = threadIdx.x; e < nx; e += kT) sx[e] = 0.0;
    __syncthreads();
    // riccati.hpp:127-141: accumulate over the children
    for (int c = cb; c < cb + cc; ++c) {
      const double pc = F.prob[c];
      const double* blk = cost_of(F, c, csz);
      const double *Ag = blk, *Bg = Ag + xx, *cg = Bg + xu, *Qg = cg + nx, *Sg = Qg + xx, *Rg = Sg + xu,
                   *qg = Rg + uu, *rg = qg + nx;
      for (int e = threadIdx.x; e < xx; e += kT) {
        V[e] = F.vq[static_cast<int64_t>(c) * xx + e];
        A[e] = Ag[e];
      }
      for (int e = threadIdx.x; e < xu; e += kT) B[e] = Bg[e];
      __syncthreads();
      gemm(nx, nu, nx, false, V, nx, false, B, nx, PB, nx, false);  // PB = V B
      gemm(nx, nx, nx, false, V, nx, false, A, nx, PA, nx, false);  // PA = V A
      for (int e = threadIdx.x; e < nx; e += kT) {                  // pc2 = 2 V c
        double s = 0.0;
        for (int z = 0; z < nx; ++z) s = fma(V[e + z * nx], cg[z], s);
        pc2[e] = 2.0 * s;
      }
      __syncthreads();
      for (int e = threadIdx.x; e < uu; e += kT) huu[e] += pc * Rg[e];
      for (int e = threadIdx.x; e < xu; e += kT) hux[e] += pc * Sg[e];
      for (int e = threadIdx.x; e < xx; e += kT) hxx[e] += pc * Qg[e];
      __syncthreads();
      gemm(nu, nu, nx, true, B, nx, false, PB, nx, huu, nu, true);   // + B' P B
      gemm(nu, nx, nx, true, B, nx, false, PA, nx, hux, nu, true);   // + B' P A
      gemm(nx, nx, nx, true, A, nx, false, PA, nx, hxx, nx, true);   // + A' P A
      for (int e = threadIdx.x; e < nu; e += kT) {
        double s = 0.0;
        for (int z = 0; z < nx; ++z) s = fma(B[z + e * nx], pc2[z], s);
        su[e] += pc * rg[e] + s;
      }
      for (int e = threadIdx.x; e < nx; e += kT) {
        double s = 0.0;
        for (int z = 0; z < nx; ++z) s = fma(A[z + e * nx], pc2[z], s);
        sx[e] += pc * qg[e] + s;
      }
      __syncthreads();
    }
    // riccati.hpp:142-150: symmetrize, strong convexity, Cholesky
    for (int e = threadIdx.x; e < uu; e += kT) {
      const int a = e % nu, b = e / nu;
      if (a > b) {
        const double s = 0.5 * (huu[a + b * nu] + huu[b + a * nu]);
        huu[a + b * nu] = s;
        huu[b + a * nu] = s;
      }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < uu; e += kT) L[e] = huu[e];
    __syncthreads();
    if (!cholesky(L, nu, 1e-10, 0.0)) {  // min eig(H) < 1e-10 <=> H - 1e-10 I not PD
      if (threadIdx.x == 0) atomicCAS(F.bad, 0, i + 1);
      continue;
    }
    for (int e = threadIdx.x; e < uu; e += kT) L[e] = huu[e];
    __syncthreads();
    cholesky(L, nu, 0.0, 0.0);
    for (int e = threadIdx.x; e < uu; e += kT) F.lchol[static_cast<int64_t>(i) * uu + e] = L[e];
    // gain K = -H^{-1} hux ; input_affine = -1/2 H^{-1} su ; costate_affine = sx + K' su
    for (int e = threadIdx.x; e < xu; e += kT) K[e] = hux[e];
    for (int e = threadIdx.x; e < nu; e += kT) T[e] = su[e];
    __syncthreads();
    chol_solve(L, nu, K, nu, nx, -1.0);
    chol_solve(L, nu, T, nu, 1, -0.5);
    __syncthreads();
    double* aff = F.aff_bw + static_cast<int64_t>(i) * W;
    for (int e = threadIdx.x; e < nu; e += kT) aff[e] = T[e];
    for (int e = threadIdx.x; e < nx; e += kT) {
      double s = sx[e];
      for (int w = 0; w < nu; ++w) s = fma(K[w + e * nu], su[w], s);
      aff[nu + e] = s;
    }
    double* Kb = F.fw_blk + F.k_off[i];  // fw K block: column j = gain row j (nxp stride)
    for (int e = threadIdx.x; e < xu; e += kT) {
      const int w = e % nu, z = e / nu;
      Kb[z + static_cast<int64_t>(w) * nxp] = K[e];
    }
    // riccati.hpp:177-178: V_i = hxx + hux' K, symmetrized
    gemm(nx, nx, nu, true, hux, nu, false, K, nu, hxx, nx, true);
    __syncthreads();
    double* Vi = F.vq + static_cast<int64_t>(i) * xx;
    for (int e = threadIdx.x; e < xx; e += kT) {
      const int a = e % nx, b = e / nx;
      Vi[e] = a == b ? hxx[e] : 0.5 * (hxx[a + b * nx] + hxx[b + a * nx]);
    }
    // riccati.hpp:157-175: children blocks
    const int M = F.dual_offset[cb + cc - 1] + F.stage_rows[cb + cc - 1] - F.dual_offset[cb];
    double* E = F.bw_blk + F.bw_off[i];  // M x W, column j over the children's rows
    for (int c = cb; c < cb + cc; ++c) {
      const int rows = F.stage_rows[c];
      const int col = F.dual_offset[c] - F.dual_offset[cb];
      const double* hc = F.hcoef + static_cast<int64_t>(F.dual_offset[c]) * W;  // [F | G] per row
      __syncthreads();
      // dual_to_input rows: -1/2 H^{-1} G' ; dual_to_costate: F + G K (transposed into E columns)
      for (int e = threadIdx.x; e < nu * rows; e += kT) {
        const int w = e % nu, rr = e / nu;
        T[w + rr * nu] = hc[static_cast<int64_t>(rr) * W + nx + w];
      }
      __syncthreads();
      chol_solve(L, nu, T, nu, rows, -0.5);
      __syncthreads();
      for (int e = threadIdx.x; e < nu * rows; e += kT) {
        const int w = e % nu, rr = e / nu;
        E[(col + rr) + static_cast<int64_t>(w) * M] = T[w + rr * nu];
      }
      for (int e = threadIdx.x; e < nx * rows; e += kT) {
        const int z = e % nx, rr = e / nx;
        const double* row = hc + static_cast<int64_t>(rr) * W;
        double s = row[z];
        for (int w = 0; w < nu; ++w) s = fma(row[nx + w], K[w + z * nu], s);
        E[(col + rr) + static_cast<int64_t>(nu + z) * M] = s;
      }
      // child_to_input_c = -1/2 H^{-1} B_c' ; closed_loop_c = A_c + B_c K  -> J_c (nxp x W)
      // (a sharded handle's top node writes the J blocks of its own children only)
      if (F.bw_j[c] < 0) continue;
      const double* blk = cost_of(F, c, csz);
      const double *Ag = blk, *Bg = Ag + xx;
      __syncthreads();
      for (int e = threadIdx.x; e < xu; e += kT) {
        const int w = e % nu, z = e / nu;
        PB[w + z * nu] = Bg[z + w * nx];  // B_c' (nu x nx)
      }
      __syncthreads();
      chol_solve(L, nu, PB, nu, nx, -0.5);
      __syncthreads();
      double* J = F.bw_blk + F.bw_j[c];
      for (int e = threadIdx.x; e < xu; e += kT) {
        const int w = e % nu, z = e / nu;
        J[z + static_cast<int64_t>(w) * nxp] = PB[w + z * nu];
      }
      for (int e = threadIdx.x; e < xx; e += kT) {
        const int a = e % nx, t = e / nx;
        double s = Ag[a + t * nx];
        for (int w = 0; w < nu; ++w) s = fma(Bg[a + w * nx], K[w + t * nu], s);
        J[a + static_cast<int64_t>(nu + t) * nxp] = s;
      }
    }
    __syncthreads();
  }
}

// riccati.hpp:187-216: new q, r, c (same matrices): every non-leaf node's
// input_affine = -1/2 H^{-1} su and costate_affine = sx + K' su from its
// children's value matrices and the stored Cholesky factor.
__global__ void __launch_bounds__(kT) factor_affine(FactorParams F) {
  const int nx = F.nx, nu = F.nu, W = nx + nu, nxp = F.nxp;
  const int64_t xx = static_cast<int64_t>(nx) * nx, xu = static_cast<int64_t>(nx) * nu,
                uu = static_cast<int64_t>(nu) * nu;
  const int64_t csz = 2 * xx + 2 * xu + uu + 2 * nx + nu;
  extern __shared__ __align__(16) double sm[];  // su (nu) | sx (nx) | pc2 (nx)
  double *su = sm, *sx = su + nu, *pc2 = sx + nx;
  const int count = F.aff_nodes ? F.n_aff_nodes : F.first_leaf;
  for (int q = blockIdx.x; q < count; q += gridDim.x) {
    const int i = F.aff_nodes ? F.aff_nodes[q] : q;
    for (int e = threadIdx.x; e < nu; e += kT) su[e] = 0.0;
    for (int e = threadIdx.x; e < nx; e += kT) sx[e] = 0.0;
    __syncthreads();
    for (int c = F.child_begin[i]; c < F.child_begin[i] + F.child_count[i]; ++c) {
      const double pc = F.prob[c];
      const double* blk = cost_of(F, c, csz);
      const double *Ag = blk, *Bg = Ag + xx, *cg = Bg + xu, *qg = cg + nx + xx + xu + uu, *rg = qg + nx;
      const double* V = F.vq + static_cast<int64_t>(c) * xx;
      for (int e = threadIdx.x; e < nx; e += kT) {
        double s = 0.0;
        for (int z = 0; z < nx; ++z) s = fma(V[e + z * nx], cg[z], s);
        pc2[e] = 2.0 * s;
      }
      __syncthreads();
      for (int e = threadIdx.x; e < nu; e += kT) {
        double s = 0.0;
        for (int z = 0; z < nx; ++z) s = fma(Bg[z + e * nx], pc2[z], s);
        su[e] += pc * rg[e] + s;
      }
      for (int e = threadIdx.x; e < nx; e += kT) {
        double s = 0.0;
        for (int z = 0; z < nx; ++z) s = fma(Ag[z + e * nx], pc2[z], s);
        sx[e] += pc * qg[e] + s;
      }
      __syncthreads();
    }
    double* aff = F.aff_bw + static_cast<int64_t>(i) * W;
    const double* Kb = F.fw_blk + F.k_off[i];
    for (int z = threadIdx.x; z < nx; z += kT) {
      double s = sx[z];
      for (int w = 0; w < nu; ++w) s = fma(Kb[z + static_cast<int64_t>(w) * nxp], su[w], s);
      aff[nu + z] = s;
    }
    __syncthreads();
    if (threadIdx.x == 0) {  // ia = -1/2 (L L')^{-1} su
      const double* L = F.lchol + static_cast<int64_t>(i) * uu;
      double* x = su;
      for (int r = 0; r < nu; ++r) {
        double s = x[r];
        for (int k = 0; k < r; ++k) s -= L[r + k * nu] * x[k];
        x[r] = s / L[r + r * nu];
      }
      for (int r = nu - 1; r >= 0; --r) {
        double s = x[r];
        for (int k = r + 1; k < nu; ++k) s -= L[k + r * nu] * x[k];
        x[r] = s / L[r + r * nu];
      }
      for (int r = 0; r < nu; ++r) aff[r] = -0.5 * x[r];
    }
    __syncthreads();
  }
}

__device__ __forceinline__ int pad2d(int l) { return l + ((2 - l % 4) + 4) % 4; }

// Flattened forward top of node c (stage k, parent p): x_c = a'_c + sum_i G_{c,i} u_off(a_i),
// stage rows z_c = h'_c + sum_i L_{c,i} u_off(a_i), with (device.cpp, host variant)
//   G_{c,i} = CL_c G_{p,i} (i < k-1), G_{c,k-1} = B_c, a'_c = CL_c a'_p + c_c,
//   L_{c,i} = Mf G_{p,i}, L_{c,k-1} = G'_c, h'_c = Mf a'_p, Mf = F_c + G'_c K_p.
__global__ void __launch_bounds__(kT) factor_flat(FactorParams F) {
  const int nx = F.nx, nu = F.nu, W = nx + nu, nxp = F.nxp;
  const int64_t xx = static_cast<int64_t>(nx) * nx, xu = static_cast<int64_t>(nx) * nu,
                uu = static_cast<int64_t>(nu) * nu;
  const int64_t csz = 2 * xx + 2 * xu + uu + 2 * nx + nu;
  extern __shared__ __align__(16) double sm[];  // Mf (m x nx) | a'_p (nx)
  for (int q = blockIdx.x; q < F.stage_count; q += gridDim.x) {
    const int c = F.stage_first + q;
    const int m = F.stage_rows[c];
    const int p = F.ancestor[c];
    int k = 0;
    for (int a = c; a > 0; a = F.ancestor[a]) ++k;  // stage of c
    const int Lp = pad2d(k * nu), Lpp = pad2d((k - 1) * nu);
    double* blk = F.fw_blk + F.flat_off[c];
    const double* pblk = k >= 2 ? F.fw_blk + F.flat_off[p] : nullptr;
    const double* J = F.bw_blk + F.bw_j[c];  // CL[a, t] = J[a + (nu + t) nxp]
    const double* cost = cost_of(F, c, csz);
    const double *Bc = cost + xx, *cc = Bc + xu;
    const double* Kb = F.fw_blk + F.k_off[p];  // K_p[w, z] = Kb[z + w nxp]
    const double* hc = F.hcoef + static_cast<int64_t>(F.dual_offset[c]) * W;
    double* Mf = sm;
    double* ap = sm + static_cast<int64_t>(m) * nx;
    for (int e = threadIdx.x; e < m * nx; e += kT) {
      const int s2 = e % m, z = e / m;
      double v = hc[static_cast<int64_t>(s2) * W + z];
      for (int w = 0; w < nu; ++w) v = fma(hc[static_cast<int64_t>(s2) * W + nx + w], Kb[z + static_cast<int64_t>(w) * nxp], v);
      Mf[e] = v;
    }
    for (int e = threadIdx.x; e < nx; e += kT) ap[e] = p == 0 ? F.root_state[e] : F.aff_fw[static_cast<int64_t>(p) * nx + e];
    __syncthreads();
    if (!F.flat_consts_only) {
      for (int e = threadIdx.x; e < (nx + m) * k * nu; e += kT) {
        const int r = e / (k * nu), ij = e - r * (k * nu), i = ij / nu, j = ij - i * nu;
        double v = 0.0;
        if (i == k - 1) {
          v = r < nx ? Bc[r + static_cast<int64_t>(j) * nx] : hc[static_cast<int64_t>(r - nx) * W + nx + j];
        } else {
          for (int z = 0; z < nx; ++z) {
            const double g = pblk[static_cast<int64_t>(z) * Lpp + i * nu + j];  // G_{p,i}[z, j]
            v = fma(r < nx ? J[r + static_cast<int64_t>(nu + z) * nxp] : Mf[(r - nx) + z * m], g, v);
          }
        }
        blk[static_cast<int64_t>(r) * Lp + ij] = v;
      }
    }
    for (int r = threadIdx.x; r < nx + m; r += kT) {
      double v = r < nx ? cc[r] : 0.0;
      for (int z = 0; z < nx; ++z) v = fma(r < nx ? J[r + static_cast<int64_t>(nu + z) * nxp] : Mf[(r - nx) + z * m], ap[z], v);
      if (r < nx)
        F.aff_fw[static_cast<int64_t>(c) * nx + r] = v;
      else
        F.aff_fwh[static_cast<int64_t>(c) * F.mmax + (r - nx)] = v;
    }
    __syncthreads();
  }
}

}  // namespace

cudaError_t factor_run_flat(const FactorParams& F, int grid, cudaStream_t st) {
  int mmax = F.mmax > 0 ? F.mmax : 1;
  const size_t smem = sizeof(double) * (static_cast<size_t>(mmax) * F.nx + F.nx);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(factor_flat, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  factor_flat<<<grid, kT, smem, st>>>(F);
  return cudaGetLastError();
}

cudaError_t factor_run_affine(const FactorParams& F, int grid, cudaStream_t st) {
  const size_t smem = sizeof(double) * (F.nu + 2 * F.nx);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(factor_affine, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  factor_affine<<<grid, kT, smem, st>>>(F);
  return cudaGetLastError();
}

int64_t factor_workspace_doubles(int nx, int nu, int max_rows) {
  const int64_t xx = static_cast<int64_t>(nx) * nx, xu = static_cast<int64_t>(nx) * nu,
                uu = static_cast<int64_t>(nu) * nu;
  const int64_t t = static_cast<int64_t>(nu > nx ? nu : nx) * (max_rows > 1 ? max_rows : 1);
  return 4 * xx + 3 * xu + 2 * uu + 2 * nx + nu + xu + (t > xu ? t : xu) + 16;
}

cudaError_t factor_run_leaves(const FactorParams& F, int grid, cudaStream_t st) {
  factor_leaves<<<grid, kT, 0, st>>>(F);
  return cudaGetLastError();
}

cudaError_t factor_run_stage(const FactorParams& F, int grid, size_t smem, cudaStream_t st) {
  if (smem) {
    cudaError_t e = cudaFuncSetAttribute(factor_stage, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  factor_stage<<<grid, kT, smem, st>>>(F);
  return cudaGetLastError();
}

}  // namespace scn
