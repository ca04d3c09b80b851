// SPDX-License-Identifier: MIT
//
// K1+K2: the dual-gradient / Hessian-vector sweep (tree_oracles.hpp:33-90)
// fused with apply_H (problem_data.hpp:144-162), as ONE persistent kernel.
//
// Work decomposition. Items (runs of same-stage nodes, see layout.hpp) are
// dispensed from a global ticket counter: first the backward items from the
// leaves to the root, then the forward items from the root to the leaves.
// Every dependency of an item therefore has a smaller ticket. A CTA processes
// its tickets in the order it grabbed them, so the smallest unfinished ticket
// always belongs to a running CTA whose dependencies are done: the scheme
// cannot deadlock and needs no grid-wide barrier, even with CTAs that are not
// co-resident. A node publishes completion through an epoch-stamped flag
// (release/acquire at gpu scope); consumers spin only on their own
// children (backward) or parent (forward).
//
// Data movement. Each CTA keeps a ring of `nslot` shared-memory slots. As
// soon as it owns a ticket, one thread issues a single cp.async.bulk (TMA 1-D)
// of the whole item (contiguous node blocks) into a free slot, completing on
// an mbarrier; the matrices are therefore in flight while the CTA is still
// waiting for the dependencies of earlier items. All matrix traffic is a
// sequential HBM stream; the small vectors (y, contributions, x, u) live in
// L2.
//
// Arithmetic. Every product is a set of "dot columns" (layout.hpp) computed
// by groups of G lanes (strided partial sums + butterfly shuffles), for all
// right-hand sides at once so a 2-RHS sweep (p-NAMA) reads the matrices once.
// fp64 throughout; the partial-sum order is fixed, so results are
// deterministic run to run and identical between 1- and 2-RHS launches.
#include <cuda_runtime.h>

#include <cstdint>

#include "layout.hpp"

namespace scn {

namespace {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void wait_flag(const unsigned* flag, unsigned epoch) {
  if (ld_acquire(flag) == epoch) return;
  unsigned ns = 32;
  while (ld_acquire(flag) != epoch) {
    __nanosleep(ns);
    if (ns < 256) ns <<= 1;
  }
}

__device__ __forceinline__ void issue_item(const SweepParams& P, unsigned t, double* slot, uint64_t* bar) {
  const Item it = P.items[t];
  const double* src = (it.pass == 0 ? P.bw_blk : P.fw_blk) + it.off;
  mbar_expect_tx(bar, static_cast<unsigned>(it.bytes));
  tma_load_1d(slot, src, static_cast<unsigned>(it.bytes), bar);
}

template <int NRHS>
__device__ __forceinline__ void group_reduce(double (&acc)[NRHS], int G) {
#pragma unroll
  for (int r = 0; r < NRHS; ++r)
    for (int o = G >> 1; o > 0; o >>= 1) acc[r] += __shfl_xor_sync(0xffffffffu, acc[r], o);
}

// ---------------------------------------------------------------- backward
// tree_oracles.hpp:44-73. For interior node c:
//   [u_off_c; w_c] = E_c' y_kids + sum_{k in kids} contrib_k (+ [sigma_c; c_hat_c])
// for a leaf: w_c = F_N' y_N (+ pi p_N); then for non-root c:
//   contrib_c = J_c' w_c = [child_to_input_c w_c ; closed_loop_c' w_c]
template <int NRHS>
__device__ void backward_item(const SweepParams& P, const Item& it, const double* blk, double* vec,
                              unsigned E, int G) {
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int nx = P.nx, nu = P.nu, W = nu + nx;
  const int first = it.first, cnt = it.count;
  const NodeMeta m0 = P.meta[first];
  const bool leaf = m0.leaf != 0;
  if (!leaf) {
    const NodeMeta ml = P.meta[first + cnt - 1];
    for (int k = m0.cb + tid; k < ml.cb + ml.cc; k += nthr) wait_flag(P.bw_flag + k, E);
  }
  __syncthreads();

  const int ngroups = nthr / G, g = tid / G, lane = tid % G;
  // phase A
  {
    const int ncols = leaf ? nx : W;
    const int ntasks = cnt * ncols;
    for (int base = 0; base < ntasks; base += ngroups) {
      const int task = base + g;
      const bool active = task < ntasks;
      double acc[NRHS];
#pragma unroll
      for (int r = 0; r < NRHS; ++r) acc[r] = 0.0;
      int ni = 0, j = 0, c = 0;
      if (active) {
        ni = task / ncols;
        j = task - ni * ncols;
        c = first + ni;
        const NodeMeta mc = P.meta[c];
        const double* nb = blk + (P.bw_off[c] - it.off);
        if (!leaf) {
          const double* col = nb + static_cast<int64_t>(j) * mc.M;
          for (int k = lane; k < mc.M; k += G) {
            const double a = col[k];
#pragma unroll
            for (int r = 0; r < NRHS; ++r) acc[r] += a * __ldg(P.y[r] + mc.cdo + k);
          }
          for (int k = lane; k < mc.cc; k += G) {
            const int64_t kid = mc.cb + k;
#pragma unroll
            for (int r = 0; r < NRHS; ++r) acc[r] += __ldcg(P.contrib[r] + kid * W + j);
          }
        } else {
          const double* col = nb + static_cast<int64_t>(j) * mc.mN;
          for (int k = lane; k < mc.mN; k += G) {
            const double a = col[k];
#pragma unroll
            for (int r = 0; r < NRHS; ++r) acc[r] += a * __ldg(P.y[r] + mc.tdo + k);
          }
        }
      }
      group_reduce<NRHS>(acc, G);
      if (active && lane == 0) {
        const int ja = leaf ? nu + j : j;
        const double aff = P.affine ? P.aff_bw[static_cast<int64_t>(c) * W + ja] : 0.0;
#pragma unroll
        for (int r = 0; r < NRHS; ++r) {
          const double v = acc[r] + aff;
          if (ja < nu)
            P.u[r][static_cast<int64_t>(c) * nu + ja] = v;  // u_off, finished by the forward pass
          else
            vec[(ni * NRHS + r) * nx + (ja - nu)] = v;  // costate w_c
        }
      }
    }
  }
  __syncthreads();
  // phase B: contributions to the parent
  if (first != 0) {
    const int ntasks = cnt * W;
    for (int base = 0; base < ntasks; base += ngroups) {
      const int task = base + g;
      const bool active = task < ntasks;
      double acc[NRHS];
#pragma unroll
      for (int r = 0; r < NRHS; ++r) acc[r] = 0.0;
      int ni = 0, j = 0, c = 0;
      if (active) {
        ni = task / W;
        j = task - ni * W;
        c = first + ni;
        const NodeMeta mc = P.meta[c];
        const double* nb = blk + (P.bw_off[c] - it.off);
        const double* col = nb + (leaf ? mc.mN * nx : mc.M * W) + static_cast<int64_t>(j) * nx;
        for (int k = lane; k < nx; k += G) {
          const double a = col[k];
#pragma unroll
          for (int r = 0; r < NRHS; ++r) acc[r] += a * vec[(ni * NRHS + r) * nx + k];
        }
      }
      group_reduce<NRHS>(acc, G);
      if (active && lane == 0) {
#pragma unroll
        for (int r = 0; r < NRHS; ++r) P.contrib[r][static_cast<int64_t>(c) * W + j] = acc[r];
      }
    }
  }
  __syncthreads();
  for (int i = tid; i < cnt; i += nthr) {
    __threadfence();
    st_release(P.bw_flag + first + i, E);
  }
}

// ---------------------------------------------------------------- forward
// tree_oracles.hpp:75-88 + apply_H. For non-root c with parent a:
//   [x_c; z_c] = W_c' [x_a; u_a] (+ [c_c; 0]);  then
//   interior: u_c = u_off_c + K_c x_c ;  leaf: z_N,c = F_N x_c
template <int NRHS>
__device__ void forward_item(const SweepParams& P, const Item& it, const double* blk, double* vec,
                             unsigned E, int G, int mmax) {
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int nx = P.nx, nu = P.nu, V = nx + nu;
  const int first = it.first, cnt = it.count;
  const NodeMeta m0 = P.meta[first];
  const bool leaf = m0.leaf != 0;
  const bool root = first == 0;
  double* vin = vec;                         // [cnt][NRHS][nx+nu]
  double* xb = vec + P.max_count * NRHS * V;  // [cnt][NRHS][nx]
  if (root) {
    if (tid == 0) wait_flag(P.bw_flag, E);
  } else {
    const int a0 = m0.anc, a1 = P.meta[first + cnt - 1].anc;
    for (int k = a0 + tid; k <= a1; k += nthr) wait_flag(P.fw_flag + k, E);
  }
  __syncthreads();
  if (root) {
    for (int idx = tid; idx < NRHS * nx; idx += nthr) {
      const int r = idx / nx, k = idx - r * nx;
      const double v = P.affine ? P.root_state[k] : 0.0;
      xb[r * nx + k] = v;
      P.x[r][k] = v;
    }
  } else {
    const int tot = cnt * NRHS * V;
    for (int idx = tid; idx < tot; idx += nthr) {
      const int ni = idx / (NRHS * V);
      const int rem = idx - ni * NRHS * V;
      const int r = rem / V, k = rem - r * V;
      const int64_t a = P.meta[first + ni].anc;
      vin[idx] = k < nx ? __ldcg(P.x[r] + a * nx + k) : __ldcg(P.u[r] + a * nu + (k - nx));
    }
  }
  __syncthreads();
  const int ngroups = nthr / G, g = tid / G, lane = tid % G;
  if (!root) {  // phase A: state + stage rows
    const int ncols = nx + mmax;
    const int ntasks = cnt * ncols;
    for (int base = 0; base < ntasks; base += ngroups) {
      const int task = base + g;
      int ni = task / ncols;
      int j = task - ni * ncols;
      const int c = first + ni;
      bool active = task < ntasks;
      NodeMeta mc{};
      if (active) {
        mc = P.meta[c];
        active = j < nx + mc.m;
      }
      double acc[NRHS];
#pragma unroll
      for (int r = 0; r < NRHS; ++r) acc[r] = 0.0;
      if (active) {
        const double* col = blk + (P.fw_off[c] - it.off) + static_cast<int64_t>(j) * V;
        const double* v = vin + ni * NRHS * V;
        for (int k = lane; k < V; k += G) {
          const double a = col[k];
#pragma unroll
          for (int r = 0; r < NRHS; ++r) acc[r] += a * v[r * V + k];
        }
      }
      group_reduce<NRHS>(acc, G);
      if (active && lane == 0) {
        if (j < nx) {
          const double aff = P.affine ? P.aff_fw[static_cast<int64_t>(c) * nx + j] : 0.0;
#pragma unroll
          for (int r = 0; r < NRHS; ++r) {
            const double xv = acc[r] + aff;
            xb[(ni * NRHS + r) * nx + j] = xv;
            P.x[r][static_cast<int64_t>(c) * nx + j] = xv;
          }
        } else {
#pragma unroll
          for (int r = 0; r < NRHS; ++r) P.Hx[r][mc.doff + (j - nx)] = acc[r];
        }
      }
    }
  }
  __syncthreads();
  {  // phase B: input (interior) or terminal rows (leaf)
    const int ncols = leaf ? P.max_mN : nu;
    const int ntasks = cnt * ncols;
    for (int base = 0; base < ntasks; base += ngroups) {
      const int task = base + g;
      const int ni = task / ncols;
      const int j = task - ni * ncols;
      const int c = first + ni;
      bool active = task < ntasks;
      NodeMeta mc{};
      if (active) {
        mc = P.meta[c];
        if (leaf) active = j < mc.mN;
      }
      double acc[NRHS];
#pragma unroll
      for (int r = 0; r < NRHS; ++r) acc[r] = 0.0;
      if (active) {
        const int64_t skip = root ? 0 : static_cast<int64_t>(V) * (nx + mc.m);
        const double* col = blk + (P.fw_off[c] - it.off) + skip + static_cast<int64_t>(j) * nx;
        const double* xv = xb + ni * NRHS * nx;
        for (int k = lane; k < nx; k += G) {
          const double a = col[k];
#pragma unroll
          for (int r = 0; r < NRHS; ++r) acc[r] += a * xv[r * nx + k];
        }
      }
      group_reduce<NRHS>(acc, G);
      if (active && lane == 0) {
#pragma unroll
        for (int r = 0; r < NRHS; ++r) {
          if (leaf) {
            P.Hx[r][mc.tdo + j] = acc[r];
          } else {
            const int64_t o = static_cast<int64_t>(c) * nu + j;
            P.u[r][o] = __ldcg(P.u[r] + o) + acc[r];
          }
        }
      }
    }
  }
  __syncthreads();
  for (int i = tid; i < cnt; i += nthr) {
    __threadfence();
    st_release(P.fw_flag + first + i, E);
  }
}

template <int NRHS>
__global__ void __launch_bounds__(256, 1) sweep_kernel(const SweepParams P, int G, int mmax) {
  extern __shared__ __align__(128) double smem[];
  __shared__ __align__(8) uint64_t mbar[kMaxSlots];
  __shared__ unsigned tick[kMaxSlots];
  __shared__ unsigned s_epoch;
  const int tid = threadIdx.x;
  const unsigned total = static_cast<unsigned>(P.items_total);
  double* slots = smem;
  double* vec = smem + static_cast<int64_t>(P.nslot) * P.slot_doubles;
  if (tid == 0) {
    s_epoch = *reinterpret_cast<volatile unsigned*>(P.ctrl) + 1u;
    for (int s = 0; s < P.nslot; ++s) mbar_init(&mbar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int s = 0; s < P.nslot; ++s) {
      const unsigned t = atomicAdd(P.ctrl + 1, 1u);
      tick[s] = t;
      if (t < total) issue_item(P, t, slots + static_cast<int64_t>(s) * P.slot_doubles, &mbar[s]);
    }
  }
  __syncthreads();
  const unsigned E = s_epoch;
  unsigned phase_bits = 0;
  for (int k = 0;; ++k) {
    const int s = k % P.nslot;
    const unsigned t = tick[s];
    if (t >= total) break;
    mbar_wait(&mbar[s], (phase_bits >> s) & 1u);
    phase_bits ^= 1u << s;
    const Item it = P.items[t];
    const double* blk = slots + static_cast<int64_t>(s) * P.slot_doubles;
    if (it.pass == 0)
      backward_item<NRHS>(P, it, blk, vec, E, G);
    else
      forward_item<NRHS>(P, it, blk, vec, E, G, mmax);
    if (tid == 0) {
      fence_proxy_async();
      const unsigned t2 = atomicAdd(P.ctrl + 1, 1u);
      tick[s] = t2;
      if (t2 < total) issue_item(P, t2, slots + static_cast<int64_t>(s) * P.slot_doubles, &mbar[s]);
    }
    __syncthreads();
  }
  if (tid == 0) {
    __threadfence();
    const unsigned prev = atomicAdd(P.ctrl + 2, 1u);
    if (prev == gridDim.x - 1) {
      P.ctrl[1] = 0u;
      P.ctrl[2] = 0u;
      __threadfence();
      atomicExch(P.ctrl, E);
    }
  }
}

}  // namespace

cudaError_t sweep_configure(int nrhs, size_t dyn_smem) {
  cudaError_t e = cudaFuncSetAttribute(sweep_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(dyn_smem));
  if (e != cudaSuccess) return e;
  (void)nrhs;
  return cudaFuncSetAttribute(sweep_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              static_cast<int>(dyn_smem));
}

cudaError_t sweep_occupancy(int* ctas_per_sm, size_t dyn_smem) {
  int a = 0, b = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, sweep_kernel<1>, 256, dyn_smem);
  if (e != cudaSuccess) return e;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, sweep_kernel<2>, 256, dyn_smem);
  *ctas_per_sm = a < b ? a : b;
  return e;
}

cudaError_t sweep_launch(const SweepParams& P, int grid, size_t dyn_smem, int G, int mmax,
                         cudaStream_t stream) {
  if (P.nrhs == 2)
    sweep_kernel<2><<<grid, 256, dyn_smem, stream>>>(P, G, mmax);
  else
    sweep_kernel<1><<<grid, 256, dyn_smem, stream>>>(P, G, mmax);
  return cudaGetLastError();
}

}  // namespace scn
