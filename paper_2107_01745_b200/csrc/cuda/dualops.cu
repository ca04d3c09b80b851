// SPDX-License-Identifier: MIT
//
// K3-K8: fused dual-vector kernels of the forward-backward machinery
// (fbe.hpp, lbfgs.hpp, prox.hpp, solvers.hpp). Dual vectors are small next
// to the sweep's matrix stream (37k doubles at C3), so these kernels are
// latency-bound: each one is a single cooperative persistent grid that does
// all the passes of one algorithmic step, with grid barriers between passes
// and a deterministic reduction (fixed per-block tree, block partials summed
// in block order by every block). Every block therefore sees bit-identical
// scalars, and decisions (L-BFGS curvature gate, first accepted line-search
// step, power-iteration stop) are taken on the device without a host round
// trip.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>

#include "dual.hpp"
#include "fbrow.cuh"

namespace scn {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kMaxRed = 32;  // scalars per reduction
constexpr int kMaxBlocks = 160;  // dual-kernel grid (one block per SM; B200: 148)
constexpr int kPartsPerLane = kMaxBlocks / 32;

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ void grid_sync(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned gen = *reinterpret_cast<volatile unsigned*>(bar + 1);
    __threadfence();
    const unsigned arrived = atomicAdd(bar, 1u);
    if (arrived == gridDim.x - 1) {
      atomicExch(bar, 0u);
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (ld_acquire(bar + 1) == gen) __nanosleep(20);
    }
  }
  __syncthreads();
}

// Deterministic grid reduction of K per-thread values (sum, or max when
// MAX; values from index MAXFROM on are max-reduced, the rest summed). Every
// thread of every block receives the totals in v.
template <int K, bool MAX = false, int MAXFROM = (MAX ? 0 : K)>
__device__ void grid_reduce(const DualCtx& c, int& ph, double (&v)[K]) {
  __shared__ double sh[kWarps][kMaxRed];
  __shared__ double tot[kMaxRed];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double t = v[k];
    const bool mx = k >= MAXFROM;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double u = __shfl_xor_sync(0xffffffffu, t, o);
      t = mx ? fmax(t, u) : t + u;
    }
    if (lane == 0) sh[warp][k] = t;
  }
  __syncthreads();
  if (threadIdx.x < K) {
    const bool mx = static_cast<int>(threadIdx.x) >= MAXFROM;
    double t = sh[0][threadIdx.x];
    for (int w = 1; w < kWarps; ++w) t = mx ? fmax(t, sh[w][threadIdx.x]) : t + sh[w][threadIdx.x];
    c.part[(static_cast<int64_t>(ph) * 64 + threadIdx.x) * c.nblk + blockIdx.x] = t;
  }
  grid_sync(c.bar);
  // The K totals are spread over the block's warps; a warp first issues every
  // load of its values' block partials (one L2 round trip instead of one per
  // partial and value), then combines them in the fixed order (lane-strided
  // over the blocks, then the xor tree): the same bits as a sequential loop.
  {
    constexpr int KW = (K + kWarps - 1) / kWarps;  // values per warp
    double ld[KW][kPartsPerLane];
#pragma unroll
    for (int j = 0; j < KW; ++j) {
      const int k = warp + j * kWarps;
      const double* p = c.part + (static_cast<int64_t>(ph) * 64 + k) * c.nblk;
#pragma unroll
      for (int u = 0; u < kPartsPerLane; ++u) {
        const int b = lane + 32 * u;
        ld[j][u] = (k < K && b < c.nblk) ? __ldcg(p + b) : 0.0;
      }
    }
#pragma unroll
    for (int j = 0; j < KW; ++j) {
      const int k = warp + j * kWarps;
      const bool mx = k >= MAXFROM;
      double t = mx ? -INFINITY : 0.0;
#pragma unroll
      for (int u = 0; u < kPartsPerLane; ++u)
        if (lane + 32 * u < c.nblk) t = mx ? fmax(t, ld[j][u]) : t + ld[j][u];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double v2 = __shfl_xor_sync(0xffffffffu, t, o);
        t = mx ? fmax(t, v2) : t + v2;
      }
      if (lane == 0 && k < K) tot[k] = t;
    }
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < K; ++k) v[k] = tot[k];
  ph ^= 1;
}

// ---- sharded handles (DualCtx: cnt / xs / xr / phase)
__device__ __forceinline__ bool counted(const DualCtx& c, int64_t i) { return !c.cnt || c.cnt[i]; }

// This rank's totals of K per-thread values into xs[off, off + K) (every
// block takes part in the grid reduction; block 0 writes).
template <int K, int MAXFROM = K>
__device__ void xsend(const DualCtx& c, int& ph, double (&v)[K], int off) {
  grid_reduce<K, false, MAXFROM>(c, ph, v);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) c.xs[off + k] = v[k];
  }
}
// The ranks' totals gathered in xr, combined in rank order (sum; max from
// MAXFROM on): bitwise the same on every rank and every block.
template <int K, int MAXFROM = K>
__device__ void xrecv(const DualCtx& c, double (&v)[K], int off) {
  __shared__ double tot[kMaxRed];
  static_assert(K <= kMaxRed, "xrecv: at most kMaxRed values");
  __syncthreads();
  if (threadIdx.x < K) {
    const int k = threadIdx.x;
    const bool mx = k >= MAXFROM;
    double t = c.xr[off + k];
    for (int q = 1; q < c.world; ++q) {
      const double u = c.xr[q * kXMax + off + k];
      t = mx ? fmax(t, u) : t + u;
    }
    tot[k] = t;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < K; ++k) v[k] = tot[k];
}
// One reduction point of a kernel. Unsharded: the grid reduction. Sharded
// phase 0: this rank's totals go to xs and the kernel must return (false);
// phase 1: the totals of all ranks from xr.
template <int K, bool MAX = false, int MAXFROM = (MAX ? 0 : K)>
__device__ bool xreduce(const DualCtx& c, int& ph, double (&v)[K]) {
  if (c.phase < 0) {
    grid_reduce<K, MAX, MAXFROM>(c, ph, v);
    return true;
  }
  if (c.phase == 0) {
    xsend<K, MAXFROM>(c, ph, v, 0);
    return false;
  }
  xrecv<K, MAXFROM>(c, v, 0);
  return true;
}

using fbrow::conj_row;
using fbrow::prox_row;

__device__ __forceinline__ int gtid() { return blockIdx.x * kThreads + threadIdx.x; }
__device__ __forceinline__ int gstride() { return gridDim.x * kThreads; }

// ---------------------------------------------------------------- K3
__global__ void __launch_bounds__(kThreads) fb_finish_kernel(DualCtx c, int st, int mode, const double* y,
                                                             const double* Hx, const double* Hx0,
                                                             const double* weight, double* z, double* R,
                                                             double* T) {
  int ph = 0;
  const double lam = c.S[st * sl::kStateStride + sl::LAM];
  const double gp = 1.0 / lam;
  double s[6] = {0, 0, 0, 0, 0, 0};  // conj, z2, Hx.R, R2, (Hx0+Hx).y; [5] weighted inf residual (max)
  if (c.phase <= 0)
    for (int i = gtid(); i < c.D; i += gstride())
      fbrow::fb_row(i, c.g.kind[i], y[i], Hx[i], c.g.lo[i], c.g.hi[i], c.g.wg[i], lam, gp, mode, Hx0, weight, z, R,
                    T, counted(c, i), s);
  if (c.phase == 1 && blockIdx.x != 0) return;  // block 0 finishes
  if (!xreduce<6, false, 5>(c, ph, s)) return;  // one barrier: five sums and the max
  if (blockIdx.x == 0 && threadIdx.x == 0) fbrow::fb_finalize(c.S, c.I, st, mode, s);
  // thread 0's S / I writes are visible to the block after publish_block's barrier
  if (c.pub && blockIdx.x == 0) fbrow::publish_block(c.S, c.I, c.pub, c.seq);
}

// ---------------------------------------------------------------- K7
__global__ void __launch_bounds__(kThreads) fbe_grad_kernel(DualCtx c, int st, const double* R,
                                                            const double* HR, double* grad) {
  int ph = 0;
  const double lam = c.S[st * sl::kStateStride + sl::LAM];
  double s[2] = {0, 0};
  if (c.phase <= 0)
    for (int i = gtid(); i < c.D; i += gstride()) {
      const double Ri = R[i];
      const double gi = Ri + lam * HR[i];
      grad[i] = gi;
      const double img = (gi - Ri) / lam;
      if (counted(c, i)) {
        s[0] += img * img;
        s[1] += Ri * Ri;
      }
    }
  if (!xreduce<2>(c, ph, s)) return;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    c.S[sl::IMG2] = s[0];
    c.S[sl::R2] = s[1];
  }
}

// ---------------------------------------------------------------- K5
__global__ void __launch_bounds__(kThreads) lbfgs_kernel(DualCtx c, int mem, double eps_curv, double scale_ref,
                                                         int do_push,
                                                         const double* a, const double* b, const double* cc,
                                                         const double* dd, const double* gv, double* out,
                                                         double* Sb, double* Qb) {
  if (c.skip && *reinterpret_cast<const volatile int*>(c.skip)) return;  // speculative launch, not needed
  int ph = 0;
  const int64_t D = c.D;
  __shared__ int order[64];
  __shared__ int count_s;
  if (threadIdx.x == 0) {
    count_s = c.I[il::LB_COUNT];
    for (int j = 0; j <= mem; ++j) order[j] = c.I[il::LB_ORDER + j];
  }
  __syncthreads();
  int count = count_s;
  double gamma0 = c.S[sl::GAMMA0];
  __shared__ double alpha[64];
  __shared__ double curv[64];
  if (threadIdx.x <= mem && threadIdx.x < 64) curv[threadIdx.x] = c.S[sl::CURV + threadIdx.x];
  __syncthreads();
  int pushed = 0;
  if (do_push) {  // lbfgs.hpp:33-44 (strict curvature gate, FIFO eviction)
    const int f = order[count];  // a free slot
    double* sv = Sb + f * D;
    double* qv = Qb + f * D;
    double s4[4] = {0, 0, 0, 0};  // <s,q>, |s|^2, |q|^2, |dd|^2 (scale_ref)
    for (int i = gtid(); i < c.D; i += gstride()) {
      const double si = a[i] - b[i];
      const double qi = cc[i] - dd[i];
      sv[i] = si;
      qv[i] = qi;
      s4[0] += si * qi;
      s4[1] += si * si;
      s4[2] += qi * qi;
      s4[3] += dd[i] * dd[i];
    }
    grid_reduce<4>(c, ph, s4);
    const double curvature = s4[0];
    const double scale = scale_ref >= 0.0 ? scale_ref : s4[3];
    if ((curvature > eps_curv * s4[1] * scale) && (s4[2] > 0.0)) {
      pushed = 1;
      if (threadIdx.x == 0) {
        if (count == mem) {  // evict the oldest pair
          const int o = order[0];
          for (int j = 0; j + 1 < mem; ++j) order[j] = order[j + 1];
          order[mem - 1] = f;
          order[mem] = o;
        } else {
          ++count_s;  // order[count] already holds f
        }
        curv[f] = curvature;
      }
      __syncthreads();
      count = count_s;
      gamma0 = curvature / s4[2];
    }
  }
  // two-loop recursion (lbfgs.hpp:48-62), fused dot/axpy passes
  if (count == 0) {
    for (int i = gtid(); i < c.D; i += gstride()) out[i] = -(gamma0 * gv[i]);
  } else {
    // first loop: newest -> oldest
    double pend = 0.0;
    int pend_slot = -1;
    for (int j = count - 1; j >= 0; --j) {
      const int sj = order[j];
      const double* s_j = Sb + sj * D;
      const double* q_p = pend_slot >= 0 ? Qb + pend_slot * D : nullptr;
      double acc[1] = {0.0};
      for (int i = gtid(); i < c.D; i += gstride()) {
        double w = (j == count - 1) ? gv[i] : out[i];
        if (q_p) w = w - pend * q_p[i];
        out[i] = w;
        acc[0] += s_j[i] * w;
      }
      grid_reduce<1>(c, ph, acc);
      const double al = acc[0] / curv[sj];
      if (threadIdx.x == 0) alpha[j] = al;
      pend = al;
      pend_slot = sj;
    }
    __syncthreads();
    // scale by gamma0 after the last pending update, then second loop
    double pb = 0.0;
    int pb_slot = -1;
    for (int j = 0; j < count; ++j) {
      const int sj = order[j];
      const double* q_j = Qb + sj * D;
      double acc[1] = {0.0};
      for (int i = gtid(); i < c.D; i += gstride()) {
        double w = out[i];
        if (j == 0) {
          w = w - alpha[0] * Qb[order[0] * D + i];
          w = w * gamma0;
        } else {
          w = w + pb * Sb[pb_slot * D + i];
        }
        out[i] = w;
        acc[0] += q_j[i] * w;
      }
      grid_reduce<1>(c, ph, acc);
      const double beta = acc[0] / curv[sj];
      pb = alpha[j] - beta;
      pb_slot = sj;
    }
    for (int i = gtid(); i < c.D; i += gstride()) out[i] = -(out[i] + pb * Sb[pb_slot * D + i]);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    c.I[il::LB_COUNT] = count;
    c.I[il::LB_PUSHED] = pushed;
    for (int j = 0; j <= mem; ++j) {
      c.I[il::LB_ORDER + j] = order[j];
      c.S[sl::CURV + j] = curv[j];
    }
    c.S[sl::GAMMA0] = gamma0;
  }
}

// L-BFGS direction in compact form (Byrd, Nocedal & Schnabel 1994; lbfgs.hpp
// restated): with the pairs oldest -> newest, R = upper(S'Y), D = diag(S'Y),
// a = S'g, b = Y'g, t = R^-1 a, u = R^-T ((D + g0 Y'Y) t - g0 b),
//   H g = g0 g + S u - g0 Y t,     direction = -H g,
// the same matrix as the two-loop recursion. One pass computes the new pair
// (the curvature gate's dots), the new pair's row of S'Y and Y'Y against the
// stored pairs, and S'g, Y'g: one grid reduction instead of 2*mem + 1. S'Y
// and Y'Y of the stored pairs persist in Mb (slot-indexed); only the free
// slot's row / column is written, which no block reads, so no barrier.
constexpr int kCompactMem = 6;
constexpr int kCompactK = 6 + 4 * kCompactMem + 2;  // 32 <= kMaxRed (last two: fused fbe_grad norms)
constexpr int kMbLd = 64;                      // Mb: STY[kMbLd][kMbLd] | YTY[kMbLd][kMbLd]

// fR != nullptr: fbe_grad (fbe.hpp:89-94) fused in front: grad = R + lam HR of
// state fstate is written to gout and used as both cc and gv; IMG2 / R2 as
// fbe_grad_kernel computes them.
__global__ void __launch_bounds__(kThreads) lbfgs_compact_kernel(DualCtx c, int mem, double eps_curv, double scale_ref,
                                                                 int do_push, const double* a, const double* b,
                                                                 const double* cc, const double* dd, const double* gv,
                                                                 double* out, double* Sb, double* Qb, double* Mb,
                                                                 const double* fR, const double* fHR, int fstate,
                                                                 double* gout) {
  if (c.skip && *reinterpret_cast<const volatile int*>(c.skip)) return;  // speculative launch, not needed
  int ph = 0;
  const int64_t D = c.D;
  __shared__ int order[kCompactMem + 1];
  __shared__ int count_s, cnt_new, pushed_s;
  __shared__ double coef_u[kCompactMem], coef_t[kCompactMem], gamma_s;
  if (threadIdx.x == 0) {
    count_s = c.I[il::LB_COUNT];
    for (int j = 0; j <= mem; ++j) order[j] = c.I[il::LB_ORDER + j];
  }
  __syncthreads();
  const int count = count_s;  // stored pairs before this call
  const int f = order[count];  // free slot (target of a push)
  // S'Y / Y'Y of the stored pairs (by age position), fetched in parallel now:
  // the small solves after the reduction then read shared memory only
  __shared__ double pSTY[kCompactMem][kCompactMem], pYTY[kCompactMem][kCompactMem];
  __shared__ double g0_in;
  if (threadIdx.x < kCompactMem * kCompactMem) {
    const int i = threadIdx.x / kCompactMem, j = threadIdx.x % kCompactMem;
    if (i < count && j < count) {
      pSTY[i][j] = Mb[order[i] * kMbLd + order[j]];
      pYTY[i][j] = Mb[kMbLd * kMbLd + order[i] * kMbLd + order[j]];
    }
  }
  if (threadIdx.x == 64) g0_in = c.S[sl::GAMMA0];
  // v: 0 <s,q> 1 |s|^2 2 |q|^2 3 |dd|^2 4 <s,g> 5 <q,g>; old pair j (order position):
  //    6+j <s_j,g>, 6+M+j <y_j,g>, 6+2M+j <s_j,q>, 6+3M+j <y_j,q>   (M = kCompactMem)
  double v[kCompactK];
#pragma unroll
  for (int k = 0; k < kCompactK; ++k) v[k] = 0.0;
  const double* sj_[kCompactMem];
  const double* yj_[kCompactMem];
#pragma unroll
  for (int j = 0; j < kCompactMem; ++j) {
    sj_[j] = Sb + static_cast<int64_t>(order[j < count ? j : 0]) * D;
    yj_[j] = Qb + static_cast<int64_t>(order[j < count ? j : 0]) * D;
  }
  double* sf = Sb + static_cast<int64_t>(f) * D;
  double* qf = Qb + static_cast<int64_t>(f) * D;
  const double flam = fR ? c.S[fstate * sl::kStateStride + sl::LAM] : 0.0;
  for (int64_t i = gtid(); c.phase <= 0 && i < D; i += gstride()) {
    const bool ci = counted(c, i);
    double gi;
    if (fR) {
      const double Ri = fR[i];
      gi = Ri + flam * fHR[i];
      gout[i] = gi;
      const double img = (gi - Ri) / flam;
      if (ci) {
        v[kCompactK - 2] += img * img;
        v[kCompactK - 1] += Ri * Ri;
      }
    } else {
      gi = gv[i];
    }
    if (!ci) {  // not this rank's row: the new pair's entries only
      if (do_push) {
        sf[i] = a[i] - b[i];
        qf[i] = (fR ? gi : cc[i]) - dd[i];
      }
      continue;
    }
    if (do_push) {
      const double si = a[i] - b[i], qi = (fR ? gi : cc[i]) - dd[i], di = dd[i];
      sf[i] = si;
      qf[i] = qi;
      v[0] += si * qi;
      v[1] += si * si;
      v[2] += qi * qi;
      v[3] += di * di;
      v[4] += si * gi;
      v[5] += qi * gi;
#pragma unroll
      for (int j = 0; j < kCompactMem; ++j)
        if (j < count) {
          const double sj = sj_[j][i], yj = yj_[j][i];
          v[6 + j] += sj * gi;
          v[6 + kCompactMem + j] += yj * gi;
          v[6 + 2 * kCompactMem + j] += sj * qi;
          v[6 + 3 * kCompactMem + j] += yj * qi;
        }
    } else {
#pragma unroll
      for (int j = 0; j < kCompactMem; ++j)
        if (j < count) {
          v[6 + j] += sj_[j][i] * gi;
          v[6 + kCompactMem + j] += yj_[j][i] * gi;
        }
    }
  }
  if (!xreduce<kCompactK>(c, ph, v)) return;
  // the serial part indexes the totals at run time: from shared memory, so
  // that v stays in registers through the accumulation above
  __shared__ double vs[kCompactK];
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k2 = 0; k2 < kCompactK; ++k2) vs[k2] = v[k2];
  }
  __syncthreads();
  // every block: gate, pair set, small triangular solves (identical results).
  // The gate is evaluated by every thread; the active pairs' S'Y / Y'Y / S'g /
  // Y'g entries are gathered into shared memory in parallel, so thread 0's
  // solves (fully unrolled over kCompactMem, predicated) run on registers and
  // shared memory only.
  const double* vv = vs;
  double gamma0 = g0_in;
  int cnt = count, pushed = 0, first = 0;
  if (do_push) {  // lbfgs.hpp:33-44 (strict curvature gate, FIFO eviction)
    const double scale = scale_ref >= 0.0 ? scale_ref : vv[3];
    if ((vv[0] > eps_curv * vv[1] * scale) && (vv[2] > 0.0)) {
      pushed = 1;
      gamma0 = vv[0] / vv[2];
      if (cnt == mem) first = 1;  // evict the oldest
      else ++cnt;
    }
  }
  // age positions: 0..count-1 the stored pairs, count the new pair; active k -> first + k
  auto sty = [&](int pi, int pj) -> double {  // age positions, pi <= pj
    if (pj == count) return pi == count ? vv[0] : vv[6 + 2 * kCompactMem + pi];
    return pSTY[pi][pj];
  };
  auto yty = [&](int pi, int pj) -> double {
    if (pi == count || pj == count) {
      if (pi == count && pj == count) return vv[2];
      return vv[6 + 3 * kCompactMem + (pi == count ? pj : pi)];
    }
    return pYTY[pi][pj];
  };
  __shared__ double aR[kCompactMem][kCompactMem], aY[kCompactMem][kCompactMem], aA[kCompactMem], aB[kCompactMem];
  if (threadIdx.x < kCompactMem * kCompactMem) {
    const int i = threadIdx.x / kCompactMem, j = threadIdx.x % kCompactMem;
    if (i < cnt && j < cnt) {
      if (i <= j) aR[i][j] = sty(first + i, first + j);
      aY[i][j] = yty(first + i, first + j);
    }
  } else if (threadIdx.x < kCompactMem * kCompactMem + kCompactMem) {
    const int i = threadIdx.x - kCompactMem * kCompactMem, p2 = first + i;
    if (i < cnt) {
      aA[i] = p2 == count ? vv[4] : vv[6 + p2];
      aB[i] = p2 == count ? vv[5] : vv[6 + kCompactMem + p2];
    }
  }
  if (pushed && blockIdx.x == 0 && threadIdx.x == 64) {  // the new pair's row / column (slot f; read by no block)
    double* STY = Mb;
    double* YTY = Mb + kMbLd * kMbLd;
    for (int k = 0; k < count; ++k) {
      const int sk = order[k];
      STY[sk * kMbLd + f] = vv[6 + 2 * kCompactMem + k];  // s_k . y_new (older k)
      YTY[sk * kMbLd + f] = vv[6 + 3 * kCompactMem + k];
      YTY[f * kMbLd + sk] = vv[6 + 3 * kCompactMem + k];
    }
    STY[f * kMbLd + f] = vv[0];
    YTY[f * kMbLd + f] = vv[2];
    c.S[sl::CURV + f] = vv[0];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t[kCompactMem], u[kCompactMem];
#pragma unroll
    for (int i = kCompactMem - 1; i >= 0; --i) {  // t = R^-1 a
      if (i < cnt) {
        double s2 = aA[i];
#pragma unroll
        for (int j = i + 1; j < kCompactMem; ++j)
          if (j < cnt) s2 -= aR[i][j] * t[j];
        t[i] = s2 / aR[i][i];
      }
    }
#pragma unroll
    for (int i = 0; i < kCompactMem; ++i) {  // u = R^-T ((D + g0 Y'Y) t - g0 b)
      if (i < cnt) {
        double w = aR[i][i] * t[i];
#pragma unroll
        for (int j = 0; j < kCompactMem; ++j)
          if (j < cnt) w += gamma0 * aY[i][j] * t[j];
        w -= gamma0 * aB[i];
#pragma unroll
        for (int j = 0; j < kCompactMem; ++j)
          if (j < i) w -= aR[j][i] * u[j];
        u[i] = w / aR[i][i];
      }
    }
#pragma unroll
    for (int i = 0; i < kCompactMem; ++i)
      if (i < cnt) {
        coef_u[i] = u[i];
        coef_t[i] = t[i];
      }
    // slot order after the push (oldest first), spare slot last
    int ord[kCompactMem + 1];
#pragma unroll
    for (int k = 0; k < kCompactMem; ++k)
      if (k < cnt) ord[k] = first + k == count ? f : order[first + k];
    int spare;
    if (pushed && first) spare = order[0];
    else if (!pushed) spare = f;
    else spare = order[cnt];
#pragma unroll
    for (int k = 0; k < kCompactMem; ++k)
      if (k < cnt) order[k] = ord[k];
    order[cnt] = spare;
    cnt_new = cnt;
    pushed_s = pushed;
    gamma_s = gamma0;
  }
  __syncthreads();
  cnt = cnt_new;
  const double g0 = gamma_s;
  const double* S_[kCompactMem];
  const double* Y_[kCompactMem];
#pragma unroll
  for (int j = 0; j < kCompactMem; ++j) {
    S_[j] = Sb + static_cast<int64_t>(order[j < cnt ? j : 0]) * D;
    Y_[j] = Qb + static_cast<int64_t>(order[j < cnt ? j : 0]) * D;
  }
  const double* gvec = fR ? gout : gv;  // fused: each thread reads back its own writes
  for (int64_t i = gtid(); i < D; i += gstride()) {  // direction = -(g0 g + S u - g0 Y t)
    double h = g0 * gvec[i];
#pragma unroll
    for (int j = 0; j < kCompactMem; ++j)
      if (j < cnt) h += coef_u[j] * S_[j][i] - g0 * coef_t[j] * Y_[j][i];
    out[i] = -h;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    c.I[il::LB_COUNT] = cnt;
    c.I[il::LB_PUSHED] = pushed_s;
    for (int j = 0; j <= mem; ++j) c.I[il::LB_ORDER + j] = order[j];
    c.S[sl::GAMMA0] = g0;
    if (fR) {
      c.S[sl::IMG2] = v[kCompactK - 2];
      c.S[sl::R2] = v[kCompactK - 1];
    }
  }
}

// ---------------------------------------------------------------- K4 / K6
// Line-search certificate (fbe.hpp:105-231) and the tau search of
// solvers.hpp:310-325 / 440-464. The row arithmetic and the scalar decisions
// live in shared helpers so that the single-launch kernel and the sharded
// phase kernel compute bit-identical values (a world-1 sharded solve equals
// the unsharded one bitwise).
struct Taus {
  double t[16];
};
// taus.t[k] by unrolled select: a run-time index into a kernel parameter
// would copy the whole array to local memory in every thread
__device__ __forceinline__ double tau_at(const Taus& taus, int k) {
  double t = taus.t[15];
#pragma unroll
  for (int m = 0; m < 16; ++m)
    if (m == k) t = taus.t[m];
  return t;
}

// Row arithmetic of the certificate with explicit round-to-nearest
// operations (no FMA contraction): the single-launch and the sharded kernel
// inline these into different code, and the compiler must not be free to
// fuse them differently. This is also the CPU oracle's arithmetic
// (-ffp-contract=off).
__device__ __forceinline__ double mul_(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add_(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub_(double a, double b) { return __dsub_rn(a, b); }

struct CertRow {
  double an, di, ha, hd;  // anchor, direction, Hx(anchor), Hx0(direction)
};
// shifted (NAMA, fbe.hpp:172-203): anchor y - lam R, direction d + lam R
__device__ __forceinline__ CertRow cert_row(int shifted, double lam, const double* y, const double* R,
                                            const double* Hx, const double* HR, const double* d,
                                            const double* Hd, int64_t i) {
  CertRow r{y[i], d[i], Hx[i], Hd[i]};
  if (shifted) {
    const double rr = mul_(-lam, R[i]);
    const double hr = mul_(-lam, HR[i]);
    r.an = add_(r.an, rr);
    r.di = sub_(r.di, rr);
    r.ha = add_(r.ha, hr);
    r.hd = sub_(r.hd, hr);
  }
  return r;
}
// trial tau of one row: z = prox(pb + tau ps), R = z - (ha + tau hd), T = (an + tau di) - lam R
struct CertTrial {
  double z, Rt, Tt, hxw;
};
__device__ __forceinline__ CertTrial cert_trial(const CertRow& r, int kd, double lo, double hi, double wg,
                                                double lam, double gp, double pb, double ps, double tau) {
  CertTrial t;
  t.z = prox_row(kd, add_(pb, mul_(tau, ps)), lo, hi, gp * wg);
  t.hxw = add_(r.ha, mul_(tau, r.hd));
  t.Rt = sub_(t.z, t.hxw);
  t.Tt = sub_(add_(r.an, mul_(tau, r.di)), mul_(lam, t.Rt));
  return t;
}
// Row i of the first pass: coefficient sums s[0..12) (fbe.hpp:136-143 and the
// shifted anchor quantities, fbe.hpp:172-203) and, when fused, the 8 trials
// tau = 2^-q (conj, |z|^2 at fx[2q], fx[2q+1]) plus the tau = 1 final-pass
// sums fx[16], fx[17] and the tau = 1 iterate into y_next.
__device__ __forceinline__ void cert_first_row(const DualCtx& c, int shifted, int tlambda, double lam, double gp,
                                               const double* y, const double* R, const double* Hx,
                                               const double* HR, const double* d, const double* Hd,
                                               double* y_next, int64_t i, bool ci, bool fused, double (&s)[12],
                                               double (&fx)[18]) {
  const CertRow r = cert_row(shifted, lam, y, R, Hx, HR, d, Hd, i);
  const int kd = c.g.kind[i];
  const double lo = c.g.lo[i], hi = c.g.hi[i], wg = c.g.wg[i];
  if (shifted && ci) {
    const double rr = mul_(-lam, R[i]);
    const double hr = mul_(-lam, HR[i]);
    s[4] = add_(s[4], mul_(Hx[i], rr));
    s[5] = add_(s[5], mul_(rr, hr));
    const double za = prox_row(kd, add_(r.an / lam, r.ha), lo, hi, gp * wg);
    const double ra = sub_(za, r.ha);
    s[6] = add_(s[6], conj_row(kd, sub_(r.an, mul_(lam, ra)), lo, hi, wg));
    s[7] = add_(s[7], mul_(za, za));
    s[8] = add_(s[8], mul_(r.ha, ra));
    s[9] = add_(s[9], mul_(ra, ra));
    s[10] = add_(s[10], mul_(HR[i], HR[i]));
    s[11] = add_(s[11], mul_(R[i], R[i]));
  }
  if (ci) {
    s[0] = add_(s[0], mul_(r.di, r.hd));
    s[1] = add_(s[1], mul_(r.hd, r.hd));
    s[2] = add_(s[2], mul_(r.ha, add_(r.di, mul_(lam, r.hd))));
    s[3] = add_(s[3], mul_(r.ha, r.di));
  }
  if (!fused) return;
  const double pb = add_(r.an / lam, r.ha), ps = add_(r.di / lam, r.hd);
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const CertTrial t = cert_trial(r, kd, lo, hi, wg, lam, gp, pb, ps, ldexp(1.0, -q));
    if (q == 0) {  // the final pass's quantities at tau = 1
      if (y_next) y_next[i] = tlambda ? t.Tt : sub_(y[i], mul_(lam, t.Rt));
      if (ci) {
        fx[16] = add_(fx[16], mul_(t.hxw, t.Rt));
        fx[17] = add_(fx[17], mul_(t.Rt, t.Rt));
      }
    }
    if (ci) {
      fx[2 * q] = add_(fx[2 * q], conj_row(kd, t.Tt, lo, hi, wg));
      fx[2 * q + 1] = add_(fx[2 * q + 1], mul_(t.z, t.z));
    }
  }
}
// Row i of a batch of 8 trials tq[q] (evaluate_cert, fbe.hpp:214-231)
__device__ __forceinline__ void cert_batch_row(const DualCtx& c, int shifted, double lam, double gp,
                                               const double* y, const double* R, const double* Hx,
                                               const double* HR, const double* d, const double* Hd, int64_t i,
                                               const double (&tq)[8], double (&acc)[16]) {
  const CertRow r = cert_row(shifted, lam, y, R, Hx, HR, d, Hd, i);
  const int kd = c.g.kind[i];
  const double lo = c.g.lo[i], hi = c.g.hi[i], wg = c.g.wg[i];
  const double pb = add_(r.an / lam, r.ha), ps = add_(r.di / lam, r.hd);
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const CertTrial t = cert_trial(r, kd, lo, hi, wg, lam, gp, pb, ps, tq[q]);
    acc[2 * q] = add_(acc[2 * q], conj_row(kd, t.Tt, lo, hi, wg));
    acc[2 * q + 1] = add_(acc[2 * q + 1], mul_(t.z, t.z));
  }
}
// Row i of the final pass at tau*: the next iterate (and the trial vectors
// on the test path), and the sums <Hx(w), R(w)>, |R(w)|^2
__device__ __forceinline__ void cert_final_row(const DualCtx& c, int shifted, int tlambda, double lam, double gp,
                                               const double* y, const double* R, const double* Hx,
                                               const double* HR, const double* d, const double* Hd,
                                               double* y_next, double* ow, double* oHxw, double* oz, double* oR,
                                               double* oT, int64_t i, bool ci, double tau, double (&f2)[2]) {
  const CertRow r = cert_row(shifted, lam, y, R, Hx, HR, d, Hd, i);
  const double pb = add_(r.an / lam, r.ha), ps = add_(r.di / lam, r.hd);
  const int kd = c.g.kind[i];
  const CertTrial t = cert_trial(r, kd, c.g.lo[i], c.g.hi[i], c.g.wg[i], lam, gp, pb, ps, tau);
  if (y_next) y_next[i] = tlambda ? t.Tt : sub_(y[i], mul_(lam, t.Rt));
  if (ow) {
    ow[i] = add_(r.an, mul_(tau, r.di));
    oHxw[i] = t.hxw;
    oz[i] = t.z;
    oR[i] = t.Rt;
    oT[i] = t.Tt;
  }
  if (ci) {
    f2[0] = add_(f2[0], mul_(t.hxw, t.Rt));
    f2[1] = add_(f2[1], mul_(t.Rt, t.Rt));
  }
}

// Scalar decisions, written with explicit round-to-nearest operations (no
// FMA contraction) so that both kernels, inlined anywhere, round alike; the
// operation order is C++'s left-to-right order of the reference's formulas
// (fbe.hpp:136-143, 189, 214-231; solvers.hpp:313-325).
struct CertScalars {
  double quad, alpha1, alpha2, fhat_a, conj_a, zn2_a, value_a, value, slack, lam;
};
__device__ __forceinline__ CertScalars cert_scalars(const double* S0, int shifted, const double* s) {
  CertScalars k;
  k.lam = S0[sl::LAM];
  k.value = S0[sl::VALUE];
  const double fhat = S0[sl::FHAT];
  const double hl = __dmul_rn(0.5, k.lam);
  k.quad = s[0];
  k.alpha2 = __dsub_rn(__dmul_rn(-0.5, k.quad), __dmul_rn(hl, s[1]));  // -q/2 - lam |Hd|^2 / 2
  k.alpha1 = -s[2];
  if (shifted) {
    k.fhat_a = __dsub_rn(__dsub_rn(fhat, s[4]), __dmul_rn(0.5, s[5]));
    k.conj_a = s[6];
    k.zn2_a = s[7];
    k.value_a = __dadd_rn(__dadd_rn(__dadd_rn(k.fhat_a, k.conj_a), __dmul_rn(k.lam, s[8])), __dmul_rn(hl, s[9]));
  } else {
    k.fhat_a = fhat;
    k.conj_a = S0[sl::CONJ];
    k.zn2_a = S0[sl::ZN2];
    k.value_a = k.value;
  }
  k.slack = __dmul_rn(1e-12, __dadd_rn(1.0, fabs(k.value)));
  return k;
}
__device__ __forceinline__ double cert_delta(const CertScalars& k, double tau, double conj, double z2) {
  const double quad = __dadd_rn(__dmul_rn(__dmul_rn(k.alpha2, tau), tau), __dmul_rn(k.alpha1, tau));
  return __dadd_rn(__dsub_rn(__dadd_rn(quad, conj), k.conj_a),
                   __dmul_rn(__dmul_rn(0.5, k.lam), __dsub_rn(z2, k.zn2_a)));
}
__device__ __forceinline__ double cert_fhat(const CertScalars& k, double s3, double tau) {
  return __dsub_rn(__dsub_rn(k.fhat_a, __dmul_rn(tau, s3)), __dmul_rn(__dmul_rn(__dmul_rn(0.5, tau), tau), k.quad));
}
// first accepted trial tau = 2^-(base+q), q < nq, of one batch (acc: conj,
// |z|^2 per trial); -1: none. The slack is 1e-12 (1 + |phi(y)|).
__device__ __forceinline__ int cert_pick(const CertScalars& k, int shifted, int base, int nq, const double* acc,
                                         double& tau_out, double& delta_out) {
  for (int q = 0; q < nq; ++q) {
    const double tau = ldexp(1.0, -(base + q));
    const double delta = cert_delta(k, tau, acc[2 * q], acc[2 * q + 1]);
    const bool ok = shifted ? (__dadd_rn(k.value_a, delta) <= __dadd_rn(k.value, k.slack)) : (delta <= k.slack);
    if (ok) {
      tau_out = tau;
      delta_out = delta;
      return base + q;
    }
  }
  return -1;
}
__device__ __forceinline__ void cert_finalize(const DualCtx& c, const CertScalars& k, const double* s, int kstar,
                                              double tau_star, double delta_star, double f20, double f21) {
  c.S[sl::TAU] = tau_star;
  c.S[sl::KSTAR] = kstar;
  c.S[sl::STALL] = kstar < 0 ? 1.0 : 0.0;
  c.S[sl::CERT_FHAT] = cert_fhat(k, s[3], tau_star);
  c.S[sl::HXW_RW] = f20;
  c.S[sl::RW2] = f21;
  c.S[sl::VALUE_A] = k.value_a;
  c.S[sl::CONJ_A] = k.conj_a;
  c.S[sl::ZN2_A] = k.zn2_a;
  c.S[sl::FHAT_A] = k.fhat_a;
  c.S[sl::ALPHA1] = k.alpha1;
  c.S[sl::ALPHA2] = k.alpha2;
  c.S[sl::DELTA] = delta_star;
  c.S[sl::HR2] = s[10];
  c.S[sl::RR2] = s[11];
}

// Single-launch certificate + tau search. In the solver path (no explicit
// taus) the first pass also evaluates the first batch of 8 trials and the
// final-pass sums and iterate for tau = 1, so when the full step is accepted
// (the common case) the whole search is this one pass and one reduction.
// Every sum keeps its own reduction tree: results are bitwise those of
// separate passes. Explicit taus (test / API path): deltas and f_hat of each
// trial, the last trial's vectors.
__global__ void __launch_bounds__(kThreads) cert_kernel(DualCtx c, int st, int shifted, int tlambda,
                                                        const double* y, const double* R, const double* Hx,
                                                        const double* HR, const double* d, const double* Hd,
                                                        double* y_next, int ntau_explicit, Taus taus,
                                                        double* deltas, double* cfh, double* ow, double* oHxw,
                                                        double* oz, double* oR, double* oT) {
  int ph = 0;
  const double* S0 = c.S + st * sl::kStateStride;
  const double lam = S0[sl::LAM], gp = 1.0 / lam;
  const bool fused = ntau_explicit <= 0;
  double s[12], fx[18];
#pragma unroll
  for (int q = 0; q < 12; ++q) s[q] = 0.0;
#pragma unroll
  for (int q = 0; q < 18; ++q) fx[q] = 0.0;
  for (int64_t i = gtid(); i < c.D; i += gstride())
    cert_first_row(c, shifted, tlambda, lam, gp, y, R, Hx, HR, d, Hd, fused ? y_next : nullptr, i, true, fused, s,
                   fx);
  double sv[30];
#pragma unroll
  for (int q = 0; q < 12; ++q) sv[q] = s[q];
#pragma unroll
  for (int q = 0; q < 18; ++q) sv[12 + q] = fx[q];
  if (fused) {
    grid_reduce<30>(c, ph, sv);
  } else {
    grid_reduce<12>(c, ph, s);
#pragma unroll
    for (int q = 0; q < 12; ++q) sv[q] = s[q];
  }
#pragma unroll
  for (int q = 0; q < 12; ++q) s[q] = sv[q];
  const CertScalars k = cert_scalars(S0, shifted, s);
  int kstar = -1;
  double tau_star = 0.0, delta_star = 0.0;
  const int ntau = ntau_explicit > 0 ? ntau_explicit : 61;
  for (int base = 0; base < ntau && kstar < 0; base += 8) {
    double acc[16];
#pragma unroll
    for (int q = 0; q < 16; ++q) acc[q] = 0.0;
    double tq[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int kk = base + q;
      tq[q] = ntau_explicit > 0 ? (kk < ntau ? tau_at(taus, kk) : 0.0) : ldexp(1.0, -kk);
    }
    if (fused && base == 0) {
#pragma unroll
      for (int q = 0; q < 16; ++q) acc[q] = sv[12 + q];
    } else {
      for (int64_t i = gtid(); i < c.D; i += gstride()) cert_batch_row(c, shifted, lam, gp, y, R, Hx, HR, d, Hd, i, tq, acc);
      grid_reduce<16>(c, ph, acc);
    }
    if (ntau_explicit > 0) {
      if (blockIdx.x == 0 && threadIdx.x == 0)
        for (int q = 0; q < 8 && base + q < ntau; ++q) {
          deltas[base + q] = cert_delta(k, tq[q], acc[2 * q], acc[2 * q + 1]);
          cfh[base + q] = cert_fhat(k, s[3], tq[q]);
        }
      continue;
    }
    kstar = cert_pick(k, shifted, base, ntau - base < 8 ? ntau - base : 8, acc, tau_star, delta_star);
  }
  if (ntau_explicit > 0) {  // vectors of the last tau (test path)
    kstar = ntau - 1;
    tau_star = tau_at(taus, ntau - 1);
  }
  // final pass at tau*: next iterate and the original-rule probes (tau = 1
  // came with the fused first pass)
  double f2[2] = {0, 0};
  const bool have_f2 = fused && kstar == 0;
  if (have_f2) {
    f2[0] = sv[28];
    f2[1] = sv[29];
  } else if (kstar >= 0) {
    for (int64_t i = gtid(); i < c.D; i += gstride())
      cert_final_row(c, shifted, tlambda, lam, gp, y, R, Hx, HR, d, Hd, y_next, ow, oHxw, oz, oR, oT, i, true,
                     tau_star, f2);
  }
  if (!have_f2) grid_reduce<2>(c, ph, f2);
  if (blockIdx.x == 0 && threadIdx.x == 0) cert_finalize(c, k, s, kstar, tau_star, delta_star, f2[0], f2[1]);
}

// ---------------------------------------------------------------- K4 / K6, sharded handles
// The same certificate and tau search with every reduction a cross-rank
// phase boundary (DualCtx). Phases (the launcher always issues four, with an
// allgather after each of the first three):
//   0: cert_kernel's fused first pass over this rank's rows;
//   1: decide in batch 0. tau* = 1 -> done. tau* in batch 0 -> final pass at
//      tau*, its two sums sent. No accept -> the sums of trials 8..60 sent;
//   2: no accept in batch 0: decide among 8..60, final pass at tau* (or
//      stall). Else finish the pending final pass;
//   3: finish a final pass started in phase 2.
// The state after phase k is I[CSTATE + k - 1]; phase k reads the previous
// one, so no block can observe a state written in its own launch. The
// coefficient totals persist in S[CERT_S ..] between phases.
constexpr int kCertDone = 0, kCertNeedF2 = 1, kCertNeedBatches = 2;

__global__ void __launch_bounds__(kThreads) cert_shard_kernel(DualCtx c, int st, int shifted, int tlambda,
                                                              const double* y, const double* R, const double* Hx,
                                                              const double* HR, const double* d, const double* Hd,
                                                              double* y_next) {
  int ph = 0;
  const double* S0 = c.S + st * sl::kStateStride;
  const double lam = S0[sl::LAM], gp = 1.0 / lam;
  const int stage = c.phase;
  const bool b0 = blockIdx.x == 0 && threadIdx.x == 0;
  auto final_pass = [&](double tau) {  // this rank's f2 sums go out
    double f2[2] = {0, 0};
    for (int64_t i = gtid(); i < c.D; i += gstride())
      cert_final_row(c, shifted, tlambda, lam, gp, y, R, Hx, HR, d, Hd, y_next, nullptr, nullptr, nullptr, nullptr,
                     nullptr, i, counted(c, i), tau, f2);
    xsend<2>(c, ph, f2, 0);
  };
  if (stage == 0) {
    double s[12], fx[18];
#pragma unroll
    for (int q = 0; q < 12; ++q) s[q] = 0.0;
#pragma unroll
    for (int q = 0; q < 18; ++q) fx[q] = 0.0;
    for (int64_t i = gtid(); i < c.D; i += gstride())
      cert_first_row(c, shifted, tlambda, lam, gp, y, R, Hx, HR, d, Hd, y_next, i, counted(c, i), true, s, fx);
    double sv[30];
#pragma unroll
    for (int q = 0; q < 12; ++q) sv[q] = s[q];
#pragma unroll
    for (int q = 0; q < 18; ++q) sv[12 + q] = fx[q];
    xsend<30>(c, ph, sv, 0);
    return;
  }
  if (stage == 1) {
    double sv[30];
    xrecv<30>(c, sv, 0);
    const CertScalars k = cert_scalars(S0, shifted, sv);
    double tau = 0.0, delta = 0.0;
    const int kstar = cert_pick(k, shifted, 0, 8, sv + 12, tau, delta);
    if (b0)
      for (int q = 0; q < 12; ++q) c.S[sl::CERT_S + q] = sv[q];
    if (kstar == 0) {
      if (b0) {
        cert_finalize(c, k, sv, 0, tau, delta, sv[28], sv[29]);
        c.I[il::CSTATE] = kCertDone;
      }
      return;
    }
    if (kstar > 0) {
      final_pass(tau);
      if (b0) {
        c.I[il::CSTATE] = kCertNeedF2;
        c.I[il::CKSTAR] = kstar;
        c.S[sl::TAU] = tau;
        c.S[sl::DELTA] = delta;
      }
      return;
    }
    // no accept in batch 0: this rank's sums of trials 8..60, 8 per pass
    for (int chunk = 0; chunk < 7; ++chunk) {
      double acc[16], tq[8];
#pragma unroll
      for (int q = 0; q < 16; ++q) acc[q] = 0.0;
#pragma unroll
      for (int q = 0; q < 8; ++q) tq[q] = ldexp(1.0, -(8 + chunk * 8 + q));
      for (int64_t i = gtid(); i < c.D; i += gstride())
        if (counted(c, i)) cert_batch_row(c, shifted, lam, gp, y, R, Hx, HR, d, Hd, i, tq, acc);
      xsend<16>(c, ph, acc, chunk * 16);
    }
    if (b0) c.I[il::CSTATE] = kCertNeedBatches;
    return;
  }
  // stages 2 and 3
  const int state = c.I[il::CSTATE + stage - 2];  // after the previous phase
  if (state == kCertDone) {
    if (b0) c.I[il::CSTATE + stage - 1] = kCertDone;
    return;
  }
  double s[12];
#pragma unroll
  for (int q = 0; q < 12; ++q) s[q] = c.S[sl::CERT_S + q];
  const CertScalars k = cert_scalars(S0, shifted, s);
  if (state == kCertNeedF2) {
    double f2[2];
    xrecv<2>(c, f2, 0);
    if (b0) {
      cert_finalize(c, k, s, c.I[il::CKSTAR], c.S[sl::TAU], c.S[sl::DELTA], f2[0], f2[1]);
      c.I[il::CSTATE + stage - 1] = kCertDone;
    }
    return;
  }
  // kCertNeedBatches (stage 2): trials 8..60 in order
  int kstar = -1;
  double tau = 0.0, delta = 0.0;
  for (int chunk = 0; chunk < 7 && kstar < 0; ++chunk) {
    double acc[16];
    xrecv<16>(c, acc, chunk * 16);
    kstar = cert_pick(k, shifted, 8 + chunk * 8, chunk == 6 ? 5 : 8, acc, tau, delta);
  }
  if (kstar < 0) {  // stall (solvers.hpp:315-325): no trial decreases the envelope
    if (b0) {
      cert_finalize(c, k, s, -1, 0.0, 0.0, 0.0, 0.0);
      c.I[il::CSTATE + stage - 1] = kCertDone;
    }
    return;
  }
  final_pass(tau);
  if (b0) {
    c.I[il::CSTATE + stage - 1] = kCertNeedF2;
    c.I[il::CKSTAR] = kstar;
    c.S[sl::TAU] = tau;
    c.S[sl::DELTA] = delta;
  }
}

// ---------------------------------------------------------------- K8
__global__ void __launch_bounds__(kThreads) power_kernel(DualCtx c, double* v, const double* Hv, double rel_tol) {
  // rounds are enqueued in batches: after the stopping round every later
  // launch (and its sweep, via SweepParams::skip) does nothing
  if (*reinterpret_cast<const volatile int*>(c.I + il::PDONE)) return;
  int ph = 0;
  double s[2] = {0, 0};
  if (c.phase <= 0)
    for (int i = gtid(); i < c.D; i += gstride()) {
      if (!counted(c, i)) continue;
      const double img = -Hv[i];
      s[0] += v[i] * img;
      s[1] += img * img;
    }
  if (!xreduce<2>(c, ph, s)) return;
  const double next = s[0], mag = sqrt(s[1]);
  const bool zero = !(mag > 0.0);
  const double rayleigh = c.S[sl::RAYLEIGH];
  const bool settled = fabs(next - rayleigh) <= rel_tol * fabs(next);
  if (!zero && !settled)
    for (int i = gtid(); i < c.D; i += gstride()) v[i] = -Hv[i] / mag;
  grid_sync(c.bar);  // every block has read S[RAYLEIGH]
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (!zero) c.S[sl::RAYLEIGH] = next;
    c.S[sl::PNEXT] = next;
    c.S[sl::PMAG] = mag;
    c.I[il::SETTLED] = settled ? 1 : 0;
    c.I[il::PZERO] = zero ? 1 : 0;
    c.I[il::PROUNDS] += 1;
    if (zero || settled || c.I[il::PROUNDS] >= c.I[il::PMAX]) c.I[il::PDONE] = 1;
  }
}

// ---------------------------------------------------------------- helpers
__global__ void extrapolate_kernel(int D, const double* yn, double* yp, double* w, double mom) {
  for (int i = gtid(); i < D; i += gstride()) {
    const double a = yn[i];
    w[i] = a + mom * (a - yp[i]);
    yp[i] = a;
  }
}

__global__ void prox_kernel(DualCtx c, const double* v, double gp, double* out) {
  for (int i = gtid(); i < c.D; i += gstride())
    out[i] = prox_row(c.g.kind[i], v[i], c.g.lo[i], c.g.hi[i], gp * c.g.wg[i]);
}

__global__ void __launch_bounds__(kThreads) conj_kernel(DualCtx c, const double* w) {
  int ph = 0;
  double s[1] = {0.0};
  if (c.phase <= 0)
    for (int i = gtid(); i < c.D; i += gstride())
      if (counted(c, i)) s[0] += conj_row(c.g.kind[i], w[i], c.g.lo[i], c.g.hi[i], c.g.wg[i]);
  if (!xreduce<1>(c, ph, s)) return;
  if (blockIdx.x == 0 && threadIdx.x == 0) c.S[sl::RED0] = s[0];
}

// prox.hpp:127-171
__global__ void __launch_bounds__(kThreads) dist_kernel(DualCtx c, const double* y, const double* z) {
  int ph = 0;
  double m[1] = {0.0};
  for (int i = gtid(); c.phase <= 0 && i < c.D; i += gstride()) {
    if (!counted(c, i)) continue;
    const int kd = c.g.kind[i];
    const double yi = y[i], zi = z[i];
    double dv = 0.0;
    if (kd == 0) {
      dv = fabs(yi);
    } else if (kd == 1) {
      const double lo = c.g.lo[i], hi = c.g.hi[i];
      const double cushion = 1e-12 * (1.0 + fabs(lo) + fabs(hi));
      const bool at_lo = zi <= lo + cushion, at_hi = zi >= hi - cushion;
      dv = (at_lo && at_hi) ? 0.0 : at_lo ? fmax(yi, 0.0) : at_hi ? fmax(-yi, 0.0) : fabs(yi);
    } else {
      const double t = c.g.wg[i];
      dv = zi > 0.0 ? fabs(yi - t) : (zi < 0.0 ? fabs(yi + t) : fmax(0.0, fabs(yi) - t));
    }
    m[0] = fmax(m[0], dv);
  }
  if (!xreduce<1, true>(c, ph, m)) return;
  if (blockIdx.x == 0 && threadIdx.x == 0) c.S[sl::RED0] = m[0];
}

__global__ void __launch_bounds__(kThreads) maxdiff_kernel(DualCtx c, const double* a, const double* b) {
  int ph = 0;
  double m[1] = {0.0};
  if (c.phase <= 0)
    for (int i = gtid(); i < c.D; i += gstride())
      if (counted(c, i)) m[0] = fmax(m[0], fabs(a[i] - b[i]));
  if (!xreduce<1, true>(c, ph, m)) return;
  if (blockIdx.x == 0 && threadIdx.x == 0) c.S[sl::RED0] = m[0];
}

__global__ void __launch_bounds__(kThreads) dot_kernel(DualCtx c, const double* a, const double* b) {
  int ph = 0;
  double s[1] = {0.0};
  if (c.phase <= 0)
    for (int i = gtid(); i < c.D; i += gstride())
      if (counted(c, i)) s[0] += a[i] * b[i];
  if (!xreduce<1>(c, ph, s)) return;
  if (blockIdx.x == 0 && threadIdx.x == 0) c.S[sl::RED0] = s[0];
}

__global__ void scale_kernel(int n, double alpha, const double* x, double beta, const double* y0, double* y) {
  for (int i = gtid(); i < n; i += gstride()) y[i] = alpha * x[i] + (y0 ? beta * y0[i] : 0.0);
}

// apply_H over packed rows
__global__ void apply_H_kernel(HRows h, const double* x, const double* u, double* z) {
  const int V = h.nx + h.nu;
  for (int r = gtid(); r < h.nrows; r += gstride()) {
    const double* cf = h.coef + static_cast<int64_t>(r) * V;
    const int64_t nd = h.row_node[r];
    const double* xv = x + nd * h.nx;
    double s = 0.0;
    for (int k = 0; k < h.nx; ++k) s = fma(cf[k], xv[k], s);
    if (!h.row_term[r]) {
      const double* uv = u + nd * h.nu;
      for (int k = 0; k < h.nu; ++k) s = fma(cf[h.nx + k], uv[k], s);
    }
    z[r] = s;
  }
}

// eval_f: one warp per node (problem_data.hpp:194-222)
__global__ void __launch_bounds__(kThreads) eval_f_kernel(DualCtx c, CostPack cp, const double* x,
                                                          const double* u, double tol) {
  int ph = 0;
  const int nx = cp.nx, nu = cp.nu;
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * kThreads + threadIdx.x) >> 5, nw = (gridDim.x * kThreads) >> 5;
  const int64_t csz = 2LL * nx * nx + 2LL * nx * nu + static_cast<int64_t>(nu) * nu + 2 * nx + nu;
  const int64_t lsz = static_cast<int64_t>(nx) * nx + nx;
  double s[1] = {0.0}, bad[1] = {0.0};
  const int NN = cp.nnodes, NL = cp.nleaves;
  for (int t = gw; c.phase <= 0 && t < NN + NL + 1; t += nw) {
    if (t == NN + NL) {  // root state check
      if (cp.check_root)
        for (int k = lane; k < nx; k += 32)
          if (fabs(x[k] - cp.root_state[k]) > tol) bad[0] = 1.0;
      continue;
    }
    if (t < NN) {
      const int nd = cp.nodes[t];
      const int64_t a = cp.anc[nd];
      const double* blk = cp.node + static_cast<int64_t>(cp.slot[nd]) * csz;
      const double *A = blk, *B = A + nx * nx, *cv = B + nx * nu, *Q = cv + nx, *Sm = Q + nx * nx,
                   *Rm = Sm + nu * nx, *q = Rm + nu * nu, *r = q + nx;
      const double* xa = x + a * nx;
      const double* ua = u + a * nu;
      const double* xc = x + static_cast<int64_t>(nd) * nx;
      double part = 0.0;
      for (int row = lane; row < nx; row += 32) {  // dynamics residual and x'Qx
        double ax = 0.0, qx = 0.0;
        for (int k = 0; k < nx; ++k) {
          ax = fma(A[row + k * nx], xa[k], ax);
          qx = fma(Q[row + k * nx], xa[k], qx);
        }
        for (int k = 0; k < nu; ++k) ax = fma(B[row + k * nx], ua[k], ax);
        if (fabs(xc[row] - ax - cv[row]) > tol) bad[0] = 1.0;
        part += xa[row] * qx + q[row] * xa[row];
      }
      for (int row = lane; row < nu; row += 32) {  // u'Ru + 2 u'Sx + r'u
        double ru = 0.0, sx = 0.0;
        for (int k = 0; k < nu; ++k) ru = fma(Rm[row + k * nu], ua[k], ru);
        for (int k = 0; k < nx; ++k) sx = fma(Sm[row + k * nu], xa[k], sx);
        part += ua[row] * ru + 2.0 * ua[row] * sx + r[row] * ua[row];
      }
      s[0] += cp.prob[nd] * part;  // per-lane partial; reduced below
    } else {
      const int l = t - NN;
      const int nd = cp.leaves[l];
      const double* P = cp.leaf + static_cast<int64_t>(cp.lslot[nd - cp.first_leaf]) * lsz;
      const double* p = P + nx * nx;
      const double* xc = x + static_cast<int64_t>(nd) * nx;
      double part = 0.0;
      for (int row = lane; row < nx; row += 32) {
        double px = 0.0;
        for (int k = 0; k < nx; ++k) px = fma(P[row + k * nx], xc[k], px);
        part += xc[row] * px + p[row] * xc[row];
      }
      s[0] += cp.prob[nd] * part;
    }
  }
  double v[2] = {s[0], bad[0]};  // the sum and the infeasibility flag (max), one barrier
  if (!xreduce<2, false, 1>(c, ph, v)) return;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    c.S[sl::EVALF] = v[0];
    c.S[sl::EVALF_INF] = v[1];
  }
}

cudaError_t coop(const void* fn, const DualCtx& c, void** args, cudaStream_t st) {
  return cudaLaunchCooperativeKernel(fn, dim3(c.nblk), dim3(kThreads), args, 0, st);
}

// Launch of a kernel whose args[0] is &cc. Unsharded: one launch. Sharded:
// `phases` launches (cc.phase = 0, 1, ...) with an allgather of the ranks'
// totals after each but the last.
cudaError_t phased(const void* fn, DualCtx& cc, void** args, cudaStream_t st, int phases = 2) {
  if (!cc.xc) {
    cc.phase = -1;
    return coop(fn, cc, args, st);
  }
  for (int p = 0; p < phases; ++p) {
    cc.phase = p;
    const cudaError_t e = coop(fn, cc, args, st);
    if (e != cudaSuccess) return e;
    if (p + 1 < phases) dual_allgather(cc.xc, cc.xs, cc.xr, kXMax, st);
  }
  return cudaSuccess;
}

}  // namespace

int dual_block_threads() { return kThreads; }
int dual_max_blocks() { return kMaxBlocks; }

cudaError_t k_fb_finish(const DualCtx& c, int state, int mode, const double* y, const double* Hx,
                        const double* Hx0, const double* weight, double* z, double* R, double* T,
                        cudaStream_t st) {
  DualCtx cc = c;
  void* args[] = {&cc, &state, &mode, &y, &Hx, &Hx0, &weight, &z, &R, &T};
  return phased(reinterpret_cast<const void*>(fb_finish_kernel), cc, args, st);
}

// Scalar block -> mapped pinned host memory in one launch, as flagged words
// (dual.hpp kPubWords): the host spins on the words themselves.
__global__ void publish_kernel(const double* S, const int* I, unsigned long long* pub, unsigned seq) {
  fbrow::publish_block(S, I, pub, seq);
}

namespace {
__global__ void exchange_pack_kernel(ExchangeDims e, double* xbuf) {
  const int64_t per = e.xbuf_rhs, total = e.nrhs * per;
  for (int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(idx / per);
    const int64_t i = idx - r * per;
    double v = 0.0;
    if (i < e.ns_w) {
      if (i >= e.own_c_lo && i < e.own_c_hi) v = e.contrib[r][e.contrib_off + i];
    } else if (i < e.ns_w + e.nys) {
      const int64_t row = e.dual_top + (i - e.ns_w);
      if (row >= e.own_y_lo && row < e.own_y_hi) v = e.y[r][row];
    }
    xbuf[idx] = v;
  }
}
__global__ void exchange_unpack_kernel(ExchangeDims e, const double* xbuf) {
  const int64_t per = e.ns_w + e.dual_top + e.nys, total = e.nrhs * per;
  for (int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(idx / per);
    const int64_t i = idx - r * per;
    const double* xb = xbuf + r * e.xbuf_rhs;
    if (i < e.ns_w)
      e.contrib[r][e.contrib_off + i] = xb[i];
    else if (i < e.ns_w + e.dual_top)
      e.ycomp[r][i - e.ns_w] = e.y[r][i - e.ns_w];
    else
      e.ycomp[r][i - e.ns_w] = xb[e.ns_w + (i - e.ns_w - e.dual_top)];
  }
}
int exchange_blocks(int64_t n) { return static_cast<int>(std::min<int64_t>((n + 255) / 256, 1184)); }
}  // namespace

cudaError_t k_exchange_pack(const ExchangeDims& e, double* xbuf, cudaStream_t st) {
  const int64_t n = e.nrhs * e.xbuf_rhs;
  if (n > 0) exchange_pack_kernel<<<exchange_blocks(n), 256, 0, st>>>(e, xbuf);
  return cudaGetLastError();
}
cudaError_t k_exchange_unpack(const ExchangeDims& e, const double* xbuf, cudaStream_t st) {
  const int64_t n = e.nrhs * (e.ns_w + e.dual_top + e.nys);
  if (n > 0) exchange_unpack_kernel<<<exchange_blocks(n), 256, 0, st>>>(e, xbuf);
  return cudaGetLastError();
}

cudaError_t k_publish(const double* S, const int* I, unsigned long long* pub_mapped, unsigned seq, cudaStream_t st) {
  publish_kernel<<<1, 256, 0, st>>>(S, I, pub_mapped, seq);
  return cudaGetLastError();
}

cudaError_t k_fbe_grad(const DualCtx& c, int state, const double* R, const double* HR, double* grad,
                       cudaStream_t st) {
  DualCtx cc = c;
  void* args[] = {&cc, &state, &R, &HR, &grad};
  return phased(reinterpret_cast<const void*>(fbe_grad_kernel), cc, args, st);
}

cudaError_t k_lbfgs(const DualCtx& c, int mem, double eps_curv, double scale_ref, int do_push, const double* a,
                    const double* b, const double* cc, const double* dd, const double* gvec,
                    double* out, double* Sbuf, double* Qbuf, cudaStream_t st, double* Mbuf, const double* fR,
                    const double* fHR, int fstate, double* gout) {
  DualCtx c2 = c;
  if (Mbuf && mem <= kCompactMem) {
    void* args[] = {&c2,  &mem,  &eps_curv, &scale_ref, &do_push, &a,  &b,   &cc,     &dd,  &gvec,
                    &out, &Sbuf, &Qbuf,     &Mbuf,      &fR,      &fHR, &fstate, &gout};
    return phased(reinterpret_cast<const void*>(lbfgs_compact_kernel), c2, args, st);
  }
  if (c2.xc) return cudaErrorNotSupported;  // sharded handles: compact form only (memory <= 6)
  void* args[] = {&c2, &mem, &eps_curv, &scale_ref, &do_push, &a, &b, &cc, &dd, &gvec, &out, &Sbuf, &Qbuf};
  return coop(reinterpret_cast<const void*>(lbfgs_kernel), c, args, st);
}

cudaError_t k_cert_search(const DualCtx& c, int state, int shifted, int tlambda, const double* y,
                          const double* R, const double* Hx, const double* HR, const double* d,
                          const double* Hd, double* y_next, cudaStream_t st) {
  DualCtx cc = c;
  if (cc.xc) {  // sharded: four phases (cert_shard_kernel)
    void* args[] = {&cc, &state, &shifted, &tlambda, &y, &R, &Hx, &HR, &d, &Hd, &y_next};
    return phased(reinterpret_cast<const void*>(cert_shard_kernel), cc, args, st, 4);
  }
  int ntau = 0;
  Taus taus{};
  double* nul = nullptr;
  void* args[] = {&cc, &state, &shifted, &tlambda, &y, &R, &Hx, &HR, &d, &Hd, &y_next, &ntau, &taus,
                  &nul, &nul, &nul, &nul, &nul, &nul, &nul};
  return coop(reinterpret_cast<const void*>(cert_kernel), c, args, st);
}

cudaError_t k_cert_eval(const DualCtx& c, int state, int shifted, const double* y, const double* R,
                        const double* Hx, const double* HR, const double* d, const double* Hd,
                        int ntau, const double* taus_host, double* deltas, double* cfh, double* w,
                        double* Hxw, double* zz, double* RR, double* TT, cudaStream_t st) {
  if (ntau < 1 || ntau > 16) return cudaErrorInvalidValue;
  if (c.xc) return cudaErrorNotSupported;  // explicit trials: unsharded handles
  DualCtx cc = c;
  Taus taus{};
  for (int k = 0; k < ntau; ++k) taus.t[k] = taus_host[k];
  int tl = 1;
  double* yn = nullptr;
  void* args[] = {&cc, &state, &shifted, &tl, &y, &R, &Hx, &HR, &d, &Hd, &yn, &ntau, &taus,
                  &deltas, &cfh, &w, &Hxw, &zz, &RR, &TT};
  return coop(reinterpret_cast<const void*>(cert_kernel), c, args, st);
}

cudaError_t k_power(const DualCtx& c, double* v, const double* Hv, double rel_tol, cudaStream_t st) {
  DualCtx cc = c;
  void* args[] = {&cc, &v, &Hv, &rel_tol};
  return phased(reinterpret_cast<const void*>(power_kernel), cc, args, st);
}

cudaError_t k_extrapolate(const DualCtx& c, const double* yn, double* yp, double* w, double mom,
                          cudaStream_t st) {
  extrapolate_kernel<<<c.nblk, kThreads, 0, st>>>(c.D, yn, yp, w, mom);
  return cudaGetLastError();
}

cudaError_t k_prox(const DualCtx& c, const double* v, double gamma_prox, double* out, cudaStream_t st) {
  prox_kernel<<<c.nblk, kThreads, 0, st>>>(c, v, gamma_prox, out);
  return cudaGetLastError();
}

cudaError_t k_conj(const DualCtx& c, const double* w, cudaStream_t st) {
  DualCtx cc = c;
  void* args[] = {&cc, &w};
  return phased(reinterpret_cast<const void*>(conj_kernel), cc, args, st);
}

cudaError_t k_dist_subdiff(const DualCtx& c, const double* y, const double* z, cudaStream_t st) {
  DualCtx cc = c;
  void* args[] = {&cc, &y, &z};
  return phased(reinterpret_cast<const void*>(dist_kernel), cc, args, st);
}

cudaError_t k_max_abs_diff(const DualCtx& c, const double* a, const double* b, cudaStream_t st) {
  DualCtx cc = c;
  void* args[] = {&cc, &a, &b};
  return phased(reinterpret_cast<const void*>(maxdiff_kernel), cc, args, st);
}

cudaError_t k_dot(const DualCtx& c, const double* a, const double* b, cudaStream_t st) {
  DualCtx cc = c;
  void* args[] = {&cc, &a, &b};
  return phased(reinterpret_cast<const void*>(dot_kernel), cc, args, st);
}

cudaError_t k_scale(const DualCtx& c, int n, double alpha, const double* x, double beta, const double* y0,
                    double* y, cudaStream_t st) {
  scale_kernel<<<c.nblk, kThreads, 0, st>>>(n, alpha, x, beta, y0, y);
  return cudaGetLastError();
}

cudaError_t k_apply_H(const HRows& h, const double* x, const double* u, double* z, cudaStream_t st) {
  const int blocks = (h.nrows + kThreads - 1) / kThreads;
  apply_H_kernel<<<blocks > 0 ? blocks : 1, kThreads, 0, st>>>(h, x, u, z);
  return cudaGetLastError();
}

cudaError_t k_eval_f(const DualCtx& c, const CostPack& cp, const double* x, const double* u,
                     double feas_tol, cudaStream_t st) {
  DualCtx cc = c;
  CostPack p = cp;
  void* args[] = {&cc, &p, &x, &u, &feas_tol};
  return phased(reinterpret_cast<const void*>(eval_f_kernel), cc, args, st);
}

}  // namespace scn
