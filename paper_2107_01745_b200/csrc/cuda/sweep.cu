// SPDX-License-Identifier: MIT
//
// K1+K2: the dual-gradient / Hessian-vector sweep (tree_oracles.hpp:33-90)
// fused with apply_H (problem_data.hpp:144-162) as ONE persistent,
// warp-specialised kernel.
//
// Schedule (built by device.cpp). Items are runs of same-stage nodes
// (layout.hpp). Below a cut stage each CTA owns a contiguous group of whole
// subtrees, so those items depend only on earlier items of the same CTA:
// the producer waits on a shared-memory retire counter (CTA-scope
// release/acquire, no gpu-scope traffic). The nodes above the cut are global
// tickets dealt round-robin; their completion (and that of the subtree
// roots they consume) is published through epoch-stamped per-node flags
// (gpu-scope fence + flag store / ld.acquire). Every CTA processes its list
// in rank order (backward leaves -> root, then forward root -> leaves) and
// every dependency has a smaller rank, so the lowest-ranked unfinished item
// can always proceed: no deadlock, no grid-wide barrier. The grid is
// co-resident (cooperative launch).
//
// Every per-item step is latency-bound (measured on B200: L2 hit ~280
// cycles, st.release ~760, dependent DFMA 8), so the kernel overlaps items
// in every role instead of shortening one item:
//   producers   warps 0..P-1 (P = 4; 6 in the geom_p6 build), items
//               k = p mod P: poll the item's dependency flags (ld.acquire)
//               and stage its small vectors (y rows, child contributions,
//               parent x/u, u_off, affine terms) with async 8-byte copies;
//               P such round trips are in flight at once.
//   teams       the next 12 warps: four consumer teams of three warps (team t
//               takes items k = t mod 4): wait for the item's matrices (slot
//               FULL) and vectors (stage FULL), compute every product from
//               shared memory, release the slot and the staging area.
//   publisher   the next warp: retires items in order (CTA-scope counter) and
//               releases the flags of publishing items, one gpu-scope fence
//               per batch of finished items.
//   issuer      the last warp: streams the CTA's items through the matrix
//               slots, one cp.async.bulk (TMA 1-D) per item once its slot is
//               released.
// Products are "dot columns" split over S in {1,2,4} threads (interleaved
// 16-byte shared loads over padded columns + xor shuffles), for all
// right-hand sides at once so a 2-RHS (p-NAMA) sweep reads each matrix once.
// fp64 throughout; the partial-sum order is fixed, so results are
// deterministic and identical between 1- and 2-RHS launches.
#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>

#include "fbrow.cuh"
#include "layout.hpp"

// One build per kernel geometry (cuda/layout.hpp SweepImpl): the default,
// and the six-producer one built with -DSCN_SWEEP_NS=geom_p6 ... (Makefile).
#ifndef SCN_SWEEP_NS
#define SCN_SWEEP_NS geom_p4
#define SCN_SWEEP_IMPL kSweepProducers4
#endif

namespace scn {
namespace SCN_SWEEP_NS {

namespace {

// Four consumer teams of three warps (the 576 threads and 96 registers of
// three 128-thread teams): one more item in flight per SM. Measured against
// 3 x 128 (profiles/ab_teams_r02.txt): C3 affine 219.9 -> 218 us, C3 2-RHS
// 238.9 -> 229 us, nx = 10 (873,813 nodes) 963 -> 939 us; 5 x 96 spills
// (C3 242 us); 4 x 128 (704 threads) caps registers at 80 and spills.
#ifndef SCN_TEAM_THREADS
#define SCN_TEAM_THREADS 96
#endif
constexpr int kTeam = SCN_TEAM_THREADS;  // threads per consumer team
#ifndef SCN_TEAMS
#define SCN_TEAMS 4
#endif
constexpr int kTeams = SCN_TEAMS;  // consumer teams (items k = team mod kTeams)
#ifndef SCN_PRODUCERS
#define SCN_PRODUCERS 4
#endif
constexpr int kProducers = SCN_PRODUCERS;  // producer warps, warp p stages items k = p (mod kProducers)
constexpr int kThreads = 32 * kProducers + kTeams * kTeam + 64;  // producers, teams, publisher, issuer
constexpr int kTeamWarp0 = kProducers;
#ifndef SCN_STAGE_Q
#define SCN_STAGE_Q ((kTeams == 3 || kTeams == 6) ? 12 : (kTeams == 5 ? 20 : 8))
#endif
constexpr int kStageQ = SCN_STAGE_Q;  // staging ring depth (items staged ahead); a multiple of kProducers
                            // and even, so each staging area always serves the same producer
                            // warp and the same team in order
static_assert(kStageQ % kProducers == 0 && kStageQ % kTeams == 0, "staging ring vs producers / teams");
constexpr int kDoneQ = 8 * kTeams;  // completion ring depth (publisher lag allowed); a multiple of kTeams
constexpr int kPublisherWarp = kProducers + kTeams * kTeam / 32;
constexpr int kIssuerWarp = kPublisherWarp + 1;
#ifndef SCN_L2_PREFETCH
#define SCN_L2_PREFETCH 8
#endif
// Items the issuer prefetches into L2 ahead of the shared-memory slots, only
// when the slot it waits for holds an item with cross-CTA dependencies (the
// serial top of the tree, where a slot stays busy for microseconds and HBM
// idles): the next items then stream into L2, so the forward pass starts
// from L2. In the steady state (CTA-local items) prefetching would compete
// with the slots' own bulk copies (measured 222 -> 233 us at C3 with 4 items).
// Gated, measured at C3: 0 -> 223.2, 8 -> 220.0, 32 -> 229.0, 64 -> 259 us
// per affine sweep (the bulk prefetches delay the slots' loads when deep).
constexpr int kL2Ahead = SCN_L2_PREFETCH;
#ifndef SCN_WARP_RELEASE
#define SCN_WARP_RELEASE 0  /* per-warp release measured 1-2% slower than one team barrier */
#endif
constexpr bool kWarpRelease = SCN_WARP_RELEASE != 0;
constexpr int kReleaseArrivals = kWarpRelease ? kTeam / 32 : 1;  // mempty / sempty / done arrivals per item
constexpr int kScratchBufs = kWarpRelease ? 2 : 1;             // w / x scratch buffers per team

#ifdef SCN_SWEEP_PROFILE
// cycle counters: [0] prod stage-empty wait [1] prod stage round trip
// [2] prod dep spin [3] team slot-full wait [4] team stage-full wait
// [5] team compute [6] team refill + publish back-pressure [7] publisher fence
__device__ unsigned long long g_prof[16];
__device__ int g_dbg;  // timing experiments only: bit0 ignore dependencies, bit1 skip compute
__device__ unsigned long long* g_timeline;  // per item: globaltimer at retirement (null: off)
__device__ long long* g_trace;              // per item: 8 clock64 stamps of the consumer team (null: off)
// light per-team counters: cycles accumulated in registers by each team's
// thread 0, flushed once per CTA (g_prof[8..15]); SCN_DBG bit 3 enables
#define LC_DECL() long long _lc[8] = {0, 0, 0, 0, 0, 0, 0, 0}; long long _lt = clock64(); const bool _lon = (g_dbg & 8) && ttid == 0
#define LC_MARK(slot) do { if (_lon) { const long long _n = clock64(); _lc[slot] += _n - _lt; _lt = _n; } } while (0)
#define LC_FLUSH() do { if (_lon) for (int _i = 0; _i < 8; ++_i) atomicAdd(&g_prof[8 + _i], (unsigned long long)_lc[_i]); } while (0)
#define TRACE_IN(i) \
  do { if (g_trace && ttid == 0 && trace_row) trace_row[i] = static_cast<long long>(gtimer()); } while (0)
#define TRACE(i) \
  do { if (g_trace && ttid == 0) g_trace[12LL * (P.cta_off[blockIdx.x] + P.items_base + k) + (i)] = static_cast<long long>(gtimer()); } while (0)
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define DBG(bit) (g_dbg & (bit))
#define PROF_T0() long long _pt = clock64()
#define PROF_T1(slot)                                                                          \
  do {                                                                                         \
    if (g_dbg & 4) {  /* SCN_DBG bit 2: per-role cycle counters (heavy: global atomics) */     \
      long long _n = clock64();                                                                \
      atomicAdd(&g_prof[slot], (unsigned long long)(_n - _pt));                                \
      _pt = _n;                                                                                \
    }                                                                                          \
  } while (0)
#else
#define DBG(bit) 0
#define LC_DECL()
#define LC_MARK(slot)
#define LC_FLUSH()
#define TRACE(i) (void)0
#define TRACE_IN(i) (void)0
#define PROF_T0() (void)0
#define PROF_T1(slot) (void)0
#endif

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
__device__ __forceinline__ int ld_acquire_cta(const int* p) {
  int v;
  asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_cta(int* p, int v) {
  asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
#ifndef SCN_MBAR_HINT_NS
#define SCN_MBAR_HINT_NS 0  /* measured: no explicit hint is ~1% faster than 32 or 256 ns */
#endif
// try_wait with an explicit suspend-time hint: a waiting warp re-checks within
// ~tens of ns instead of the implementation's default suspend interval (the
// item pipeline is latency-bound; every wake-up is on some item's path).
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
#if SCN_MBAR_HINT_NS > 0
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity), "n"(SCN_MBAR_HINT_NS)
      : "memory");
#else
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
#endif
}
__device__ __forceinline__ bool mbar_test(uint64_t* bar, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
      "selp.u32 %0, 1, 0, P1;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// L2 prefetch of a global range (cp.async.bulk.prefetch; no completion to wait for)
__device__ __forceinline__ void prefetch_l2(const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void team_sync(int team) {
  asm volatile("bar.sync %0, %1;" ::"r"(1 + team), "r"(kTeam) : "memory");
}
__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
}

__device__ __forceinline__ const unsigned* dep_flags(const SweepParams& P, const Item& it) {
  return (it.pass == 0 || it.first == 0 || (it.direct & kFlatTop)) ? P.bw_flag : P.fw_flag;
}
// padded dot length of a flattened top node of depth k (== 2 mod 4, as pad2 on the host)
__device__ __forceinline__ int flat_len(int k, int nu) {
  const int l = k * nu;
  return l + ((2 - l % 4) + 4) % 4;
}

__device__ __forceinline__ bool flags_ready(const unsigned* flags, const Item& it, unsigned E, int lane) {
  bool ok = true;
  for (int k = it.dep_lo + lane; k < it.dep_hi; k += 32) ok &= (ld_acquire(flags + k) == E);
  return __all_sync(0xffffffffu, ok);
}

// Staged-vector layout of one item for NRHS right-hand sides:
//   bw: Y_r at r*v0n ; C_r at NRHS*v0n + r*v1n*W ; AFF at NRHS*(v0n+v1n*W)  (count*W)
//   fw: PV_r[p] = [x_a; u_a; 0-pad] at (r*v0n + p)*Vp ; UO_r at NRHS*v0n*Vp + r*v1n*nu ;
//       AFF at NRHS*(v0n*Vp + v1n*nu)  (count*nx)
// Issued as asynchronous 8-byte copies (LDGSTS) program-ordered after the
// acquire that observed this item's flags (ld.acquire.gpu also invalidates
// L1), so they read the published values. PART: 3 stages everything; the
// host-output kernels split a backward item into 1 (the y rows and affine
// terms, which no item produces, issued before the dependency wait so their
// PCIe reads from the caller's pinned y overlap it) and 2 (the children's
// contributions; a forward item stages everything as 2).
template <int NRHS, int nt = 32, int PART = 3>
__device__ void stage_issue(const SweepParams& P, const Item& it, double* st, int lane) {
  const int nx = P.nx, nu = P.nu, W = nx + nu, Vp = P.Vp;
  if (it.pass == 0) {
    const int nc = it.v1_n * W;
#pragma unroll
    for (int r = 0; r < NRHS; ++r) {
      const double* ys = P.y[r] + it.v0_lo;
      double* yd = st + r * it.v0_n;
      if (PART & 1)
        for (int i = lane; i < it.v0_n; i += nt) cp_async8(yd + i, ys + i);
      if ((PART & 2) && !(it.direct & kDirectContrib)) {
        const double* cs = P.contrib[r] + static_cast<int64_t>(it.v1_lo) * W;
        double* cd = st + NRHS * it.v0_n + r * nc;
        for (int i = lane; i < nc; i += nt) cp_async8(cd + i, cs + i);
      }
    }
    if ((PART & 1) && P.affine) {
      const int na = it.count * W;
      const double* as = P.aff_bw + static_cast<int64_t>(it.first) * W;
      double* ad = st + NRHS * (it.v0_n + ((it.direct & kDirectContrib) ? 0 : nc));
      for (int i = lane; i < na; i += nt) cp_async8(ad + i, as + i);
    }
  } else if (!(PART & 2)) {
    return;
  } else if (it.direct & kFlatTop) {
    // flattened top: PV_r = [u_off(root); u_off(a_1); u_off(a_2); 0-pad] shared by the
    // item's siblings, then UO_r (own u_off), AFX (a'), AFH (stage-row constants)
    const int k = it.direct >> 8, Lp = flat_len(k, nu), nuo = it.v1_n * nu;
#pragma unroll
    for (int r = 0; r < NRHS; ++r) {
      double* pd = st + r * Lp;
      for (int e = lane; e < Lp; e += nt) {
        const int i = e / nu, j = e - i * nu;
        if (i < k) {
          const int a = i == 0 ? 0 : (i == 1 ? it.v0_lo : it.v0_n);
          cp_async8(pd + e, P.uoff[r] + static_cast<int64_t>(a) * nu + j);
        } else {
          pd[e] = 0.0;
        }
      }
      const double* os = P.uoff[r] + static_cast<int64_t>(it.v1_lo) * nu;
      double* od = st + NRHS * Lp + r * nuo;
      for (int i = lane; i < nuo; i += nt) cp_async8(od + i, os + i);
    }
    if (P.affine) {
      double* ad = st + NRHS * (Lp + nuo);
      const int na = it.count * nx;
      const double* as = P.aff_fw + static_cast<int64_t>(it.first) * nx;
      for (int i = lane; i < na; i += nt) cp_async8(ad + i, as + i);
      const int nh = it.count * P.mmax;
      const double* hs = P.aff_fwh + static_cast<int64_t>(it.first) * P.mmax;
      for (int i = lane; i < nh; i += nt) cp_async8(ad + na + i, hs + i);
    }
  } else {
    const int tot = it.v0_n * Vp, nuo = it.v1_n * nu;
#pragma unroll
    for (int r = 0; r < NRHS; ++r) {
      for (int pp = 0; pp < it.v0_n; ++pp) {
        double* pd = st + r * tot + pp * Vp;
        const double* xs = P.x[r] + static_cast<int64_t>(it.v0_lo + pp) * nx;
        const double* us = P.u[r] + static_cast<int64_t>(it.v0_lo + pp) * nu;
        for (int e = lane; e < Vp; e += nt) {
          if (e < nx)
            cp_async8(pd + e, xs + e);
          else if (e < W)
            cp_async8(pd + e, us + (e - nx));
          else
            pd[e] = 0.0;
        }
      }
      const double* os = P.uoff[r] + static_cast<int64_t>(it.v1_lo) * nu;
      double* od = st + NRHS * tot + r * nuo;
      for (int i = lane; i < nuo; i += nt) cp_async8(od + i, os + i);
    }
    if (P.affine) {
      const int na = it.count * nx;
      const double* as = P.aff_fw + static_cast<int64_t>(it.first) * nx;
      double* ad = st + NRHS * (tot + nuo);
      for (int i = lane; i < na; i += nt) cp_async8(ad + i, as + i);
    }
  }
}

// out[r] = <col, vec_r> over a padded length (even; 16-byte aligned operands)
// by S consecutive threads (q = 0..S-1) taking interleaved 16-byte chunks,
// two accumulators each, then an xor-shuffle reduction. All threads of a
// warp call it (inactive ones with lenp = 0).
#ifndef SCN_DOT_UNROLL
#define SCN_DOT_UNROLL 4
#endif
// Dot tasks are split over at most SCN_TASK_S_MAX threads: the 8-way split's
// extra instantiations cost instruction-cache room, measured at C3 2-RHS
// 255.7 -> 237.7 us with the cap at 4 (1-RHS unchanged; nx = 10: 978 -> 964 us;
// a cap of 2: 242 us). A smaller dot unroll shrinks code further but slows
// the loops (unroll 2: 1-RHS 225 us).
#ifndef SCN_TASK_S_MAX
#define SCN_TASK_S_MAX 4
#endif
constexpr int kDotUnroll = SCN_DOT_UNROLL;
template <int NRHS, int S>
__device__ __forceinline__ void dot_split(const double* __restrict__ col, const double* __restrict__ v0,
                                          int vstride, int lenp, int q, double (&out)[NRHS]) {
  double a[NRHS], bq[NRHS];
#pragma unroll
  for (int r = 0; r < NRHS; ++r) a[r] = bq[r] = 0.0;
#pragma unroll kDotUnroll
  for (int k = 2 * q; k < lenp; k += 2 * S) {
    const double2 m = *reinterpret_cast<const double2*>(col + k);
#pragma unroll
    for (int r = 0; r < NRHS; ++r) {
      const double2 v = *reinterpret_cast<const double2*>(v0 + r * vstride + k);
      a[r] = fma(m.x, v.x, a[r]);
      bq[r] = fma(m.y, v.y, bq[r]);
    }
  }
#pragma unroll
  for (int r = 0; r < NRHS; ++r) {
    double t = a[r] + bq[r];
#pragma unroll
    for (int o = S >> 1; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    out[r] = t;
  }
}

// Runs body.run<S>(task, q, active) over ntasks dot tasks on one team, S
// threads per task, S chosen so one round covers the tasks when possible.
template <class Body>
__device__ __forceinline__ void for_tasks(int ntasks, int ttid, const Body& body) {
  if (SCN_TASK_S_MAX >= 8 && ntasks * 8 <= kTeam) {
    const int g = ttid >> 3, q = ttid & 7;
    body.template run<(SCN_TASK_S_MAX >= 8 ? 8 : 4)>(g, q, g < ntasks);
  } else if (SCN_TASK_S_MAX >= 4 && ntasks * 4 <= kTeam) {
    const int g = ttid >> 2, q = ttid & 3;
    body.template run<(SCN_TASK_S_MAX >= 4 ? 4 : 2)>(g, q, g < ntasks);
  } else if (ntasks * 2 <= kTeam) {
    const int g = ttid >> 1, q = ttid & 1;
    body.template run<2>(g, q, g < ntasks);
  } else {
    for (int base = 0; base < ntasks; base += kTeam) body.template run<1>(base + ttid, 0, base + ttid < ntasks);
  }
}

// ---------------------------------------------------------------- backward
// tree_oracles.hpp:54-73, phase B: contrib_c = J_c' w_c
//   = [child_to_input_c w_c ; closed_loop_c' w_c] (non-root c).
template <int NRHS>
struct BwPhaseB {
  const SweepParams& P;
  const NodeMeta* meta;
  const double* slot;
  const double* wbuf;
  int nx, W, nxp, leaf, single;
  template <int S>
  __device__ __forceinline__ void run(int task, int q, bool active) const {
    int ni = 0, j = 0;
    const double* col = slot;
    if (active) {
      ni = single ? 0 : task / W;
      j = task - ni * W;
      const NodeMeta& mc = meta[ni];
      const int e = leaf ? mc.mN * nx : mc.M * W;
      col = slot + mc.blk + ((e + 1) & ~1) + j * nxp;
    }
    double acc[NRHS];
    dot_split<NRHS, S>(col, wbuf + ni * NRHS * nxp, nxp, active ? nxp : 0, q, acc);
    if (active && q == 0) {
      const int64_t c = meta[ni].c;
#pragma unroll
      for (int r = 0; r < NRHS; ++r) P.contrib[r][c * W + j] = acc[r];
    }
  }
};

// tree_oracles.hpp:44-73. Interior c: [u_off_c; w_c] = E_c' y_kids +
// sum_kids contrib_k (+[sigma_c; c_hat_c]); leaf: w_c = F_N' y_N (+pi p_N);
// then phase B for non-root c.
template <int NRHS>
__device__ void consume_backward(const SweepParams& P, const Item& it, const double* slot, const double* mat,
                                 const double* st, double* wbuf, int ttid, int team, long long* trace_row) {
  const int nx = P.nx, nu = P.nu, W = nx + nu, nxp = P.nxp;
  const int cnt = it.count;
  const bool leaf = it.leaf != 0;
  const NodeMeta* meta = reinterpret_cast<const NodeMeta*>(slot);
  const double* Y = st;
  const double* Cn = st + NRHS * it.v0_n;
  const double* AF = st + NRHS * (it.v0_n + ((it.direct & kDirectContrib) ? 0 : it.v1_n * W));
  PROF_T0();
  {  // phase A: short dot columns (len M or mN), child sums, affine terms
    const int ncols = leaf ? nx : W;
    const int ntasks = cnt * ncols;
    for (int task = ttid; task < ntasks; task += kTeam) {
      const int ni = cnt == 1 ? 0 : task / ncols;
      const int j = task - ni * ncols;
      const NodeMeta& mc = meta[ni];
      const int len = leaf ? mc.mN : mc.M;
      const double* col = mat + mc.blk + j * len;
      const double* yv = Y + mc.yoff;
      double acc[NRHS];
#pragma unroll
      for (int r = 0; r < NRHS; ++r) acc[r] = 0.0;
      for (int k = 0; k < len; ++k) {
        const double a = col[k];
#pragma unroll
        for (int r = 0; r < NRHS; ++r) acc[r] = fma(a, yv[r * it.v0_n + k], acc[r]);
      }
      if (!leaf) {
        if (it.direct & kDirectContrib) {  // many children: read the published contributions from L2,
                          // eight loads in flight, summed in child order (as when staged)
          const int64_t base = static_cast<int64_t>(it.v1_lo + mc.kid0) * W + j;
          for (int k0 = 0; k0 < mc.nkid; k0 += 8) {
            double v[NRHS][8];
#pragma unroll
            for (int u = 0; u < 8; ++u)
#pragma unroll
              for (int r = 0; r < NRHS; ++r)
                v[r][u] = k0 + u < mc.nkid ? __ldcg(P.contrib[r] + base + static_cast<int64_t>(k0 + u) * W) : 0.0;
#pragma unroll
            for (int u = 0; u < 8; ++u)
#pragma unroll
              for (int r = 0; r < NRHS; ++r)
                if (k0 + u < mc.nkid) acc[r] += v[r][u];
          }
        } else {
          for (int k = 0; k < mc.nkid; ++k) {
#pragma unroll
            for (int r = 0; r < NRHS; ++r) acc[r] += Cn[r * it.v1_n * W + (mc.kid0 + k) * W + j];
          }
        }
      }
      const int ja = leaf ? nu + j : j;
      const double aff = P.affine ? AF[ni * W + ja] : 0.0;
#pragma unroll
      for (int r = 0; r < NRHS; ++r) {
        const double v = acc[r] + aff;
        if (ja < nu)
          P.uoff[r][static_cast<int64_t>(mc.c) * nu + ja] = v;  // u_off, completed by the forward pass
        else
          wbuf[(ni * NRHS + r) * nxp + (ja - nu)] = v;  // costate w_c
      }
    }
  }
  if (ttid == 0) PROF_T1(8);
  TRACE_IN(3);
  team_sync(team);
  if (ttid == 0) PROF_T1(9);
  TRACE_IN(4);
  if (it.first != 0) {
    const BwPhaseB<NRHS> body{P, meta, mat, wbuf, nx, W, nxp, leaf ? 1 : 0, cnt == 1 ? 1 : 0};
    for_tasks(cnt * W, ttid, body);
  }
  if (ttid == 0) PROF_T1(10);
}

// ---------------------------------------------------------------- forward
// tree_oracles.hpp:75-88 + apply_H, phase A: [x_c; z_c] = W_c' [x_a; u_a]
// (+[c_c; 0]) for non-root c.
template <int NRHS, bool HOST = false>
struct FwPhaseA {
  const SweepParams& P;
  const NodeMeta* meta;
  const double* slot;
  const double* PV;
  const double* AF;
  double* xbuf;
  int nx, Vp, nxp, ncols, tot, single;
  int flat;             // flattened top: one shared vector PV (ancestors' u_off), column stride Vp = Lp
  const double* AFH;    // flattened top: stage-row constants [count][mmaxh]
  int mmaxh;
  template <int S>
  __device__ __forceinline__ void run(int task, int q, bool active) const {
    int ni = 0, j = 0;
    const double* col = slot;
    const double* v = PV;
    if (active) {
      ni = single ? 0 : task / ncols;
      j = task - ni * ncols;
      const NodeMeta& mc = meta[ni];
      active = j < nx + mc.m;
      col = slot + mc.blk + j * Vp;
      v = flat ? PV : PV + mc.par * Vp;
    }
    double acc[NRHS];
    dot_split<NRHS, S>(col, v, tot, active ? Vp : 0, q, acc);
    if (active && q == 0) {
      const NodeMeta& mc = meta[ni];
      const int64_t c = mc.c;
      if (j < nx) {
        const double aff = P.affine ? AF[ni * nx + j] : 0.0;
#pragma unroll
        for (int r = 0; r < NRHS; ++r) {
          const double xv = acc[r] + aff;
          xbuf[(ni * NRHS + r) * nxp + j] = xv;
          P.x[r][c * nx + j] = xv;
          if constexpr (!HOST)
            if (P.hx[r]) P.hx[r][c * nx + j] = xv;  // host-output kernels write whole rows instead
        }
      } else {
        const double h = (flat && P.affine) ? AFH[ni * mmaxh + (j - nx)] : 0.0;
#pragma unroll
        for (int r = 0; r < NRHS; ++r) P.Hx[r][mc.doff + (j - nx)] = acc[r] + h;
      }
    }
  }
};

// phase B: interior u_c = u_off_c + K_c x_c ; leaf z_N,c = F_N x_c.
// Host-output kernels (HOST) also leave u in the staged u_off entry it was
// computed from (each task reads and overwrites its own entry), so whole u
// rows can go to the caller's mapped buffer after the phase (16-byte stores).
#ifndef SCN_HOST_U_ROWS
#define SCN_HOST_U_ROWS 1
#endif
template <int NRHS, bool HOST = false>
struct FwPhaseB {
  const SweepParams& P;
  const NodeMeta* meta;
  const double* slot;
  double* UO;
  const double* xbuf;
  int nx, nu, Vp, nxp, ncols, v1nu, leaf, root, single;
  template <int S>
  __device__ __forceinline__ void run(int task, int q, bool active) const {
    int ni = 0, j = 0;
    const double* col = slot;
    if (active) {
      ni = single ? 0 : task / ncols;
      j = task - ni * ncols;
      const NodeMeta& mc = meta[ni];
      if (leaf) active = j < mc.mN;
      const int skip = root ? 0 : Vp * (nx + mc.m);
      col = slot + mc.blk + skip + j * nxp;
    }
    double acc[NRHS];
    dot_split<NRHS, S>(col, xbuf + ni * NRHS * nxp, nxp, active ? nxp : 0, q, acc);
    if (active && q == 0) {
      const NodeMeta& mc = meta[ni];
#pragma unroll
      for (int r = 0; r < NRHS; ++r) {
        if (leaf) {
          P.Hx[r][mc.tdo + j] = acc[r];
        } else {
          const double uv = UO[r * v1nu + ni * nu + j] + acc[r];
          P.u[r][static_cast<int64_t>(mc.c) * nu + j] = uv;
          if constexpr (HOST) {
            if (SCN_HOST_U_ROWS)
              UO[r * v1nu + ni * nu + j] = uv;  // whole rows leave after the phase (consume_forward)
            else if (P.hu[r])
              P.hu[r][static_cast<int64_t>(mc.c) * nu + j] = uv;
          }
        }
      }
    }
  }
};

template <int NRHS, bool HOST = false>
__device__ void consume_forward(const SweepParams& P, const Item& it, const double* slot, const double* mat,
                                const double* st, double* xbuf, int ttid, int team, int mmax,
                                int mNmax, long long* trace_row) {
  const int nx = P.nx, nu = P.nu, Vp = P.Vp, nxp = P.nxp;
  const int cnt = it.count;
  const bool leaf = it.leaf != 0;
  const bool root = it.first == 0;
  const NodeMeta* meta = reinterpret_cast<const NodeMeta*>(slot);
  const bool flat = (it.direct & kFlatTop) != 0;
  const int cstride = flat ? flat_len(it.direct >> 8, nu) : Vp;  // phase-A column length
  const int tot = flat ? cstride : it.v0_n * Vp;
  const double* PV = st;
  double* UO = const_cast<double*>(st) + NRHS * tot;  // host-output kernels leave u here (FwPhaseB)
  const double* AF = st + NRHS * (tot + it.v1_n * nu);
  PROF_T0();
  if (root) {  // x_0 = p (affine) or 0
    for (int idx = ttid; idx < NRHS * nx; idx += kTeam) {
      const int r = idx / nx, k = idx - r * nx;
      const double v = P.affine ? P.root_state[k] : 0.0;
      xbuf[r * nxp + k] = v;
      P.x[r][k] = v;
      if (P.hx[r]) P.hx[r][k] = v;
    }
  } else {
    const FwPhaseA<NRHS, HOST> body{P,    meta, mat, PV, AF, xbuf, nx, cstride, nxp, nx + mmax, tot,
                                    cnt == 1 ? 1 : 0, flat ? 1 : 0, AF + cnt * nx, P.mmax};
    for_tasks(cnt * (nx + mmax), ttid, body);
  }
  if (ttid == 0) PROF_T1(11);
  TRACE_IN(3);
  team_sync(team);
  if (ttid == 0) PROF_T1(12);
  TRACE_IN(4);
  // mapped host output (host I/O): the item's x rows leave shared memory as
  // whole 16-byte stores (full PCIe write transactions), alongside phase B
  if constexpr (HOST)
  if (!root && (P.hx[0] || (NRHS > 1 && P.hx[NRHS - 1]))) {
    if ((nx & 1) == 0) {
      const int n2 = nx >> 1;
      for (int idx = ttid; idx < NRHS * cnt * n2; idx += kTeam) {
        const int r = idx / (cnt * n2), rem = idx - r * cnt * n2, ni = rem / n2, k = rem - ni * n2;
        if (P.hx[r])
          reinterpret_cast<double2*>(P.hx[r] + static_cast<int64_t>(meta[ni].c) * nx)[k] =
              *reinterpret_cast<const double2*>(xbuf + (ni * NRHS + r) * nxp + 2 * k);
      }
    } else {
      for (int idx = ttid; idx < NRHS * cnt * nx; idx += kTeam) {
        const int r = idx / (cnt * nx), rem = idx - r * cnt * nx, ni = rem / nx, k = rem - ni * nx;
        if (P.hx[r]) P.hx[r][static_cast<int64_t>(meta[ni].c) * nx + k] = xbuf[(ni * NRHS + r) * nxp + k];
      }
    }
  }
  const FwPhaseB<NRHS, HOST> body{P,  meta, mat, UO, xbuf, nx, nu, cstride, nxp, leaf ? mNmax : nu, it.v1_n * nu,
                                  leaf ? 1 : 0, root ? 1 : 0, cnt == 1 ? 1 : 0};
  for_tasks(cnt * (leaf ? mNmax : nu), ttid, body);
  if constexpr (HOST)
  if (SCN_HOST_U_ROWS && !leaf && (P.hu[0] || (NRHS > 1 && P.hu[NRHS - 1]))) {
    team_sync(team);  // every u of the item is in UO
    const int v1nu = it.v1_n * nu;
    if ((nu & 1) == 0) {
      const int n2 = nu >> 1;
      for (int idx = ttid; idx < NRHS * cnt * n2; idx += kTeam) {
        const int r = idx / (cnt * n2), rem = idx - r * cnt * n2, ni = rem / n2, k = rem - ni * n2;
        if (P.hu[r])
          reinterpret_cast<double2*>(P.hu[r] + static_cast<int64_t>(meta[ni].c) * nu)[k] =
              *reinterpret_cast<const double2*>(UO + r * v1nu + ni * nu + 2 * k);
      }
    } else {
      for (int idx = ttid; idx < NRHS * cnt * nu; idx += kTeam) {
        const int r = idx / (cnt * nu), rem = idx - r * cnt * nu, ni = rem / nu, k = rem - ni * nu;
        if (P.hu[r]) P.hu[r][static_cast<int64_t>(meta[ni].c) * nu + k] = UO[r * v1nu + ni * nu + k];
      }
    }
  }
  if (ttid == 0) PROF_T1(13);
}

// ---------------------------------------------------------------- fused FB-step finish
// The dual rows of this CTA's forward items (each row's Hx was written by one
// of this CTA's teams; visible after the block barrier), listed per CTA by the
// host (P.fb_rows): one row per thread, so every row's loads are in flight at
// once, then a fixed-order block reduction into this CTA's partial.
__device__ void fb_epilogue_cta(const SweepParams& P) {
  __shared__ double red[kThreads / 32][8];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double lam = P.fb_S[P.fb_state * sl::kStateStride + sl::LAM];
  const double gp = 1.0 / lam;
  const double* y = P.y[0];
  const double* Hx = P.Hx[0];
  double s[6] = {0, 0, 0, 0, 0, 0};
  const int lo = P.fb_rows_off[blockIdx.x], hi = P.fb_rows_off[blockIdx.x + 1];
  for (int q = lo + tid; q < hi; q += kThreads) {
    const int64_t i = P.fb_rows[q];
    fbrow::fb_row(i, P.fb_kind[i], y[i], Hx[i], P.fb_lo[i], P.fb_hi[i], P.fb_wg[i], lam, gp, 0, P.fb_Hx0,
                  P.fb_weight, P.fb_z, P.fb_R, P.fb_T, true, s);
  }
#pragma unroll
  for (int q = 0; q < 6; ++q) {
    double t = s[q];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double u = __shfl_xor_sync(0xffffffffu, t, o);
      t = q == 5 ? fmax(t, u) : t + u;
    }
    if (lane == 0) red[warp][q] = t;
  }
  __syncthreads();
  if (tid < 6) {
    double t = red[0][tid];
    for (int w = 1; w < kThreads / 32; ++w) t = tid == 5 ? fmax(t, red[w][tid]) : t + red[w][tid];
    P.fb_part[static_cast<int64_t>(blockIdx.x) * 8 + tid] = t;
    __threadfence();  // before thread 0's arrival on the grid counter
  }
}

// The last CTA: the grid's partials combined in CTA order (the order of
// grid_reduce's second stage), the step's scalars, the publish.
__device__ void fb_epilogue_last(const SweepParams& P) {
  __shared__ double tot[8];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (warp < 6) {
    const int q = warp;
    double t = q == 5 ? -INFINITY : 0.0;
    for (int b = lane; b < static_cast<int>(gridDim.x); b += 32) {
      const double v = __ldcg(P.fb_part + static_cast<int64_t>(b) * 8 + q);
      t = q == 5 ? fmax(t, v) : t + v;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double u = __shfl_xor_sync(0xffffffffu, t, o);
      t = q == 5 ? fmax(t, u) : t + u;
    }
    if (lane == 0) tot[q] = t;
  }
  __syncthreads();
  if (tid == 0) {
    const double s[6] = {tot[0], tot[1], tot[2], tot[3], tot[4], tot[5]};
    fbrow::fb_finalize(P.fb_S, P.fb_I, P.fb_state, 0, s);
  }
  if (P.pub) fbrow::publish_block(P.fb_S, P.fb_I, P.pub, P.seq);
}

// MODE bits (one instantiation per combination, so the common layout's
// kernel carries no fallback code): kModeConsumerStage = teams stage their own
// vectors; kModeGlobalBlocks = some items read their node blocks from HBM.
constexpr int kModeConsumerStage = 1, kModeGlobalBlocks = 2;
// kModeHostOut: forward x rows to mapped host memory as 16-byte row stores
// (only instantiated for the default layout; other layouts store per element)
constexpr int kModeHostOut = 4;
template <int NRHS, int MODE>
__global__ void __launch_bounds__(kThreads, 1) sweep_kernel(const SweepParams P, int mmax, int mNmax) {
  extern __shared__ __align__(128) double smem[];
  // full[k mod kTeams*NS]: the matrix-slot barrier of item k. kTeams per
  // slot, so a barrier always serves the same consumer team in order (k and
  // k + kTeams*NS go to the same team) whatever NS is: a team can never test
  // the phase parity of a use that has not started yet.
  __shared__ __align__(8) uint64_t full[kTeams * kMaxSlots], sfull[kStageQ], sempty[kStageQ], done[kDoneQ],
      pdone[kDoneQ];
  __shared__ __align__(8) uint64_t mempty[kMaxSlots];  // slot consumed (team -> issuer)
  __shared__ __align__(16) Item sitem[kMaxSlots];
  __shared__ __align__(16) int4 sdone[kDoneQ];  // {first, count, pass, publish} of finished items
  __shared__ unsigned s_epoch;
  __shared__ int s_retired;  // items [0, s_retired) of this CTA are complete
  // a skipped launch touches nothing: the epoch stays, so the next sweep is
  // as if this one had not been enqueued (every CTA reads the same flag)
  if (P.skip && *reinterpret_cast<const volatile int*>(P.skip)) return;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int NS = P.nslot;  // matrix slots
  double* slots = smem;
  double* stages = smem + static_cast<int64_t>(NS) * P.slot_doubles;  // kStageQ (or kTeams) staging areas
  constexpr bool kConsumerStage = (MODE & kModeConsumerStage) != 0;
  double* scratch = stages + static_cast<int64_t>(kConsumerStage ? kTeams : kStageQ) * P.stage_doubles;
  const int b = blockIdx.x;
  const Item* items = P.items + P.cta_off[b];
  const int K = P.cta_off[b + 1] - P.cta_off[b];

  auto issue = [&](int k, const Item& it) {  // one thread
    const int s = k % NS;
    sitem[s] = it;
    uint64_t* fb = &full[k % (kTeams * NS)];
    mbar_arrive_expect_tx(fb, static_cast<unsigned>(it.bytes));
    tma_load_1d(slots + static_cast<int64_t>(s) * P.slot_doubles, (it.pass == 0 ? P.bw_blk : P.fw_blk) + it.off,
                static_cast<unsigned>(it.bytes), fb);
  };

  if (tid == 0) {
    s_epoch = *reinterpret_cast<volatile unsigned*>(P.ctrl) + 1u;
    s_retired = 0;
    for (int s = 0; s < kTeams * NS; ++s) mbar_init(&full[s], 1);
    for (int s = 0; s < NS; ++s) mbar_init(&mempty[s], kReleaseArrivals);
    for (int q = 0; q < kStageQ; ++q) {
      mbar_init(&sfull[q], 1);
      mbar_init(&sempty[q], kReleaseArrivals);
    }
    for (int q = 0; q < kDoneQ; ++q) {
      mbar_init(&done[q], kReleaseArrivals);
      mbar_init(&pdone[q], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = tid; i < kScratchBufs * kTeams * P.scratch_doubles; i += kThreads) scratch[i] = 0.0;  // zero pads of w / x
  __syncthreads();
  const unsigned E = s_epoch;
  if (warp < kProducers) {
    // ------------------------------------------------------------ producers
    // Producer warp p stages items k = p (mod kProducers) into staging area
    // q = k mod kStageQ (a ring twice as deep as the matrix slots, so staging
    // runs ahead of slot recycling): wait for the area to be consumed, poll
    // the item's dependency flags (ld.acquire), stage its vectors, arrive.
    const int p = warp;
    for (int k = p; k < K; k += kProducers) {
      const int q = k % kStageQ;
      const Item it = items[k];
      PROF_T0();
      if (k >= kStageQ) mbar_wait(&sempty[q], static_cast<unsigned>((k / kStageQ - 1) & 1));
      if (lane == 0 && p == 0) PROF_T1(0);
#ifdef SCN_SWEEP_PROFILE
      if (g_trace && lane == 0) g_trace[12LL * (P.cta_off[blockIdx.x] + P.items_base + k) + 8] = static_cast<long long>(gtimer());
#endif
      // host-output kernels: a backward item's y rows (the caller's pinned
      // memory, over PCIe) and affine terms go out before the dependency wait
      constexpr bool kSplitStage = (MODE & kModeHostOut) != 0 && !kConsumerStage;
      if constexpr (kSplitStage)
        if (it.pass == 0) stage_issue<NRHS, 32, 1>(P, it, stages + static_cast<int64_t>(q) * P.stage_doubles, lane);
      if (!DBG(1)) {
        if (it.ldep >= 0)
          while (ld_acquire_cta(&s_retired) <= it.ldep) __nanosleep(16);
        if (it.dep_lo < it.dep_hi)
          while (!flags_ready(dep_flags(P, it), it, E, lane)) __nanosleep(32);
      }
      if (lane == 0 && p == 0) PROF_T1(2);
#ifdef SCN_SWEEP_PROFILE
      if (g_trace && lane == 0) g_trace[12LL * (P.cta_off[blockIdx.x] + P.items_base + k) + 9] = static_cast<long long>(gtimer());
#endif
      if constexpr (kSplitStage) {
        stage_issue<NRHS, 32, 2>(P, it, stages + static_cast<int64_t>(q) * P.stage_doubles, lane);
      } else if (!kConsumerStage) {
        stage_issue<NRHS>(P, it, stages + static_cast<int64_t>(q) * P.stage_doubles, lane);
      }
      cp_async_wait_all();
      __syncwarp();
#ifdef SCN_SWEEP_PROFILE
      if (g_trace && lane == 0) g_trace[12LL * (P.cta_off[blockIdx.x] + P.items_base + k) + 10] = static_cast<long long>(gtimer());
#endif
      if (lane == 0) mbar_arrive(&sfull[q]);
      if (lane == 0 && p == 0) PROF_T1(1);
    }
  } else if (warp < kPublisherWarp) {
    // ------------------------------------------------------------ consumer teams
    const int team = (warp - kTeamWarp0) / (kTeam / 32);
    const int ttid = tid - 32 * kTeamWarp0 - team * kTeam;
    double* const tbuf0 = scratch + static_cast<int64_t>(team) * kScratchBufs * P.scratch_doubles;
    LC_DECL();
    for (int k = team; k < K; k += kTeams) {
      const int s = k % NS;
      PROF_T0();
      TRACE(0);
      LC_MARK(7);  // loop overhead
      mbar_wait(&full[k % (kTeams * NS)], static_cast<unsigned>((k / (kTeams * NS)) & 1));
      if (ttid == 0) PROF_T1(3);
      TRACE(1);
      LC_MARK(0);  // wait matrices
      const int q = k % kStageQ;
      mbar_wait(&sfull[q], static_cast<unsigned>((k / kStageQ) & 1));
      if (ttid == 0) PROF_T1(4);
      TRACE(2);
      LC_MARK(1);  // wait vectors
      const Item it = sitem[s];
      // w / x scratch of this item: double-buffered by item parity when the
      // team's warps release items independently (they may run one item apart)
      double* tbuf = tbuf0 + ((kScratchBufs == 2) ? ((k / kTeams) & 1) * P.scratch_doubles : 0);
      const double* slot = slots + static_cast<int64_t>(s) * P.slot_doubles;
      // node blocks: in the slot, or (an item larger than a slot) read from
      // HBM/L2 in place; the slot then holds only the item's node headers.
      // Separate call sites keep the slot path's loads in the shared space.
      const bool gblocks = (it.direct & kGlobalBlocks) != 0;
      const double* gmat = (it.pass == 0 ? P.bw_blk : P.fw_blk) + it.off;
      const double* st = stages + static_cast<int64_t>(q) * P.stage_doubles;
      if constexpr (kConsumerStage) {  // large vectors: the team stages its own item after the producer's
                               // dependency check (acquire) into a per-team area
        double* tst = stages + static_cast<int64_t>(team) * P.stage_doubles;
        stage_issue<NRHS, kTeam>(P, it, tst, ttid);
        cp_async_wait_all();
        team_sync(team);
        st = tst;
      }
      long long* trace_row = nullptr;
#ifdef SCN_SWEEP_PROFILE
      if (g_trace) trace_row = g_trace + 12LL * (P.cta_off[blockIdx.x] + P.items_base + k);
#endif
      if (DBG(2)) {
      } else if (it.pass == 0) {
        if ((MODE & kModeGlobalBlocks) && gblocks)
          consume_backward<NRHS>(P, it, slot, gmat, st, tbuf, ttid, team, trace_row);
        else
          consume_backward<NRHS>(P, it, slot, slot, st, tbuf, ttid, team, trace_row);
      } else {
        if ((MODE & kModeGlobalBlocks) && gblocks)
          consume_forward<NRHS, (MODE & kModeHostOut) != 0>(P, it, slot, gmat, st, tbuf, ttid, team, mmax, mNmax,
                                                          trace_row);
        else
          consume_forward<NRHS, (MODE & kModeHostOut) != 0>(P, it, slot, slot, st, tbuf, ttid, team, mmax, mNmax,
                                                          trace_row);
      }
      TRACE(5);
      LC_MARK(2);  // compute (phases A + barrier + B)
      if (!kWarpRelease || kConsumerStage) team_sync(team);
      LC_MARK(3);  // end barrier
      if (ttid == 0) PROF_T1(5);
      TRACE(6);
      // release: slot reads done -> the issuer may refill the slot; staging
      // area free; item complete -> the publisher. Per warp (kWarpRelease:
      // a warp done with phase B moves on without waiting for the others),
      // else once per team after the barrier above.
      if (kWarpRelease ? (lane == 0) : (ttid == 0)) {
        mbar_arrive(&mempty[s]);
        mbar_arrive(&sempty[q]);
        // the publisher must have retired item k-kDoneQ before its DONE phase reuses
        const int dq = k % kDoneQ;
        if (k >= kDoneQ) mbar_wait(&pdone[dq], static_cast<unsigned>((k / kDoneQ - 1) & 1));
        if (ttid == 0) sdone[dq] = make_int4(it.first, it.count, it.pass, it.publish);
        mbar_arrive(&done[dq]);
      }
      if (ttid == 0) PROF_T1(6);
      TRACE(7);
      LC_MARK(4);  // release
    }
    LC_FLUSH();
  }
  if (warp == kIssuerWarp) {
    // ------------------------------------------------------------ issuer
    // One thread streams the CTA's items through the matrix slots in order:
    // item k goes to slot k mod NS once the team holding item k - NS has
    // released it (mbarrier, so generic reads precede the async-proxy
    // write), as one 1-D bulk copy completing on full[k mod 2NS].
    // The next item's record is prefetched while waiting for the slot.
    Item nxt{};
    if (lane == 0 && K > 0) nxt = items[0];
    int pf = 0;                // items [0, pf) are issued or prefetched into L2
    unsigned gdep = 0;         // bit k % NS: item k (in its slot) waits on other CTAs
    for (int k = 0; k < K; ++k) {
      if (lane == 0) {
        const Item it = nxt;
        if (k + 1 < K) nxt = items[k + 1];
        if (k >= NS) {
          if (kL2Ahead > 0 && ((gdep >> (k % NS)) & 1u)) {  // a long wait ahead: the next items into L2
            const int lim = min(K, k + 1 + kL2Ahead);
            for (pf = max(pf, k + 1); pf < lim; ++pf) {
              const Item& q = items[pf];
              if (!(q.direct & kGlobalBlocks)) prefetch_l2((q.pass == 0 ? P.bw_blk : P.fw_blk) + q.off, q.bytes);
            }
          }
          mbar_wait(&mempty[k % NS], static_cast<unsigned>((k / NS - 1) & 1));
        }
        issue(k, it);
        gdep = (gdep & ~(1u << (k % NS))) | ((it.dep_lo < it.dep_hi ? 1u : 0u) << (k % NS));
      }
      __syncwarp();
    }
  }
  if (warp == kPublisherWarp) {
    // ------------------------------------------------------------ publisher
    // Retires items in order. Items consumed by other CTAs get their flags
    // released; one gpu-scope fence covers every item finished since the
    // previous one (the fence is the expensive part; it is cumulative over
    // the teams' writes observed through DONE). Local-only batches need just
    // the CTA-scope release of the retire counter.
    int k = 0;
    while (k < K) {
      mbar_wait(&done[k % kDoneQ], static_cast<unsigned>((k / kDoneQ) & 1));
      int j = k + 1;
      if (lane == 0)
        while (j < K && j - k < kDoneQ &&
               mbar_test(&done[j % kDoneQ], static_cast<unsigned>((j / kDoneQ) & 1)))
          ++j;
      j = __shfl_sync(0xffffffffu, j, 0);
      PROF_T0();
      bool pub = false;
      for (int q2 = k; q2 < j; ++q2) pub |= (sdone[q2 % kDoneQ].w & 1) != 0;
      if (pub) {
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        for (int q2 = k; q2 < j; ++q2) {
          const int4 dn = sdone[q2 % kDoneQ];
          if (!(dn.w & 1)) continue;
          unsigned* flags = dn.z == 0 ? P.bw_flag : P.fw_flag;
          for (int i = lane; i < dn.y; i += 32)
            asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(flags + dn.x + i), "r"(E) : "memory");
        }
      }
      __syncwarp();
      if (lane == 0) {
        st_release_cta(&s_retired, j);
#ifdef SCN_SWEEP_PROFILE
        if (g_timeline || g_trace) {
          const unsigned long long now = gtimer();
          for (int q2 = k; q2 < j; ++q2) {
            if (g_timeline) g_timeline[P.cta_off[b] + q2 + P.items_base] = now;
            if (g_trace) g_trace[12LL * (P.cta_off[b] + P.items_base + q2) + 11] = static_cast<long long>(now);
          }
        }
#endif
        PROF_T1(7);
        for (int q2 = k; q2 < j; ++q2) mbar_arrive(&pdone[q2 % kDoneQ]);
      }
      k = j;
    }
  }
  __syncthreads();
  // the fused FB finish exists only in the 1-RHS instantiations: carrying
  // its code made the 2-RHS kernel 10 us slower (258 -> 268 us at C3)
  const bool fb = NRHS == 1 && P.fb_S != nullptr;
  if constexpr (NRHS == 1)
    if (fb) fb_epilogue_cta(P);  // this CTA's partial, written by threads < 6 (after a barrier)
  __shared__ int s_last;
  if (fb) __syncthreads();
  if (tid == 0) {
    __threadfence();
    const unsigned prev = atomicAdd(P.ctrl + 1, 1u);
    s_last = prev == gridDim.x - 1;
  }
  __syncthreads();
  if (s_last) {
    if constexpr (NRHS == 1)
      if (fb) {
        __threadfence();
        fb_epilogue_last(P);
      }
    if (tid == 0) {
      P.ctrl[1] = 0u;
      __threadfence();
      atomicExch(P.ctrl, E);
    }
  }
}

}  // namespace

namespace {
#define SCN_K(R, M) reinterpret_cast<const void*>(sweep_kernel<R, M>)
const void* const kKernels[3][4] = {
    {SCN_K(1, 0), SCN_K(1, 1), SCN_K(1, 2), SCN_K(1, 3)},
    {SCN_K(2, 0), SCN_K(2, 1), SCN_K(2, 2), SCN_K(2, 3)},
    // host-output variants of the default layout (row [nrhs-1]); the rest of the row repeats them
    {SCN_K(1, 4), SCN_K(2, 4), SCN_K(1, 4), SCN_K(2, 4)}};
#undef SCN_K
}  // namespace

size_t static_smem() {
  size_t m = 0;
  for (auto& row : kKernels)
    for (const void* fn : row) {
      cudaFuncAttributes a{};
      cudaFuncGetAttributes(&a, fn);
      m = a.sharedSizeBytes > m ? a.sharedSizeBytes : m;
    }
  return m;
}
cudaError_t configure(size_t dyn_smem);
cudaError_t occupancy(int* ctas_per_sm, size_t dyn_smem);
cudaError_t launch(const SweepParams& P, int grid, size_t dyn_smem, int mmax, int mNmax, cudaStream_t stream);
}  // namespace SCN_SWEEP_NS

#define SCN_STR2(x) #x
#define SCN_STR(x) SCN_STR2(x)
extern const SweepImpl SCN_SWEEP_IMPL = {
    SCN_STR(SCN_SWEEP_NS), SCN_SWEEP_NS::kProducers, SCN_SWEEP_NS::kTeams, SCN_SWEEP_NS::kThreads,
    SCN_SWEEP_NS::kStageQ, SCN_SWEEP_NS::kScratchBufs, &SCN_SWEEP_NS::static_smem,
    &SCN_SWEEP_NS::configure, &SCN_SWEEP_NS::occupancy, &SCN_SWEEP_NS::launch};

#ifndef SCN_SWEEP_SECONDARY  // diagnostics (profiling build of the default geometry)
cudaError_t sweep_trace(long long* dev_buf) {
#ifdef SCN_SWEEP_PROFILE
  return cudaMemcpyToSymbol(SCN_SWEEP_NS::g_trace, &dev_buf, sizeof(dev_buf));
#else
  (void)dev_buf;
  return cudaErrorNotSupported;
#endif
}

cudaError_t sweep_timeline(unsigned long long* dev_buf) {
#ifdef SCN_SWEEP_PROFILE
  return cudaMemcpyToSymbol(SCN_SWEEP_NS::g_timeline, &dev_buf, sizeof(dev_buf));
#else
  (void)dev_buf;
  return cudaErrorNotSupported;
#endif
}

cudaError_t sweep_profile_read(unsigned long long* out, bool reset) {
#ifdef SCN_SWEEP_PROFILE
  cudaError_t e = cudaMemcpyFromSymbol(out, SCN_SWEEP_NS::g_prof, sizeof(unsigned long long) * 16);
  if (e == cudaSuccess && reset) {
    unsigned long long z[16] = {0};
    e = cudaMemcpyToSymbol(SCN_SWEEP_NS::g_prof, z, sizeof(z));
  }
  return e;
#else
  for (int i = 0; i < 16; ++i) out[i] = 0;
  (void)reset;
  return cudaSuccess;
#endif
}

#endif

namespace SCN_SWEEP_NS {
cudaError_t configure(size_t dyn_smem) {
  // The cap is a per-function, per-device attribute shared by every handle of
  // the process: only ever raise it (a lower value would break the launches
  // of handles with larger slots).
  static std::mutex mu;
  static size_t configured[64] = {};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  if (dev >= 0 && dev < 64) {
    if (dyn_smem <= configured[dev]) return cudaSuccess;
    configured[dev] = dyn_smem;
  }
  for (auto& row : kKernels)
    for (const void* fn : row) {
      e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(dyn_smem));
      if (e != cudaSuccess) return e;
    }
  return cudaSuccess;
}

cudaError_t occupancy(int* ctas_per_sm, size_t dyn_smem) {
  int lo = 1 << 30;
  for (auto& row : kKernels)
    for (const void* fn : row) {
      int a = 0;
      cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, fn, kThreads, dyn_smem);
      if (e != cudaSuccess) return e;
      lo = a < lo ? a : lo;
    }
  *ctas_per_sm = lo;
  return cudaSuccess;
}

cudaError_t launch(const SweepParams& P, int grid, size_t dyn_smem, int mmax, int mNmax, cudaStream_t stream) {
  SweepParams p = P;
  void* args[] = {&p, &mmax, &mNmax};
#ifdef SCN_SWEEP_PROFILE
  static int dbg_set = [] {
    const char* e = getenv("SCN_DBG");
    int v = e ? atoi(e) : 0;
    cudaMemcpyToSymbol(g_dbg, &v, sizeof(int));
    return 1;
  }();
  (void)dbg_set;
#endif
  const int mode = (P.consumer_stage ? kModeConsumerStage : 0) | (P.global_blocks ? kModeGlobalBlocks : 0);
  const bool host_out = P.hx[0] || (P.nrhs == 2 && P.hx[1]);
  const void* fn = (host_out && mode == 0) ? kKernels[2][P.nrhs == 2 ? 1 : 0] : kKernels[P.nrhs == 2 ? 1 : 0][mode];
  return cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kThreads), args, dyn_smem, stream);
}
}  // namespace SCN_SWEEP_NS

}  // namespace scn
