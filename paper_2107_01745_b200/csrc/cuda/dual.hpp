// SPDX-License-Identifier: MIT
// Shared declarations of the fused dual-vector kernels (dualops.cu) and the
// device scalar block used by the solver loops (solver.cpp).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace scn {

// Scalar block slots (doubles). Per-state scalars live at state*kStateStride.
namespace sl {
constexpr int kStateStride = 8;
constexpr int LAM = 0, FHAT = 1, CONJ = 2, ZN2 = 3, VALUE = 4, RESID = 5;
constexpr int FHAT0 = 32;
constexpr int IMG2 = 33, R2 = 34;                   // simple-rule norms (MINFBE)
constexpr int RAYLEIGH = 35, PMAG = 36, PNEXT = 37;  // power iteration
constexpr int GAMMA0 = 38;                          // L-BFGS gamma0
constexpr int TAU = 40, KSTAR = 41, STALL = 42, CERT_FHAT = 43, HXW_RW = 44, RW2 = 45, VALUE_A = 46,
              CONJ_A = 47, ZN2_A = 48, FHAT_A = 49, ALPHA1 = 50, ALPHA2 = 51, HR2 = 52, RR2 = 53,
              DELTA = 54;
constexpr int EVALF = 56, EVALF_INF = 57, RED0 = 58, RED1 = 59;  // API reductions
// fb_finish's skip word I[CONV] for a speculative MINFBE sweep: 1 when the
// step met the stop tolerance or the backtracking rule in S[GATE_RULE]
// (0 original, 1 MINFBE simple, 3 NAMA simple; 2 none) would reject it
// (solvers.hpp:279-302, 329-346, 424-438, 467-483)
constexpr int EPS_STOP = 60, GATE_RULE = 61, BETA_BT = 62, EPS_BT = 63;
constexpr int CURV = 64;  // L-BFGS curvatures [64, 64 + mem + 1)
constexpr int CERT_S = 120;  // sharded certificate: coefficient totals [120, 132) between phases
constexpr int kScalars = 192;
}  // namespace sl
// Int block slots.
// Host publication of the scalar block (mapped pinned memory), in the manner
// of NCCL's low-latency protocol: every 8-byte word carries 4 bytes of data in
// its low half and the publish sequence number in its high half, written as
// one store, so the host validates each word by its own flag and the device
// needs no system-scope fence before it can move on. Layout: S as two words
// per double (low, high 32 bits), then I one word per int.
namespace il {
constexpr int LB_COUNT = 0, LB_PUSHED = 1, SETTLED = 2, PZERO = 3;
constexpr int PDONE = 4, PROUNDS = 5, PMAX = 6;  // batched power iteration: sticky stop flag, rounds run, cap
constexpr int CONV = 7;  // last fb_finish met the stop tolerance: skip word of a speculative sweep
constexpr int LB_ORDER = 8;  // [8, 8 + mem + 1): slot ids, oldest first, then free slots
constexpr int REJECT = 100;  // last fb_finish: the backtracking rule in S[GATE_RULE] rejects the step
constexpr int CSTATE = 101;  // sharded certificate: state after phase k at CSTATE + k - 1 (k = 1..3)
constexpr int CKSTAR = 105;  // sharded certificate: accepted trial between phases
constexpr int kInts = 128;
}  // namespace il
constexpr int kPubWords = 2 * sl::kScalars + il::kInts;

// Per-dual-row nonsmooth data (prox.hpp:15-52 flattened).
struct RowG {
  const int8_t* kind;  // 0 none, 1 box, 2 scaled l1
  const double* lo;
  const double* hi;
  const double* wg;  // weight * gamma
};

struct DualCtx {
  int D;
  int nblk;
  RowG g;
  double* S;       // scalar block
  int* I;          // int block
  double* part;    // partial sums [2][64][nblk]
  unsigned* bar;   // grid barrier {count, generation}
  const int* skip = nullptr;  // L-BFGS kernels: non-null and *skip != 0 -> return at once (speculation)
  // fb_finish: when pub is set, block 0 also publishes S / I into mapped
  // host memory (publish_kernel's protocol, one launch fewer)
  unsigned long long* pub = nullptr;
  unsigned seq = 0;
  // Subtree-sharded handles. Reductions count only the rows
  // with cnt[i] != 0 (this rank's own rows; the replicated top on rank 0),
  // and every reduction becomes a phase boundary: phase 0 ends with this
  // rank's totals in xs, the launcher allgathers them over the ranks (xc,
  // a Comm*), and phase 1 combines xr in rank order and carries on. Every
  // rank then holds bitwise-identical scalars.
  const uint8_t* cnt = nullptr;
  void* xc = nullptr;     // host: the handle's communicator (null: single-launch kernels)
  int world = 1;
  double* xs = nullptr;   // [kXMax] this rank's totals
  double* xr = nullptr;   // [world][kXMax] gathered totals
  int phase = -1;         // set by the launchers
};
constexpr int kXMax = 160;  // doubles exchanged per rank and phase
// allgather of n doubles per rank through a Comm* (comm.cpp), on st
void dual_allgather(void* xc, const double* send, double* recv, size_t n, cudaStream_t st);

// fb_step / rescale_state finish (fbe.hpp:38-67). mode 0: fhat from the
// quadratic identity fhat(y) = fhat(0) - 1/2 <Hx(0) + Hx(y), y>; mode 1: keep
// S[FHAT] of the state.
cudaError_t k_fb_finish(const DualCtx& c, int state, int mode, const double* y, const double* Hx,
                        const double* Hx0, const double* weight, double* z, double* R, double* T,
                        cudaStream_t st);
cudaError_t k_publish(const double* S, const int* I, unsigned long long* pub_mapped, unsigned seq, cudaStream_t st);
// Sharded sweep exchange (device.cpp phase_a / phase_b). Per right-hand side
// the exchange buffer is [ns_w contributions of the shard-stage nodes | nys
// dual rows of those nodes]. Pack (after launch A): this rank's own entries,
// zero elsewhere, ready for the sum-allreduce. Unpack (before launch B): the
// summed contributions into the contribution array, and launch B's dual input
// = the top rows of y followed by the summed shard-stage rows.
struct ExchangeDims {
  int64_t ns_w, nys, xbuf_rhs, contrib_off, dual_top;
  int64_t own_c_lo, own_c_hi;  // this rank's contributions, buffer coordinates
  int64_t own_y_lo, own_y_hi;  // this rank's shard-stage dual rows, y coordinates
  int nrhs;
  double* contrib[2];
  const double* y[2];
  double* ycomp[2];
};
cudaError_t k_exchange_pack(const ExchangeDims& e, double* xbuf, cudaStream_t st);
cudaError_t k_exchange_unpack(const ExchangeDims& e, const double* xbuf, cudaStream_t st);
// MINFBE fbe_grad epilogue (fbe.hpp:89-94): grad = R + lam HR, and the simple
// backtracking norms ||(grad - R)/lam||^2, ||R||^2 (solvers.hpp:215-222, 279-302).
cudaError_t k_fbe_grad(const DualCtx& c, int state, const double* R, const double* HR, double* grad,
                       cudaStream_t st);
// L-BFGS (lbfgs.hpp:33-62): optional push of (a - b, cc - dd) with scale_ref
// ||dd||^2 (or the given scale_ref when >= 0), then the two-loop recursion
// out = -B g.
// Mbuf (2 * 64 * 64 doubles, persistent per buffer): compact form when mem <= 6
cudaError_t k_lbfgs(const DualCtx& c, int mem, double eps_curv, double scale_ref, int do_push, const double* a,
                    const double* b, const double* cc, const double* dd, const double* gvec,
                    double* out, double* Sbuf, double* Qbuf, cudaStream_t st, double* Mbuf = nullptr,
                    const double* fR = nullptr, const double* fHR = nullptr, int fstate = 0, double* gout = nullptr);
// compact form (and the fused fbe_grad) applies when Mbuf is given and mem <= this
constexpr int kLbfgsCompactMaxMem = 6;
// Line-search certificate + speculative multi-tau search (fbe.hpp:136-231,
// solvers.hpp:310-325 / 440-464). shifted = 0: MINFBE (anchor y); 1: NAMA
// (anchor y - lam R, dir d + lam R). Writes y_next = T(tau*) (or
// y - lam R(tau*) when tlambda == 0) and the accepted-trial scalars.
cudaError_t k_cert_search(const DualCtx& c, int state, int shifted, int tlambda, const double* y,
                          const double* R, const double* Hx, const double* HR, const double* d,
                          const double* Hd, double* y_next, cudaStream_t st);
// Evaluate the certificate at explicit taus (test/API path): deltas[k] and
// cert_fhat[k] into S-independent outputs, the last tau's vectors into w..T.
cudaError_t k_cert_eval(const DualCtx& c, int state, int shifted, const double* y, const double* R,
                        const double* Hx, const double* HR, const double* d, const double* Hd,
                        int ntau, const double* taus_host, double* deltas, double* cfh, double* w,
                        double* Hxw, double* zz, double* RR, double* TT, cudaStream_t st);
// Power-iteration round (solvers.hpp:101-111) on v with Hv = H x0(v).
cudaError_t k_power(const DualCtx& c, double* v, const double* Hv, double rel_tol, cudaStream_t st);
// GPAD extrapolation (solvers.hpp:532-536): w = yn + mom (yn - yp); yp = yn.
cudaError_t k_extrapolate(const DualCtx& c, const double* yn, double* yp, double* w, double mom,
                          cudaStream_t st);
// prox_g / conj_value_g / dist_subdiff_inf (prox.hpp:58-171).
cudaError_t k_prox(const DualCtx& c, const double* v, double gamma_prox, double* out, cudaStream_t st);
cudaError_t k_conj(const DualCtx& c, const double* w, cudaStream_t st);                // -> S[RED0]
cudaError_t k_dist_subdiff(const DualCtx& c, const double* y, const double* z, cudaStream_t st);  // S[RED0]
// max |z - Hx| (verify_report, solvers.hpp:630-639) -> S[RED0]
cudaError_t k_max_abs_diff(const DualCtx& c, const double* a, const double* b, cudaStream_t st);
// <a, b> -> S[RED0]
cudaError_t k_dot(const DualCtx& c, const double* a, const double* b, cudaStream_t st);
// elementwise y = alpha * x (+ beta * y0)
cudaError_t k_scale(const DualCtx& c, int n, double alpha, const double* x, double beta, const double* y0,
                    double* y, cudaStream_t st);
int dual_block_threads();
int dual_max_blocks();  // grid_reduce's bound on the dual kernels' grid

// apply_H over packed rows (problem_data.hpp:144-162): z = H [x; u].
struct HRows {
  int nx, nu, nrows;
  const int32_t* row_node;    // ancestor (stage rows) or leaf node (terminal rows) per dual row
  const int8_t* row_term;     // 1 for terminal rows
  const double* coef;         // per row: nx + nu coefficients (terminal rows: nx, rest 0)
};
cudaError_t k_apply_H(const HRows& h, const double* x, const double* u, double* z, cudaStream_t st);

// eval_f (problem_data.hpp:194-222) over packed node cost blocks.
struct CostPack {
  int nx, nu, n, first_leaf;
  const int32_t* anc;
  const double* prob;
  const int32_t* nodes;  // non-root nodes evaluated here (all, or a rank's share)
  int nnodes;
  const double* node;    // cost blocks [A | B | c | Q | S | R | q | r] of the handle's nodes
  const int32_t* slot;   // [n]: block of node i in `node` (-1: not on this handle)
  const int32_t* leaves; // leaves evaluated here
  int nleaves;
  const double* leaf;    // blocks [P | p] of the handle's leaves
  const int32_t* lslot;  // [L]: block of leaf l in `leaf` (-1: not on this handle)
  const double* root_state;
  int check_root;        // 1: include the x^0 = p check
};
cudaError_t k_eval_f(const DualCtx& c, const CostPack& cp, const double* x, const double* u,
                     double feas_tol, cudaStream_t st);  // -> S[EVALF], S[EVALF_INF]

}  // namespace scn
