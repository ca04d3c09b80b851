// SPDX-License-Identifier: MIT
// Row arithmetic of the forward-backward step shared by the dual-space
// kernels (dualops.cu) and the fused FB-step epilogue of the sweep
// (sweep.cu): prox / conjugate of one dual row (prox.hpp:58-113), one row of
// finish_fb_fields (fbe.hpp:38-50) and the step's scalar finish, so both
// paths compute the same values with the same operations.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "dual.hpp"

namespace scn {
namespace fbrow {

// prox of gamma_prox * g on one row (prox.hpp:58-81).
__device__ __forceinline__ double prox_row(int kind, double v, double lo, double hi, double thr) {
  if (kind == 1) return fmin(fmax(v, lo), hi);
  if (kind == 2) return v > thr ? v - thr : (v < -thr ? v + thr : 0.0);
  return v;
}
// g* on one row (prox.hpp:90-113); +inf where the conjugate is infinite.
__device__ __forceinline__ double conj_row(int kind, double w, double lo, double hi, double wg) {
  constexpr double slack = 1e-9;
  if (kind == 1) return fmax(w * lo, w * hi);
  if (kind == 2) return fabs(w) > wg * (1.0 + slack) + slack ? INFINITY : 0.0;
  return fabs(w) > slack ? INFINITY : 0.0;
}

// One row of finish_fb_fields: z, R, T written; s accumulates conj, |z|^2,
// <Hx,R>, |R|^2, <Hx0 + Hx, y> (mode 0) and the weighted max |R| (s[5]).
__device__ __forceinline__ void fb_row(int64_t i, int kd, double yi, double hi, double lo, double up, double wg,
                                       double lam, double gp, int mode, const double* Hx0, const double* weight,
                                       double* z, double* R, double* T, bool counted, double (&s)[6]) {
  const double zi = prox_row(kd, yi / lam + hi, lo, up, gp * wg);
  const double Ri = zi - hi;
  const double Ti = yi - lam * Ri;
  z[i] = zi;
  R[i] = Ri;
  T[i] = Ti;
  if (counted) {
    s[0] += conj_row(kd, Ti, lo, up, wg);
    s[1] += zi * zi;
    s[2] += hi * Ri;
    s[3] += Ri * Ri;
    if (mode == 0) s[4] += (Hx0[i] + hi) * yi;
    s[5] = fmax(s[5], fabs(weight ? Ri * weight[i] : Ri));
  }
}

// The step's scalars from the reduced sums (one thread): f_hat by the
// quadratic identity (mode 0) or kept (mode 1), g*(T), |z|^2, the envelope
// value and the weighted residual; then the backtracking verdict of the
// rule in S[GATE_RULE] (I[REJECT]) and the skip word of speculative work
// (I[CONV]: converged or rejected).
__device__ __forceinline__ void fb_finalize(double* Sg, int* I, int state, int mode, const double (&s)[6]) {
  double* S = Sg + state * sl::kStateStride;
  // Every scalar is read before the first store: the stores go through the
  // same block, so a load after one would be ordered behind it (one L2 round
  // trip per load on the step's critical path). Same operations as before.
  const double lam = S[sl::LAM], fhat_state = S[sl::FHAT], fhat0 = Sg[sl::FHAT0];
  const double rule_d = Sg[sl::GATE_RULE], cert_fhat = Sg[sl::CERT_FHAT], hxw_rw = Sg[sl::HXW_RW],
               beta_bt = Sg[sl::BETA_BT], rw2 = Sg[sl::RW2], img2 = Sg[sl::IMG2], eps_bt = Sg[sl::EPS_BT],
               r2 = Sg[sl::R2], hr2 = Sg[sl::HR2], rr2 = Sg[sl::RR2], eps_stop = Sg[sl::EPS_STOP];
  const double fhat = mode == 0 ? fhat0 - 0.5 * s[4] : fhat_state;
  S[sl::FHAT] = fhat;
  S[sl::CONJ] = s[0];
  S[sl::ZN2] = s[1];
  S[sl::VALUE] = fhat + s[0] + lam * s[2] + 0.5 * lam * s[3];
  S[sl::RESID] = s[5];
  const int rule = static_cast<int>(rule_d);
  int reject = 0;
  if (rule == 0) {  // original rule: candidate fhat above the model (the host takes this verdict)
    const double model = __dadd_rn(__dadd_rn(cert_fhat, __dmul_rn(lam, hxw_rw)),
                                   __dmul_rn(__dmul_rn(__dmul_rn(0.5, __dadd_rn(1.0, -beta_bt)), lam), rw2));
    reject = fhat > model;
  } else if (rule == 1) {  // MINFBE simple rule: lambda |img| > eps_bt |R| halves lambda
    reject = __dmul_rn(lam, sqrt(img2)) > __dmul_rn(eps_bt, sqrt(r2));
  } else if (rule == 3) {  // NAMA simple rule on the certificate's norms
    reject = __dmul_rn(lam, sqrt(hr2)) > __dmul_rn(eps_bt, sqrt(rr2));
  }
  I[il::REJECT] = reject;
  I[il::CONV] = (s[5] <= eps_stop || reject) ? 1 : 0;
}

// S / I into mapped host memory as flagged words (dual.hpp kPubWords; all
// threads of one block). The barrier makes thread 0's scalar writes visible
// to the block; no fence follows: each word carries its own flag.
__device__ __forceinline__ void publish_block(const double* S, const int* I, unsigned long long* pub, unsigned seq) {
  __syncthreads();
  volatile unsigned long long* w = pub;
  const unsigned long long f = static_cast<unsigned long long>(seq) << 32;
  for (int t = threadIdx.x; t < sl::kScalars; t += blockDim.x) {
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(S[t]));
    w[2 * t] = f | (b & 0xffffffffull);
    w[2 * t + 1] = f | (b >> 32);
  }
  for (int t = threadIdx.x; t < il::kInts; t += blockDim.x)
    w[2 * sl::kScalars + t] = f | static_cast<unsigned>(I[t]);
}

}  // namespace fbrow
}  // namespace scn
