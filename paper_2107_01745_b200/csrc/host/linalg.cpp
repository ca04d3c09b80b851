// SPDX-License-Identifier: MIT
// Small dense kernels for the host setup path (factor + generator + checks).
#include <algorithm>
#include <cmath>
#include <limits>
#include <vector>

#include "model.hpp"

namespace scn {

bool cholesky(std::vector<double>& a, int n) {
  for (int j = 0; j < n; ++j) {
    double d = a[j + j * n];
    for (int k = 0; k < j; ++k) d -= a[j + k * n] * a[j + k * n];
    if (!(d > 0.0)) return false;
    d = std::sqrt(d);
    a[j + j * n] = d;
    for (int i = j + 1; i < n; ++i) {
      double s = a[i + j * n];
      for (int k = 0; k < j; ++k) s -= a[i + k * n] * a[j + k * n];
      a[i + j * n] = s / d;
    }
    for (int i = 0; i < j; ++i) a[i + j * n] = 0.0;
  }
  return true;
}

void chol_solve(const std::vector<double>& Lm, int n, double* B, int k) {
  for (int c = 0; c < k; ++c) {
    double* b = B + static_cast<size_t>(c) * n;
    for (int i = 0; i < n; ++i) {
      double s = b[i];
      for (int t = 0; t < i; ++t) s -= Lm[i + t * n] * b[t];
      b[i] = s / Lm[i + i * n];
    }
    for (int i = n - 1; i >= 0; --i) {
      double s = b[i];
      for (int t = i + 1; t < n; ++t) s -= Lm[t + i * n] * b[t];
      b[i] = s / Lm[i + i * n];
    }
  }
}

// Two-sided cyclic Jacobi; the eigenvalues are the converged diagonal.
double sym_min_eig(const double* S, int n) {
  std::vector<double> a(S, S + static_cast<size_t>(n) * n);
  auto at = [&a, n](int i, int j) -> double& { return a[i + static_cast<size_t>(j) * n]; };
  for (int sweep = 0; sweep < 64; ++sweep) {
    double off = 0.0, diag = 0.0;
    for (int j = 0; j < n; ++j) {
      diag += at(j, j) * at(j, j);
      for (int i = j + 1; i < n; ++i) off += 2.0 * at(i, j) * at(i, j);
    }
    if (off == 0.0 || off <= 1e-30 * (diag + off)) break;
    for (int pp = 0; pp < n - 1; ++pp)
      for (int qq = pp + 1; qq < n; ++qq) {
        const double apq = at(pp, qq);
        if (apq == 0.0) continue;
        const double tau = (at(qq, qq) - at(pp, pp)) / (2.0 * apq);
        const double t = std::copysign(1.0, tau) / (std::fabs(tau) + std::sqrt(1.0 + tau * tau));
        const double cs = 1.0 / std::sqrt(1.0 + t * t), sn = t * cs;
        for (int k = 0; k < n; ++k) {
          const double x = at(k, pp), y = at(k, qq);
          at(k, pp) = cs * x - sn * y;
          at(k, qq) = sn * x + cs * y;
        }
        for (int k = 0; k < n; ++k) {
          const double x = at(pp, k), y = at(qq, k);
          at(pp, k) = cs * x - sn * y;
          at(qq, k) = sn * x + cs * y;
        }
      }
  }
  double mn = std::numeric_limits<double>::infinity();
  for (int i = 0; i < n; ++i) mn = std::min(mn, at(i, i));
  return mn;
}

// max |lambda| of a general real matrix: Householder Hessenberg form, then
// implicit double-shift Francis QR with deflation (real Schur form).
double spectral_radius(const double* A0, int n) {
  if (n == 1) return std::fabs(A0[0]);
  std::vector<double> h(A0, A0 + static_cast<size_t>(n) * n);
  auto H = [&h, n](int i, int j) -> double& { return h[i + static_cast<size_t>(j) * n]; };
  std::vector<double> v(static_cast<size_t>(n));
  for (int k = 0; k + 2 < n; ++k) {
    double norm = 0.0;
    for (int i = k + 1; i < n; ++i) norm += H(i, k) * H(i, k);
    norm = std::sqrt(norm);
    if (norm == 0.0) continue;
    const double alpha = H(k + 1, k) > 0 ? -norm : norm;
    double vv = 0.0;
    for (int i = k + 1; i < n; ++i) {
      v[i] = H(i, k) - (i == k + 1 ? alpha : 0.0);
      vv += v[i] * v[i];
    }
    if (vv == 0.0) continue;
    const double beta = 2.0 / vv;
    for (int j = 0; j < n; ++j) {
      double s = 0.0;
      for (int i = k + 1; i < n; ++i) s += v[i] * H(i, j);
      s *= beta;
      for (int i = k + 1; i < n; ++i) H(i, j) -= s * v[i];
    }
    for (int i = 0; i < n; ++i) {
      double s = 0.0;
      for (int j = k + 1; j < n; ++j) s += H(i, j) * v[j];
      s *= beta;
      for (int j = k + 1; j < n; ++j) H(i, j) -= s * v[j];
    }
    for (int i = k + 2; i < n; ++i) H(i, k) = 0.0;
  }
  const double eps = std::numeric_limits<double>::epsilon();
  double norm1 = 0.0;
  for (int i = 0; i < n; ++i)
    for (int j = std::max(i - 1, 0); j < n; ++j) norm1 += std::fabs(H(i, j));
  double radius = 0.0;
  int hi = n - 1;
  double shift_acc = 0.0;
  int iter = 0;
  while (hi >= 0) {
    int lo = hi;
    for (; lo > 0; --lo) {
      double s = std::fabs(H(lo - 1, lo - 1)) + std::fabs(H(lo, lo));
      if (s == 0.0) s = norm1;
      if (std::fabs(H(lo, lo - 1)) <= eps * s) {
        H(lo, lo - 1) = 0.0;
        break;
      }
    }
    double x = H(hi, hi);
    if (lo == hi) {  // 1x1 block
      radius = std::max(radius, std::fabs(x + shift_acc));
      --hi;
      iter = 0;
      continue;
    }
    double y = H(hi - 1, hi - 1);
    double w = H(hi, hi - 1) * H(hi - 1, hi);
    if (lo == hi - 1) {  // 2x2 block
      const double pp = 0.5 * (y - x), qq = pp * pp + w;
      const double z = std::sqrt(std::fabs(qq));
      const double xs = x + shift_acc;
      if (qq >= 0.0) {
        const double zz = pp + std::copysign(z, pp);
        const double e1 = xs + zz;
        const double e2 = zz != 0.0 ? xs - w / zz : e1;
        radius = std::max(radius, std::max(std::fabs(e1), std::fabs(e2)));
      } else {
        radius = std::max(radius, std::hypot(xs + pp, z));
      }
      hi -= 2;
      iter = 0;
      continue;
    }
    // LAPACK dlahqr budget: 30 max(10, n) sweeps per block, exceptional shift
    // every 10 (the classic 10/20 shifts for every block converging within 30)
    if (iter == 30 * std::max(10, n)) fail(SCENOPT_E_ERROR, "spectral_radius: QR iteration did not converge");
    if (iter > 0 && iter % 10 == 0) {  // exceptional shift
      shift_acc += x;
      for (int i = 0; i <= hi; ++i) H(i, i) -= x;
      const double s = std::fabs(H(hi, hi - 1)) + std::fabs(H(hi - 1, hi - 2));
      x = y = 0.75 * s;
      w = -0.4375 * s * s;
    }
    ++iter;
    int m = hi - 2;
    double p = 0, q = 0, r = 0;
    for (; m >= lo; --m) {
      const double z = H(m, m);
      const double rr = x - z, ss = y - z;
      p = (rr * ss - w) / H(m + 1, m) + H(m, m + 1);
      q = H(m + 1, m + 1) - z - rr - ss;
      r = H(m + 2, m + 1);
      const double s = std::fabs(p) + std::fabs(q) + std::fabs(r);
      p /= s;
      q /= s;
      r /= s;
      if (m == lo) break;
      const double u = std::fabs(H(m, m - 1)) * (std::fabs(q) + std::fabs(r));
      const double vv = std::fabs(p) * (std::fabs(H(m - 1, m - 1)) + std::fabs(z) + std::fabs(H(m + 1, m + 1)));
      if (u <= eps * vv) break;
    }
    for (int i = m + 2; i <= hi; ++i) {
      H(i, i - 2) = 0.0;
      if (i != m + 2) H(i, i - 3) = 0.0;
    }
    for (int k = m; k < hi; ++k) {
      double scale = 0.0;
      if (k != m) {
        p = H(k, k - 1);
        q = H(k + 1, k - 1);
        r = (k + 1 != hi) ? H(k + 2, k - 1) : 0.0;
        scale = std::fabs(p) + std::fabs(q) + std::fabs(r);
        if (scale != 0.0) {
          p /= scale;
          q /= scale;
          r /= scale;
        }
      }
      const double s = std::copysign(std::sqrt(p * p + q * q + r * r), p);
      if (s == 0.0) continue;
      if (k == m) {
        if (lo != m) H(k, k - 1) = -H(k, k - 1);
      } else {
        H(k, k - 1) = -s * scale;
      }
      p += s;
      const double xk = p / s, yk = q / s, zk = r / s;
      q /= p;
      r /= p;
      for (int j = k; j <= hi; ++j) {
        double t = H(k, j) + q * H(k + 1, j);
        if (k + 1 != hi) {
          t += r * H(k + 2, j);
          H(k + 2, j) -= t * zk;
        }
        H(k + 1, j) -= t * yk;
        H(k, j) -= t * xk;
      }
      const int top = std::min(hi, k + 3);
      for (int i = lo; i <= top; ++i) {
        double t = xk * H(i, k) + yk * H(i, k + 1);
        if (k + 1 != hi) {
          t += zk * H(i, k + 2);
          H(i, k + 2) -= t * r;
        }
        H(i, k + 1) -= t * q;
        H(i, k) -= t;
      }
    }
  }
  return radius;
}

}  // namespace scn

namespace scn {
namespace {
using Dm = std::vector<double>;
Dm mm(const Dm& A, const Dm& B, int n) {
  Dm C(static_cast<size_t>(n) * n, 0.0);
  for (int j = 0; j < n; ++j)
    for (int k = 0; k < n; ++k) {
      const double b = B[k + static_cast<size_t>(j) * n];
      if (b == 0.0) continue;
      for (int i = 0; i < n; ++i) C[i + static_cast<size_t>(j) * n] += A[i + static_cast<size_t>(k) * n] * b;
    }
  return C;
}
// X = P^{-1} Q by LU with partial pivoting (P overwritten)
Dm lu_solve(Dm P, Dm Q, int n) {
  for (int k = 0; k < n; ++k) {
    int piv = k;
    for (int i = k + 1; i < n; ++i)
      if (std::fabs(P[i + static_cast<size_t>(k) * n]) > std::fabs(P[piv + static_cast<size_t>(k) * n])) piv = i;
    if (piv != k) {
      for (int j = 0; j < n; ++j) std::swap(P[k + static_cast<size_t>(j) * n], P[piv + static_cast<size_t>(j) * n]);
      for (int j = 0; j < n; ++j) std::swap(Q[k + static_cast<size_t>(j) * n], Q[piv + static_cast<size_t>(j) * n]);
    }
    const double d = P[k + static_cast<size_t>(k) * n];
    for (int i = k + 1; i < n; ++i) {
      const double l = P[i + static_cast<size_t>(k) * n] / d;
      if (l == 0.0) continue;
      for (int j = k; j < n; ++j) P[i + static_cast<size_t>(j) * n] -= l * P[k + static_cast<size_t>(j) * n];
      for (int j = 0; j < n; ++j) Q[i + static_cast<size_t>(j) * n] -= l * Q[k + static_cast<size_t>(j) * n];
    }
  }
  for (int j = 0; j < n; ++j)
    for (int i = n - 1; i >= 0; --i) {
      double s = Q[i + static_cast<size_t>(j) * n];
      for (int k = i + 1; k < n; ++k) s -= P[i + static_cast<size_t>(k) * n] * Q[k + static_cast<size_t>(j) * n];
      Q[i + static_cast<size_t>(j) * n] = s / P[i + static_cast<size_t>(i) * n];
    }
  return Q;
}
}  // namespace

// Matrix exponential by scaling and squaring with the [m/m] Pade approximant,
// m in {3, 5, 7, 9, 13} chosen by the 1-norm (Higham 2005, the method behind
// Eigen's MatrixBase::exp() that generators.hpp:108 calls).
std::vector<double> expm(const std::vector<double>& A0, int n) {
  static const double th[5] = {1.495585217958292e-2, 2.539398330063230e-1, 9.504178996162932e-1,
                               2.097847961257068e0, 5.371920351148152e0};
  static const double b3[4] = {120., 60., 12., 1.};
  static const double b5[6] = {30240., 15120., 3360., 420., 30., 1.};
  static const double b7[8] = {17297280., 8648640., 1995840., 277200., 25200., 1512., 56., 1.};
  static const double b9[10] = {17643225600., 8821612800., 2075673600., 302702400., 30270240.,
                                2162160.,     110880.,     3960.,       90.,         1.};
  static const double b13[14] = {64764752532480000., 32382376266240000., 7771770303897600., 1187353796428800.,
                                 129060195264000.,   10559470521600.,    670442572800.,    33522128640.,
                                 1323241920.,        40840800.,          960960.,          16380.,
                                 182.,               1.};
  const size_t nn = static_cast<size_t>(n) * n;
  double norm1 = 0.0;
  for (int j = 0; j < n; ++j) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += std::fabs(A0[i + static_cast<size_t>(j) * n]);
    norm1 = std::max(norm1, s);
  }
  Dm I(nn, 0.0);
  for (int i = 0; i < n; ++i) I[i + static_cast<size_t>(i) * n] = 1.0;
  auto pade = [&](const Dm& A, const double* b, int m, Dm& U, Dm& V) {  // m in {3,5,7,9}
    const Dm A2 = mm(A, A, n);
    Dm pw = I, Uo(nn, 0.0);
    V.assign(nn, 0.0);
    for (int k = 0; k <= m; k += 2) {  // even powers A^k: V += b_k A^k, Uo += b_{k+1} A^k
      for (size_t t = 0; t < nn; ++t) {
        V[t] += b[k] * pw[t];
        Uo[t] += b[k + 1] * pw[t];
      }
      if (k + 2 <= m) pw = mm(pw, A2, n);
    }
    U = mm(A, Uo, n);
  };
  int s = 0;
  Dm A = A0, U, V;
  if (norm1 <= th[0]) pade(A, b3, 3, U, V);
  else if (norm1 <= th[1]) pade(A, b5, 5, U, V);
  else if (norm1 <= th[2]) pade(A, b7, 7, U, V);
  else if (norm1 <= th[3]) pade(A, b9, 9, U, V);
  else {
    if (norm1 > th[4]) s = std::max(0, static_cast<int>(std::ceil(std::log2(norm1 / th[4]))));
    const double sc = std::ldexp(1.0, -s);
    for (double& v : A) v *= sc;
    const Dm A2 = mm(A, A, n), A4 = mm(A2, A2, n), A6 = mm(A4, A2, n);
    Dm t1(nn), t2(nn), t3(nn), t4(nn);
    for (size_t t = 0; t < nn; ++t) {
      t1[t] = b13[13] * A6[t] + b13[11] * A4[t] + b13[9] * A2[t];
      t2[t] = b13[7] * A6[t] + b13[5] * A4[t] + b13[3] * A2[t] + b13[1] * I[t];
      t3[t] = b13[12] * A6[t] + b13[10] * A4[t] + b13[8] * A2[t];
      t4[t] = b13[6] * A6[t] + b13[4] * A4[t] + b13[2] * A2[t] + b13[0] * I[t];
    }
    Dm inner = mm(A6, t1, n);
    for (size_t t = 0; t < nn; ++t) inner[t] += t2[t];
    U = mm(A, inner, n);
    V = mm(A6, t3, n);
    for (size_t t = 0; t < nn; ++t) V[t] += t4[t];
  }
  Dm P(nn), Q(nn);
  for (size_t t = 0; t < nn; ++t) {
    P[t] = V[t] - U[t];
    Q[t] = V[t] + U[t];
  }
  Dm X = lu_solve(std::move(P), std::move(Q), n);
  for (int k = 0; k < s; ++k) X = mm(X, X, n);
  return X;
}

}  // namespace scn
