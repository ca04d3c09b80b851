// SPDX-License-Identifier: MIT
// TEST INFRASTRUCTURE ONLY — dense kernels of the CPU parity oracle.
// Stand-ins for the Eigen calls the reference makes (SURVEY §8c "third-party
// boundary"): GEMV (tree_oracles.hpp:48-50,60-61,68-70,80,84), GEMM/LLT/
// SelfAdjointEigenSolver (riccati.hpp:132-154,170,174), EigenSolver for the
// generator's spectral radius (generators.hpp:281-283).
#include <algorithm>
#include <cmath>
#include <limits>

#include "oracle_core.hpp"

namespace orc {

void gemv(const Mat& A, const double* x, double* y, bool accumulate) {
  if (!accumulate) std::fill(y, y + A.r, 0.0);
  for (int j = 0; j < A.c; ++j) {
    const double xj = x[j];
    const double* a = A.col(j);
    for (int i = 0; i < A.r; ++i) y[i] += a[i] * xj;
  }
}

void gemv_t(const Mat& A, const double* x, double* y, bool accumulate) {
  for (int j = 0; j < A.c; ++j) {
    const double* a = A.col(j);
    double s = 0.0;
    for (int i = 0; i < A.r; ++i) s += a[i] * x[i];
    y[j] = accumulate ? y[j] + s : s;
  }
}

Mat matmul(const Mat& A, const Mat& B) {
  Mat C(A.r, B.c);
  for (int j = 0; j < B.c; ++j)
    for (int k = 0; k < A.c; ++k) {
      const double b = B(k, j);
      const double* a = A.col(k);
      double* c = C.col(j);
      for (int i = 0; i < A.r; ++i) c[i] += a[i] * b;
    }
  return C;
}

Mat matmul_tn(const Mat& A, const Mat& B) {
  Mat C(A.c, B.c);
  for (int j = 0; j < B.c; ++j)
    for (int i = 0; i < A.c; ++i) C(i, j) = dot(A.col(i), B.col(j), static_cast<size_t>(A.r));
  return C;
}

Mat matmul_nt(const Mat& A, const Mat& B) {
  Mat C(A.r, B.r);
  for (int k = 0; k < A.c; ++k)
    for (int j = 0; j < B.r; ++j) {
      const double b = B(j, k);
      const double* a = A.col(k);
      double* c = C.col(j);
      for (int i = 0; i < A.r; ++i) c[i] += a[i] * b;
    }
  return C;
}

Mat transpose(const Mat& A) {
  Mat T(A.c, A.r);
  for (int j = 0; j < A.c; ++j)
    for (int i = 0; i < A.r; ++i) T(j, i) = A(i, j);
  return T;
}

double dot(const double* a, const double* b, size_t n) {
  double s = 0.0;
  for (size_t i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}
double dot(const Vec& a, const Vec& b) { return dot(a.data(), b.data(), a.size()); }
double sqnorm(const Vec& a) { return dot(a, a); }
double inf_norm(const Vec& a) {
  double m = 0.0;
  for (double v : a) m = std::max(m, std::abs(v));
  return m;
}

Llt::Llt(const Mat& A) : L(A.r, A.c) {
  const int n = A.r;
  for (int j = 0; j < n; ++j) {
    double s = A(j, j);
    for (int k = 0; k < j; ++k) s -= L(j, k) * L(j, k);
    const double d = std::sqrt(s);
    L(j, j) = d;
    for (int i = j + 1; i < n; ++i) {
      double t = A(i, j);
      for (int k = 0; k < j; ++k) t -= L(i, k) * L(j, k);
      L(i, j) = t / d;
    }
  }
}

Vec Llt::solve(const Vec& b) const {
  const int n = L.r;
  Vec x(b);
  for (int i = 0; i < n; ++i) {
    double s = x[static_cast<size_t>(i)];
    for (int k = 0; k < i; ++k) s -= L(i, k) * x[static_cast<size_t>(k)];
    x[static_cast<size_t>(i)] = s / L(i, i);
  }
  for (int i = n - 1; i >= 0; --i) {
    double s = x[static_cast<size_t>(i)];
    for (int k = i + 1; k < n; ++k) s -= L(k, i) * x[static_cast<size_t>(k)];
    x[static_cast<size_t>(i)] = s / L(i, i);
  }
  return x;
}

Mat Llt::solve(const Mat& B) const {
  Mat X(B.r, B.c);
  for (int j = 0; j < B.c; ++j) {
    const Vec col(B.col(j), B.col(j) + B.r);
    const Vec s = solve(col);
    std::copy(s.begin(), s.end(), X.col(j));
  }
  return X;
}

// Cyclic Jacobi eigenvalues of a symmetric matrix.
static std::vector<double> sym_eigs(const Mat& S) {
  const int n = S.r;
  Mat a = S;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i) {
        tot += a(i, j) * a(i, j);
        if (i != j) off += a(i, j) * a(i, j);
      }
    if (off <= 1e-32 * tot || off == 0.0) break;
    for (int p = 0; p < n; ++p)
      for (int q = p + 1; q < n; ++q) {
        const double apq = a(p, q);
        if (apq == 0.0) continue;
        const double theta = (a(q, q) - a(p, p)) / (2.0 * apq);
        const double t = (theta >= 0 ? 1.0 : -1.0) /
                         (std::abs(theta) + std::sqrt(theta * theta + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < n; ++k) {
          const double akp = a(k, p), akq = a(k, q);
          a(k, p) = c * akp - s * akq;
          a(k, q) = s * akp + c * akq;
        }
        for (int k = 0; k < n; ++k) {
          const double apk = a(p, k), aqk = a(q, k);
          a(p, k) = c * apk - s * aqk;
          a(q, k) = s * apk + c * aqk;
        }
      }
  }
  std::vector<double> ev(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) ev[static_cast<size_t>(i)] = a(i, i);
  return ev;
}
double sym_min_eig(const Mat& S) {
  const auto ev = sym_eigs(S);
  return *std::min_element(ev.begin(), ev.end());
}
double sym_max_eig(const Mat& S) {
  const auto ev = sym_eigs(S);
  return *std::max_element(ev.begin(), ev.end());
}

// Spectral radius through Householder Hessenberg reduction and the Francis
// double-shift QR iteration (real Schur form), as Eigen::EigenSolver does.
double spectral_radius(const Mat& A0) {
  const int n = A0.r;
  if (n == 1) return std::abs(A0(0, 0));
  Mat a = A0;
  // Householder reduction to upper Hessenberg form.
  std::vector<double> v(static_cast<size_t>(n));
  for (int k = 0; k < n - 2; ++k) {
    double alpha = 0.0;
    for (int i = k + 1; i < n; ++i) alpha += a(i, k) * a(i, k);
    alpha = std::sqrt(alpha);
    if (alpha == 0.0) continue;
    if (a(k + 1, k) > 0) alpha = -alpha;
    double vnorm2 = 0.0;
    for (int i = k + 1; i < n; ++i) {
      v[static_cast<size_t>(i)] = a(i, k);
      if (i == k + 1) v[static_cast<size_t>(i)] -= alpha;
      vnorm2 += v[static_cast<size_t>(i)] * v[static_cast<size_t>(i)];
    }
    if (vnorm2 == 0.0) continue;
    for (int j = 0; j < n; ++j) {  // a = (I - 2vv'/v'v) a
      double s = 0.0;
      for (int i = k + 1; i < n; ++i) s += v[static_cast<size_t>(i)] * a(i, j);
      s = 2.0 * s / vnorm2;
      for (int i = k + 1; i < n; ++i) a(i, j) -= s * v[static_cast<size_t>(i)];
    }
    for (int i = 0; i < n; ++i) {  // a = a (I - 2vv'/v'v)
      double s = 0.0;
      for (int j = k + 1; j < n; ++j) s += a(i, j) * v[static_cast<size_t>(j)];
      s = 2.0 * s / vnorm2;
      for (int j = k + 1; j < n; ++j) a(i, j) -= s * v[static_cast<size_t>(j)];
    }
    for (int i = k + 2; i < n; ++i) a(i, k) = 0.0;
  }
  // Francis QR on the Hessenberg matrix (EISPACK/NR hqr structure).
  std::vector<double> wr(static_cast<size_t>(n), 0.0), wi(static_cast<size_t>(n), 0.0);
  const double EPS = std::numeric_limits<double>::epsilon();
  double anorm = 0.0;
  for (int i = 0; i < n; ++i)
    for (int j = std::max(i - 1, 0); j < n; ++j) anorm += std::abs(a(i, j));
  int nn = n - 1;
  double t = 0.0;
  auto sgn = [](double mag, double s) { return s >= 0 ? std::abs(mag) : -std::abs(mag); };
  while (nn >= 0) {
    int its = 0, l = 0;
    do {
      for (l = nn; l > 0; --l) {
        double s = std::abs(a(l - 1, l - 1)) + std::abs(a(l, l));
        if (s == 0.0) s = anorm;
        if (std::abs(a(l, l - 1)) <= EPS * s) {
          a(l, l - 1) = 0.0;
          break;
        }
      }
      double x = a(nn, nn);
      if (l == nn) {
        wr[static_cast<size_t>(nn)] = x + t;
        wi[static_cast<size_t>(nn)] = 0.0;
        --nn;
      } else {
        double y = a(nn - 1, nn - 1);
        double w = a(nn, nn - 1) * a(nn - 1, nn);
        if (l == nn - 1) {
          const double p = 0.5 * (y - x);
          const double q = p * p + w;
          double z = std::sqrt(std::abs(q));
          x += t;
          if (q >= 0.0) {
            z = p + sgn(z, p);
            wr[static_cast<size_t>(nn - 1)] = wr[static_cast<size_t>(nn)] = x + z;
            if (z != 0.0) wr[static_cast<size_t>(nn)] = x - w / z;
            wi[static_cast<size_t>(nn - 1)] = wi[static_cast<size_t>(nn)] = 0.0;
          } else {
            wr[static_cast<size_t>(nn)] = wr[static_cast<size_t>(nn - 1)] = x + p;
            wi[static_cast<size_t>(nn)] = -z;
            wi[static_cast<size_t>(nn - 1)] = z;
          }
          nn -= 2;
        } else {
          // LAPACK dlahqr budget: 30 max(10, n) sweeps per block, exceptional
          // shift every 10 (identical to the classic 10/20 shifts for every
          // block that converges within 30 sweeps)
          if (its == 30 * std::max(10, n)) ORC_THROW(kError, "spectral_radius: QR iteration did not converge");
          if (its > 0 && its % 10 == 0) {
            t += x;
            for (int i = 0; i < nn + 1; ++i) a(i, i) -= x;
            const double s = std::abs(a(nn, nn - 1)) + std::abs(a(nn - 1, nn - 2));
            y = x = 0.75 * s;
            w = -0.4375 * s * s;
          }
          ++its;
          int m;
          double p = 0, q = 0, r = 0, z = 0;
          for (m = nn - 2; m >= l; --m) {
            z = a(m, m);
            r = x - z;
            double s = y - z;
            p = (r * s - w) / a(m + 1, m) + a(m, m + 1);
            q = a(m + 1, m + 1) - z - r - s;
            r = a(m + 2, m + 1);
            s = std::abs(p) + std::abs(q) + std::abs(r);
            p /= s;
            q /= s;
            r /= s;
            if (m == l) break;
            const double u = std::abs(a(m, m - 1)) * (std::abs(q) + std::abs(r));
            const double v = std::abs(p) * (std::abs(a(m - 1, m - 1)) + std::abs(z) +
                                            std::abs(a(m + 1, m + 1)));
            if (u <= EPS * v) break;
          }
          for (int i = m; i < nn - 1; ++i) {
            a(i + 2, i) = 0.0;
            if (i != m) a(i + 2, i - 1) = 0.0;
          }
          for (int k = m; k < nn; ++k) {
            if (k != m) {
              p = a(k, k - 1);
              q = a(k + 1, k - 1);
              r = 0.0;
              if (k + 1 != nn) r = a(k + 2, k - 1);
              if ((x = std::abs(p) + std::abs(q) + std::abs(r)) != 0.0) {
                p /= x;
                q /= x;
                r /= x;
              }
            }
            const double s = sgn(std::sqrt(p * p + q * q + r * r), p);
            if (s != 0.0) {
              if (k == m) {
                if (l != m) a(k, k - 1) = -a(k, k - 1);
              } else {
                a(k, k - 1) = -s * x;
              }
              p += s;
              x = p / s;
              y = q / s;
              z = r / s;
              q /= p;
              r /= p;
              for (int j = k; j < nn + 1; ++j) {
                p = a(k, j) + q * a(k + 1, j);
                if (k + 1 != nn) {
                  p += r * a(k + 2, j);
                  a(k + 2, j) -= p * z;
                }
                a(k + 1, j) -= p * y;
                a(k, j) -= p * x;
              }
              const int mmin = nn < k + 3 ? nn : k + 3;
              for (int i = l; i < mmin + 1; ++i) {
                p = x * a(i, k) + y * a(i, k + 1);
                if (k + 1 != nn) {
                  p += z * a(i, k + 2);
                  a(i, k + 2) -= p * r;
                }
                a(i, k + 1) -= p * q;
                a(i, k) -= p;
              }
            }
          }
        }
      }
    } while (l + 1 < nn);
  }
  double rad = 0.0;
  for (int i = 0; i < n; ++i)
    rad = std::max(rad, std::hypot(wr[static_cast<size_t>(i)], wi[static_cast<size_t>(i)]));
  return rad;
}

}  // namespace orc
