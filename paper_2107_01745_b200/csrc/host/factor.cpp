// SPDX-License-Identifier: MIT
// Offline Riccati factorization (riccati.hpp:82-216) on the host worker pool.
//
// Nodes of one stage are independent given the stage below, so each stage
// is a parallel_for over its nodes (the reference loops serially,
// riccati.hpp:115-180). The arithmetic per node follows the reference
// exactly: accumulate the eliminated-input Hessian, check its smallest
// eigenvalue, Cholesky-solve for the gain and affine terms, build the child
// blocks and the symmetrized value matrix.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>

#include "model.hpp"

namespace scn {

namespace {
// C = A^T B  : A is r x m, B is r x k -> C m x k
void gemm_tn(const double* A, const double* B, int r, int m, int k, double* C, bool acc) {
  for (int j = 0; j < k; ++j)
    for (int i = 0; i < m; ++i) {
      const double* a = A + static_cast<size_t>(i) * r;
      const double* b = B + static_cast<size_t>(j) * r;
      double s = 0.0;
      for (int t = 0; t < r; ++t) s += a[t] * b[t];
      C[i + static_cast<size_t>(j) * m] = acc ? C[i + static_cast<size_t>(j) * m] + s : s;
    }
}
// C = A B : A m x r, B r x k -> C m x k
void gemm_nn(const double* A, const double* B, int m, int r, int k, double* C) {
  std::fill(C, C + static_cast<size_t>(m) * k, 0.0);
  for (int j = 0; j < k; ++j)
    for (int t = 0; t < r; ++t) {
      const double bt = B[t + static_cast<size_t>(j) * r];
      const double* a = A + static_cast<size_t>(t) * m;
      double* c = C + static_cast<size_t>(j) * m;
      for (int i = 0; i < m; ++i) c[i] += a[i] * bt;
    }
}
}  // namespace

void check_factor_shape(const Factor& f, const Problem& p, const char* who) {
  // riccati.hpp:67-74
  if (f.n != p.n || f.nx != p.nx || f.nu != p.nu || f.dual_dim != p.dual_dim ||
      f.first_leaf != p.first_leaf)
    fail(SCENOPT_E_CACHE_MISMATCH, std::string(who) + ": cache was built for a different problem shape");
}

Factor factor_shape(const Problem& p, bool lite) {
  require_valid(p);
  const int nx = p.nx, nu = p.nu, n = p.n, Fn = p.first_leaf;
  Factor f;
  f.nx = nx;
  f.nu = nu;
  f.n = n;
  f.first_leaf = Fn;
  f.dual_dim = p.dual_dim;
  f.L = p.L;
  f.stage_total = p.stage_total;
  f.child_dual_offset.assign(static_cast<size_t>(Fn), 0);
  f.child_dual_rows.assign(static_cast<size_t>(Fn), 0);
  for (int i = 0; i < Fn; ++i) {
    const int cb = p.child_begin[i], cc = p.child_count[i];
    int rows = 0;
    for (int c = cb; c < cb + cc; ++c) rows += p.stage_rows[c];
    f.child_dual_rows[i] = rows;
    f.child_dual_offset[i] = p.dual_offset[cb];
  }
  if (lite) return f;  // dimensions and child offsets only (device factor layout)
  f.gain.assign(static_cast<size_t>(Fn) * p.sxu(), 0.0);
  f.dual_to_input.assign(static_cast<size_t>(p.stage_total) * nu, 0.0);
  f.dual_to_costate.assign(static_cast<size_t>(p.stage_total) * nx, 0.0);
  f.input_affine.assign(static_cast<size_t>(Fn) * nu, 0.0);
  f.costate_affine.assign(static_cast<size_t>(Fn) * nx, 0.0);
  f.child_to_input.assign(static_cast<size_t>(n) * p.sxu(), 0.0);
  f.closed_loop.assign(static_cast<size_t>(n) * p.sxx(), 0.0);
  f.value_quad.assign(static_cast<size_t>(n) * p.sxx(), 0.0);
  f.leaf_costate_affine.assign(static_cast<size_t>(p.L) * nx, 0.0);
  return f;
}

Factor factor(const Problem& p) {
  require_full(p, "factor");
  require_valid(p);
  const int nx = p.nx, nu = p.nu, n = p.n, Fn = p.first_leaf;
  const size_t sxx = p.sxx(), sxu = p.sxu(), suu = p.suu();
  Factor f;
  f.nx = nx;
  f.nu = nu;
  f.n = n;
  f.first_leaf = Fn;
  f.dual_dim = p.dual_dim;
  f.L = p.L;
  f.stage_total = p.stage_total;
  f.child_dual_offset.assign(static_cast<size_t>(Fn), 0);
  f.child_dual_rows.assign(static_cast<size_t>(Fn), 0);
  f.gain.assign(static_cast<size_t>(Fn) * sxu, 0.0);
  f.dual_to_input.assign(static_cast<size_t>(p.stage_total) * nu, 0.0);
  f.dual_to_costate.assign(static_cast<size_t>(p.stage_total) * nx, 0.0);
  f.input_affine.assign(static_cast<size_t>(Fn) * nu, 0.0);
  f.costate_affine.assign(static_cast<size_t>(Fn) * nx, 0.0);
  f.input_hessian.assign(static_cast<size_t>(Fn) * suu, 0.0);
  f.child_to_input.assign(static_cast<size_t>(n) * sxu, 0.0);
  f.closed_loop.assign(static_cast<size_t>(n) * sxx, 0.0);
  f.value_quad.assign(static_cast<size_t>(n) * sxx, 0.0);
  f.leaf_costate_affine.assign(static_cast<size_t>(p.L) * nx, 0.0);

  // riccati.hpp:106-113
  for (int l = 0; l < p.L; ++l) {
    const int i = Fn + l;
    const double pi = p.probability[i];
    const double* P = p.Pl(l);
    double* V = f.value_quad.data() + i * sxx;
    for (size_t k = 0; k < sxx; ++k) V[k] = pi * P[k];
    for (int k = 0; k < nx; ++k) f.leaf_costate_affine[static_cast<size_t>(l) * nx + k] = pi * p.pl(l)[k];
  }

  for (int t = p.N - 1; t >= 0; --t) {
    const int first = p.stage_offsets[t], past = p.stage_offsets[t + 1];
    std::vector<std::string> errors(static_cast<size_t>(past - first));
    parallel_for(past - first, 4, [&](int b, int e) {
      std::vector<double> huu(suu), hux(sxu), hxx(sxx), su(nu), sx(nx), PB(sxu), PA(sxx), pc2(nx),
          llt(suu), tmp(std::max(sxu, suu));
      for (int k = b; k < e; ++k) {
        const int i = first + k;
        std::fill(huu.begin(), huu.end(), 0.0);
        std::fill(hux.begin(), hux.end(), 0.0);
        std::fill(hxx.begin(), hxx.end(), 0.0);
        std::fill(su.begin(), su.end(), 0.0);
        std::fill(sx.begin(), sx.end(), 0.0);
        const int cb = p.child_begin[i], cc = p.child_count[i];
        int mrows = 0;
        // riccati.hpp:127-141
        for (int c = cb; c < cb + cc; ++c) {
          const double pc = p.probability[c];
          const double* A = p.Ai(c);
          const double* B = p.Bi(c);
          const double* V = f.value_quad.data() + c * sxx;
          gemm_nn(V, B, nx, nx, nu, PB.data());
          gemm_nn(V, A, nx, nx, nx, PA.data());
          const double* R = p.Ri(c);
          const double* S = p.Si(c);
          const double* Q = p.Qi(c);
          gemm_tn(B, PB.data(), nx, nu, nu, tmp.data(), false);
          for (size_t z = 0; z < suu; ++z) huu[z] += pc * R[z] + tmp[z];
          gemm_tn(B, PA.data(), nx, nu, nx, tmp.data(), false);
          for (size_t z = 0; z < sxu; ++z) hux[z] += pc * S[z] + tmp[z];
          for (int j = 0; j < nx; ++j)
            for (int ii = 0; ii < nx; ++ii) {
              const double* a = A + static_cast<size_t>(ii) * nx;
              const double* pa = PA.data() + static_cast<size_t>(j) * nx;
              double s = 0.0;
              for (int z = 0; z < nx; ++z) s += a[z] * pa[z];
              hxx[ii + static_cast<size_t>(j) * nx] += pc * Q[ii + static_cast<size_t>(j) * nx] + s;
            }
          const double* cv = p.ci(c);
          for (int ii = 0; ii < nx; ++ii) {
            double s = 0.0;
            for (int z = 0; z < nx; ++z) s += V[ii + static_cast<size_t>(z) * nx] * cv[z];
            pc2[ii] = 2.0 * s;
          }
          const double* rv = p.ri(c);
          const double* qv = p.qi(c);
          for (int ii = 0; ii < nu; ++ii) {
            double s = 0.0;
            for (int z = 0; z < nx; ++z) s += B[z + static_cast<size_t>(ii) * nx] * pc2[z];
            su[ii] += pc * rv[ii] + s;
          }
          for (int ii = 0; ii < nx; ++ii) {
            double s = 0.0;
            for (int z = 0; z < nx; ++z) s += A[z + static_cast<size_t>(ii) * nx] * pc2[z];
            sx[ii] += pc * qv[ii] + s;
          }
          mrows += p.stage_rows[c];
        }
        // riccati.hpp:142-150
        for (int j = 0; j < nu; ++j)
          for (int ii = j; ii < nu; ++ii) {
            const double s = 0.5 * (huu[ii + j * nu] + huu[j + ii * nu]);
            huu[ii + j * nu] = s;
            huu[j + ii * nu] = s;
          }
        if (sym_min_eig(huu.data(), nu) < 1e-10) {
          errors[static_cast<size_t>(k)] = "factor: eliminated input Hessian at node " +
                                           std::to_string(i) + " has min eigenvalue below 1e-10";
          continue;
        }
        std::copy(huu.begin(), huu.end(), f.input_hessian.begin() + i * suu);
        llt = huu;
        if (!cholesky(llt, nu)) {
          errors[static_cast<size_t>(k)] = "factor: eliminated input Hessian at node " +
                                           std::to_string(i) + " is not positive definite";
          continue;
        }
        // gain = -H^{-1} hux ; input_affine = -1/2 H^{-1} su
        double* K = f.gain.data() + i * sxu;
        std::copy(hux.begin(), hux.end(), K);
        chol_solve(llt, nu, K, nx);
        for (size_t z = 0; z < sxu; ++z) K[z] = -K[z];
        double* ia = f.input_affine.data() + static_cast<size_t>(i) * nu;
        std::copy(su.begin(), su.end(), ia);
        chol_solve(llt, nu, ia, 1);
        for (int z = 0; z < nu; ++z) ia[z] *= -0.5;
        double* ca = f.costate_affine.data() + static_cast<size_t>(i) * nx;
        for (int ii = 0; ii < nx; ++ii) {
          double s = 0.0;
          for (int z = 0; z < nu; ++z) s += K[z + static_cast<size_t>(ii) * nu] * su[z];
          ca[ii] = sx[ii] + s;
        }
        // riccati.hpp:157-175: children blocks
        f.child_dual_rows[i] = mrows;
        const int cdo = p.dual_offset[cb];
        f.child_dual_offset[i] = cdo;
        double* d2i = f.dual_to_input.data() + static_cast<size_t>(cdo) * nu;   // nu x mrows
        double* d2c = f.dual_to_costate.data() + static_cast<size_t>(cdo) * nx;  // nx x mrows
        int col = 0;
        for (int c = cb; c < cb + cc; ++c) {
          const int rows = p.stage_rows[c];
          const double* Fc = p.Fi(c);
          const double* Gc = p.Gi(c);
          for (int rr = 0; rr < rows; ++rr) {
            for (int z = 0; z < nu; ++z) d2i[z + static_cast<size_t>(col + rr) * nu] = Gc[rr + z * rows];
            for (int z = 0; z < nx; ++z) {
              double s = Fc[rr + static_cast<size_t>(z) * rows];
              for (int w = 0; w < nu; ++w) s += Gc[rr + w * rows] * K[w + static_cast<size_t>(z) * nu];
              d2c[z + static_cast<size_t>(col + rr) * nx] = s;
            }
          }
          // child_to_input = -1/2 H^{-1} B_c'
          const double* Bc = p.Bi(c);
          double* c2i = f.child_to_input.data() + c * sxu;  // nu x nx
          for (int z = 0; z < nx; ++z)
            for (int w = 0; w < nu; ++w) c2i[w + static_cast<size_t>(z) * nu] = Bc[z + static_cast<size_t>(w) * nx];
          chol_solve(llt, nu, c2i, nx);
          for (size_t z = 0; z < sxu; ++z) c2i[z] *= -0.5;
          // closed_loop = A_c + B_c K
          const double* Ac = p.Ai(c);
          double* cl = f.closed_loop.data() + c * sxx;
          for (int j = 0; j < nx; ++j)
            for (int ii = 0; ii < nx; ++ii) {
              double s = Ac[ii + static_cast<size_t>(j) * nx];
              for (int w = 0; w < nu; ++w)
                s += Bc[ii + static_cast<size_t>(w) * nx] * K[w + static_cast<size_t>(j) * nu];
              cl[ii + static_cast<size_t>(j) * nx] = s;
            }
          col += rows;
        }
        chol_solve(llt, nu, d2i, mrows);
        for (size_t z = 0; z < static_cast<size_t>(nu) * mrows; ++z) d2i[z] *= -0.5;
        // riccati.hpp:177-178: value = hxx + hux' K, symmetrized
        double* V = f.value_quad.data() + i * sxx;
        for (int j = 0; j < nx; ++j)
          for (int ii = 0; ii < nx; ++ii) {
            double s = hxx[ii + static_cast<size_t>(j) * nx];
            for (int w = 0; w < nu; ++w)
              s += hux[w + static_cast<size_t>(ii) * nu] * K[w + static_cast<size_t>(j) * nu];
            V[ii + static_cast<size_t>(j) * nx] = s;
          }
        for (int j = 0; j < nx; ++j)
          for (int ii = j + 1; ii < nx; ++ii) {
            const double s = 0.5 * (V[ii + static_cast<size_t>(j) * nx] + V[j + static_cast<size_t>(ii) * nx]);
            V[ii + static_cast<size_t>(j) * nx] = s;
            V[j + static_cast<size_t>(ii) * nx] = s;
          }
      }
    });
    for (const auto& e : errors)
      if (!e.empty()) fail(SCENOPT_E_NOT_STRONGLY_CONVEX, e);
  }
  return f;
}

// riccati.hpp:187-216
void refactor_affine(Factor& f, const Problem& p) {
  if (f.n != p.n || f.nx != p.nx || f.nu != p.nu || f.dual_dim != p.dual_dim || f.first_leaf != p.first_leaf)
    fail(SCENOPT_E_SHAPE_CHANGED, "refactor_affine: problem shape changed since factor()");
  const int nx = p.nx, nu = p.nu;
  const size_t sxx = p.sxx(), suu = p.suu();
  for (int l = 0; l < p.L; ++l) {
    const double pi = p.probability[p.first_leaf + l];
    for (int k = 0; k < nx; ++k) f.leaf_costate_affine[static_cast<size_t>(l) * nx + k] = pi * p.pl(l)[k];
  }
  parallel_for(p.first_leaf, 64, [&](int b, int e) {
    std::vector<double> su(nu), sx(nx), pc2(nx), llt(suu);
    for (int i = b; i < e; ++i) {
      std::fill(su.begin(), su.end(), 0.0);
      std::fill(sx.begin(), sx.end(), 0.0);
      for (int c = p.child_begin[i]; c < p.child_begin[i] + p.child_count[i]; ++c) {
        const double pc = p.probability[c];
        const double* V = f.value_quad.data() + c * sxx;
        const double* cv = p.ci(c);
        for (int ii = 0; ii < nx; ++ii) {
          double s = 0.0;
          for (int z = 0; z < nx; ++z) s += V[ii + static_cast<size_t>(z) * nx] * cv[z];
          pc2[ii] = 2.0 * s;
        }
        const double* A = p.Ai(c);
        const double* B = p.Bi(c);
        for (int ii = 0; ii < nu; ++ii) {
          double s = 0.0;
          for (int z = 0; z < nx; ++z) s += B[z + static_cast<size_t>(ii) * nx] * pc2[z];
          su[ii] += pc * p.ri(c)[ii] + s;
        }
        for (int ii = 0; ii < nx; ++ii) {
          double s = 0.0;
          for (int z = 0; z < nx; ++z) s += A[z + static_cast<size_t>(ii) * nx] * pc2[z];
          sx[ii] += pc * p.qi(c)[ii] + s;
        }
      }
      std::copy(f.input_hessian.begin() + i * suu, f.input_hessian.begin() + (i + 1) * suu, llt.begin());
      cholesky(llt, nu);
      double* ia = f.input_affine.data() + static_cast<size_t>(i) * nu;
      std::copy(su.begin(), su.end(), ia);
      chol_solve(llt, nu, ia, 1);
      for (int z = 0; z < nu; ++z) ia[z] *= -0.5;
      const double* K = f.gain.data() + i * p.sxu();
      double* ca = f.costate_affine.data() + static_cast<size_t>(i) * nx;
      for (int ii = 0; ii < nx; ++ii) {
        double s = 0.0;
        for (int z = 0; z < nu; ++z) s += K[z + static_cast<size_t>(ii) * nu] * su[z];
        ca[ii] = sx[ii] + s;
      }
    }
  });
}

}  // namespace scn
