// SPDX-License-Identifier: MIT
// Host-side data model of the scenopt_b200 library: the flat, node-indexed
// problem (ProblemInstance, problem_data.hpp:95-141) and the factor cache
// (FactorCache, riccati.hpp:38-63) in contiguous arrays that the packer
// (pack.cpp) turns into the device layout.
#pragma once

#include <cstdint>
#include <functional>
#include <stdexcept>
#include <sys/mman.h>

#include <memory>
#include <new>
#include <string>
#include <utility>
#include <vector>

#include "scenopt_b200.h"

namespace scn {

// errors.hpp:9-80 as status-carrying exceptions; the C-ABI converts them.
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }

// Allocator for the per-node matrices. Blocks of kLazyBytes or more come
// straight from an anonymous mapping (zero pages, backed on first write), and
// value-less construction writes nothing, so zeros() of a large array touches
// no page: a shard's instance never writes the matrices of the nodes it does
// not hold, and those pages never become resident (host RAM ~1/N per rank).
template <class T>
struct NoInitAlloc : std::allocator<T> {
  static constexpr size_t kLazyBytes = size_t{64} << 20;
  template <class U>
  struct rebind {
    using other = NoInitAlloc<U>;
  };
  NoInitAlloc() = default;
  template <class U>
  NoInitAlloc(const NoInitAlloc<U>&) noexcept {}
  T* allocate(size_t n) {
    if (n * sizeof(T) < kLazyBytes) return std::allocator<T>::allocate(n);
    void* p = mmap(nullptr, n * sizeof(T), PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    if (p == MAP_FAILED) throw std::bad_alloc();
    return static_cast<T*>(p);
  }
  void deallocate(T* p, size_t n) noexcept {
    if (n * sizeof(T) < kLazyBytes)
      std::allocator<T>::deallocate(p, n);
    else
      munmap(p, n * sizeof(T));
  }
  template <class U>
  void construct(U*) noexcept {}  // default-init: no write
  template <class U, class... Args>
  void construct(U* p, Args&&... args) {
    ::new (static_cast<void*>(p)) U(std::forward<Args>(args)...);
  }
};
using BigVec = std::vector<double, NoInitAlloc<double>>;  // per-node matrices (GBs at C4)
template <class U, class V>
bool operator==(const NoInitAlloc<U>&, const NoInitAlloc<V>&) noexcept {
  return true;
}

// v = n zeros; a large array stays unbacked until written
inline void zeros(BigVec& v, size_t n) {
  BigVec().swap(v);
  if (n * sizeof(double) >= NoInitAlloc<double>::kLazyBytes)
    v.resize(n);  // fresh anonymous mapping: reads as zero
  else
    v.assign(n, 0.0);
}

struct Problem {
  int nx = 0, nu = 0, N = 0, n = 0, L = 0, first_leaf = 0, dual_dim = 0, stage_total = 0;
  std::vector<int32_t> ancestor, stage_offsets, stage_rows, terminal_rows, g_kind, tg_kind;
  std::vector<int32_t> mode;  // Markov mode per node (-1 root); empty when unknown (scenario_tree.hpp:41)
  std::vector<double> probability, root_state, c, q, r, F, G, g_gamma, p, FN, tg_gamma, zmin, zmax;
  BigVec A, B, Q, R, S, P;
  // derived (finalize)
  std::vector<int32_t> node_stage, child_begin, child_count, dual_offset, tdual_offset;
  // Nodes whose problem data this instance holds (empty: all). A shard's
  // instance (gen_random with a keep mask) holds its subtrees, the top and
  // the shard-stage nodes; the dual-row data (F, G, bounds, F_N) are always
  // complete. Such an instance can only build that shard's handle.
  std::vector<char> held;

  void finalize();  // layout + child ranges (problem_data.hpp:126-140)
  size_t sxx() const { return static_cast<size_t>(nx) * nx; }
  size_t sxu() const { return static_cast<size_t>(nx) * nu; }
  size_t suu() const { return static_cast<size_t>(nu) * nu; }
  const double* Ai(int i) const { return A.data() + i * sxx(); }
  const double* Bi(int i) const { return B.data() + i * sxu(); }
  const double* ci(int i) const { return c.data() + static_cast<size_t>(i) * nx; }
  const double* Qi(int i) const { return Q.data() + i * sxx(); }
  const double* Ri(int i) const { return R.data() + i * suu(); }
  const double* Si(int i) const { return S.data() + i * sxu(); }
  const double* qi(int i) const { return q.data() + static_cast<size_t>(i) * nx; }
  const double* ri(int i) const { return r.data() + static_cast<size_t>(i) * nu; }
  const double* Fi(int i) const { return F.data() + static_cast<size_t>(dual_offset[i]) * nx; }
  const double* Gi(int i) const { return G.data() + static_cast<size_t>(dual_offset[i]) * nu; }
  const double* Pl(int l) const { return P.data() + l * sxx(); }
  const double* pl(int l) const { return p.data() + static_cast<size_t>(l) * nx; }
  const double* FNl(int l) const {
    return FN.data() + static_cast<size_t>(tdual_offset[l] - stage_total) * nx;
  }
  int primal_dim() const { return first_leaf * nu + (n - 1) * nx; }
};

Problem problem_from_view(const scenopt_problem_view& v);
void problem_to_view(const Problem& p, scenopt_problem_view* v);
std::vector<std::string> validate(const Problem& p);
std::vector<std::string> validate_tree(const Problem& p);  // scenario_tree.hpp:128-240 only
void markov_tree(const std::vector<double>& transition, int rows, int cols, const std::vector<double>& initial,
                 int horizon, Problem& p);
void require_valid(const Problem& p);
Problem precondition(const Problem& p);                 // solvers.hpp:569-602
std::vector<double> probability_roots(const Problem& p);  // solvers.hpp:608-623
// keep: the nodes whose data are built (null: all); the random stream is
// drawn in full either way, so kept nodes get the full instance's values.
Problem gen_random(uint64_t seed, int nx, int nu, int horizon, const std::vector<int>& br,
                   const std::vector<char>* keep = nullptr);
// the tree of gen_random (shapes and layout only, no data)
Problem gen_random_tree(int nx, int nu, int horizon, const std::vector<int>& br);
// an instance holding every node (a shard's instance cannot be factored,
// saved or packed into an unsharded handle)
void require_full(const Problem& p, const char* who);

// generators.hpp:39-234: spring-mass-damper array on the Markov mode tree.
// Empty vectors take the reference defaults; transition is row-major.
struct SpringMass {
  double mass_kg = 5.0, stiffness = 1.0, damping = 0.1, input_bound = 2.0, velocity_bound = 5.0;
  int horizon = 11;
  double sampling = 0.5, state_weight = 5.0, input_weight = 2.0, terminal_weight = 100.0;
  std::vector<double> initial_probs, transition, mode_values, root_state;
  int transition_rows = 0, transition_cols = 0;
};
Problem gen_spring_mass(int masses, const SpringMass& par);
void spring_mass_continuous(int masses, const SpringMass& par, std::vector<double>& A, std::vector<double>& B);
std::vector<double> expm(const std::vector<double>& A, int n);  // column-major n x n
void discretize_zoh(const double* A, const double* B, int n, int m, double period, double* Ad, double* Bd);

struct Factor {
  int nx = 0, nu = 0, n = 0, first_leaf = 0, dual_dim = 0, L = 0, stage_total = 0;
  std::vector<int32_t> child_dual_offset, child_dual_rows;
  std::vector<double> gain;             // [F][nu*nx]
  std::vector<double> dual_to_input;    // by child_dual_offset: nu x M_i
  std::vector<double> dual_to_costate;  // by child_dual_offset: nx x M_i
  std::vector<double> input_affine;     // [F][nu]
  std::vector<double> costate_affine;   // [F][nx]
  std::vector<double> input_hessian;    // [F][nu*nu]
  std::vector<double> child_to_input;   // [n][nu*nx]
  std::vector<double> closed_loop;      // [n][nx*nx]
  std::vector<double> value_quad;       // [n][nx*nx]
  std::vector<double> leaf_costate_affine;  // [L][nx]
};

Factor factor(const Problem& p);                // riccati.hpp:82-182
// dimensions and child offsets; zero blocks unless lite (device factor layout)
Factor factor_shape(const Problem& p, bool lite = false);
void refactor_affine(Factor& f, const Problem& p);  // riccati.hpp:187-216
void check_factor_shape(const Factor& f, const Problem& p, const char* who);

// small dense helpers (column-major)
double sym_min_eig(const double* S, int n);
double spectral_radius(const double* A, int n);
// Cholesky in place (lower); returns false when not SPD
bool cholesky(std::vector<double>& a, int n);
// solve L L' X = B in place, B is n x k column-major
void chol_solve(const std::vector<double>& L, int n, double* B, int k);

// Parallel-for over [0, count) on the host worker pool (setup code only).
void parallel_for(int count, int grain, const std::function<void(int, int)>& body);

}  // namespace scn
