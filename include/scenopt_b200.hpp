// SPDX-License-Identifier: MIT
//
// scenopt_b200.hpp: the reference's C++ API (namespace scenopt), header-only,
// forwarding to the C-ABI of scenopt_b200.h.
//
// Reference code written against /root/reference/proj/include/scenopt/*.hpp
// (ProblemInstance, FactorCache, dual_grad, hessian_vec, fb_step,
// solve_minfbe, solve_nama, solve, ...) compiles against this header with
// the same names, argument meanings and exception types. Differences:
//   * Mat / Vec are small in-house column-major types with the subset of the
//     Eigen API the callers use (the reference's Eigen types are not
//     available in this image).
//   * factor() fills FactorCache's matrix members as the reference does;
//     factor(prob, FactorMembers::on_demand) keeps the factor on the C side
//     only (no host copy: 1.2 GB at C3) until load_matrices() is called.
//   * The device handle of a (ProblemInstance, FactorCache) pair is created
//     on first use and snapshots the instance. After changing an instance's
//     affine data call refactor_affine(cache, prob), as with the reference.
//   * SeparableNonsmooth must come from make_nonsmooth(prob); it carries
//     the device-side row data of that instance.
//   * CUDA / NCCL / allocation / no-device failures throw DeviceError (a
//     scenopt::Error); there is no CPU fallback.
// Every function cites the reference function it replaces.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <initializer_list>
#include <limits>
#include <memory>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "scenopt_b200.h"

namespace scenopt {

// ------------------------------------------------------------------ errors.hpp:9-80
struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NonStochasticMatrix : Error { using Error::Error; };
struct StageOutOfRange : Error { using Error::Error; };
struct DimensionMismatch : Error { using Error::Error; };
struct UnsupportedSpec : Error { using Error::Error; };
struct NotStronglyConvex : Error { using Error::Error; };
struct ShapeChanged : Error { using Error::Error; };
struct CacheMismatch : Error { using Error::Error; };
struct LineSearchStalled : Error { using Error::Error; };
struct StepUnderflow : Error { using Error::Error; };
struct ZeroProbability : Error { using Error::Error; };
struct InvalidParams : Error { using Error::Error; };
struct InfiniteConjugate : Error { using Error::Error; };
struct ParseError : Error { using Error::Error; };
/// CUDA, NCCL, allocation and no-device failures (no reference counterpart).
struct DeviceError : Error { using Error::Error; };

namespace detail {
[[noreturn]] inline void throw_status(int code, const std::string& what) {
  switch (code) {
    case SCENOPT_E_NON_STOCHASTIC_MATRIX: throw NonStochasticMatrix(what);
    case SCENOPT_E_STAGE_OUT_OF_RANGE: throw StageOutOfRange(what);
    case SCENOPT_E_DIMENSION_MISMATCH: throw DimensionMismatch(what);
    case SCENOPT_E_UNSUPPORTED_SPEC: throw UnsupportedSpec(what);
    case SCENOPT_E_NOT_STRONGLY_CONVEX: throw NotStronglyConvex(what);
    case SCENOPT_E_SHAPE_CHANGED: throw ShapeChanged(what);
    case SCENOPT_E_CACHE_MISMATCH: throw CacheMismatch(what);
    case SCENOPT_E_LINE_SEARCH_STALLED: throw LineSearchStalled(what);
    case SCENOPT_E_STEP_UNDERFLOW: throw StepUnderflow(what);
    case SCENOPT_E_ZERO_PROBABILITY: throw ZeroProbability(what);
    case SCENOPT_E_INVALID_PARAMS: throw InvalidParams(what);
    case SCENOPT_E_INFINITE_CONJUGATE: throw InfiniteConjugate(what);
    case SCENOPT_E_PARSE_ERROR: throw ParseError(what);
    case SCENOPT_E_CUDA:
    case SCENOPT_E_NCCL:
    case SCENOPT_E_NOMEM:
    case SCENOPT_E_NODEVICE: throw DeviceError(what);
    default: throw Error(what);
  }
}
inline int check(int rc) {
  if (rc < 0) throw_status(rc, scenopt_last_error());
  return rc;
}
}  // namespace detail

// ------------------------------------------------------------------ value types
/// Dense vector (the subset of Eigen::VectorXd the reference's callers use).
class Vec {
 public:
  Vec() = default;
  explicit Vec(int n) : v_(static_cast<size_t>(n), 0.0) {}
  Vec(std::initializer_list<double> l) : v_(l) {}
  explicit Vec(std::vector<double> v) : v_(std::move(v)) {}
  static Vec Zero(int n) { return Vec(n); }
  static Vec Constant(int n, double c) { return Vec(std::vector<double>(static_cast<size_t>(n), c)); }
  int size() const { return static_cast<int>(v_.size()); }
  void resize(int n) { v_.assign(static_cast<size_t>(n), 0.0); }
  void setZero() { std::fill(v_.begin(), v_.end(), 0.0); }
  double* data() { return v_.data(); }
  const double* data() const { return v_.data(); }
  double& operator()(int i) { return v_[static_cast<size_t>(i)]; }
  double operator()(int i) const { return v_[static_cast<size_t>(i)]; }
  double& operator[](int i) { return v_[static_cast<size_t>(i)]; }
  double operator[](int i) const { return v_[static_cast<size_t>(i)]; }
  double dot(const Vec& o) const {
    need(o);
    double s = 0.0;
    for (size_t i = 0; i < v_.size(); ++i) s += v_[i] * o.v_[i];
    return s;
  }
  double squaredNorm() const { return dot(*this); }
  double norm() const { return std::sqrt(squaredNorm()); }
  double lpNormInf() const {
    double m = 0.0;
    for (double x : v_) m = std::max(m, std::abs(x));
    return m;
  }
  Vec segment(int off, int n) const {
    return Vec(std::vector<double>(v_.begin() + off, v_.begin() + off + n));
  }
  Vec& operator+=(const Vec& o) { need(o); for (size_t i = 0; i < v_.size(); ++i) v_[i] += o.v_[i]; return *this; }
  Vec& operator-=(const Vec& o) { need(o); for (size_t i = 0; i < v_.size(); ++i) v_[i] -= o.v_[i]; return *this; }
  Vec& operator*=(double a) { for (double& x : v_) x *= a; return *this; }
  Vec& operator/=(double a) { for (double& x : v_) x /= a; return *this; }
  friend Vec operator+(Vec a, const Vec& b) { return a += b; }
  friend Vec operator-(Vec a, const Vec& b) { return a -= b; }
  friend Vec operator-(Vec a) { return a *= -1.0; }
  friend Vec operator*(Vec a, double s) { return a *= s; }
  friend Vec operator*(double s, Vec a) { return a *= s; }
  friend Vec operator/(Vec a, double s) { return a /= s; }
  const std::vector<double>& std() const { return v_; }
  double sum() const {
    double s = 0.0;
    for (double x : v_) s += x;
    return s;
  }
  double minCoeff() const { return *std::min_element(v_.begin(), v_.end()); }
  double maxCoeff() const { return *std::max_element(v_.begin(), v_.end()); }
  /// Eigen-style comma initializer: v << a, b, c;
  struct Comma {
    Vec& v;
    int i;
    Comma& operator,(double x) {
      if (i >= v.size()) throw DimensionMismatch("Vec: too many coefficients in comma initializer");
      v(i++) = x;
      return *this;
    }
  };
  Comma operator<<(double x) {
    Comma c{*this, 0};
    return c, x;
  }

 private:
  void need(const Vec& o) const {
    if (o.v_.size() != v_.size()) throw DimensionMismatch("Vec: length mismatch");
  }
  std::vector<double> v_;
};

/// Dense column-major matrix (the subset of Eigen::MatrixXd the callers use).
class Mat {
 public:
  Mat() = default;
  Mat(int r, int c) : r_(r), c_(c), v_(static_cast<size_t>(r) * c, 0.0) {}
  static Mat Zero(int r, int c) { return Mat(r, c); }
  static Mat Constant(int r, int c, double v) {
    Mat m(r, c);
    std::fill(m.v_.begin(), m.v_.end(), v);
    return m;
  }
  static Mat Identity(int n) { return Identity(n, n); }
  static Mat Identity(int r, int c) {
    Mat m(r, c);
    for (int i = 0; i < std::min(r, c); ++i) m(i, i) = 1.0;
    return m;
  }
  /// Eigen-style comma initializer, row-major order: m << a, b, c, d;
  struct Comma {
    Mat& m;
    int k;
    Comma& operator,(double x) {
      if (k >= m.size()) throw DimensionMismatch("Mat: too many coefficients in comma initializer");
      m(k / m.c_, k % m.c_) = x;
      ++k;
      return *this;
    }
  };
  Comma operator<<(double x) {
    Comma c{*this, 0};
    return c, x;
  }
  Mat& operator*=(double a) {
    for (double& x : v_) x *= a;
    return *this;
  }
  friend Mat operator*(double a, Mat m) { return m *= a; }
  friend Mat operator*(Mat m, double a) { return m *= a; }
  friend Mat operator+(Mat a, const Mat& b) {
    if (a.r_ != b.r_ || a.c_ != b.c_) throw DimensionMismatch("Mat + Mat: size mismatch");
    for (size_t i = 0; i < a.v_.size(); ++i) a.v_[i] += b.v_[i];
    return a;
  }
  Vec row(int i) const {
    Vec r(c_);
    for (int j = 0; j < c_; ++j) r(j) = (*this)(i, j);
    return r;
  }
  int rows() const { return r_; }
  int cols() const { return c_; }
  int size() const { return r_ * c_; }
  void resize(int r, int c) { *this = Mat(r, c); }
  double* data() { return v_.data(); }
  const double* data() const { return v_.data(); }
  double& operator()(int i, int j) { return v_[static_cast<size_t>(j) * r_ + i]; }
  double operator()(int i, int j) const { return v_[static_cast<size_t>(j) * r_ + i]; }
  Vec col(int j) const {
    return Vec(std::vector<double>(v_.begin() + static_cast<long>(j) * r_, v_.begin() + static_cast<long>(j + 1) * r_));
  }
  Mat transpose() const {
    Mat t(c_, r_);
    for (int j = 0; j < c_; ++j)
      for (int i = 0; i < r_; ++i) t(j, i) = (*this)(i, j);
    return t;
  }
  friend Vec operator*(const Mat& m, const Vec& x) {
    if (x.size() != m.c_) throw DimensionMismatch("Mat * Vec: size mismatch");
    Vec y(m.r_);
    for (int j = 0; j < m.c_; ++j)
      for (int i = 0; i < m.r_; ++i) y(i) += m(i, j) * x(j);
    return y;
  }

 private:
  int r_ = 0, c_ = 0;
  std::vector<double> v_;
};

using DualVector = Vec;

// ------------------------------------------------------------------ scenario_tree.hpp:21-45
struct ScenarioTree {
  int num_stages = 0;
  std::vector<int> node_stage;
  std::vector<int> ancestor;  ///< -1 at the root
  std::vector<std::vector<int>> children;
  std::vector<double> probability;
  std::vector<int> stage_offsets;  ///< size num_stages + 2
  std::vector<int> mode;

  int num_nodes() const { return static_cast<int>(node_stage.size()); }
  int num_leaves() const { return num_nodes() - stage_offsets[static_cast<size_t>(num_stages)]; }
  bool is_leaf(int i) const { return node_stage[static_cast<size_t>(i)] == num_stages; }
  int first_leaf() const { return stage_offsets[static_cast<size_t>(num_stages)]; }
};

/// scenario_tree.hpp:46-63
struct NodeRange {
  int first = 0;
  int past = 0;
  int size() const { return past - first; }
};
inline NodeRange nodes_at(const ScenarioTree& tree, int t1, int t2) {
  if (t1 < 0 || t2 > tree.num_stages || t1 > t2)
    throw StageOutOfRange("nodes_at: stage range [" + std::to_string(t1) + ", " + std::to_string(t2) +
                          "] outside [0, " + std::to_string(tree.num_stages) + "]");
  return NodeRange{tree.stage_offsets[static_cast<size_t>(t1)], tree.stage_offsets[static_cast<size_t>(t2) + 1]};
}
inline NodeRange nodes_at(const ScenarioTree& tree, int t) { return nodes_at(tree, t, t); }

/// build_from_markov, scenario_tree.hpp:72-126: the tree of all
/// positive-probability mode paths of a Markov chain, BFS numbered; the root
/// branches on `initial`, later nodes on their mode's transition row.
inline ScenarioTree build_from_markov(const Mat& transition, const Vec& initial, int horizon) {
  const int modes = initial.size();
  if (horizon < 1) throw InvalidParams("build_from_markov: horizon must be >= 1");
  if (transition.rows() != modes || transition.cols() != modes)
    throw DimensionMismatch("build_from_markov: transition must be square and match the initial distribution size");
  const double tol = 1e-9;
  if (initial.minCoeff() < 0.0 || std::abs(initial.sum() - 1.0) > tol)
    throw NonStochasticMatrix("build_from_markov: initial distribution");
  for (int w = 0; w < modes; ++w) {
    const Vec row = transition.row(w);
    if (row.minCoeff() < 0.0 || std::abs(row.sum() - 1.0) > tol)
      throw NonStochasticMatrix("build_from_markov: transition row " + std::to_string(w));
  }
  ScenarioTree t;
  t.num_stages = horizon;
  t.node_stage = {0};
  t.ancestor = {-1};
  t.children = {{}};
  t.probability = {1.0};
  t.mode = {-1};
  t.stage_offsets = {0, 1};
  for (int s = 0; s < horizon; ++s) {
    const int lo = t.stage_offsets[static_cast<size_t>(s)], hi = t.stage_offsets[static_cast<size_t>(s) + 1];
    for (int a = lo; a < hi; ++a)
      for (int w = 0; w < modes; ++w) {
        const double pr = s == 0 ? initial(w) : transition(t.mode[static_cast<size_t>(a)], w);
        if (!(pr > 0.0)) continue;
        t.children[static_cast<size_t>(a)].push_back(t.num_nodes());
        t.node_stage.push_back(s + 1);
        t.ancestor.push_back(a);
        t.children.emplace_back();
        t.probability.push_back(t.probability[static_cast<size_t>(a)] * pr);
        t.mode.push_back(w);
      }
    t.stage_offsets.push_back(t.num_nodes());
  }
  return t;
}

// ------------------------------------------------------------------ problem_data.hpp:16-141
struct NodeDynamics { Mat A, B; Vec c; };
struct NodeCost { Mat Q, R, S; Vec q, r; };
struct TerminalCost { Mat P; Vec p; };
enum class NonsmoothKind { None, Box, ScaledL1 };
struct NonsmoothSpec {
  NonsmoothKind kind = NonsmoothKind::None;
  Vec zmin, zmax;
  double gamma = 0.0;
};
struct ConstraintBlock { Mat F, G; NonsmoothSpec g; };
struct TerminalBlock { Mat F; NonsmoothSpec g; };

struct PrimalPoint {
  Mat x;  ///< nx by num_nodes
  Mat u;  ///< nu by first_leaf
  Vec flatten() const {
    std::vector<double> out(u.data(), u.data() + u.size());
    out.insert(out.end(), x.data(), x.data() + x.size());
    return Vec(std::move(out));
  }
  double dot(const PrimalPoint& o) const {
    double s = 0.0;
    for (int i = 0; i < u.size(); ++i) s += u.data()[i] * o.u.data()[i];
    for (int i = 0; i < x.size(); ++i) s += x.data()[i] * o.x.data()[i];
    return s;
  }
};

inline PrimalPoint zero_primal(int nx, int nu, const ScenarioTree& tree) {
  return PrimalPoint{Mat::Zero(nx, tree.num_nodes()), Mat::Zero(nu, tree.first_leaf())};
}

struct ProblemInstance {
  ScenarioTree tree;
  int nx = 0, nu = 0;
  Vec root_state;
  std::vector<NodeDynamics> dyn;
  std::vector<NodeCost> cost;
  std::vector<TerminalCost> tcost;
  std::vector<ConstraintBlock> con;
  std::vector<TerminalBlock> tcon;
  std::vector<int> dual_offset;   ///< per node; -1 at the root
  std::vector<int> tdual_offset;  ///< per leaf ordinal
  int dual_dim = 0;

  int num_nodes() const { return tree.num_nodes(); }
  int leaf_ordinal(int node) const { return node - tree.first_leaf(); }
  int primal_dim() const { return tree.first_leaf() * nu + (tree.num_nodes() - 1) * nx; }
  int stage_rows(int node) const { return con[static_cast<size_t>(node)].F.rows(); }
  int terminal_rows(int leaf_ord) const { return tcon[static_cast<size_t>(leaf_ord)].F.rows(); }
  void finalize_layout() {
    const int n = num_nodes();
    dual_offset.assign(static_cast<size_t>(n), -1);
    int off = 0;
    for (int i = 1; i < n; ++i) {
      dual_offset[static_cast<size_t>(i)] = off;
      off += stage_rows(i);
    }
    tdual_offset.assign(static_cast<size_t>(tree.num_leaves()), 0);
    for (int l = 0; l < tree.num_leaves(); ++l) {
      tdual_offset[static_cast<size_t>(l)] = off;
      off += terminal_rows(l);
    }
    dual_dim = off;
  }
};

// ------------------------------------------------------------------ C-handle plumbing
namespace detail {

struct ProblemDeleter { void operator()(scenopt_problem* p) const { scenopt_problem_destroy(p); } };
struct FactorDeleter { void operator()(scenopt_factor* f) const { scenopt_factor_destroy(f); } };
struct DevDeleter { void operator()(scenopt_dev* d) const { scenopt_dev_destroy(d); } };
struct ReportDeleter { void operator()(scenopt_report* r) const { scenopt_report_destroy(r); } };
using ProblemPtr = std::shared_ptr<scenopt_problem>;

inline void copy_block(const Mat& m, int rows, int cols, double* dst, const char* what, int node,
                       std::vector<std::string>* bad) {
  if (m.rows() != rows || m.cols() != cols) {
    if (bad)
      bad->push_back("node " + std::to_string(node) + ": " + what + " must be " + std::to_string(rows) + " x " +
                     std::to_string(cols));
    return;
  }
  std::copy(m.data(), m.data() + m.size(), dst);
}
inline void copy_vec(const Vec& v, int n, double* dst, const char* what, int node, std::vector<std::string>* bad) {
  if (v.size() != n) {
    if (bad) bad->push_back("node " + std::to_string(node) + ": " + what + " must have length " + std::to_string(n));
    return;
  }
  std::copy(v.data(), v.data() + n, dst);
}

/// ProblemInstance flattened into the C view (scenopt_problem_view).
struct FlatProblem {
  std::vector<int32_t> ancestor, stage_offsets, stage_rows, g_kind, terminal_rows, tg_kind;
  std::vector<double> probability, root_state, A, B, c, Q, R, S, q, r, F, G, g_gamma, P, p, FN, tg_gamma, zmin,
      zmax;
  scenopt_problem_view view{};
  std::vector<std::string> shape_errors;

  explicit FlatProblem(const ProblemInstance& pi) {
    const int n = pi.num_nodes(), nx = pi.nx, nu = pi.nu, N = pi.tree.num_stages;
    const int F0 = n > 0 ? pi.tree.first_leaf() : 0, L = n - F0;
    auto* bad = &shape_errors;
    if (static_cast<int>(pi.dyn.size()) != n || static_cast<int>(pi.cost.size()) != n ||
        static_cast<int>(pi.con.size()) != n || static_cast<int>(pi.tcost.size()) != L ||
        static_cast<int>(pi.tcon.size()) != L)
      throw DimensionMismatch("ProblemInstance: per-node / per-leaf containers do not match the tree");
    ancestor.assign(pi.tree.ancestor.begin(), pi.tree.ancestor.end());
    stage_offsets.assign(pi.tree.stage_offsets.begin(), pi.tree.stage_offsets.end());
    probability = pi.tree.probability;
    root_state.assign(static_cast<size_t>(nx), 0.0);
    copy_vec(pi.root_state, nx, root_state.data(), "root_state", 0, bad);
    const size_t un = static_cast<size_t>(n);
    A.assign(un * nx * nx, 0.0); B.assign(un * nx * nu, 0.0); c.assign(un * nx, 0.0);
    Q.assign(un * nx * nx, 0.0); R.assign(un * nu * nu, 0.0); S.assign(un * nu * nx, 0.0);
    q.assign(un * nx, 0.0); r.assign(un * nu, 0.0);
    stage_rows.assign(un, 0); g_kind.assign(un, 0); g_gamma.assign(un, 0.0);
    int stage_total = 0;
    for (int i = 1; i < n; ++i) stage_rows[i] = pi.con[i].F.rows(), stage_total += stage_rows[i];
    terminal_rows.assign(static_cast<size_t>(L), 0);
    int term_total = 0;
    for (int l = 0; l < L; ++l) terminal_rows[l] = pi.tcon[l].F.rows(), term_total += terminal_rows[l];
    const int D = stage_total + term_total;
    F.assign(static_cast<size_t>(stage_total) * nx, 0.0);
    G.assign(static_cast<size_t>(stage_total) * nu, 0.0);
    FN.assign(static_cast<size_t>(term_total) * nx, 0.0);
    zmin.assign(static_cast<size_t>(D), 0.0);
    zmax.assign(static_cast<size_t>(D), 0.0);
    tg_kind.assign(static_cast<size_t>(L), 0);
    tg_gamma.assign(static_cast<size_t>(L), 0.0);
    auto put_spec = [&](const NonsmoothSpec& g, int off, int rows, int node) {
      if (g.kind == NonsmoothKind::Box) {
        copy_vec(g.zmin, rows, zmin.data() + off, "zmin", node, bad);
        copy_vec(g.zmax, rows, zmax.data() + off, "zmax", node, bad);
      }
    };
    int off = 0;
    for (int i = 1; i < n; ++i) {
      const size_t si = static_cast<size_t>(i);
      copy_block(pi.dyn[si].A, nx, nx, A.data() + si * nx * nx, "A", i, bad);
      copy_block(pi.dyn[si].B, nx, nu, B.data() + si * nx * nu, "B", i, bad);
      copy_vec(pi.dyn[si].c, nx, c.data() + si * nx, "c", i, bad);
      copy_block(pi.cost[si].Q, nx, nx, Q.data() + si * nx * nx, "Q", i, bad);
      copy_block(pi.cost[si].R, nu, nu, R.data() + si * nu * nu, "R", i, bad);
      copy_block(pi.cost[si].S, nu, nx, S.data() + si * nu * nx, "S", i, bad);
      copy_vec(pi.cost[si].q, nx, q.data() + si * nx, "q", i, bad);
      copy_vec(pi.cost[si].r, nu, r.data() + si * nu, "r", i, bad);
      const int m = stage_rows[si];
      copy_block(pi.con[si].F, m, nx, F.data() + static_cast<size_t>(off) * nx, "F", i, bad);
      copy_block(pi.con[si].G, m, nu, G.data() + static_cast<size_t>(off) * nu, "G", i, bad);
      g_kind[si] = static_cast<int32_t>(pi.con[si].g.kind);
      g_gamma[si] = pi.con[si].g.gamma;
      put_spec(pi.con[si].g, off, m, i);
      off += m;
    }
    int toff = 0;
    for (int l = 0; l < L; ++l) {
      const size_t sl = static_cast<size_t>(l);
      P.resize(static_cast<size_t>(L) * nx * nx);
      p.resize(static_cast<size_t>(L) * nx);
      copy_block(pi.tcost[sl].P, nx, nx, P.data() + sl * nx * nx, "P", F0 + l, bad);
      copy_vec(pi.tcost[sl].p, nx, p.data() + sl * nx, "p", F0 + l, bad);
      const int m = terminal_rows[sl];
      copy_block(pi.tcon[sl].F, m, nx, FN.data() + static_cast<size_t>(toff) * nx, "F_N", F0 + l, bad);
      tg_kind[sl] = static_cast<int32_t>(pi.tcon[sl].g.kind);
      tg_gamma[sl] = pi.tcon[sl].g.gamma;
      put_spec(pi.tcon[sl].g, stage_total + toff, m, F0 + l);
      toff += m;
    }
    view.nx = nx;
    view.nu = nu;
    view.num_stages = N;
    view.num_nodes = n;
    view.ancestor = ancestor.data();
    view.probability = probability.data();
    view.stage_offsets = stage_offsets.data();
    view.root_state = root_state.data();
    view.A = A.data(); view.B = B.data(); view.c = c.data();
    view.Q = Q.data(); view.R = R.data(); view.S = S.data();
    view.q = q.data(); view.r = r.data();
    view.stage_rows = stage_rows.data();
    view.F = F.data(); view.G = G.data();
    view.g_kind = g_kind.data(); view.g_gamma = g_gamma.data();
    view.P = P.data(); view.p = p.data();
    view.terminal_rows = terminal_rows.data();
    view.FN = FN.data();
    view.tg_kind = tg_kind.data(); view.tg_gamma = tg_gamma.data();
    view.zmin = zmin.data(); view.zmax = zmax.data();
  }
};

/// C handle of an instance (problem_data.hpp:95-141 + finalize_layout).
inline ProblemPtr to_handle(const ProblemInstance& pi) {
  FlatProblem fp(pi);
  if (!fp.shape_errors.empty()) throw DimensionMismatch(fp.shape_errors.front());
  scenopt_problem* h = nullptr;
  check(scenopt_problem_create(&fp.view, &h));
  ProblemPtr out(h, ProblemDeleter{});
  if (static_cast<int>(pi.tree.mode.size()) == pi.num_nodes()) {
    std::vector<int32_t> mode(pi.tree.mode.begin(), pi.tree.mode.end());
    check(scenopt_problem_set_mode(h, mode.data(), static_cast<int>(mode.size())));
  }
  return out;
}

/// Structured instance from a C handle (inverse of to_handle).
inline ProblemInstance from_handle(scenopt_problem* h) {
  scenopt_problem_view v{};
  int32_t D = 0;
  check(scenopt_problem_get_view(h, &v, &D));
  ProblemInstance pi;
  const int n = v.num_nodes, nx = v.nx, nu = v.nu, N = v.num_stages;
  pi.nx = nx;
  pi.nu = nu;
  ScenarioTree& t = pi.tree;
  t.num_stages = N;
  t.ancestor.assign(v.ancestor, v.ancestor + n);
  t.probability.assign(v.probability, v.probability + n);
  t.stage_offsets.assign(v.stage_offsets, v.stage_offsets + N + 2);
  t.node_stage.assign(static_cast<size_t>(n), 0);
  for (int s = 0; s <= N; ++s)
    for (int i = t.stage_offsets[s]; i < t.stage_offsets[s + 1]; ++i) t.node_stage[i] = s;
  t.children.assign(static_cast<size_t>(n), {});
  for (int i = 1; i < n; ++i) t.children[static_cast<size_t>(t.ancestor[i])].push_back(i);
  {
    std::vector<int32_t> mode(static_cast<size_t>(n));
    const int k = check(scenopt_problem_get_mode(h, mode.data(), n));
    t.mode.assign(mode.begin(), mode.begin() + k);
  }
  pi.root_state = Vec(std::vector<double>(v.root_state, v.root_state + nx));
  const int F0 = t.first_leaf(), L = n - F0;
  pi.dyn.resize(static_cast<size_t>(n));
  pi.cost.resize(static_cast<size_t>(n));
  pi.con.resize(static_cast<size_t>(n));
  pi.tcost.resize(static_cast<size_t>(L));
  pi.tcon.resize(static_cast<size_t>(L));
  auto mat = [](const double* src, int r, int c) {
    Mat m(r, c);
    std::copy(src, src + static_cast<size_t>(r) * c, m.data());
    return m;
  };
  auto vec = [](const double* src, int k) { return Vec(std::vector<double>(src, src + k)); };
  auto spec = [&](int kind, double gamma, int off, int rows) {
    NonsmoothSpec s;
    s.kind = static_cast<NonsmoothKind>(kind);
    s.gamma = gamma;
    if (s.kind == NonsmoothKind::Box) {
      s.zmin = vec(v.zmin + off, rows);
      s.zmax = vec(v.zmax + off, rows);
    }
    return s;
  };
  int off = 0;
  for (int i = 0; i < n; ++i) {
    const size_t si = static_cast<size_t>(i);
    if (i == 0) {
      pi.con[0].F = Mat(0, nx);
      pi.con[0].G = Mat(0, nu);
      continue;
    }
    pi.dyn[si] = NodeDynamics{mat(v.A + si * nx * nx, nx, nx), mat(v.B + si * nx * nu, nx, nu), vec(v.c + si * nx, nx)};
    pi.cost[si] = NodeCost{mat(v.Q + si * nx * nx, nx, nx), mat(v.R + si * nu * nu, nu, nu),
                           mat(v.S + si * nu * nx, nu, nx), vec(v.q + si * nx, nx), vec(v.r + si * nu, nu)};
    const int m = v.stage_rows[i];
    pi.con[si].F = mat(v.F + static_cast<size_t>(off) * nx, m, nx);
    pi.con[si].G = mat(v.G + static_cast<size_t>(off) * nu, m, nu);
    pi.con[si].g = spec(v.g_kind[i], v.g_gamma[i], off, m);
    off += m;
  }
  const int stage_total = off;
  int toff = 0;
  for (int l = 0; l < L; ++l) {
    const size_t sl = static_cast<size_t>(l);
    pi.tcost[sl] = TerminalCost{mat(v.P + sl * nx * nx, nx, nx), vec(v.p + sl * nx, nx)};
    const int m = v.terminal_rows[l];
    pi.tcon[sl].F = mat(v.FN + static_cast<size_t>(toff) * nx, m, nx);
    pi.tcon[sl].g = spec(v.tg_kind[l], v.tg_gamma[l], stage_total + toff, m);
    toff += m;
  }
  pi.finalize_layout();
  return pi;
}

/// Device handle of one instance (factor-less: apply_H, prox, conj, dist).
struct RowDevice {
  ProblemPtr prob;
  std::shared_ptr<scenopt_dev> dev;
  scenopt_dev* get() {
    if (!dev) {
      scenopt_dev* d = nullptr;
      check(scenopt_dev_create(prob.get(), nullptr, 0, &d));
      dev = std::shared_ptr<scenopt_dev>(d, DevDeleter{});
    }
    return dev.get();
  }
};

/// Factor + device handle behind a FactorCache.
struct FactorState {
  ProblemPtr prob;                 // instance snapshot the factor was built from
  const ProblemInstance* src = nullptr;
  std::shared_ptr<scenopt_factor> fac;
  std::shared_ptr<scenopt_dev> dev;
  // a second instance of the same shape used with this cache (reference
  // semantics: the sweep reads the cache's matrices and the instance's data)
  const ProblemInstance* alt_src = nullptr;
  std::shared_ptr<scenopt_dev> alt_dev;
  ProblemPtr alt_prob;

  bool on_device = false;  // factored by factor_device(): no host factor, one device handle
  scenopt_dev* device_for(const ProblemInstance& pi) {
    if (on_device) return dev.get();
    if (&pi == src || src == nullptr) {
      if (!dev) {
        scenopt_dev* d = nullptr;
        check(scenopt_dev_create(prob.get(), fac.get(), 0, &d));
        dev = std::shared_ptr<scenopt_dev>(d, DevDeleter{});
      }
      return dev.get();
    }
    if (&pi != alt_src || !alt_dev) {
      alt_prob = to_handle(pi);
      scenopt_dev* d = nullptr;
      check(scenopt_dev_create(alt_prob.get(), fac.get(), 0, &d));
      alt_dev = std::shared_ptr<scenopt_dev>(d, DevDeleter{});
      alt_src = &pi;
    }
    return alt_dev.get();
  }
};

}  // namespace detail

// ------------------------------------------------------------------ validate (problem_data.hpp:233-314)
inline std::vector<std::string> validate(const ProblemInstance& prob) {
  detail::FlatProblem fp(prob);
  if (!fp.shape_errors.empty()) return fp.shape_errors;
  scenopt_problem* h = nullptr;
  const int rc = scenopt_problem_create(&fp.view, &h);
  if (rc < 0) return {scenopt_last_error()};
  std::unique_ptr<scenopt_problem, detail::ProblemDeleter> hp(h);
  std::vector<char> buf(1 << 16);
  const int nbad = detail::check(scenopt_problem_validate(h, buf.data(), static_cast<int>(buf.size())));
  std::vector<std::string> out;
  if (nbad == 0) return out;
  std::string all(buf.data());
  size_t pos = 0;
  while (pos <= all.size()) {
    const size_t nl = all.find('\n', pos);
    const std::string line = all.substr(pos, nl == std::string::npos ? std::string::npos : nl - pos);
    if (!line.empty()) out.push_back(line);
    if (nl == std::string::npos) break;
    pos = nl + 1;
  }
  return out;
}

// ------------------------------------------------------------------ generators.hpp:236-328
struct RandomDims {
  int nx = 3;
  int nu = 2;
};
struct RandomTreeShape {
  int horizon = 3;
  int branching = 2;
};
/// gen_random_instance (generators.hpp:255): full branching tree.
inline ProblemInstance gen_random_instance(std::uint64_t seed, RandomDims dims = {}, RandomTreeShape shape = {}) {
  if (dims.nx < 1 || dims.nu < 1) throw InvalidParams("gen_random_instance: dims must be positive");
  if (shape.horizon < 1 || shape.branching < 1)
    throw InvalidParams("gen_random_instance: tree shape must be positive");
  std::vector<int32_t> br(static_cast<size_t>(shape.horizon), shape.branching);
  scenopt_problem* h = nullptr;
  detail::check(scenopt_problem_gen_random(seed, dims.nx, dims.nu, shape.horizon, br.data(),
                                           static_cast<int>(br.size()), &h));
  std::unique_ptr<scenopt_problem, detail::ProblemDeleter> hp(h);
  return detail::from_handle(h);
}
/// Extension (BASELINE configs): per-stage branching br[t], 1 after the list.
inline ProblemInstance gen_random_instance(std::uint64_t seed, RandomDims dims, int horizon,
                                           const std::vector<int>& branching) {
  std::vector<int32_t> br(branching.begin(), branching.end());
  scenopt_problem* h = nullptr;
  detail::check(scenopt_problem_gen_random(seed, dims.nx, dims.nu, horizon, br.data(), static_cast<int>(br.size()),
                                           &h));
  std::unique_ptr<scenopt_problem, detail::ProblemDeleter> hp(h);
  return detail::from_handle(h);
}

// ------------------------------------------------------------------ generators.hpp:39-234
/// Spring-mass-damper array benchmark parameters (generators.hpp:49-64).
/// Empty members take the reference defaults.
struct SpringMassParams {
  double mass_kg = 5.0;
  double stiffness = 1.0;
  double damping = 0.1;
  double input_bound = 2.0;
  double velocity_bound = 5.0;
  int horizon = 11;
  double sampling = 0.5;
  double state_weight = 5.0;
  double input_weight = 2.0;
  double terminal_weight = 100.0;
  Vec initial_probs;
  Mat transition;
  Vec mode_values;
  Vec root_state;
};
namespace detail {
struct SpringMassC {
  scenopt_spring_mass_params c{};
  std::vector<double> t;  // transition, row-major
  explicit SpringMassC(const SpringMassParams& p) {
    c.mass_kg = p.mass_kg;
    c.stiffness = p.stiffness;
    c.damping = p.damping;
    c.input_bound = p.input_bound;
    c.velocity_bound = p.velocity_bound;
    c.horizon = p.horizon;
    c.sampling = p.sampling;
    c.state_weight = p.state_weight;
    c.input_weight = p.input_weight;
    c.terminal_weight = p.terminal_weight;
    c.initial_len = p.initial_probs.size();
    c.initial_probs = p.initial_probs.data();
    c.mode_values_len = p.mode_values.size();
    c.mode_values = p.mode_values.data();
    c.root_state_len = p.root_state.size();
    c.root_state = p.root_state.data();
    if (p.transition.size() > 0) {
      for (int i = 0; i < p.transition.rows(); ++i)
        for (int j = 0; j < p.transition.cols(); ++j) t.push_back(p.transition(i, j));
      c.transition_rows = p.transition.rows();
      c.transition_cols = p.transition.cols();
      c.transition = t.data();
    }
  }
};
/// detail::spring_mass_continuous (generators.hpp:70-91).
inline void spring_mass_continuous(int masses, const SpringMassParams& par, Mat& A, Mat& B) {
  SpringMassC c(par);
  A = Mat(2 * masses, 2 * masses);
  B = Mat(2 * masses, masses - 1);
  check(scenopt_spring_mass_continuous(masses, &c.c, A.data(), B.data()));
}
}  // namespace detail

/// discretize_zoh (generators.hpp:97-112).
inline void discretize_zoh(const Mat& A, const Mat& B, double period, Mat& Ad, Mat& Bd) {
  if (A.rows() != A.cols() || B.rows() != A.rows())
    throw DimensionMismatch("discretize_zoh: A must be square and match B");
  Ad = Mat(A.rows(), A.cols());
  Bd = Mat(B.rows(), B.cols());
  detail::check(scenopt_discretize_zoh(A.data(), B.data(), A.rows(), B.cols(), period, Ad.data(), Bd.data()));
}

/// gen_spring_mass (generators.hpp:119-218).
inline ProblemInstance gen_spring_mass(int masses, const SpringMassParams& params = {}) {
  detail::SpringMassC c(params);
  scenopt_problem* h = nullptr;
  detail::check(scenopt_problem_gen_spring_mass(masses, &c.c, &h));
  std::unique_ptr<scenopt_problem, detail::ProblemDeleter> hp(h);
  return detail::from_handle(h);
}

/// sample_initial_state (generators.hpp:223-234): one draw of the caller's engine per component.
inline Vec sample_initial_state(int masses, const SpringMassParams& params, std::mt19937_64& gen) {
  if (masses < 2) throw InvalidParams("sample_initial_state: masses must be >= 2");
  const double half = 0.5 * params.velocity_bound, pos_box = 1.0 * params.velocity_bound;
  auto sym = [&gen]() { return 2.0 * (static_cast<double>(gen() >> 11) * 0x1.0p-53) - 1.0; };
  Vec state(2 * masses);
  for (int i = 0; i < masses; ++i) state(i) = pos_box * sym();
  for (int i = masses; i < state.size(); ++i) state(i) = half * sym();
  return state;
}

// ------------------------------------------------------------------ problem_io.hpp:18-559
/// Problem files: JSON documents with schema "scenopt-problem-v1" (the
/// canonical text of the library's serializer; nlohmann DOM entry points
/// problem_to_json / problem_from_json are text-based here).
inline constexpr const char* kProblemSchema = "scenopt-problem-v1";

inline std::string serialize_problem(const ProblemInstance& prob) {
  auto h = detail::to_handle(prob);
  size_t n = 0;
  detail::check(scenopt_problem_serialize(h.get(), nullptr, 0, &n));
  std::string out(n + 1, '\0');
  detail::check(scenopt_problem_serialize(h.get(), out.data(), n + 1, &n));
  out.resize(n);
  return out;
}
inline ProblemInstance parse_problem(const std::string& text) {
  scenopt_problem* h = nullptr;
  detail::check(scenopt_problem_parse(text.data(), text.size(), &h));
  std::unique_ptr<scenopt_problem, detail::ProblemDeleter> hp(h);
  return detail::from_handle(h);
}
inline void save_problem(const ProblemInstance& prob, const std::string& path) {
  auto h = detail::to_handle(prob);
  detail::check(scenopt_problem_save(h.get(), path.c_str()));
}
inline ProblemInstance load_problem(const std::string& path) {
  scenopt_problem* h = nullptr;
  detail::check(scenopt_problem_load(path.c_str(), &h));
  std::unique_ptr<scenopt_problem, detail::ProblemDeleter> hp(h);
  return detail::from_handle(h);
}
inline std::vector<std::string> validate_problem_text(const std::string& text) {
  std::vector<char> buf(1 << 16);
  const int k = detail::check(scenopt_problem_validate_text(text.data(), text.size(), buf.data(),
                                                            static_cast<int>(buf.size())));
  std::vector<std::string> out;
  std::string all(buf.data());
  for (size_t pos = 0; k > 0 && pos < all.size();) {
    const size_t nl = all.find('\n', pos);
    const std::string line = all.substr(pos, nl == std::string::npos ? std::string::npos : nl - pos);
    if (!line.empty()) out.push_back(line);
    if (nl == std::string::npos) break;
    pos = nl + 1;
  }
  return out;
}
inline std::uint64_t content_hash(const ProblemInstance& prob) {
  auto h = detail::to_handle(prob);
  std::uint64_t c = 0;
  detail::check(scenopt_problem_hashes(h.get(), &c, nullptr));
  return c;
}
inline std::uint64_t factor_hash(const ProblemInstance& prob) {
  auto h = detail::to_handle(prob);
  std::uint64_t f = 0;
  detail::check(scenopt_problem_hashes(h.get(), nullptr, &f));
  return f;
}

// ------------------------------------------------------------------ riccati.hpp:38-216
struct FactorCache {
  int nx = 0, nu = 0;
  int num_nodes = 0;
  int first_leaf = 0;
  int dual_dim = 0;
  // The reference's matrix members, filled by load_matrices() only.
  std::vector<Mat> gain, dual_to_input, dual_to_costate;
  std::vector<Vec> input_affine, costate_affine;
  std::vector<int> child_dual_offset, child_dual_rows;
  std::vector<Mat> child_to_input, closed_loop, value_quad;
  std::vector<Vec> leaf_costate_affine;

  std::shared_ptr<detail::FactorState> state;
  bool members_loaded = false;  // the fields above hold the current factor

  /// Copies the factor's matrices into the reference's fields.
  void load_matrices(const ProblemInstance& prob) {
    const int n = num_nodes, F = first_leaf, L = n - F;
    std::vector<double> g(static_cast<size_t>(F) * nu * nx), c2i(static_cast<size_t>(n) * nu * nx),
        cl(static_cast<size_t>(n) * nx * nx), ia(static_cast<size_t>(F) * nu), ca(static_cast<size_t>(F) * nx),
        vq(static_cast<size_t>(n) * nx * nx), lca(static_cast<size_t>(L) * nx);
    int S = 0;
    for (int i = 1; i < n; ++i) S += prob.stage_rows(i);
    std::vector<double> d2i(static_cast<size_t>(std::max(S, 1)) * nu), d2c(static_cast<size_t>(std::max(S, 1)) * nx);
    if (state->on_device)
      detail::check(scenopt_dev_factor_export(state->dev.get(), state->prob.get(), g.data(), c2i.data(), cl.data(),
                                              d2i.data(), d2c.data(), ia.data(), ca.data(), vq.data(), lca.data()));
    else
      detail::check(scenopt_factor_export(state->fac.get(), g.data(), c2i.data(), cl.data(), d2i.data(), d2c.data(),
                                          ia.data(), ca.data(), vq.data(), lca.data()));
    auto mat = [](const double* src, int r, int c) {
      Mat m(r, c);
      std::copy(src, src + static_cast<size_t>(r) * c, m.data());
      return m;
    };
    auto vec = [](const double* src, int k) { return Vec(std::vector<double>(src, src + k)); };
    gain.assign(static_cast<size_t>(F), Mat());
    dual_to_input.assign(static_cast<size_t>(F), Mat());
    dual_to_costate.assign(static_cast<size_t>(F), Mat());
    input_affine.assign(static_cast<size_t>(F), Vec());
    costate_affine.assign(static_cast<size_t>(F), Vec());
    child_dual_offset.assign(static_cast<size_t>(F), 0);
    child_dual_rows.assign(static_cast<size_t>(F), 0);
    for (int i = 0; i < F; ++i) {
      const auto& kids = prob.tree.children[static_cast<size_t>(i)];
      const int off = kids.empty() ? 0 : prob.dual_offset[static_cast<size_t>(kids.front())];
      int rows = 0;
      for (int c : kids) rows += prob.stage_rows(c);
      child_dual_offset[i] = off;
      child_dual_rows[i] = rows;
      gain[i] = mat(g.data() + static_cast<size_t>(i) * nu * nx, nu, nx);
      dual_to_input[i] = mat(d2i.data() + static_cast<size_t>(off) * nu, nu, rows);
      dual_to_costate[i] = mat(d2c.data() + static_cast<size_t>(off) * nx, nx, rows);
      input_affine[i] = vec(ia.data() + static_cast<size_t>(i) * nu, nu);
      costate_affine[i] = vec(ca.data() + static_cast<size_t>(i) * nx, nx);
    }
    child_to_input.assign(static_cast<size_t>(n), Mat());
    closed_loop.assign(static_cast<size_t>(n), Mat());
    value_quad.assign(static_cast<size_t>(n), Mat());
    for (int c = 0; c < n; ++c) {
      if (c > 0) {
        child_to_input[c] = mat(c2i.data() + static_cast<size_t>(c) * nu * nx, nu, nx);
        closed_loop[c] = mat(cl.data() + static_cast<size_t>(c) * nx * nx, nx, nx);
      }
      value_quad[c] = mat(vq.data() + static_cast<size_t>(c) * nx * nx, nx, nx);
    }
    leaf_costate_affine.assign(static_cast<size_t>(L), Vec());
    for (int l = 0; l < L; ++l) leaf_costate_affine[l] = vec(lca.data() + static_cast<size_t>(l) * nx, nx);
    members_loaded = true;
  }
};

/// Whether factor() copies the factor into FactorCache's matrix members.
enum class FactorMembers { full, on_demand };

namespace detail {
/// riccati.hpp:67-74
inline void check_shapes(const FactorCache& cache, const ProblemInstance& prob, const char* who) {
  if (cache.num_nodes != prob.num_nodes() || cache.nx != prob.nx || cache.nu != prob.nu ||
      cache.dual_dim != prob.dual_dim || cache.first_leaf != prob.tree.first_leaf())
    throw CacheMismatch(std::string(who) + ": cache was built for a different problem shape");
  if (!cache.state) throw CacheMismatch(std::string(who) + ": cache was not built by factor()");
}
inline void need_dual(const ProblemInstance& prob, const Vec& y, const char* who) {
  if (y.size() != prob.dual_dim) throw DimensionMismatch(std::string(who) + ": dual vector has wrong length");
}
}  // namespace detail

/// factor(), riccati.hpp:82-182 (host, offline; the device handle is built
/// on first use).
inline FactorCache factor(const ProblemInstance& prob, FactorMembers members = FactorMembers::full) {
  auto st = std::make_shared<detail::FactorState>();
  st->prob = detail::to_handle(prob);
  st->src = &prob;
  scenopt_factor* f = nullptr;
  detail::check(scenopt_factor_create(st->prob.get(), &f));
  st->fac = std::shared_ptr<scenopt_factor>(f, detail::FactorDeleter{});
  FactorCache c;
  c.nx = prob.nx;
  c.nu = prob.nu;
  c.num_nodes = prob.num_nodes();
  c.first_leaf = prob.tree.first_leaf();
  c.dual_dim = prob.dual_dim;
  c.state = st;
  if (members == FactorMembers::full) c.load_matrices(prob);
  return c;
}

/// factor() on the device (K9; B200 extension): the Riccati factor is computed
/// by a GPU kernel directly into the sweep layout, with no host factor and no
/// factor upload. Use with refactor_affine() for receding-horizon re-solves.
inline FactorCache factor_device(const ProblemInstance& prob) {
  auto st = std::make_shared<detail::FactorState>();
  st->prob = detail::to_handle(prob);
  st->src = &prob;
  st->on_device = true;
  scenopt_dev* d = nullptr;
  detail::check(scenopt_dev_create_device_factor(st->prob.get(), 0, &d));
  st->dev = std::shared_ptr<scenopt_dev>(d, detail::DevDeleter{});
  FactorCache c;
  c.nx = prob.nx;
  c.nu = prob.nu;
  c.num_nodes = prob.num_nodes();
  c.first_leaf = prob.tree.first_leaf();
  c.dual_dim = prob.dual_dim;
  c.state = st;
  return c;
}

/// refactor_affine(), riccati.hpp:187-216: recomputes the affine members for
/// new q, r, c, p (same matrices) and refreshes the device handle. On a
/// factor_device() cache only the linear terms and the root state move to
/// the device and the affine terms are recomputed there.
inline void refactor_affine(FactorCache& cache, const ProblemInstance& prob) {
  detail::check_shapes(cache, prob, "refactor_affine");
  if (cache.state->on_device) {
    auto ph = detail::to_handle(prob);
    detail::check(scenopt_dev_refactor_affine(cache.state->dev.get(), ph.get()));
    if (cache.members_loaded) cache.load_matrices(prob);
    return;
  }
  auto st = std::make_shared<detail::FactorState>(*cache.state);
  auto ph = detail::to_handle(prob);
  detail::check(scenopt_refactor_affine(st->fac.get(), ph.get()));
  st->prob = ph;
  st->src = &prob;
  st->dev.reset();
  st->alt_dev.reset();
  st->alt_src = nullptr;
  cache.state = st;
  if (cache.members_loaded) cache.load_matrices(prob);  // the affine members changed
}

// ------------------------------------------------------------------ tree_oracles.hpp:14-129
struct OracleStats {
  std::uint64_t dual_grad_calls = 0;
  std::uint64_t hessian_vec_calls = 0;
  std::uint64_t prox_calls = 0;
  std::uint64_t conj_calls = 0;
  std::uint64_t sweep_total() const { return dual_grad_calls + hessian_vec_calls; }
};

/// dual_grad, tree_oracles.hpp:96-102: x(y) by one fused device sweep.
inline PrimalPoint dual_grad(const FactorCache& cache, const ProblemInstance& prob, const DualVector& y,
                             OracleStats* stats = nullptr) {
  detail::check_shapes(cache, prob, "dual_grad");
  detail::need_dual(prob, y, "riccati_sweep");
  scenopt_dev* d = cache.state->device_for(prob);
  PrimalPoint pt = zero_primal(prob.nx, prob.nu, prob.tree);
  detail::check(scenopt_dual_grad(d, y.data(), pt.x.data(), pt.u.data(), SCENOPT_HOST_IO));
  if (stats) ++stats->dual_grad_calls;
  return pt;
}

/// hessian_vec, tree_oracles.hpp:107-114: x0(r), the homogeneous part.
inline PrimalPoint hessian_vec(const FactorCache& cache, const ProblemInstance& prob, const DualVector& r,
                               OracleStats* stats = nullptr) {
  detail::check_shapes(cache, prob, "hessian_vec");
  detail::need_dual(prob, r, "riccati_sweep");
  scenopt_dev* d = cache.state->device_for(prob);
  PrimalPoint pt = zero_primal(prob.nx, prob.nu, prob.tree);
  detail::check(scenopt_hessian_vec(d, r.data(), pt.x.data(), pt.u.data(), SCENOPT_HOST_IO));
  if (stats) ++stats->hessian_vec_calls;
  return pt;
}

/// apply_H, problem_data.hpp:144-162 (device; factor-less handle of prob).
inline DualVector apply_H(const ProblemInstance& prob, const PrimalPoint& pt) {
  if (pt.x.rows() != prob.nx || pt.x.cols() != prob.num_nodes() || pt.u.rows() != prob.nu ||
      pt.u.cols() != prob.tree.first_leaf())
    throw DimensionMismatch("apply_H: point does not match the instance");
  detail::RowDevice rd{detail::to_handle(prob), nullptr};
  DualVector z(prob.dual_dim);
  detail::check(scenopt_apply_H(rd.get(), pt.x.data(), pt.u.data(), z.data(), SCENOPT_HOST_IO));
  return z;
}

/// grad_fhat, tree_oracles.hpp:117-122: -H x(y).
inline DualVector grad_fhat(const FactorCache& cache, const ProblemInstance& prob, const DualVector& y,
                            OracleStats* stats = nullptr) {
  detail::check_shapes(cache, prob, "grad_fhat");
  detail::need_dual(prob, y, "riccati_sweep");
  scenopt_dev* d = cache.state->device_for(prob);
  const double* ys[1] = {y.data()};
  DualVector Hx(prob.dual_dim);
  double* hs[1] = {Hx.data()};
  detail::check(scenopt_dev_sweep(d, 1, 1, ys, nullptr, nullptr, hs, SCENOPT_HOST_IO));
  if (stats) ++stats->dual_grad_calls;
  return -Hx;
}

/// fhat_value, tree_oracles.hpp:125-129.
inline double fhat_value(const FactorCache& cache, const ProblemInstance& prob, const DualVector& y,
                         OracleStats* stats = nullptr) {
  detail::check_shapes(cache, prob, "fhat_value");
  detail::need_dual(prob, y, "riccati_sweep");
  double v = 0.0;
  detail::check(scenopt_fhat_value(cache.state->device_for(prob), y.data(), &v, SCENOPT_HOST_IO));
  if (stats) ++stats->dual_grad_calls;
  return v;
}

// ------------------------------------------------------------------ prox.hpp:15-171
struct GBlock {
  int offset = 0;
  int size = 0;
  double weight = 1.0;
  NonsmoothKind kind = NonsmoothKind::None;
  Vec zmin, zmax;
  double gamma = 0.0;
};
struct SeparableNonsmooth {
  std::vector<GBlock> blocks;
  int dim = 0;
  std::shared_ptr<detail::RowDevice> device;  ///< row data of the instance (make_nonsmooth)
};

/// make_nonsmooth, prox.hpp:30-52.
inline SeparableNonsmooth make_nonsmooth(const ProblemInstance& prob) {
  SeparableNonsmooth g;
  g.dim = prob.dual_dim;
  auto add = [&g](int offset, int rows, double weight, const NonsmoothSpec& s) {
    if (weight <= 0.0) throw ZeroProbability("make_nonsmooth: block with nonpositive weight");
    g.blocks.push_back(GBlock{offset, rows, weight, s.kind, s.zmin, s.zmax, s.gamma});
  };
  for (int i = 1; i < prob.num_nodes(); ++i)
    add(prob.dual_offset[static_cast<size_t>(i)], prob.stage_rows(i), prob.tree.probability[static_cast<size_t>(i)],
        prob.con[static_cast<size_t>(i)].g);
  for (int i = prob.tree.first_leaf(); i < prob.num_nodes(); ++i) {
    const int l = prob.leaf_ordinal(i);
    add(prob.tdual_offset[static_cast<size_t>(l)], prob.terminal_rows(l), prob.tree.probability[static_cast<size_t>(i)],
        prob.tcon[static_cast<size_t>(l)].g);
  }
  g.device = std::make_shared<detail::RowDevice>(detail::RowDevice{detail::to_handle(prob), nullptr});
  return g;
}

namespace detail {
inline scenopt_dev* rows_of(const SeparableNonsmooth& g, const Vec& v, const char* who) {
  if (!g.device) throw UnsupportedSpec(std::string(who) + ": SeparableNonsmooth must come from make_nonsmooth()");
  if (v.size() != g.dim) throw DimensionMismatch(std::string(who) + ": vector length does not match g");
  return g.device->get();
}
}  // namespace detail

/// prox_g, prox.hpp:58-81.
inline Vec prox_g(const SeparableNonsmooth& g, const Vec& v, double gamma_prox) {
  Vec out(v.size());
  detail::check(scenopt_prox_g(detail::rows_of(g, v, "prox_g"), v.data(), gamma_prox, out.data(), SCENOPT_HOST_IO));
  return out;
}
/// conj_value_g, prox.hpp:90-113.
inline double conj_value_g(const SeparableNonsmooth& g, const Vec& w) {
  double v = 0.0;
  detail::check(scenopt_conj_value_g(detail::rows_of(g, w, "conj_value_g"), w.data(), &v, SCENOPT_HOST_IO));
  return v;
}
/// prox_g_conj, prox.hpp:117-121 (Moreau: v - gamma prox_{g/gamma}(v/gamma)).
inline Vec prox_g_conj(const SeparableNonsmooth& g, const Vec& v, double gamma) {
  return v - gamma * prox_g(g, v / gamma, 1.0 / gamma);
}
/// dist_subdiff_inf, prox.hpp:127-171.
inline double dist_subdiff_inf(const SeparableNonsmooth& g, const Vec& y, const Vec& z) {
  if (y.size() != z.size()) throw DimensionMismatch("dist_subdiff_inf: length mismatch");
  double v = 0.0;
  detail::check(scenopt_dist_subdiff_inf(detail::rows_of(g, y, "dist_subdiff_inf"), y.data(), z.data(), &v,
                                         SCENOPT_HOST_IO));
  return v;
}

// ------------------------------------------------------------------ fbe.hpp:22-94
struct FbState {
  DualVector y;
  double lambda = 0.0;
  PrimalPoint x;
  DualVector Hx;
  DualVector z;
  DualVector T;
  DualVector R;
  double fhat = 0.0;
  double conj_T = 0.0;
  double znorm_sq = 0.0;
  double value = 0.0;
};

/// fb_step, fbe.hpp:55-67: one fused sweep + prox + conj on the device.
inline FbState fb_step(const FactorCache& cache, const ProblemInstance& prob, const SeparableNonsmooth& g,
                       const DualVector& y, double lambda, OracleStats* stats = nullptr) {
  if (!(lambda > 0.0)) throw InvalidParams("fb_step: lambda must be > 0");
  detail::check_shapes(cache, prob, "dual_grad");
  detail::need_dual(prob, y, "riccati_sweep");
  (void)g;
  FbState s;
  s.y = y;
  s.lambda = lambda;
  s.x = zero_primal(prob.nx, prob.nu, prob.tree);
  s.Hx = s.z = s.R = s.T = DualVector(prob.dual_dim);
  double sc[4] = {0, 0, 0, 0};
  detail::check(scenopt_fb_step(cache.state->device_for(prob), y.data(), lambda, s.x.x.data(), s.x.u.data(),
                                s.Hx.data(), s.z.data(), s.R.data(), s.T.data(), sc, SCENOPT_HOST_IO));
  s.fhat = sc[0];
  s.conj_T = sc[1];
  s.znorm_sq = sc[2];
  s.value = sc[3];
  if (stats) {
    ++stats->dual_grad_calls;
    ++stats->prox_calls;
    ++stats->conj_calls;
  }
  return s;
}

/// rescale_state, fbe.hpp:72-77: lambda-dependent fields at a new step
/// (one prox and one conj on the device; no sweep).
inline void rescale_state(FbState& state, const SeparableNonsmooth& g, double lambda, OracleStats* stats = nullptr) {
  if (!(lambda > 0.0)) throw InvalidParams("rescale_state: lambda must be > 0");
  state.lambda = lambda;
  state.z = prox_g(g, state.y / lambda + state.Hx, 1.0 / lambda);
  if (stats) ++stats->prox_calls;
  state.R = state.z - state.Hx;
  state.T = state.y - lambda * state.R;
  state.conj_T = conj_value_g(g, state.T);
  if (stats) ++stats->conj_calls;
  state.znorm_sq = state.z.squaredNorm();
  state.value = state.fhat + state.conj_T + lambda * state.Hx.dot(state.R) + 0.5 * lambda * state.R.squaredNorm();
}

/// fbe_value, fbe.hpp:82-87.
inline double fbe_value(const FbState& state) {
  if (!std::isfinite(state.value)) throw InfiniteConjugate("fbe_value: g*(T) is infinite");
  return state.value;
}

/// fbe_grad, fbe.hpp:89-94: R + lambda H x0(R) (one homogeneous sweep).
inline DualVector fbe_grad(const FbState& state, const FactorCache& cache, const ProblemInstance& prob,
                           OracleStats* stats = nullptr) {
  detail::check_shapes(cache, prob, "hessian_vec");
  detail::need_dual(prob, state.R, "riccati_sweep");
  DualVector grad(prob.dual_dim);
  detail::check(scenopt_fbe_grad(cache.state->device_for(prob), state.R.data(), state.lambda, grad.data(),
                                 SCENOPT_HOST_IO));
  if (stats) ++stats->hessian_vec_calls;
  return grad;
}

// ------------------------------------------------------------------ lbfgs.hpp:22-84
/// L-BFGS buffer with device-resident pairs (standalone handle on device 0,
/// created on first use so parameter validation needs no device).
class LbfgsBuffer {
 public:
  LbfgsBuffer(int memory, double eps_curv) : memory_(memory), eps_curv_(eps_curv) {
    if (memory < 1) throw InvalidParams("LbfgsBuffer: memory must be >= 1");
    if (!(eps_curv > 0.0)) throw InvalidParams("LbfgsBuffer: eps_curv must be > 0");
  }
  bool push(const DualVector& step, const DualVector& change, double scale_ref) {
    if (step.size() != change.size()) throw DimensionMismatch("LbfgsBuffer::push: length mismatch");
    return detail::check(scenopt_lbfgs_push(h(), step.size(), step.data(), change.data(), scale_ref)) == 1;
  }
  DualVector apply_direction(const DualVector& grad) const {
    DualVector out(grad.size());
    detail::check(scenopt_lbfgs_apply(h(), grad.size(), grad.data(), out.data()));
    return out;
  }
  void clear() {
    if (h_) detail::check(scenopt_lbfgs_clear(h_.get()));
  }
  int size() const { return h_ ? detail::check(scenopt_lbfgs_size(h_.get())) : 0; }
  int memory() const { return memory_; }
  double gamma0() const { return h_ ? scenopt_lbfgs_gamma0(h_.get()) : 1.0; }

 private:
  struct Deleter { void operator()(scenopt_lbfgs* b) const { scenopt_lbfgs_destroy(b); } };
  scenopt_lbfgs* h() const {
    if (!h_) {
      scenopt_lbfgs* b = nullptr;
      detail::check(scenopt_lbfgs_create(nullptr, memory_, eps_curv_, &b));
      h_ = std::shared_ptr<scenopt_lbfgs>(b, Deleter{});
    }
    return h_.get();
  }
  int memory_;
  double eps_curv_;
  mutable std::shared_ptr<scenopt_lbfgs> h_;
};

// ------------------------------------------------------------------ solvers.hpp:20-720
enum class BacktrackingRule { Original, Simple, None };
enum class SolverKind { Minfbe, Nama, Gpad };
enum class SolverStatus { Converged, MaxItersExceeded };

struct SolverConfig {
  double lambda0 = 0.0;
  double eps = 5e-4;
  double eps_curv = 1e-12;
  double eps_bt = 0.25;
  double beta_bt = 0.05;
  int memory = 5;
  int max_iters = 20000;
  BacktrackingRule backtracking_rule = BacktrackingRule::Simple;
  bool warm_start = false;
  int warm_start_iters = 5;
  bool precondition = false;
  bool nama_parallel_linesearch = false;
  bool nama_update_tlambda = true;
};

/// validate_config, solvers.hpp:48-63.
inline void validate_config(const SolverConfig& cfg) {
  if (cfg.lambda0 < 0.0) throw InvalidParams("lambda0 must be >= 0");
  if (!(cfg.eps > 0.0)) throw InvalidParams("eps must be > 0");
  if (!(cfg.eps_curv > 0.0)) throw InvalidParams("eps_curv must be > 0");
  if (!(cfg.eps_bt > 0.0 && cfg.eps_bt < 0.5)) throw InvalidParams("eps_bt must lie in (0, 1/2)");
  if (cfg.beta_bt < 0.0 || cfg.beta_bt >= 1.0) throw InvalidParams("beta_bt must lie in [0, 1)");
  if (cfg.memory < 1) throw InvalidParams("memory must be >= 1");
  if (cfg.max_iters < 1) throw InvalidParams("max_iters must be >= 1");
  if (cfg.warm_start_iters < 0) throw InvalidParams("warm_start_iters must be >= 0");
}

struct SolverReport {
  SolverStatus status = SolverStatus::MaxItersExceeded;
  PrimalPoint x;
  DualVector y;
  DualVector z;
  double residual_inf = std::numeric_limits<double>::infinity();
  int iterations = 0;
  OracleStats stats;
  std::uint64_t lipschitz_calls = 0;
  double lipschitz_estimate = 0.0;
  double lambda_final = 0.0;
  double eps = 0.0;
  std::vector<double> residual_trace;
  std::vector<double> fbe_trace;
  double wall_ms = 0.0;
  bool verified = false;
  double verify_residual_inf = std::numeric_limits<double>::infinity();
  double verify_subdiff_dist = std::numeric_limits<double>::infinity();
};

namespace detail {
inline scenopt_solver_config c_config(const SolverConfig& c) {
  scenopt_solver_config o{};
  o.lambda0 = c.lambda0;
  o.eps = c.eps;
  o.eps_curv = c.eps_curv;
  o.eps_bt = c.eps_bt;
  o.beta_bt = c.beta_bt;
  o.memory = c.memory;
  o.max_iters = c.max_iters;
  o.backtracking_rule = static_cast<int32_t>(c.backtracking_rule);
  o.warm_start = c.warm_start;
  o.warm_start_iters = c.warm_start_iters;
  o.precondition = c.precondition;
  o.nama_parallel_linesearch = c.nama_parallel_linesearch;
  o.nama_update_tlambda = c.nama_update_tlambda;
  return o;
}
inline SolverReport take_report(scenopt_report* raw, const ProblemInstance& prob) {
  std::unique_ptr<scenopt_report, ReportDeleter> r(raw);
  scenopt_report_summary s{};
  check(scenopt_report_summary_get(r.get(), &s));
  SolverReport rep;
  rep.status = s.status == 0 ? SolverStatus::Converged : SolverStatus::MaxItersExceeded;
  rep.iterations = s.iterations;
  rep.verified = s.verified != 0;
  rep.stats.dual_grad_calls = s.dual_grad_calls;
  rep.stats.hessian_vec_calls = s.hessian_vec_calls;
  rep.stats.prox_calls = s.prox_calls;
  rep.stats.conj_calls = s.conj_calls;
  rep.lipschitz_calls = s.lipschitz_calls;
  rep.lipschitz_estimate = s.lipschitz_estimate;
  rep.lambda_final = s.lambda_final;
  rep.eps = s.eps;
  rep.residual_inf = s.residual_inf;
  rep.wall_ms = s.wall_ms;
  rep.verify_residual_inf = s.verify_residual_inf;
  rep.verify_subdiff_dist = s.verify_subdiff_dist;
  rep.x = zero_primal(prob.nx, prob.nu, prob.tree);
  rep.y = DualVector(prob.dual_dim);
  rep.z = DualVector(prob.dual_dim);
  rep.residual_trace.assign(static_cast<size_t>(s.trace_len), 0.0);
  rep.fbe_trace.assign(static_cast<size_t>(s.trace_len), 0.0);
  check(scenopt_report_arrays(r.get(), rep.x.x.data(), rep.x.u.data(), rep.y.data(), rep.z.data(),
                              rep.residual_trace.data(), rep.fbe_trace.data()));
  return rep;
}
inline SolverReport run_solver(const ProblemInstance& prob, const FactorCache& cache, const SeparableNonsmooth& g,
                               const SolverConfig& cfg, const DualVector& y0, const Vec* residual_weight, int kind,
                               const char* who) {
  validate_config(cfg);
  check_shapes(cache, prob, who);
  if (g.dim != prob.dual_dim) throw DimensionMismatch(std::string(who) + ": g does not match the instance");
  need_dual(prob, y0, who);
  if (residual_weight) need_dual(prob, *residual_weight, who);
  const scenopt_solver_config c = c_config(cfg);
  scenopt_report* r = nullptr;
  check(scenopt_dev_solve(cache.state->device_for(prob), &c, kind, y0.data(),
                          residual_weight ? residual_weight->data() : nullptr, &r));
  return take_report(r, prob);
}
}  // namespace detail

/// estimate_dual_lipschitz, solvers.hpp:89-113 (power iteration on the device).
inline double estimate_dual_lipschitz(const FactorCache& cache, const ProblemInstance& prob,
                                      std::uint64_t* calls = nullptr, double rel_tol = 1e-6, int max_rounds = 100) {
  detail::check_shapes(cache, prob, "estimate_dual_lipschitz");
  std::uint64_t n = 0;
  double L = 0.0;
  detail::check(scenopt_estimate_lipschitz_ex(cache.state->device_for(prob), rel_tol, max_rounds, &n, &L));
  if (calls) *calls += n;
  return L;
}

/// solve_minfbe, solvers.hpp:234-356.
inline SolverReport solve_minfbe(const ProblemInstance& prob, const FactorCache& cache, const SeparableNonsmooth& g,
                                 const SolverConfig& cfg, const DualVector& y0, const Vec* residual_weight = nullptr) {
  return detail::run_solver(prob, cache, g, cfg, y0, residual_weight, 0, "solve_minfbe");
}
/// solve_nama, solvers.hpp:362-492.
inline SolverReport solve_nama(const ProblemInstance& prob, const FactorCache& cache, const SeparableNonsmooth& g,
                               const SolverConfig& cfg, const DualVector& y0, const Vec* residual_weight = nullptr) {
  return detail::run_solver(prob, cache, g, cfg, y0, residual_weight, 1, "solve_nama");
}
/// solve_gpad, solvers.hpp:498-540.
inline SolverReport solve_gpad(const ProblemInstance& prob, const FactorCache& cache, const SeparableNonsmooth& g,
                               const SolverConfig& cfg, const DualVector& y0, const Vec* residual_weight = nullptr) {
  return detail::run_solver(prob, cache, g, cfg, y0, residual_weight, 2, "solve_gpad");
}

/// warm_start, solvers.hpp:545-564.
inline DualVector warm_start(const ProblemInstance& prob, const FactorCache& cache, const SeparableNonsmooth& g,
                             const SolverConfig& cfg, double lambda, OracleStats* stats = nullptr) {
  (void)g;
  detail::check_shapes(cache, prob, "warm_start");
  DualVector y = DualVector::Zero(prob.dual_dim);
  if (cfg.warm_start_iters <= 0) return y;
  if (!(lambda > 0.0)) throw InvalidParams("warm_start: lambda must be > 0");
  const scenopt_solver_config c = detail::c_config(cfg);
  std::uint64_t calls = 0;
  detail::check(scenopt_warm_start(cache.state->device_for(prob), &c, lambda, y.data(), &calls));
  if (stats) {
    stats->dual_grad_calls += calls;
    stats->prox_calls += calls;
    stats->conj_calls += calls;
  }
  return y;
}

/// precondition, solvers.hpp:569-602.
inline ProblemInstance precondition(const ProblemInstance& prob) {
  auto h = detail::to_handle(prob);
  scenopt_problem* out = nullptr;
  detail::check(scenopt_problem_precondition(h.get(), &out));
  std::unique_ptr<scenopt_problem, detail::ProblemDeleter> o(out);
  return detail::from_handle(out);
}

/// probability_roots, solvers.hpp:608-623.
inline Vec probability_roots(const ProblemInstance& prob) {
  Vec roots(prob.dual_dim);
  for (int i = 1; i < prob.num_nodes(); ++i) {
    const double r = std::sqrt(prob.tree.probability[static_cast<size_t>(i)]);
    for (int k = 0; k < prob.stage_rows(i); ++k) roots(prob.dual_offset[static_cast<size_t>(i)] + k) = r;
  }
  for (int i = prob.tree.first_leaf(); i < prob.num_nodes(); ++i) {
    const int l = prob.leaf_ordinal(i);
    const double r = std::sqrt(prob.tree.probability[static_cast<size_t>(i)]);
    for (int k = 0; k < prob.terminal_rows(l); ++k) roots(prob.tdual_offset[static_cast<size_t>(l)] + k) = r;
  }
  return roots;
}

/// verify_report, solvers.hpp:630-639 (apply_H and dist on the device).
inline void verify_report(const ProblemInstance& prob, const SeparableNonsmooth& g, SolverReport& rep) {
  const DualVector Hx = apply_H(prob, rep.x);
  rep.verify_residual_inf = (rep.z - Hx).lpNormInf();
  rep.verify_subdiff_dist = dist_subdiff_inf(g, rep.y, rep.z);
  const double slop = 1.0 + 1e-9;
  rep.verified = rep.status == SolverStatus::Converged && rep.verify_residual_inf <= rep.eps * slop &&
                 rep.verify_subdiff_dist <= rep.lambda_final * rep.eps * slop;
}

/// solve, solvers.hpp:645-720: precondition, factor (unless shared), the
/// Lipschitz estimate, warm start, the solver run and verify_report.
inline SolverReport solve(const ProblemInstance& prob, const SolverConfig& cfg, SolverKind kind,
                          const FactorCache* shared_cache = nullptr) {
  validate_config(cfg);
  auto h = detail::to_handle(prob);
  if (shared_cache) detail::check_shapes(*shared_cache, prob, "solve");
  const scenopt_solver_config c = detail::c_config(cfg);
  scenopt_report* r = nullptr;
  detail::check(scenopt_solve(h.get(), &c, static_cast<int>(kind),
                              (shared_cache && !shared_cache->state->on_device) ? shared_cache->state->fac.get()
                                                                                : nullptr,
                              0, &r));
  return detail::take_report(r, prob);
}

// ------------------------------------------------------------------ experiment.hpp:22-283
/// One solver column of an experiment (p-NAMA: NAMA with the parallel line search).
struct SolverSpec {
  std::string name;
  SolverKind kind = SolverKind::Nama;
  bool parallel_linesearch = false;
};
inline SolverSpec solver_spec_from_name(const std::string& name) {
  if (name == "minfbe") return {"minfbe", SolverKind::Minfbe, false};
  if (name == "nama") return {"nama", SolverKind::Nama, false};
  if (name == "pnama") return {"pnama", SolverKind::Nama, true};
  if (name == "gpad") return {"gpad", SolverKind::Gpad, false};
  throw InvalidParams("unknown solver \"" + name + "\"; expected minfbe, nama, pnama, or gpad");
}
inline std::vector<SolverSpec> default_solver_set() {
  return {solver_spec_from_name("minfbe"), solver_spec_from_name("nama"), solver_spec_from_name("gpad")};
}
struct BatchEntry {
  std::string id;
  ProblemInstance prob;
};
struct ExperimentConfig {
  SolverConfig solver;
  bool include_timing = true;  ///< false zeroes wall_ms: byte-deterministic reports
  bool reuse_factors = true;   ///< one factor per factor_hash
};
struct ExperimentRow {
  std::string instance_id;
  std::string solver;
  int iterations = 0;
  std::uint64_t dual_grad_calls = 0, hessian_vec_calls = 0, prox_calls = 0;
  double final_residual_inf = std::numeric_limits<double>::infinity();
  double wall_ms = 0.0;
  bool converged = false;
  bool fbe_monotone = true;
  std::string error;
  std::vector<double> residual_trace;
  std::uint64_t oracle_calls() const { return dual_grad_calls + hessian_vec_calls; }
};
struct SolverSummary {
  std::string solver;
  int count = 0, converged = 0;
  double median_calls = 0.0, p84_calls = 0.0, p95_calls = 0.0, frac_within_50 = 0.0;
  int fbe_violations = 0;
  double total_wall_ms = 0.0;
};
inline constexpr const char* kResultsCsvHeader =
    "instance_id,solver,iterations,dual_grad_calls,hessian_vec_calls,prox_calls,final_residual_inf,wall_ms,converged";

namespace detail {
struct ExperimentDeleter { void operator()(scenopt_experiment* x) const { scenopt_experiment_destroy(x); } };
}  // namespace detail

/// RunReport (experiment.hpp:136-214). `metadata` is a JSON object text
/// (nlohmann::json in the reference); summary_json() returns the dump(2) text.
struct RunReport {
  std::vector<ExperimentRow> rows;
  std::string metadata = "{}";
  std::shared_ptr<scenopt_experiment> native;

  std::string text(int which) const {
    size_t n = 0;
    detail::check(scenopt_experiment_text(native.get(), which, metadata.c_str(), nullptr, 0, &n));
    std::string out(n + 1, '\0');
    detail::check(scenopt_experiment_text(native.get(), which, metadata.c_str(), out.data(), n + 1, &n));
    out.resize(n);
    return out;
  }
  std::string csv() const { return text(0); }
  std::string traces_csv() const { return text(1); }
  std::string summary_json() const {  // dump(2), no trailing newline
    std::string t = text(2);
    if (!t.empty() && t.back() == '\n') t.pop_back();
    return t;
  }
  std::vector<SolverSummary> summaries() const {
    std::vector<scenopt_solver_summary> raw(16);
    const int k = detail::check(scenopt_experiment_summaries(native.get(), raw.data(), 16));
    std::vector<SolverSummary> out;
    for (int i = 0; i < k; ++i) {
      const auto& s = raw[static_cast<size_t>(i)];
      out.push_back({s.solver, s.count, s.converged, s.median_calls, s.p84_calls, s.p95_calls, s.frac_within_50,
                     s.fbe_violations, s.total_wall_ms});
    }
    return out;
  }
};

/// run_experiment (experiment.hpp:222-283): every solver on every instance, in order.
inline RunReport run_experiment(const std::vector<BatchEntry>& instances, const std::vector<SolverSpec>& solvers,
                                const ExperimentConfig& cfg = {}) {
  validate_config(cfg.solver);
  std::vector<detail::ProblemPtr> hs;
  std::vector<const scenopt_problem*> ps;
  std::vector<const char*> ids;
  for (const auto& e : instances) {
    hs.push_back(detail::to_handle(e.prob));
    ps.push_back(hs.back().get());
    ids.push_back(e.id.c_str());
  }
  std::vector<const char*> names;
  for (const auto& s : solvers) names.push_back(s.name.c_str());
  const scenopt_solver_config c = detail::c_config(cfg.solver);
  scenopt_experiment* x = nullptr;
  detail::check(scenopt_run_experiment(ps.data(), ids.data(), static_cast<int>(ps.size()), names.data(),
                                       static_cast<int>(names.size()), &c, cfg.include_timing ? 1 : 0,
                                       cfg.reuse_factors ? 1 : 0, 0, &x));
  RunReport rep;
  rep.native.reset(x, detail::ExperimentDeleter{});
  const int k = scenopt_experiment_row_count(x);
  for (int i = 0; i < k; ++i) {
    scenopt_experiment_row r{};
    detail::check(scenopt_experiment_row_get(x, i, &r));
    ExperimentRow row;
    row.instance_id = r.instance_id;
    row.solver = r.solver;
    row.iterations = r.iterations;
    row.dual_grad_calls = r.dual_grad_calls;
    row.hessian_vec_calls = r.hessian_vec_calls;
    row.prox_calls = r.prox_calls;
    row.final_residual_inf = r.final_residual_inf;
    row.wall_ms = r.wall_ms;
    row.converged = r.converged != 0;
    row.fbe_monotone = r.fbe_monotone != 0;
    row.error = r.error;
    row.residual_trace.assign(r.residual_trace, r.residual_trace + r.trace_len);
    rep.rows.push_back(std::move(row));
  }
  return rep;
}

}  // namespace scenopt
