// SPDX-License-Identifier: MIT
//
// TEST INFRASTRUCTURE ONLY — CPU parity oracle for the scenopt hot path.
//
// This is an Eigen-free restatement of the reference library's algorithms
// (arXiv 2107.01745 reference, /root/reference/proj/include/scenopt/*.hpp).
// Every function cites the reference file:line it follows. It is used by
//   * tests/ (as the checker the CUDA path is compared against),
//   * __graft_entry__.smoke() (one small parity check),
//   * bench.py's cpu_baseline leg and `--impl reference` arm (timed CPU
//     implementation, "kind": "port").
// It is never linked into, loaded by, or called from the product library
// (paper_2107_01745_b200/lib/libscenopt_b200.so).
//
// Parity pinning: the reference cannot be compiled here (Eigen/Catch2 are
// absent). The restatement is pinned against every
// known-answer test the reference suite holds for this path (test_prox.cpp,
// test_scenario_tree.cpp, test_lbfgs.cpp, SPEC.md examples) and against the
// reference's own ground-truth property oracles (dense KKT solve of the
// dual-gradient subproblem, dense BFGS inverse, dense-reduction ADMM), which
// tests/ restate independently in numpy.
#pragma once

#include <cmath>
#include <cstdint>
#include <deque>
#include <limits>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

namespace orc {

// ---------------------------------------------------------------- errors
// errors.hpp:9-80. Codes are the C-ABI convention shared with the product.
enum ErrCode {
  kOk = 0,
  kError = -1,
  kNonStochasticMatrix = -2,
  kStageOutOfRange = -3,
  kDimensionMismatch = -4,
  kUnsupportedSpec = -5,
  kNotStronglyConvex = -6,
  kShapeChanged = -7,
  kCacheMismatch = -8,
  kLineSearchStalled = -9,
  kStepUnderflow = -10,
  kZeroProbability = -11,
  kInvalidParams = -12,
  kInfiniteConjugate = -13,
  kParseError = -14,
};

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
#define ORC_THROW(code, msg) throw ::orc::Error((code), (msg))

// ---------------------------------------------------------------- dense
// Minimal column-major dense matrix; the reference uses Eigen::MatrixXd
// (problem_data.hpp:13-14) which is column-major by default.
using Vec = std::vector<double>;

struct Mat {
  int r = 0, c = 0;
  std::vector<double> d;
  Mat() = default;
  Mat(int rows, int cols, double v = 0.0)
      : r(rows), c(cols), d(static_cast<size_t>(rows) * cols, v) {}
  double& operator()(int i, int j) { return d[static_cast<size_t>(i) + static_cast<size_t>(j) * r]; }
  double operator()(int i, int j) const { return d[static_cast<size_t>(i) + static_cast<size_t>(j) * r]; }
  const double* col(int j) const { return d.data() + static_cast<size_t>(j) * r; }
  double* col(int j) { return d.data() + static_cast<size_t>(j) * r; }
  static Mat identity(int n) {
    Mat m(n, n);
    for (int i = 0; i < n; ++i) m(i, i) = 1.0;
    return m;
  }
};

// y = A x (overwrite) / y += A x
void gemv(const Mat& A, const double* x, double* y, bool accumulate);
// y = A' x / y += A' x
void gemv_t(const Mat& A, const double* x, double* y, bool accumulate);
Mat matmul(const Mat& A, const Mat& B);      // A B
Mat matmul_tn(const Mat& A, const Mat& B);   // A' B
Mat matmul_nt(const Mat& A, const Mat& B);   // A B'
Mat transpose(const Mat& A);
double dot(const Vec& a, const Vec& b);
double dot(const double* a, const double* b, size_t n);
double sqnorm(const Vec& a);
double inf_norm(const Vec& a);

// Cholesky L L' of an SPD matrix (Eigen::LLT); solve(B) returns A^{-1} B.
struct Llt {
  Mat L;
  explicit Llt(const Mat& A);
  Mat solve(const Mat& B) const;
  Vec solve(const Vec& b) const;
};
double sym_min_eig(const Mat& S);   // SelfAdjointEigenSolver min eigenvalue
double sym_max_eig(const Mat& S);
double spectral_radius(const Mat& A);  // max |eig| of a general matrix

// ---------------------------------------------------------------- tree
// scenario_tree.hpp:21-43
struct ScenarioTree {
  int num_stages = 0;
  std::vector<int> node_stage;
  std::vector<int> ancestor;
  std::vector<std::vector<int>> children;
  std::vector<double> probability;
  std::vector<int> stage_offsets;
  std::vector<int> mode;
  int num_nodes() const { return static_cast<int>(node_stage.size()); }
  int num_leaves() const { return num_nodes() - stage_offsets[static_cast<size_t>(num_stages)]; }
  bool is_leaf(int i) const { return node_stage[static_cast<size_t>(i)] == num_stages; }
  int first_leaf() const { return stage_offsets[static_cast<size_t>(num_stages)]; }
};
struct NodeRange {
  int first = 0, past = 0;
  int size() const { return past - first; }
};
NodeRange nodes_at(const ScenarioTree& tree, int t1, int t2);
inline NodeRange nodes_at(const ScenarioTree& tree, int t) { return nodes_at(tree, t, t); }
ScenarioTree build_from_markov(const Mat& transition, const Vec& initial, int horizon);
std::vector<std::string> validate_tree(const ScenarioTree& tree);

// ---------------------------------------------------------------- problem
// problem_data.hpp:17-141
struct NodeDynamics { Mat A, B; Vec c; };
struct NodeCost { Mat Q, R, S; Vec q, r; };
struct TerminalCost { Mat P; Vec p; };
enum class NonsmoothKind : int { None = 0, Box = 1, ScaledL1 = 2 };
struct NonsmoothSpec {
  NonsmoothKind kind = NonsmoothKind::None;
  Vec zmin, zmax;
  double gamma = 0.0;
};
struct ConstraintBlock { Mat F, G; NonsmoothSpec g; };
struct TerminalBlock { Mat F; NonsmoothSpec g; };

struct PrimalPoint {
  Mat x;  // nx x num_nodes
  Mat u;  // nu x first_leaf
  double dot(const PrimalPoint& o) const;
};
PrimalPoint zero_primal(int nx, int nu, const ScenarioTree& tree);

struct ProblemInstance {
  ScenarioTree tree;
  int nx = 0, nu = 0;
  Vec root_state;
  std::vector<NodeDynamics> dyn;
  std::vector<NodeCost> cost;
  std::vector<TerminalCost> tcost;
  std::vector<ConstraintBlock> con;
  std::vector<TerminalBlock> tcon;
  std::vector<int> dual_offset;
  std::vector<int> tdual_offset;
  int dual_dim = 0;
  int num_nodes() const { return tree.num_nodes(); }
  int leaf_ordinal(int node) const { return node - tree.first_leaf(); }
  int primal_dim() const { return tree.first_leaf() * nu + (tree.num_nodes() - 1) * nx; }
  int stage_rows(int node) const { return con[static_cast<size_t>(node)].F.r; }
  int terminal_rows(int l) const { return tcon[static_cast<size_t>(l)].F.r; }
  void finalize_layout();
};

Vec apply_H(const ProblemInstance& prob, const PrimalPoint& pt);
PrimalPoint apply_H_adjoint(const ProblemInstance& prob, const Vec& y);
double eval_f(const ProblemInstance& prob, const PrimalPoint& pt, double feas_tol = 1e-8);
std::vector<std::string> validate_problem(const ProblemInstance& prob);

// ---------------------------------------------------------------- factor
// riccati.hpp:38-63
struct FactorCache {
  int nx = 0, nu = 0, num_nodes = 0, first_leaf = 0, dual_dim = 0;
  std::vector<Mat> gain, dual_to_input, dual_to_costate;
  std::vector<Vec> input_affine, costate_affine;
  std::vector<Mat> input_hessian;
  std::vector<int> child_dual_offset, child_dual_rows;
  std::vector<Mat> child_to_input, closed_loop, value_quad;
  std::vector<Vec> leaf_costate_affine;
};
FactorCache factor(const ProblemInstance& prob);
void refactor_affine(FactorCache& cache, const ProblemInstance& prob);

// ---------------------------------------------------------------- oracles
// tree_oracles.hpp:14-129
struct OracleStats {
  std::uint64_t dual_grad_calls = 0, hessian_vec_calls = 0, prox_calls = 0, conj_calls = 0;
  std::uint64_t sweep_total() const { return dual_grad_calls + hessian_vec_calls; }
};
PrimalPoint riccati_sweep(const FactorCache& cache, const ProblemInstance& prob,
                          const Vec& y, bool affine);
PrimalPoint dual_grad(const FactorCache& cache, const ProblemInstance& prob,
                      const Vec& y, OracleStats* stats = nullptr);
PrimalPoint hessian_vec(const FactorCache& cache, const ProblemInstance& prob,
                        const Vec& r, OracleStats* stats = nullptr);
Vec grad_fhat(const FactorCache& cache, const ProblemInstance& prob, const Vec& y,
              OracleStats* stats = nullptr);
double fhat_value(const FactorCache& cache, const ProblemInstance& prob, const Vec& y,
                  OracleStats* stats = nullptr);

// ---------------------------------------------------------------- prox
// prox.hpp:15-171
struct GBlock {
  int offset = 0, size = 0;
  double weight = 1.0;
  NonsmoothKind kind = NonsmoothKind::None;
  Vec zmin, zmax;
  double gamma = 0.0;
};
struct SeparableNonsmooth {
  std::vector<GBlock> blocks;
  int dim = 0;
};
SeparableNonsmooth make_nonsmooth(const ProblemInstance& prob);
Vec prox_g(const SeparableNonsmooth& g, const Vec& v, double gamma_prox);
double conj_value_g(const SeparableNonsmooth& g, const Vec& w, double slack = 1e-9);
Vec prox_g_conj(const SeparableNonsmooth& g, const Vec& v, double lambda);
double dist_subdiff_inf(const SeparableNonsmooth& g, const Vec& y, const Vec& z);

// ---------------------------------------------------------------- fbe
// fbe.hpp:22-231
struct FbState {
  Vec y;
  double lambda = 0.0;
  PrimalPoint x;
  Vec Hx, z, T, R;
  double fhat = 0.0, conj_T = 0.0, znorm_sq = 0.0, value = 0.0;
};
FbState fb_step(const FactorCache& cache, const ProblemInstance& prob,
                const SeparableNonsmooth& g, const Vec& y, double lambda,
                OracleStats* stats = nullptr);
void rescale_state(FbState& state, const SeparableNonsmooth& g, double lambda,
                   OracleStats* stats = nullptr);
double fbe_value(const FbState& state);
Vec fbe_grad(const FbState& state, const FactorCache& cache, const ProblemInstance& prob,
             OracleStats* stats = nullptr);

struct LineSearchCert {
  Vec anchor, dir;
  double lambda = 0.0;
  Vec Hx_anchor, Hx_dir, prox_base, prox_slope;
  double alpha1 = 0.0, alpha2 = 0.0, conj_anchor = 0.0, znorm_sq_anchor = 0.0,
         value_anchor = 0.0, fhat_anchor = 0.0;
};
struct CertEval {
  double tau = 0.0, delta = 0.0;
  Vec w, Hx_w, z, R, T;
};
LineSearchCert linesearch_cert(const FbState& state, const Vec& dir,
                               const PrimalPoint& hom_dir, const ProblemInstance& prob);
LineSearchCert linesearch_cert_shifted(const FbState& state, const SeparableNonsmooth& g,
                                       const Vec& r, const Vec& dir, const PrimalPoint& hom_r,
                                       const PrimalPoint& hom_dir, const ProblemInstance& prob,
                                       OracleStats* stats = nullptr);
double cert_fhat(const LineSearchCert& cert, double tau);
CertEval evaluate_cert(const LineSearchCert& cert, const SeparableNonsmooth& g, double tau,
                       OracleStats* stats = nullptr);

// ---------------------------------------------------------------- lbfgs
// lbfgs.hpp:22-84
class LbfgsBuffer {
 public:
  LbfgsBuffer(int memory, double eps_curv);
  bool push(const Vec& step, const Vec& change, double scale_ref);
  Vec apply_direction(const Vec& grad) const;
  void clear();
  int size() const { return static_cast<int>(pairs_.size()); }
  int memory() const { return memory_; }
  double gamma0() const { return gamma0_; }

 private:
  struct Pair { Vec step, change; double curvature; };
  int memory_;
  double eps_curv_;
  double gamma0_ = 1.0;
  std::deque<Pair> pairs_;
};

// ---------------------------------------------------------------- solvers
// solvers.hpp:21-84
enum class BacktrackingRule : int { Original = 0, Simple = 1, None = 2 };
enum class SolverKind : int { Minfbe = 0, Nama = 1, Gpad = 2 };
enum class SolverStatus : int { Converged = 0, MaxItersExceeded = 1 };
struct SolverConfig {
  double lambda0 = 0.0, eps = 5e-4, eps_curv = 1e-12, eps_bt = 0.25, beta_bt = 0.05;
  int memory = 5, max_iters = 20000;
  BacktrackingRule backtracking_rule = BacktrackingRule::Simple;
  bool warm_start = false;
  int warm_start_iters = 5;
  bool precondition = false;
  bool nama_parallel_linesearch = false;
  bool nama_update_tlambda = true;
};
void validate_config(const SolverConfig& cfg);
struct SolverReport {
  SolverStatus status = SolverStatus::MaxItersExceeded;
  PrimalPoint x;
  Vec y, z;
  double residual_inf = std::numeric_limits<double>::infinity();
  int iterations = 0;
  OracleStats stats;
  std::uint64_t lipschitz_calls = 0;
  double lipschitz_estimate = 0.0, lambda_final = 0.0, eps = 0.0;
  std::vector<double> residual_trace, fbe_trace;
  double wall_ms = 0.0;
  bool verified = false;
  double verify_residual_inf = std::numeric_limits<double>::infinity();
  double verify_subdiff_dist = std::numeric_limits<double>::infinity();
};
double estimate_dual_lipschitz(const FactorCache& cache, const ProblemInstance& prob,
                               std::uint64_t* calls = nullptr, double rel_tol = 1e-6,
                               int max_rounds = 100);
SolverReport solve_minfbe(const ProblemInstance& prob, const FactorCache& cache,
                          const SeparableNonsmooth& g, const SolverConfig& cfg, const Vec& y0,
                          const Vec* residual_weight = nullptr);
SolverReport solve_nama(const ProblemInstance& prob, const FactorCache& cache,
                        const SeparableNonsmooth& g, const SolverConfig& cfg, const Vec& y0,
                        const Vec* residual_weight = nullptr);
SolverReport solve_gpad(const ProblemInstance& prob, const FactorCache& cache,
                        const SeparableNonsmooth& g, const SolverConfig& cfg, const Vec& y0,
                        const Vec* residual_weight = nullptr);
Vec warm_start(const ProblemInstance& prob, const FactorCache& cache, const SeparableNonsmooth& g,
               const SolverConfig& cfg, double lambda, OracleStats* stats = nullptr);
ProblemInstance precondition(const ProblemInstance& prob);
Vec probability_roots(const ProblemInstance& prob);
void verify_report(const ProblemInstance& prob, const SeparableNonsmooth& g, SolverReport& rep);
SolverReport solve(const ProblemInstance& prob, const SolverConfig& cfg, SolverKind kind,
                   const FactorCache* shared_cache = nullptr);

// ---------------------------------------------------------------- generators
// generators.hpp:20-35, 236-328, extended with per-stage branching
ProblemInstance gen_random_instance(std::uint64_t seed, int nx, int nu, int horizon,
                                    const std::vector<int>& branching);

// generators.hpp:39-234: spring-mass-damper array benchmark. Empty vectors take
// the reference defaults (generators.hpp:149-162).
struct SpringMassParams {
  double mass_kg = 5.0, stiffness = 1.0, damping = 0.1, input_bound = 2.0, velocity_bound = 5.0;
  int horizon = 11;
  double sampling = 0.5, state_weight = 5.0, input_weight = 2.0, terminal_weight = 100.0;
  Vec initial_probs;
  Mat transition;
  Vec mode_values;
  Vec root_state;
};
void spring_mass_continuous(int masses, const SpringMassParams& par, Mat& A, Mat& B);
// matrix exponential by the series oracle of test_generators.cpp:23-38
// (scaling and squaring around a Taylor sum), independent of the product's Pade
Mat expm_series(Mat X);
void discretize_zoh(const Mat& A, const Mat& B, double period, Mat& Ad, Mat& Bd);
ProblemInstance gen_spring_mass(int masses, const SpringMassParams& params);
Vec sample_initial_state(int masses, const SpringMassParams& params, std::mt19937_64& gen);

// ---------------------------------------------------------------- test support
// tests/support.hpp:24-209
struct Rng {
  std::mt19937_64 gen;
  explicit Rng(std::uint64_t seed) : gen(seed) {}
  double uniform() { return static_cast<double>(gen() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
  int integer(int lo, int hi) {
    return lo + static_cast<int>(gen() % static_cast<std::uint64_t>(hi - lo + 1));
  }
  Mat matrix(int rows, int cols, double scale = 1.0);
  Vec vector(int size, double scale = 1.0);
};
ScenarioTree random_tree(Rng& rng, int stages, int max_nodes, int max_children = 3);
struct InstanceOptions {
  bool with_box = true, with_l1 = false, with_none = false, affine = true;
  int stage_rows_lo = 1, stage_rows_hi = 3;
  bool feasible_boxes = false;
};
ProblemInstance random_instance(Rng& rng, ScenarioTree tree, int nx, int nu,
                                const InstanceOptions& opt);

}  // namespace orc
