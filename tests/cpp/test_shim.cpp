// SPDX-License-Identifier: MIT
// Tests of the C++ drop-in layer (include/scenopt_b200.hpp), written against
// the reference's API exactly as the reference's own Catch2 tests use it
// (proj/tests/test_tree_oracles.cpp, test_fbe.cpp, test_lbfgs.cpp,
// test_solvers.cpp). A minimal harness replaces Catch2 (not in the image).
//   test_shim            all cases (needs an sm_100 device)
//   test_shim --host     host-only cases (no device: layout, validation,
//                        generators, errors)
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <random>
#include <string>
#include <vector>

#include "scenopt_b200.hpp"

using scenopt::Vec;

namespace {
struct Case {
  const char* name;
  bool host;
  std::function<void()> fn;
};
std::vector<Case>& cases() {
  static std::vector<Case> c;
  return c;
}
struct Reg {
  Reg(const char* n, bool host, std::function<void()> f) { cases().push_back({n, host, std::move(f)}); }
};
int g_fail = 0;
#define CAT2(a, b) a##b
#define CAT(a, b) CAT2(a, b)
#define TEST_CASE(name, host) \
  static void CAT(tc_, __LINE__)(); \
  static Reg CAT(reg_, __LINE__)(name, host, CAT(tc_, __LINE__)); \
  static void CAT(tc_, __LINE__)()
#define CHECK(cond)                                                              \
  do {                                                                           \
    if (!(cond)) {                                                               \
      std::printf("    CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond);    \
      ++g_fail;                                                                  \
    }                                                                            \
  } while (0)
#define REQUIRE(cond)                                                            \
  do {                                                                           \
    if (!(cond)) {                                                               \
      std::printf("    REQUIRE failed %s:%d: %s\n", __FILE__, __LINE__, #cond);  \
      ++g_fail;                                                                  \
      return;                                                                    \
    }                                                                            \
  } while (0)
#define CHECK_THROWS_AS(expr, type)                                              \
  do {                                                                           \
    bool ok_ = false;                                                            \
    try {                                                                        \
      (void)(expr);                                                              \
    } catch (const type&) {                                                      \
      ok_ = true;                                                                \
    } catch (...) {                                                              \
    }                                                                            \
    if (!ok_) {                                                                  \
      std::printf("    CHECK_THROWS_AS failed %s:%d: %s\n", __FILE__, __LINE__, #expr); \
      ++g_fail;                                                                  \
    }                                                                            \
  } while (0)

struct Rng {  // tests/support.hpp-style uniform draws
  std::mt19937_64 gen;
  explicit Rng(uint64_t s) : gen(s) {}
  double uniform(double lo, double hi) { return std::uniform_real_distribution<double>(lo, hi)(gen); }
  Vec vector(int n, double scale = 1.0) {
    Vec v(n);
    for (int i = 0; i < n; ++i) v(i) = uniform(-scale, scale);
    return v;
  }
};

double max_abs(const Vec& v) { return v.lpNormInf(); }
Vec flat_x(const scenopt::PrimalPoint& p) { return p.flatten(); }

scenopt::ProblemInstance small(uint64_t seed, int nx = 3, int nu = 2, int horizon = 3, int br = 2) {
  return scenopt::gen_random_instance(seed, scenopt::RandomDims{nx, nu}, scenopt::RandomTreeShape{horizon, br});
}
}  // namespace

// ---------------------------------------------------------------- host-only
TEST_CASE("generated instances are valid and laid out like the reference", true) {
  const auto prob = small(7, 3, 2, 3, 2);
  CHECK(scenopt::validate(prob).empty());
  CHECK(prob.num_nodes() == 15);
  CHECK(prob.tree.first_leaf() == 7);
  CHECK(prob.tree.stage_offsets == std::vector<int>({0, 1, 3, 7, 15}));  // test_scenario_tree.cpp:20-50
  CHECK(prob.dual_offset[0] == -1 && prob.dual_offset[1] == 0);
  int rows = 0;
  for (int i = 1; i < prob.num_nodes(); ++i) rows += prob.stage_rows(i);
  for (int l = 0; l < prob.tree.num_leaves(); ++l) rows += prob.terminal_rows(l);
  CHECK(rows == prob.dual_dim);
  CHECK(prob.primal_dim() == 7 * 2 + 14 * 3);
  // equal seeds give identical instances (generators.hpp:247-249)
  const auto again = small(7, 3, 2, 3, 2);
  CHECK(again.con[5].F(1, 2) == prob.con[5].F(1, 2) && again.cost[9].Q(2, 1) == prob.cost[9].Q(2, 1));
}

TEST_CASE("markov build: full two-mode chain is a binary tree", true) {
  scenopt::Mat P(2, 2);  // test_scenario_tree.cpp:20-50 known answers
  P << 0.1, 0.9, 0.9, 0.1;
  Vec p0(2);
  p0 << 0.5, 0.5;
  const auto tree = scenopt::build_from_markov(P, p0, 3);
  CHECK(tree.num_nodes() == 15 && tree.num_leaves() == 8 && tree.first_leaf() == 7);
  CHECK(tree.stage_offsets == std::vector<int>({0, 1, 3, 7, 15}));
  CHECK(tree.mode[0] == -1 && tree.mode[1] == 0 && tree.probability[1] == 0.5);
  const int stay = tree.children[1][0], flip = tree.children[1][1];
  CHECK(tree.mode[stay] == 0 && std::abs(tree.probability[stay] - 0.05) < 1e-15);
  CHECK(std::abs(tree.probability[flip] - 0.45) < 1e-15);
  const auto r = scenopt::nodes_at(tree, 2);
  CHECK(r.first == 3 && r.past == 7 && r.size() == 4);
  CHECK_THROWS_AS(scenopt::nodes_at(tree, 4), scenopt::StageOutOfRange);
  scenopt::Mat bad(2, 2);
  bad << 0.5, 0.6, 0.5, 0.5;
  CHECK_THROWS_AS(scenopt::build_from_markov(bad, p0, 2), scenopt::NonStochasticMatrix);
}

TEST_CASE("spring-mass defaults and documented structure (test_generators.cpp:42-93)", true) {
  const auto def = scenopt::gen_spring_mass(5);
  CHECK(def.nx == 10 && def.nu == 4 && def.tree.num_stages == 11);
  CHECK(def.num_nodes() == 4095 && def.tree.num_leaves() == 2048);
  scenopt::SpringMassParams par;
  par.horizon = 3;
  const auto prob = scenopt::gen_spring_mass(5, par);
  REQUIRE(prob.num_nodes() == 15);
  CHECK(scenopt::validate(prob).empty());
  CHECK(prob.dual_dim == 14 * 9 + 8 * 5);
  CHECK(prob.tree.probability[1] == 0.5 && prob.tree.probability[2] == 0.5);
  for (int i = 1; i < prob.num_nodes(); ++i) {
    CHECK(prob.stage_rows(i) == 9);
    CHECK(prob.cost[i].Q(3, 3) == 5.0 && prob.cost[i].Q(3, 4) == 0.0 && prob.cost[i].R(2, 2) == 2.0);
    const auto& g = prob.con[i].g;
    CHECK(g.zmin(0) == -5.0 && g.zmax(4) == 5.0 && g.zmin(5) == -2.0 && g.zmax(8) == 2.0);
  }
  CHECK(prob.dyn[1].c.lpNormInf() == 0.0 && prob.dyn[2].c(7) == 0.1);  // modes 0 / 1 at stage 1
  CHECK(prob.tcost[3].P(9, 9) == 100.0 && prob.terminal_rows(3) == 5);
}

TEST_CASE("spring-mass ZOH, free particles and parameter checks (test_generators.cpp:95-145)", true) {
  scenopt::SpringMassParams par;
  par.horizon = 1;
  for (const int masses : {2, 3, 5}) {
    const auto prob = scenopt::gen_spring_mass(masses, par);
    scenopt::Mat Ac, Bc, Ad, Bd;
    scenopt::detail::spring_mass_continuous(masses, par, Ac, Bc);
    scenopt::discretize_zoh(Ac, Bc, par.sampling, Ad, Bd);
    double d = 0.0;
    for (int j = 0; j < Ad.cols(); ++j)
      for (int i = 0; i < Ad.rows(); ++i) d = std::max(d, std::abs(Ad(i, j) - prob.dyn[1].A(i, j)));
    CHECK(d == 0.0);
  }
  par.stiffness = 0.0;
  par.damping = 0.0;
  const auto free = scenopt::gen_spring_mass(4, par);
  for (int i = 0; i < 4; ++i) {
    CHECK(std::abs(free.dyn[1].A(i, i) - 1.0) < 1e-12 && std::abs(free.dyn[1].A(4 + i, 4 + i) - 1.0) < 1e-12);
    CHECK(std::abs(free.dyn[1].A(i, 4 + i) - par.sampling) < 1e-12 && std::abs(free.dyn[1].A(4 + i, i)) < 1e-12);
  }
  CHECK_THROWS_AS(scenopt::gen_spring_mass(1), scenopt::InvalidParams);
  scenopt::SpringMassParams bad;
  bad.mass_kg = 0.0;
  CHECK_THROWS_AS(scenopt::gen_spring_mass(5, bad), scenopt::InvalidParams);
  bad = {};
  bad.mode_values = Vec::Zero(3);
  CHECK_THROWS_AS(scenopt::gen_spring_mass(5, bad), scenopt::DimensionMismatch);
  bad = {};
  bad.root_state = Vec::Zero(3);
  CHECK_THROWS_AS(scenopt::gen_spring_mass(5, bad), scenopt::DimensionMismatch);
  std::mt19937_64 ga(7), gb(7);
  const Vec sa = scenopt::sample_initial_state(5, {}, ga), sb = scenopt::sample_initial_state(5, {}, gb);
  CHECK(sa.size() == 10 && (sa - sb).lpNormInf() == 0.0 && sa.segment(5, 5).lpNormInf() <= 2.5);
}

TEST_CASE("problem files: canonical round trip, shared fields, hashes (test_io.cpp)", true) {
  const std::string chain = R"json({
  "schema": "scenopt-problem-v1", "dims": {"nx": 2, "nu": 1}, "root_state": [0.25, -0.5],
  "tree": {"stage": [0, 1, 2], "ancestor": [-1, 0, 1], "probability": [1.0, 1.0, 1.0]},
  "dynamics": {"A": [[0.9, 0.1], [0.0, 0.8]], "B": [[0.5], [1.0]], "c": [0.0, 0.0]},
  "cost": {"Q": [[1.0, 0.0], [0.0, 1.0]], "R": [[1.0]], "S": [[0.0, 0.0]], "q": [0.0, 0.0], "r": [0.0]},
  "constraints": {"F": [[1.0, 0.0]], "G": [[1.0]], "kind": "box", "zmin": [[-1.0], [-2.0]],
                  "zmax": [[1.0], [2.0]], "gamma": 0.0},
  "terminal_cost": {"P": [[1.0, 0.0], [0.0, 1.0]], "p": [0.0, 0.0]},
  "terminal_constraints": {"F": [[0.0, 1.0]], "kind": "box", "zmin": [-1.0], "zmax": [1.0], "gamma": 0.0}})json";
  const auto prob = scenopt::parse_problem(chain);
  REQUIRE(prob.num_nodes() == 3 && prob.tree.num_leaves() == 1);
  CHECK(prob.root_state(0) == 0.25 && prob.dyn[1].A(0, 0) == 0.9 && prob.dyn[2].A(0, 1) == 0.1);
  CHECK(prob.con[1].g.zmin(0) == -1.0 && prob.con[2].g.zmax(0) == 2.0);
  CHECK(scenopt::validate(prob).empty());
  for (const auto& p : {small(7), scenopt::gen_spring_mass(3, [] {
                          scenopt::SpringMassParams par;
                          par.horizon = 3;
                          return par;
                        }())}) {
    const std::string first = scenopt::serialize_problem(p);
    CHECK(scenopt::serialize_problem(scenopt::parse_problem(first)) == first);
  }
  CHECK_THROWS_AS(scenopt::parse_problem("not json at all"), scenopt::ParseError);
  CHECK(!scenopt::validate_problem_text("{\"schema\": 3}").empty());
  CHECK(scenopt::validate_problem_text(chain).empty());
  const auto base = small(5);
  auto moved = base;
  moved.root_state = Vec::Constant(base.nx, 0.01);
  CHECK(scenopt::content_hash(moved) != scenopt::content_hash(base));
  CHECK(scenopt::factor_hash(moved) == scenopt::factor_hash(base));
  auto redyn = base;
  redyn.dyn[1].A(0, 0) += 0.125;
  CHECK(scenopt::factor_hash(redyn) != scenopt::factor_hash(base));
  CHECK(scenopt::content_hash(base) == scenopt::content_hash(small(5)));
}

TEST_CASE("validate reports broken instances", true) {
  auto prob = small(8);
  prob.tree.probability[1] = 0.9;  // children no longer sum to the parent
  CHECK(!scenopt::validate(prob).empty());
  auto bad = small(8);
  bad.dyn[3].A = scenopt::Mat(2, 2);
  const auto msgs = scenopt::validate(bad);
  CHECK(!msgs.empty() && msgs.front().find("A must be") != std::string::npos);
}

TEST_CASE("preconditioning scales rows by square-root probabilities", true) {
  const auto prob = small(9);
  const auto pre = scenopt::precondition(prob);
  const Vec roots = scenopt::probability_roots(prob);
  CHECK(roots.size() == prob.dual_dim);
  const int i = 4;
  const double r = std::sqrt(prob.tree.probability[i]);
  CHECK(std::abs(pre.con[i].F(0, 1) - r * prob.con[i].F(0, 1)) < 1e-15);
  CHECK(std::abs(roots(prob.dual_offset[i]) - r) < 1e-15);
}

TEST_CASE("configuration and buffer parameters are validated", true) {
  scenopt::SolverConfig cfg;
  cfg.eps = 0.0;
  CHECK_THROWS_AS(scenopt::validate_config(cfg), scenopt::InvalidParams);
  cfg = {};
  cfg.eps_bt = 0.5;
  CHECK_THROWS_AS(scenopt::validate_config(cfg), scenopt::InvalidParams);
  CHECK_THROWS_AS(scenopt::LbfgsBuffer(0, 1e-12), scenopt::InvalidParams);  // test_lbfgs.cpp:194
  CHECK_THROWS_AS(scenopt::LbfgsBuffer(3, 0.0), scenopt::InvalidParams);
  CHECK_THROWS_AS(scenopt::gen_random_instance(1, scenopt::RandomDims{0, 2}), scenopt::InvalidParams);
}

TEST_CASE("factor() fills the reference's FactorCache members; refactor_affine refreshes them", true) {
  const auto prob = small(10);
  auto cache = scenopt::factor(prob);
  const int F = prob.tree.first_leaf(), nx = prob.nx, nu = prob.nu;
  REQUIRE(static_cast<int>(cache.gain.size()) == F && cache.members_loaded);
  REQUIRE(static_cast<int>(cache.closed_loop.size()) == prob.num_nodes());
  // closed_loop_c = A_c + B_c gain_parent (riccati.hpp:171)
  double gap = 0.0;
  for (int c = 1; c < prob.num_nodes(); ++c) {
    const int a = prob.tree.ancestor[static_cast<size_t>(c)];
    for (int i = 0; i < nx; ++i)
      for (int j = 0; j < nx; ++j) {
        double v = prob.dyn[c].A(i, j);
        for (int k = 0; k < nu; ++k) v += prob.dyn[c].B(i, k) * cache.gain[a](k, j);
        gap = std::max(gap, std::abs(v - cache.closed_loop[c](i, j)));
      }
  }
  CHECK(gap < 1e-12);
  const auto lazy = scenopt::factor(prob, scenopt::FactorMembers::on_demand);
  CHECK(lazy.gain.empty() && !lazy.members_loaded);
  const Vec before = cache.costate_affine[0];
  auto prob2 = prob;
  for (int i = 1; i < prob2.num_nodes(); ++i) prob2.cost[i].q = prob2.cost[i].q * 1.5;
  scenopt::refactor_affine(cache, prob2);
  const auto fresh = scenopt::factor(prob2);
  double agap = 0.0;
  for (int i = 0; i < F; ++i) agap = std::max(agap, max_abs(cache.costate_affine[i] - fresh.costate_affine[i]));
  CHECK(agap < 1e-12);
  CHECK(max_abs(cache.costate_affine[0] - before) > 1e-9);  // the members moved with the affine data
}

// ---------------------------------------------------------------- device
TEST_CASE("dual_grad output is dynamics-feasible", false) {
  Rng rng(41);
  const auto prob = small(11, 4, 2, 4, 2);
  const auto cache = scenopt::factor(prob);
  for (int trial = 0; trial < 5; ++trial) {
    const Vec y = rng.vector(prob.dual_dim, 2.0);
    const auto pt = scenopt::dual_grad(cache, prob, y);
    CHECK(max_abs(pt.x.col(0) - prob.root_state) < 1e-12);
    for (int i = 1; i < prob.num_nodes(); ++i) {
      const int a = prob.tree.ancestor[i];
      const Vec res = pt.x.col(i) - prob.dyn[i].A * pt.x.col(a) - prob.dyn[i].B * pt.u.col(a) - prob.dyn[i].c;
      CHECK(max_abs(res) < 1e-9 * (1.0 + max_abs(pt.x.col(i))));
    }
  }
}

TEST_CASE("hessian_vec is the homogeneous part of the affine solution map", false) {
  Rng rng(43);  // test_tree_oracles.cpp:64-81
  const auto prob = small(12, 3, 2, 4, 2);
  const auto cache = scenopt::factor(prob);
  for (int trial = 0; trial < 5; ++trial) {
    const Vec y = rng.vector(prob.dual_dim, 2.0), r = rng.vector(prob.dual_dim, 2.0);
    const Vec d = flat_x(scenopt::dual_grad(cache, prob, y + r)) - flat_x(scenopt::dual_grad(cache, prob, y));
    const Vec h = flat_x(scenopt::hessian_vec(cache, prob, r));
    REQUIRE(max_abs(d - h) < 1e-9 * (1.0 + max_abs(h)));
  }
}

TEST_CASE("dual Hessian-vector products: exactness, symmetry, curvature sign", false) {
  Rng rng(44);  // test_tree_oracles.cpp:83-109
  const auto prob = small(13, 3, 2, 3, 3);
  const auto cache = scenopt::factor(prob);
  for (int trial = 0; trial < 5; ++trial) {
    const Vec y = rng.vector(prob.dual_dim, 2.0), r = rng.vector(prob.dual_dim, 2.0);
    const Vec lhs = scenopt::grad_fhat(cache, prob, y + r) - scenopt::grad_fhat(cache, prob, y);
    const Vec rhs = -scenopt::apply_H(prob, scenopt::hessian_vec(cache, prob, r));
    REQUIRE(max_abs(lhs - rhs) < 1e-9 * (1.0 + max_abs(rhs)));
    const Vec a = rng.vector(prob.dual_dim), b = rng.vector(prob.dual_dim);
    const double ab = a.dot(-scenopt::apply_H(prob, scenopt::hessian_vec(cache, prob, b)));
    const double ba = b.dot(-scenopt::apply_H(prob, scenopt::hessian_vec(cache, prob, a)));
    CHECK(std::abs(ab - ba) <= 1e-9 * std::abs(ba) + 1e-12);
    CHECK(r.dot(rhs) > -1e-10);
  }
}

TEST_CASE("fhat gradient matches central differences of fhat_value", false) {
  Rng rng(45);  // test_tree_oracles.cpp:111-126
  const auto prob = small(14, 2, 2, 2, 2);
  const auto cache = scenopt::factor(prob);
  for (int trial = 0; trial < 5; ++trial) {
    const Vec y = rng.vector(prob.dual_dim);
    Vec d = rng.vector(prob.dual_dim);
    d /= d.norm();
    const double h = 1e-4;
    const double fd =
        (scenopt::fhat_value(cache, prob, y + h * d) - scenopt::fhat_value(cache, prob, y - h * d)) / (2.0 * h);
    const double an = scenopt::grad_fhat(cache, prob, y).dot(d);
    CHECK(std::abs(fd - an) <= 1e-6 * std::abs(an) + 1e-8);
  }
}

TEST_CASE("oracle call counters", false) {
  const auto prob = small(46, 2, 2, 2, 2);  // test_tree_oracles.cpp:128-141
  const auto cache = scenopt::factor(prob);
  scenopt::OracleStats stats;
  const Vec y = Vec::Zero(prob.dual_dim);
  scenopt::dual_grad(cache, prob, y, &stats);
  scenopt::hessian_vec(cache, prob, y, &stats);
  scenopt::hessian_vec(cache, prob, y, &stats);
  scenopt::grad_fhat(cache, prob, y, &stats);
  CHECK(stats.dual_grad_calls == 2);
  CHECK(stats.hessian_vec_calls == 2);
  CHECK(stats.sweep_total() == 4);
}

TEST_CASE("oracles reject foreign caches and bad dual lengths", false) {
  const auto prob = small(47, 2, 2, 2, 2);  // test_tree_oracles.cpp:143-152
  const auto other = small(48, 3, 2, 2, 2);
  const auto cache = scenopt::factor(prob);
  CHECK_THROWS_AS(scenopt::dual_grad(cache, other, Vec::Zero(other.dual_dim)), scenopt::CacheMismatch);
  CHECK_THROWS_AS(scenopt::hessian_vec(cache, prob, Vec::Zero(prob.dual_dim + 1)), scenopt::DimensionMismatch);
}

TEST_CASE("a second instance of the same shape is swept with the cache's matrices", false) {
  const auto prob = small(49, 3, 2, 3, 2);
  const auto twin = small(49, 3, 2, 3, 2);  // identical bytes, different object
  const auto cache = scenopt::factor(prob);
  Rng rng(50);
  const Vec y = rng.vector(prob.dual_dim);
  const Vec a = flat_x(scenopt::dual_grad(cache, prob, y)), b = flat_x(scenopt::dual_grad(cache, twin, y));
  CHECK(max_abs(a - b) == 0.0);
}

TEST_CASE("fb_step populates a consistent state", false) {
  Rng rng(51);  // test_fbe.cpp:44-79
  const auto prob = small(52, 3, 2, 3, 2);
  const auto cache = scenopt::factor(prob);
  const auto g = scenopt::make_nonsmooth(prob);
  const Vec y = rng.vector(prob.dual_dim);
  const double lambda = 0.7;
  scenopt::OracleStats stats;
  const auto s = scenopt::fb_step(cache, prob, g, y, lambda, &stats);
  CHECK(stats.dual_grad_calls == 1 && stats.prox_calls == 1 && stats.conj_calls == 1);
  CHECK(max_abs(s.Hx - scenopt::apply_H(prob, s.x)) < 1e-12 * (1.0 + max_abs(s.Hx)));
  const Vec z = scenopt::prox_g(g, y / lambda + s.Hx, 1.0 / lambda);
  CHECK(max_abs(s.z - z) < 1e-12 * (1.0 + max_abs(z)));
  CHECK(max_abs(s.R - (s.z - s.Hx)) < 1e-13 * (1.0 + max_abs(s.R)));
  CHECK(max_abs(s.T - (y - lambda * s.R)) < 1e-13 * (1.0 + max_abs(s.T)));
  const double fhat = scenopt::fhat_value(cache, prob, y);
  CHECK(std::abs(s.fhat - fhat) <= 1e-9 * (1.0 + std::abs(fhat)));
  const double value = s.fhat + s.conj_T + lambda * s.Hx.dot(s.R) + 0.5 * lambda * s.R.squaredNorm();
  CHECK(std::abs(scenopt::fbe_value(s) - value) <= 1e-9 * (1.0 + std::abs(value)));
  CHECK_THROWS_AS(scenopt::fb_step(cache, prob, g, y, 0.0), scenopt::InvalidParams);  // test_fbe.cpp:81-89
  // rescale_state at the same lambda reproduces the state (fbe.hpp:72-77)
  auto t = s;
  scenopt::rescale_state(t, g, lambda);
  CHECK(std::abs(t.value - s.value) <= 1e-12 * (1.0 + std::abs(s.value)));
  // fbe_grad = R + lambda H x0(R)
  const Vec grad = scenopt::fbe_grad(s, cache, prob);
  const Vec want = s.R + lambda * scenopt::apply_H(prob, scenopt::hessian_vec(cache, prob, s.R));
  CHECK(max_abs(grad - want) < 1e-9 * (1.0 + max_abs(want)));
}

TEST_CASE("lbfgs: empty buffer, clear resets scaling and contents", false) {
  Rng rng(87);  // test_lbfgs.cpp:31-38, 177-192
  scenopt::LbfgsBuffer buf(4, 1e-12);
  const Vec g0 = rng.vector(5);
  CHECK(max_abs(buf.apply_direction(g0) + g0) < 1e-15);
  for (int k = 0; k < 4; ++k) {
    const Vec step = rng.vector(5);
    buf.push(step, Vec(2.5 * step), 1.0);
  }
  REQUIRE(buf.size() > 0);
  CHECK(std::abs(buf.gamma0() - 0.4) < 1e-14);
  buf.clear();
  CHECK(buf.size() == 0);
  CHECK(buf.gamma0() == 1.0);
  const Vec grad = rng.vector(5);
  CHECK(max_abs(buf.apply_direction(grad) + grad) < 1e-15);
}

TEST_CASE("termination reports verify independently", false) {
  for (int trial = 0; trial < 2; ++trial) {  // test_solvers.cpp:248-270
    const auto prob = small(1203 + trial, 3, 2, 4, 2);
    const auto g = scenopt::make_nonsmooth(prob);
    scenopt::SolverConfig cfg;
    for (const auto kind : {scenopt::SolverKind::Minfbe, scenopt::SolverKind::Nama, scenopt::SolverKind::Gpad}) {
      auto rep = scenopt::solve(prob, cfg, kind);
      REQUIRE(rep.status == scenopt::SolverStatus::Converged);
      CHECK(rep.verified);
      CHECK(rep.verify_residual_inf <= cfg.eps * (1.0 + 1e-9));
      CHECK(rep.verify_subdiff_dist <= rep.lambda_final * cfg.eps * (1.0 + 1e-9));
      scenopt::verify_report(prob, g, rep);
      CHECK(rep.verified);
      for (int i = 0; i < rep.z.size(); ++i) rep.z(i) += 10.0 * cfg.eps;
      scenopt::verify_report(prob, g, rep);
      CHECK(!rep.verified);
    }
  }
}

TEST_CASE("the solver entry points agree with solve() and each other", false) {
  const auto prob = small(1300, 3, 2, 4, 2);  // test_solvers.cpp:368-386
  const auto cache = scenopt::factor(prob);
  const auto g = scenopt::make_nonsmooth(prob);
  scenopt::SolverConfig cfg;
  std::uint64_t calls = 0;
  const double L = scenopt::estimate_dual_lipschitz(cache, prob, &calls);
  CHECK(L > 0.0 && calls > 0);
  cfg.lambda0 = 0.9 / L;
  const Vec y0 = Vec::Zero(prob.dual_dim);
  const auto a = scenopt::solve_minfbe(prob, cache, g, cfg, y0);
  const auto b = scenopt::solve_nama(prob, cache, g, cfg, y0);
  REQUIRE(a.status == scenopt::SolverStatus::Converged && b.status == scenopt::SolverStatus::Converged);
  scenopt::SolverConfig dflt;
  const auto c = scenopt::solve(prob, dflt, scenopt::SolverKind::Minfbe, &cache);
  CHECK(c.iterations == a.iterations);  // solve() computes the same lambda0 = 0.9 / L
  const Vec xa = flat_x(a.x), xb = flat_x(b.x);
  CHECK(max_abs(xa - xb) < 1e-2 * (1.0 + max_abs(xa)));
  CHECK(a.stats.dual_grad_calls >= static_cast<std::uint64_t>(a.iterations));
  scenopt::SolverConfig bad;
  bad.memory = 0;
  CHECK_THROWS_AS(scenopt::solve_minfbe(prob, cache, g, bad, y0), scenopt::InvalidParams);
}

TEST_CASE("factor_device and refactor_affine (receding horizon)", false) {
  auto prob = small(61, 4, 2, 4, 2);
  auto cache = scenopt::factor_device(prob);
  const auto host = scenopt::factor(prob);
  Rng rng(62);
  const Vec y = rng.vector(prob.dual_dim);
  const Vec a = flat_x(scenopt::dual_grad(cache, prob, y)), b = flat_x(scenopt::dual_grad(host, prob, y));
  CHECK(max_abs(a - b) < 1e-10 * (1.0 + max_abs(b)));
  // new initial state and linear costs, same matrices
  auto prob2 = prob;
  prob2.root_state = rng.vector(prob.nx, 0.1);
  for (int i = 1; i < prob2.num_nodes(); ++i) prob2.cost[i].q = prob2.cost[i].q * 1.05;
  scenopt::refactor_affine(cache, prob2);
  const auto fresh = scenopt::factor(prob2);
  const Vec c2 = flat_x(scenopt::dual_grad(cache, prob2, y)), d2 = flat_x(scenopt::dual_grad(fresh, prob2, y));
  CHECK(max_abs(c2 - d2) < 1e-10 * (1.0 + max_abs(d2)));
  CHECK(max_abs(c2.segment(prob.tree.first_leaf() * prob.nu, prob.nx) - prob2.root_state) < 1e-14);
  cache.load_matrices(prob2);
  CHECK(static_cast<int>(cache.gain.size()) == prob.tree.first_leaf());
}

TEST_CASE("run_experiment: rows, pinned csv header, byte-stable reports (test_experiment.cpp)", false) {
  std::vector<scenopt::BatchEntry> batch;
  for (int k = 0; k < 3; ++k) batch.push_back({"r" + std::to_string(k + 1), small(static_cast<uint64_t>(k + 1))});
  scenopt::ExperimentConfig cfg;
  cfg.include_timing = false;
  const auto a = scenopt::run_experiment(batch, scenopt::default_solver_set(), cfg);
  const auto b = scenopt::run_experiment(batch, scenopt::default_solver_set(), cfg);
  REQUIRE(a.rows.size() == 9);
  for (const auto& r : a.rows) {
    CHECK(r.converged && r.error.empty());
    if (r.solver != "gpad") CHECK(r.fbe_monotone);  // GPAD records the envelope too, not monotone (solvers.hpp:518)
  }
  const std::string csv = a.csv();
  CHECK(csv.substr(0, csv.find('\n')) == scenopt::kResultsCsvHeader);
  CHECK(csv == b.csv() && a.traces_csv() == b.traces_csv() && a.summary_json() == b.summary_json());
  const auto sums = a.summaries();
  REQUIRE(sums.size() == 3);
  CHECK(sums[0].solver == "minfbe" && sums[0].count == 3 && sums[0].converged == 3);
  CHECK_THROWS_AS(scenopt::solver_spec_from_name("bfgs"), scenopt::InvalidParams);
}

int main(int argc, char** argv) {
  const bool host_only = argc > 1 && std::strcmp(argv[1], "--host") == 0;
  int run = 0;
  for (const Case& c : cases()) {
    if (host_only && !c.host) continue;
    const int before = g_fail;
    try {
      c.fn();
    } catch (const std::exception& e) {
      std::printf("    unexpected exception: %s\n", e.what());
      ++g_fail;
    }
    std::printf("%s %s\n", g_fail == before ? "ok  " : "FAIL", c.name);
    ++run;
  }
  std::printf("%d cases, %d failed checks\n", run, g_fail);
  return g_fail == 0 ? 0 : 1;
}
