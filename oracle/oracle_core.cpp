// SPDX-License-Identifier: MIT
// TEST INFRASTRUCTURE ONLY — CPU parity oracle, see oracle_core.hpp header.
// Each function names the reference file:line it restates
// (/root/reference/proj/include/scenopt/...).
#include "oracle_core.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <thread>
#include <utility>

namespace orc {

namespace {
void axpy(double a, const Vec& x, Vec& y) {
  for (size_t i = 0; i < y.size(); ++i) y[i] += a * x[i];
}
Vec lincomb(const Vec& a, double s, const Vec& b) {  // a + s b
  Vec out(a.size());
  for (size_t i = 0; i < a.size(); ++i) out[i] = a[i] + s * b[i];
  return out;
}
Vec sub(const Vec& a, const Vec& b) {
  Vec out(a.size());
  for (size_t i = 0; i < a.size(); ++i) out[i] = a[i] - b[i];
  return out;
}
Vec scaled(const Vec& a, double s) {
  Vec out(a.size());
  for (size_t i = 0; i < a.size(); ++i) out[i] = a[i] * s;
  return out;
}
Mat scaled(const Mat& a, double s) {
  Mat out = a;
  for (auto& v : out.d) v *= s;
  return out;
}
void add_into(Mat& a, const Mat& b) {
  for (size_t i = 0; i < a.d.size(); ++i) a.d[i] += b.d[i];
}
}  // namespace

// ============================================================ tree
// scenario_tree.hpp:52-59
NodeRange nodes_at(const ScenarioTree& tree, int t1, int t2) {
  if (t1 < 0 || t2 > tree.num_stages || t1 > t2)
    ORC_THROW(kStageOutOfRange, "nodes_at: stage range [" + std::to_string(t1) + ", " +
                                    std::to_string(t2) + "] outside [0, " +
                                    std::to_string(tree.num_stages) + "]");
  return NodeRange{tree.stage_offsets[static_cast<size_t>(t1)],
                   tree.stage_offsets[static_cast<size_t>(t2) + 1]};
}

// scenario_tree.hpp:72-123
ScenarioTree build_from_markov(const Mat& transition, const Vec& initial, int horizon) {
  const int num_modes = static_cast<int>(initial.size());
  if (horizon < 1) ORC_THROW(kInvalidParams, "build_from_markov: horizon must be >= 1");
  if (transition.r != num_modes || transition.c != num_modes)
    ORC_THROW(kDimensionMismatch,
              "build_from_markov: transition must be square and match the initial "
              "distribution size");
  constexpr double kStochTol = 1e-9;
  double isum = 0.0, imin = 1e300;
  for (double v : initial) {
    isum += v;
    imin = std::min(imin, v);
  }
  if (imin < 0.0 || std::abs(isum - 1.0) > kStochTol)
    ORC_THROW(kNonStochasticMatrix, "build_from_markov: initial distribution");
  for (int w = 0; w < num_modes; ++w) {
    double s = 0.0, mn = 1e300;
    for (int j = 0; j < num_modes; ++j) {
      s += transition(w, j);
      mn = std::min(mn, transition(w, j));
    }
    if (mn < 0.0 || std::abs(s - 1.0) > kStochTol)
      ORC_THROW(kNonStochasticMatrix, "build_from_markov: transition row " + std::to_string(w));
  }
  ScenarioTree tree;
  tree.num_stages = horizon;
  tree.node_stage = {0};
  tree.ancestor = {-1};
  tree.children = {{}};
  tree.probability = {1.0};
  tree.mode = {-1};
  tree.stage_offsets = {0, 1};
  int stage_begin = 0, stage_end = 1;
  for (int t = 0; t < horizon; ++t) {
    for (int i = stage_begin; i < stage_end; ++i) {
      for (int w = 0; w < num_modes; ++w) {
        const double branch =
            (t == 0) ? initial[static_cast<size_t>(w)]
                     : transition(tree.mode[static_cast<size_t>(i)], w);
        if (branch <= 0.0) continue;
        const int id = tree.num_nodes();
        tree.node_stage.push_back(t + 1);
        tree.ancestor.push_back(i);
        tree.children.emplace_back();
        tree.probability.push_back(tree.probability[static_cast<size_t>(i)] * branch);
        tree.mode.push_back(w);
        tree.children[static_cast<size_t>(i)].push_back(id);
      }
    }
    stage_begin = stage_end;
    stage_end = tree.num_nodes();
    tree.stage_offsets.push_back(stage_end);
  }
  return tree;
}

// scenario_tree.hpp:128-240
std::vector<std::string> validate_tree(const ScenarioTree& tree) {
  std::vector<std::string> bad;
  auto complain = [&bad](const std::string& m) { bad.push_back(m); };
  constexpr double kTol = 1e-9;
  const int n = tree.num_nodes();
  if (tree.num_stages < 1) complain("tree: num_stages must be >= 1");
  if (n == 0) {
    complain("tree: empty");
    return bad;
  }
  if (static_cast<int>(tree.ancestor.size()) != n ||
      static_cast<int>(tree.children.size()) != n ||
      static_cast<int>(tree.probability.size()) != n) {
    complain("tree: per-node array sizes disagree");
    return bad;
  }
  if (static_cast<int>(tree.stage_offsets.size()) != tree.num_stages + 2) {
    complain("tree: stage_offsets must have num_stages + 2 entries");
    return bad;
  }
  if (!tree.mode.empty() && static_cast<int>(tree.mode.size()) != n)
    complain("tree: mode labels present but not one per node");
  if (tree.stage_offsets.front() != 0 || tree.stage_offsets.back() != n)
    complain("tree: stage_offsets must start at 0 and end at num_nodes");
  for (int t = 0; t <= tree.num_stages; ++t)
    if (tree.stage_offsets[static_cast<size_t>(t)] >= tree.stage_offsets[static_cast<size_t>(t) + 1])
      complain("stage " + std::to_string(t) + ": empty stage");
  if (tree.node_stage[0] != 0) complain("node 0: root must have stage 0");
  if (tree.ancestor[0] != -1) complain("node 0: root must have ancestor -1");
  if (std::abs(tree.probability[0] - 1.0) > kTol) complain("node 0: root probability must be 1");
  for (int i = 0; i < n; ++i) {
    const auto si = static_cast<size_t>(i);
    const int t = tree.node_stage[si];
    if (t < 0 || t > tree.num_stages) {
      complain("node " + std::to_string(i) + ": stage out of range");
      continue;
    }
    if (i < tree.stage_offsets[static_cast<size_t>(t)] ||
        i >= tree.stage_offsets[static_cast<size_t>(t) + 1])
      complain("node " + std::to_string(i) + ": id not inside its stage's offset range");
    if (!(tree.probability[si] > 0.0) || tree.probability[si] > 1.0 + kTol)
      complain("node " + std::to_string(i) + ": probability not in (0, 1]");
    if (i > 0) {
      const int a = tree.ancestor[si];
      if (a < 0 || a >= i) {
        complain("node " + std::to_string(i) + ": ancestor id must be smaller than the node's own id");
      } else {
        if (tree.node_stage[static_cast<size_t>(a)] != t - 1)
          complain("node " + std::to_string(i) + ": ancestor is not one stage earlier");
        const auto& sibs = tree.children[static_cast<size_t>(a)];
        if (std::find(sibs.begin(), sibs.end(), i) == sibs.end())
          complain("node " + std::to_string(i) + ": missing from its ancestor's child list");
      }
    }
    if (t == tree.num_stages) {
      if (!tree.children[si].empty()) complain("node " + std::to_string(i) + ": leaf with children");
    } else {
      if (tree.children[si].empty())
        complain("node " + std::to_string(i) +
                 ": interior node without children (leaves must sit at the final stage)");
      double mass = 0.0;
      for (int c : tree.children[si]) {
        if (c <= i || c >= n) {
          complain("node " + std::to_string(i) + ": child id out of range");
          continue;
        }
        if (tree.ancestor[static_cast<size_t>(c)] != i)
          complain("node " + std::to_string(i) + ": child " + std::to_string(c) +
                   " does not point back");
        mass += tree.probability[static_cast<size_t>(c)];
      }
      if (std::abs(mass - tree.probability[si]) > kTol)
        complain("node " + std::to_string(i) +
                 ": children probabilities do not sum to the node's own");
    }
  }
  for (int t = 0; t <= tree.num_stages; ++t) {
    double mass = 0.0;
    for (int i = tree.stage_offsets[static_cast<size_t>(t)];
         i < tree.stage_offsets[static_cast<size_t>(t) + 1]; ++i)
      mass += tree.probability[static_cast<size_t>(i)];
    if (std::abs(mass - 1.0) > kTol)
      complain("stage " + std::to_string(t) + ": probabilities do not sum to 1");
  }
  for (int i = 1; i + 1 < n; ++i)
    if (tree.node_stage[static_cast<size_t>(i)] == tree.node_stage[static_cast<size_t>(i) + 1] &&
        tree.ancestor[static_cast<size_t>(i)] > tree.ancestor[static_cast<size_t>(i) + 1])
      complain("node " + std::to_string(i + 1) +
               ": siblings out of BFS order (ancestor ids must be nondecreasing within a stage)");
  return bad;
}

// ============================================================ problem
double PrimalPoint::dot(const PrimalPoint& o) const {  // problem_data.hpp:74-76
  return orc::dot(u.d, o.u.d) + orc::dot(x.d, o.x.d);
}
PrimalPoint zero_primal(int nx, int nu, const ScenarioTree& tree) {  // problem_data.hpp:79-82
  return PrimalPoint{Mat(nx, tree.num_nodes()), Mat(nu, tree.first_leaf())};
}

// problem_data.hpp:126-140
void ProblemInstance::finalize_layout() {
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

// problem_data.hpp:144-162
Vec apply_H(const ProblemInstance& prob, const PrimalPoint& pt) {
  if (pt.x.r != prob.nx || pt.x.c != prob.num_nodes() || pt.u.r != prob.nu ||
      pt.u.c != prob.tree.first_leaf())
    ORC_THROW(kDimensionMismatch, "apply_H: point does not match the instance");
  Vec z(static_cast<size_t>(prob.dual_dim), 0.0);
  for (int i = 1; i < prob.num_nodes(); ++i) {
    const auto& blk = prob.con[static_cast<size_t>(i)];
    const int a = prob.tree.ancestor[static_cast<size_t>(i)];
    double* zi = z.data() + prob.dual_offset[static_cast<size_t>(i)];
    gemv(blk.F, pt.x.col(a), zi, false);
    gemv(blk.G, pt.u.col(a), zi, true);
  }
  for (int i = prob.tree.first_leaf(); i < prob.num_nodes(); ++i) {
    const int l = prob.leaf_ordinal(i);
    const auto& blk = prob.tcon[static_cast<size_t>(l)];
    gemv(blk.F, pt.x.col(i), z.data() + prob.tdual_offset[static_cast<size_t>(l)], false);
  }
  return z;
}

// problem_data.hpp:168-189
PrimalPoint apply_H_adjoint(const ProblemInstance& prob, const Vec& y) {
  if (static_cast<int>(y.size()) != prob.dual_dim)
    ORC_THROW(kDimensionMismatch, "apply_H_adjoint: dual vector has wrong length");
  PrimalPoint out = zero_primal(prob.nx, prob.nu, prob.tree);
  for (int i = 1; i < prob.num_nodes(); ++i) {
    const auto& blk = prob.con[static_cast<size_t>(i)];
    const int a = prob.tree.ancestor[static_cast<size_t>(i)];
    const double* yi = y.data() + prob.dual_offset[static_cast<size_t>(i)];
    gemv_t(blk.F, yi, out.x.col(a), true);
    gemv_t(blk.G, yi, out.u.col(a), true);
  }
  for (int i = prob.tree.first_leaf(); i < prob.num_nodes(); ++i) {
    const int l = prob.leaf_ordinal(i);
    const auto& blk = prob.tcon[static_cast<size_t>(l)];
    gemv_t(blk.F, y.data() + prob.tdual_offset[static_cast<size_t>(l)], out.x.col(i), true);
  }
  return out;
}

// problem_data.hpp:194-222
double eval_f(const ProblemInstance& prob, const PrimalPoint& pt, double feas_tol) {
  constexpr double kInf = std::numeric_limits<double>::infinity();
  const int nx = prob.nx, nu = prob.nu;
  for (int k = 0; k < nx; ++k)
    if (std::abs(pt.x(k, 0) - prob.root_state[static_cast<size_t>(k)]) > feas_tol) return kInf;
  Vec res(static_cast<size_t>(nx));
  for (int i = 1; i < prob.num_nodes(); ++i) {
    const auto& d = prob.dyn[static_cast<size_t>(i)];
    const int a = prob.tree.ancestor[static_cast<size_t>(i)];
    gemv(d.A, pt.x.col(a), res.data(), false);
    gemv(d.B, pt.u.col(a), res.data(), true);
    for (int k = 0; k < nx; ++k)
      if (std::abs(pt.x(k, i) - res[static_cast<size_t>(k)] - d.c[static_cast<size_t>(k)]) > feas_tol)
        return kInf;
  }
  double total = 0.0;
  Vec tx(static_cast<size_t>(nx)), tu(static_cast<size_t>(nu));
  for (int i = 1; i < prob.num_nodes(); ++i) {
    const auto& c = prob.cost[static_cast<size_t>(i)];
    const int a = prob.tree.ancestor[static_cast<size_t>(i)];
    const double pi = prob.tree.probability[static_cast<size_t>(i)];
    const double* xa = pt.x.col(a);
    const double* ua = pt.u.col(a);
    gemv(c.Q, xa, tx.data(), false);
    const double xQx = dot(xa, tx.data(), static_cast<size_t>(nx));
    gemv(c.R, ua, tu.data(), false);
    const double uRu = dot(ua, tu.data(), static_cast<size_t>(nu));
    gemv(c.S, xa, tu.data(), false);
    const double uSx = dot(ua, tu.data(), static_cast<size_t>(nu));
    total += pi * (xQx + uRu + 2.0 * uSx + dot(c.q.data(), xa, static_cast<size_t>(nx)) +
                   dot(c.r.data(), ua, static_cast<size_t>(nu)));
  }
  for (int i = prob.tree.first_leaf(); i < prob.num_nodes(); ++i) {
    const auto& c = prob.tcost[static_cast<size_t>(prob.leaf_ordinal(i))];
    const double pi = prob.tree.probability[static_cast<size_t>(i)];
    const double* xi = pt.x.col(i);
    gemv(c.P, xi, tx.data(), false);
    total += pi * (dot(xi, tx.data(), static_cast<size_t>(nx)) +
                   dot(c.p.data(), xi, static_cast<size_t>(nx)));
  }
  return total;
}

// problem_data.hpp:233-314
std::vector<std::string> validate_problem(const ProblemInstance& prob) {
  std::vector<std::string> bad = validate_tree(prob.tree);
  auto complain = [&bad](const std::string& m) { bad.push_back(m); };
  const int n = prob.num_nodes();
  const int nx = prob.nx, nu = prob.nu;
  if (nx <= 0 || nu <= 0) complain("instance: nx and nu must be positive");
  if (static_cast<int>(prob.root_state.size()) != nx)
    complain("instance: root_state must have length nx");
  if (static_cast<int>(prob.dyn.size()) != n || static_cast<int>(prob.cost.size()) != n ||
      static_cast<int>(prob.con.size()) != n) {
    complain("instance: per-node containers must have one entry per node");
    return bad;
  }
  if (static_cast<int>(prob.tcost.size()) != prob.tree.num_leaves() ||
      static_cast<int>(prob.tcon.size()) != prob.tree.num_leaves()) {
    complain("instance: per-leaf containers must have one entry per leaf");
    return bad;
  }
  auto check_spec = [&](const NonsmoothSpec& g, int rows, const std::string& where) {
    switch (g.kind) {
      case NonsmoothKind::None:
        break;
      case NonsmoothKind::Box:
        if (static_cast<int>(g.zmin.size()) != rows || static_cast<int>(g.zmax.size()) != rows) {
          complain(where + ": box bounds must match the block's row count");
        } else {
          double mn = 1e300;
          for (int j = 0; j < rows; ++j)
            mn = std::min(mn, g.zmax[static_cast<size_t>(j)] - g.zmin[static_cast<size_t>(j)]);
          if (rows > 0 && mn < 0.0) complain(where + ": box needs zmin <= zmax");
        }
        break;
      case NonsmoothKind::ScaledL1:
        if (!(g.gamma > 0.0)) complain(where + ": scaled_l1 needs gamma > 0");
        break;
    }
  };
  for (int i = 1; i < n; ++i) {
    const auto si = static_cast<size_t>(i);
    const std::string where = "node " + std::to_string(i);
    const auto& d = prob.dyn[si];
    if (d.A.r != nx || d.A.c != nx || d.B.r != nx || d.B.c != nu ||
        static_cast<int>(d.c.size()) != nx)
      complain(where + ": dynamics dimensions");
    const auto& c = prob.cost[si];
    if (c.Q.r != nx || c.Q.c != nx || c.R.r != nu || c.R.c != nu || c.S.r != nu || c.S.c != nx ||
        static_cast<int>(c.q.size()) != nx || static_cast<int>(c.r.size()) != nu) {
      complain(where + ": cost dimensions");
    } else {
      if (sym_min_eig(c.R) < 1e-10) complain(where + ": R must be positive definite");
      Mat blk(nx + nu, nx + nu);
      for (int j = 0; j < nx; ++j)
        for (int k = 0; k < nx; ++k) blk(k, j) = c.Q(k, j);
      for (int j = 0; j < nu; ++j)
        for (int k = 0; k < nx; ++k) blk(k, nx + j) = c.S(j, k);
      for (int j = 0; j < nx; ++j)
        for (int k = 0; k < nu; ++k) blk(nx + k, j) = c.S(k, j);
      for (int j = 0; j < nu; ++j)
        for (int k = 0; k < nu; ++k) blk(nx + k, nx + j) = c.R(k, j);
      if (sym_min_eig(blk) < -1e-10)
        complain(where + ": cost block [[Q, S'], [S, R]] must be positive semidefinite");
    }
    const auto& b = prob.con[si];
    if (b.F.c != nx || b.G.c != nu || b.F.r != b.G.r) complain(where + ": constraint block dimensions");
    check_spec(b.g, b.F.r, where + " stage block");
  }
  for (int l = 0; l < prob.tree.num_leaves(); ++l) {
    const auto sl = static_cast<size_t>(l);
    const std::string where = "leaf " + std::to_string(l);
    const auto& c = prob.tcost[sl];
    if (c.P.r != nx || c.P.c != nx || static_cast<int>(c.p.size()) != nx)
      complain(where + ": terminal cost dimensions");
    else if (sym_min_eig(c.P) < 1e-10)
      complain(where + ": P_N must be positive definite");
    const auto& b = prob.tcon[sl];
    if (b.F.c != nx) complain(where + ": terminal block dimensions");
    check_spec(b.g, b.F.r, where + " terminal block");
  }
  if (prob.dual_offset.size() != static_cast<size_t>(n))
    complain("instance: finalize_layout() has not been run");
  return bad;
}

// ============================================================ factor
static void check_shapes(const FactorCache& cache, const ProblemInstance& prob, const char* who) {
  // riccati.hpp:67-74
  if (cache.num_nodes != prob.num_nodes() || cache.nx != prob.nx || cache.nu != prob.nu ||
      cache.dual_dim != prob.dual_dim || cache.first_leaf != prob.tree.first_leaf())
    ORC_THROW(kCacheMismatch, std::string(who) + ": cache was built for a different problem shape");
}

// riccati.hpp:82-182
FactorCache factor(const ProblemInstance& prob) {
  const int nx = prob.nx, nu = prob.nu;
  const int n = prob.num_nodes();
  const auto& tree = prob.tree;
  FactorCache cache;
  cache.nx = nx;
  cache.nu = nu;
  cache.num_nodes = n;
  cache.first_leaf = tree.first_leaf();
  cache.dual_dim = prob.dual_dim;
  const auto nl = static_cast<size_t>(cache.first_leaf);
  cache.gain.resize(nl);
  cache.dual_to_input.resize(nl);
  cache.dual_to_costate.resize(nl);
  cache.input_affine.resize(nl);
  cache.costate_affine.resize(nl);
  cache.input_hessian.resize(nl);
  cache.child_dual_offset.resize(nl);
  cache.child_dual_rows.resize(nl);
  cache.child_to_input.resize(static_cast<size_t>(n));
  cache.closed_loop.resize(static_cast<size_t>(n));
  cache.value_quad.resize(static_cast<size_t>(n));
  cache.leaf_costate_affine.resize(static_cast<size_t>(tree.num_leaves()));

  for (int i = cache.first_leaf; i < n; ++i) {
    const auto si = static_cast<size_t>(i);
    const int l = prob.leaf_ordinal(i);
    const auto& tc = prob.tcost[static_cast<size_t>(l)];
    const double pi = tree.probability[si];
    cache.value_quad[si] = scaled(tc.P, pi);
    cache.leaf_costate_affine[static_cast<size_t>(l)] = scaled(tc.p, pi);
  }

  for (int t = tree.num_stages - 1; t >= 0; --t) {
    const NodeRange rng = nodes_at(tree, t);
    // Nodes of one stage are independent (riccati.hpp:115-180 loops them in
    // order); the oracle runs them on host threads to keep setup time
    // bounded. Each node's arithmetic is the serial restatement below, so
    // results are identical to a serial run.
    auto node = [&](int i) {
      const auto si = static_cast<size_t>(i);
      const auto& kids = tree.children[si];
      Mat huu(nu, nu), hux(nu, nx), hxx(nx, nx);
      Vec su(static_cast<size_t>(nu), 0.0), sx(static_cast<size_t>(nx), 0.0);
      int mrows = 0;
      for (int c : kids) {
        const auto sc = static_cast<size_t>(c);
        const double pc = tree.probability[sc];
        const auto& d = prob.dyn[sc];
        const auto& cc = prob.cost[sc];
        const Mat PB = matmul(cache.value_quad[sc], d.B);
        const Mat PA = matmul(cache.value_quad[sc], d.A);
        Mat t1 = scaled(cc.R, pc);
        add_into(t1, matmul_tn(d.B, PB));
        add_into(huu, t1);
        Mat t2 = scaled(cc.S, pc);
        add_into(t2, matmul_tn(d.B, PA));
        add_into(hux, t2);
        Mat t3 = scaled(cc.Q, pc);
        add_into(t3, matmul_tn(d.A, PA));
        add_into(hxx, t3);
        Vec pc2(static_cast<size_t>(nx));
        gemv(cache.value_quad[sc], d.c.data(), pc2.data(), false);
        for (auto& v : pc2) v *= 2.0;
        Vec tu = scaled(cc.r, pc);
        gemv_t(d.B, pc2.data(), tu.data(), true);
        axpy(1.0, tu, su);
        Vec tx = scaled(cc.q, pc);
        gemv_t(d.A, pc2.data(), tx.data(), true);
        axpy(1.0, tx, sx);
        mrows += prob.stage_rows(c);
      }
      {
        Mat h2(nu, nu);
        for (int j = 0; j < nu; ++j)
          for (int k = 0; k < nu; ++k) h2(k, j) = 0.5 * (huu(k, j) + huu(j, k));
        huu = h2;
      }
      if (sym_min_eig(huu) < 1e-10)
        ORC_THROW(kNotStronglyConvex, "factor: eliminated input Hessian at node " +
                                          std::to_string(i) + " has min eigenvalue below 1e-10");
      const Llt llt(huu);
      cache.input_hessian[si] = huu;
      cache.gain[si] = scaled(llt.solve(hux), -1.0);
      cache.input_affine[si] = scaled(llt.solve(su), -0.5);
      {
        Vec ca = sx;
        gemv_t(cache.gain[si], su.data(), ca.data(), true);
        cache.costate_affine[si] = ca;
      }
      cache.child_dual_rows[si] = mrows;
      cache.child_dual_offset[si] = prob.dual_offset[static_cast<size_t>(kids.front())];
      Mat gt(nu, mrows), dt(nx, mrows);
      int col = 0;
      for (int c : kids) {
        const auto sc = static_cast<size_t>(c);
        const auto& blk = prob.con[sc];
        const int rows = blk.F.r;
        Mat fg = blk.F;  // F + G gain
        add_into(fg, matmul(blk.G, cache.gain[si]));
        for (int r = 0; r < rows; ++r) {
          for (int k = 0; k < nu; ++k) gt(k, col + r) = blk.G(r, k);
          for (int k = 0; k < nx; ++k) dt(k, col + r) = fg(r, k);
        }
        cache.child_to_input[sc] = scaled(llt.solve(transpose(prob.dyn[sc].B)), -0.5);
        Mat cl = prob.dyn[sc].A;
        add_into(cl, matmul(prob.dyn[sc].B, cache.gain[si]));
        cache.closed_loop[sc] = cl;
        col += rows;
      }
      cache.dual_to_input[si] = scaled(llt.solve(gt), -0.5);
      cache.dual_to_costate[si] = dt;
      Mat value = hxx;
      add_into(value, matmul_tn(hux, cache.gain[si]));
      Mat vq(nx, nx);
      for (int j = 0; j < nx; ++j)
        for (int k = 0; k < nx; ++k) vq(k, j) = 0.5 * (value(k, j) + value(j, k));
      cache.value_quad[si] = vq;
    };
    const int cnt = rng.past - rng.first;
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const int nth = static_cast<int>(std::min<unsigned>(hw, static_cast<unsigned>((cnt + 15) / 16)));
    std::vector<std::string> errs(static_cast<size_t>(std::max(nth, 1)));
    auto run = [&](int tix) {
      try {
        for (int i = rng.first + tix; i < rng.past; i += std::max(nth, 1)) node(i);
      } catch (const Error& e) {
        errs[static_cast<size_t>(tix)] = e.what();
      }
    };
    if (nth <= 1) {
      run(0);
    } else {
      std::vector<std::thread> pool;
      for (int tix = 0; tix < nth; ++tix) pool.emplace_back(run, tix);
      for (auto& th : pool) th.join();
    }
    for (const auto& e : errs)
      if (!e.empty()) ORC_THROW(kNotStronglyConvex, e);
  }
  return cache;
}

// riccati.hpp:187-216
void refactor_affine(FactorCache& cache, const ProblemInstance& prob) {
  if (cache.num_nodes != prob.num_nodes() || cache.nx != prob.nx || cache.nu != prob.nu ||
      cache.dual_dim != prob.dual_dim || cache.first_leaf != prob.tree.first_leaf())
    ORC_THROW(kShapeChanged, "refactor_affine: problem shape changed since factor()");
  const auto& tree = prob.tree;
  for (int i = cache.first_leaf; i < cache.num_nodes; ++i) {
    const int l = prob.leaf_ordinal(i);
    cache.leaf_costate_affine[static_cast<size_t>(l)] =
        scaled(prob.tcost[static_cast<size_t>(l)].p, tree.probability[static_cast<size_t>(i)]);
  }
  for (int i = 0; i < cache.first_leaf; ++i) {
    const auto si = static_cast<size_t>(i);
    Vec su(static_cast<size_t>(cache.nu), 0.0), sx(static_cast<size_t>(cache.nx), 0.0);
    for (int c : tree.children[si]) {
      const auto sc = static_cast<size_t>(c);
      const double pc = tree.probability[sc];
      const auto& d = prob.dyn[sc];
      Vec pc2(static_cast<size_t>(cache.nx));
      gemv(cache.value_quad[sc], d.c.data(), pc2.data(), false);
      for (auto& v : pc2) v *= 2.0;
      Vec tu = scaled(prob.cost[sc].r, pc);
      gemv_t(d.B, pc2.data(), tu.data(), true);
      axpy(1.0, tu, su);
      Vec tx = scaled(prob.cost[sc].q, pc);
      gemv_t(d.A, pc2.data(), tx.data(), true);
      axpy(1.0, tx, sx);
    }
    const Llt llt(cache.input_hessian[si]);
    cache.input_affine[si] = scaled(llt.solve(su), -0.5);
    Vec ca = sx;
    gemv_t(cache.gain[si], su.data(), ca.data(), true);
    cache.costate_affine[si] = ca;
  }
}

// ============================================================ oracles
// tree_oracles.hpp:33-90
PrimalPoint riccati_sweep(const FactorCache& cache, const ProblemInstance& prob, const Vec& y,
                          bool affine) {
  if (static_cast<int>(y.size()) != cache.dual_dim)
    ORC_THROW(kDimensionMismatch, "riccati_sweep: dual vector has wrong length");
  const auto& tree = prob.tree;
  const int n = cache.num_nodes;
  Mat costate(cache.nx, n);
  PrimalPoint out = zero_primal(cache.nx, cache.nu, tree);
  for (int i = cache.first_leaf; i < n; ++i) {  // :44-52
    const int l = prob.leaf_ordinal(i);
    const auto sl = static_cast<size_t>(l);
    const auto& blk = prob.tcon[sl];
    gemv_t(blk.F, y.data() + prob.tdual_offset[sl], costate.col(i), false);
    if (affine)
      for (int k = 0; k < cache.nx; ++k) costate(k, i) += cache.leaf_costate_affine[sl][static_cast<size_t>(k)];
  }
  for (int t = tree.num_stages - 1; t >= 0; --t) {  // :54-73
    const NodeRange rng = nodes_at(tree, t);
    for (int i = rng.first; i < rng.past; ++i) {
      const auto si = static_cast<size_t>(i);
      const double* ydual = y.data() + cache.child_dual_offset[si];
      gemv(cache.dual_to_input[si], ydual, out.u.col(i), false);
      gemv(cache.dual_to_costate[si], ydual, costate.col(i), false);
      if (affine) {
        for (int k = 0; k < cache.nu; ++k) out.u(k, i) += cache.input_affine[si][static_cast<size_t>(k)];
        for (int k = 0; k < cache.nx; ++k) costate(k, i) += cache.costate_affine[si][static_cast<size_t>(k)];
      }
      for (int c : tree.children[si]) {
        const auto sc = static_cast<size_t>(c);
        gemv(cache.child_to_input[sc], costate.col(c), out.u.col(i), true);
        gemv_t(cache.closed_loop[sc], costate.col(c), costate.col(i), true);
      }
    }
  }
  if (affine)  // :75
    for (int k = 0; k < cache.nx; ++k) out.x(k, 0) = prob.root_state[static_cast<size_t>(k)];
  for (int t = 0; t < tree.num_stages; ++t) {  // :76-88
    const NodeRange rng = nodes_at(tree, t);
    for (int i = rng.first; i < rng.past; ++i) {
      const auto si = static_cast<size_t>(i);
      gemv(cache.gain[si], out.x.col(i), out.u.col(i), true);
      for (int c : tree.children[si]) {
        const auto& d = prob.dyn[static_cast<size_t>(c)];
        gemv(d.A, out.x.col(i), out.x.col(c), false);
        gemv(d.B, out.u.col(i), out.x.col(c), true);
        if (affine)
          for (int k = 0; k < cache.nx; ++k) out.x(k, c) += d.c[static_cast<size_t>(k)];
      }
    }
  }
  return out;
}

// tree_oracles.hpp:96-102
PrimalPoint dual_grad(const FactorCache& cache, const ProblemInstance& prob, const Vec& y,
                      OracleStats* stats) {
  check_shapes(cache, prob, "dual_grad");
  if (stats) ++stats->dual_grad_calls;
  return riccati_sweep(cache, prob, y, true);
}
// tree_oracles.hpp:107-114
PrimalPoint hessian_vec(const FactorCache& cache, const ProblemInstance& prob, const Vec& r,
                        OracleStats* stats) {
  check_shapes(cache, prob, "hessian_vec");
  if (stats) ++stats->hessian_vec_calls;
  return riccati_sweep(cache, prob, r, false);
}
// tree_oracles.hpp:117-121
Vec grad_fhat(const FactorCache& cache, const ProblemInstance& prob, const Vec& y,
              OracleStats* stats) {
  return scaled(apply_H(prob, dual_grad(cache, prob, y, stats)), -1.0);
}
// tree_oracles.hpp:125-129
double fhat_value(const FactorCache& cache, const ProblemInstance& prob, const Vec& y,
                  OracleStats* stats) {
  const PrimalPoint x = dual_grad(cache, prob, y, stats);
  return -dot(apply_H(prob, x), y) - eval_f(prob, x);
}

// ============================================================ prox
// prox.hpp:30-52
SeparableNonsmooth make_nonsmooth(const ProblemInstance& prob) {
  SeparableNonsmooth g;
  g.dim = prob.dual_dim;
  auto add = [&g](int offset, int rows, double weight, const NonsmoothSpec& spec) {
    if (weight <= 0.0) ORC_THROW(kZeroProbability, "make_nonsmooth: block with nonpositive weight");
    g.blocks.push_back(GBlock{offset, rows, weight, spec.kind, spec.zmin, spec.zmax, spec.gamma});
  };
  for (int i = 1; i < prob.num_nodes(); ++i) {
    const auto si = static_cast<size_t>(i);
    add(prob.dual_offset[si], prob.stage_rows(i), prob.tree.probability[si], prob.con[si].g);
  }
  for (int i = prob.tree.first_leaf(); i < prob.num_nodes(); ++i) {
    const int l = prob.leaf_ordinal(i);
    add(prob.tdual_offset[static_cast<size_t>(l)], prob.terminal_rows(l),
        prob.tree.probability[static_cast<size_t>(i)], prob.tcon[static_cast<size_t>(l)].g);
  }
  return g;
}

// prox.hpp:58-81
Vec prox_g(const SeparableNonsmooth& g, const Vec& v, double gamma_prox) {
  if (static_cast<int>(v.size()) != g.dim) ORC_THROW(kDimensionMismatch, "prox_g: vector length");
  if (!(gamma_prox > 0.0)) ORC_THROW(kInvalidParams, "prox_g: gamma_prox must be > 0");
  Vec out = v;
  for (const auto& b : g.blocks) {
    double* seg = out.data() + b.offset;
    switch (b.kind) {
      case NonsmoothKind::None:
        break;
      case NonsmoothKind::Box:
        for (int j = 0; j < b.size; ++j)
          seg[j] = std::min(std::max(seg[j], b.zmin[static_cast<size_t>(j)]), b.zmax[static_cast<size_t>(j)]);
        break;
      case NonsmoothKind::ScaledL1: {
        const double t = gamma_prox * b.weight * b.gamma;
        for (int j = 0; j < b.size; ++j) {
          const double a = seg[j];
          seg[j] = (a > t) ? a - t : (a < -t ? a + t : 0.0);
        }
        break;
      }
    }
  }
  return out;
}

// prox.hpp:90-113
double conj_value_g(const SeparableNonsmooth& g, const Vec& w, double slack) {
  if (static_cast<int>(w.size()) != g.dim) ORC_THROW(kDimensionMismatch, "conj_value_g: vector length");
  constexpr double kInf = std::numeric_limits<double>::infinity();
  double total = 0.0;
  for (const auto& b : g.blocks) {
    const double* seg = w.data() + b.offset;
    switch (b.kind) {
      case NonsmoothKind::None:
        for (int j = 0; j < b.size; ++j)
          if (std::abs(seg[j]) > slack) return kInf;
        break;
      case NonsmoothKind::Box: {
        double s = 0.0;
        for (int j = 0; j < b.size; ++j)
          s += std::max(seg[j] * b.zmin[static_cast<size_t>(j)], seg[j] * b.zmax[static_cast<size_t>(j)]);
        total += s;
        break;
      }
      case NonsmoothKind::ScaledL1: {
        const double radius = b.weight * b.gamma;
        for (int j = 0; j < b.size; ++j)
          if (std::abs(seg[j]) > radius * (1.0 + slack) + slack) return kInf;
        break;
      }
    }
  }
  return total;
}

// prox.hpp:117-121
Vec prox_g_conj(const SeparableNonsmooth& g, const Vec& v, double lambda) {
  if (!(lambda > 0.0)) ORC_THROW(kInvalidParams, "prox_g_conj: lambda must be > 0");
  const Vec p = prox_g(g, scaled(v, 1.0 / lambda), 1.0 / lambda);
  return lincomb(v, -lambda, p);
}

// prox.hpp:127-171
double dist_subdiff_inf(const SeparableNonsmooth& g, const Vec& y, const Vec& z) {
  if (static_cast<int>(y.size()) != g.dim || static_cast<int>(z.size()) != g.dim)
    ORC_THROW(kDimensionMismatch, "dist_subdiff_inf: vector length");
  double worst = 0.0;
  for (const auto& b : g.blocks) {
    for (int j = 0; j < b.size; ++j) {
      const double yj = y[static_cast<size_t>(b.offset + j)];
      const double zj = z[static_cast<size_t>(b.offset + j)];
      double d = 0.0;
      switch (b.kind) {
        case NonsmoothKind::None:
          d = std::abs(yj);
          break;
        case NonsmoothKind::Box: {
          const double lo = b.zmin[static_cast<size_t>(j)], hi = b.zmax[static_cast<size_t>(j)];
          const double cushion = 1e-12 * (1.0 + std::abs(lo) + std::abs(hi));
          const bool at_lo = zj <= lo + cushion;
          const bool at_hi = zj >= hi - cushion;
          if (at_lo && at_hi) d = 0.0;
          else if (at_lo) d = std::max(yj, 0.0);
          else if (at_hi) d = std::max(-yj, 0.0);
          else d = std::abs(yj);
          break;
        }
        case NonsmoothKind::ScaledL1: {
          const double t = b.weight * b.gamma;
          if (zj > 0.0) d = std::abs(yj - t);
          else if (zj < 0.0) d = std::abs(yj + t);
          else d = std::max(0.0, std::abs(yj) - t);
          break;
        }
      }
      worst = std::max(worst, d);
    }
  }
  return worst;
}

// ============================================================ fbe
// fbe.hpp:38-50
static void finish_fb_fields(FbState& state, const SeparableNonsmooth& g, OracleStats* stats) {
  const double lambda = state.lambda;
  Vec v(state.y.size());
  for (size_t i = 0; i < v.size(); ++i) v[i] = state.y[i] / lambda + state.Hx[i];
  state.z = prox_g(g, v, 1.0 / lambda);
  if (stats) ++stats->prox_calls;
  state.R = sub(state.z, state.Hx);
  state.T = lincomb(state.y, -lambda, state.R);
  state.conj_T = conj_value_g(g, state.T);
  if (stats) ++stats->conj_calls;
  state.znorm_sq = sqnorm(state.z);
  state.value = state.fhat + state.conj_T + lambda * dot(state.Hx, state.R) +
                0.5 * lambda * sqnorm(state.R);
}

// fbe.hpp:55-67
FbState fb_step(const FactorCache& cache, const ProblemInstance& prob, const SeparableNonsmooth& g,
                const Vec& y, double lambda, OracleStats* stats) {
  if (!(lambda > 0.0)) ORC_THROW(kInvalidParams, "fb_step: lambda must be > 0");
  FbState state;
  state.y = y;
  state.lambda = lambda;
  state.x = dual_grad(cache, prob, y, stats);
  state.Hx = apply_H(prob, state.x);
  state.fhat = -dot(state.Hx, y) - eval_f(prob, state.x);
  finish_fb_fields(state, g, stats);
  return state;
}

// fbe.hpp:72-77
void rescale_state(FbState& state, const SeparableNonsmooth& g, double lambda, OracleStats* stats) {
  if (!(lambda > 0.0)) ORC_THROW(kInvalidParams, "rescale_state: lambda must be > 0");
  state.lambda = lambda;
  finish_fb_fields(state, g, stats);
}

// fbe.hpp:82-86
double fbe_value(const FbState& state) {
  if (!std::isfinite(state.value)) ORC_THROW(kInfiniteConjugate, "fbe_value: g*(T) is infinite");
  return state.value;
}

// fbe.hpp:89-94
Vec fbe_grad(const FbState& state, const FactorCache& cache, const ProblemInstance& prob,
             OracleStats* stats) {
  const PrimalPoint hom = hessian_vec(cache, prob, state.R, stats);
  return lincomb(state.R, state.lambda, apply_H(prob, hom));
}

// fbe.hpp:136-143
static void fill_cert_coefficients(LineSearchCert& cert) {
  const double quad = dot(cert.dir, cert.Hx_dir);
  cert.alpha2 = -0.5 * quad - 0.5 * cert.lambda * sqnorm(cert.Hx_dir);
  cert.alpha1 = -dot(cert.Hx_anchor, lincomb(cert.dir, cert.lambda, cert.Hx_dir));
  cert.prox_base.resize(cert.anchor.size());
  cert.prox_slope.resize(cert.anchor.size());
  for (size_t i = 0; i < cert.anchor.size(); ++i) {
    cert.prox_base[i] = cert.anchor[i] / cert.lambda + cert.Hx_anchor[i];
    cert.prox_slope[i] = cert.dir[i] / cert.lambda + cert.Hx_dir[i];
  }
}

// fbe.hpp:149-165
LineSearchCert linesearch_cert(const FbState& state, const Vec& dir, const PrimalPoint& hom_dir,
                               const ProblemInstance& prob) {
  LineSearchCert cert;
  cert.anchor = state.y;
  cert.dir = dir;
  cert.lambda = state.lambda;
  cert.Hx_anchor = state.Hx;
  cert.Hx_dir = apply_H(prob, hom_dir);
  cert.conj_anchor = state.conj_T;
  cert.znorm_sq_anchor = state.znorm_sq;
  cert.value_anchor = state.value;
  cert.fhat_anchor = state.fhat;
  fill_cert_coefficients(cert);
  return cert;
}

// fbe.hpp:172-203
LineSearchCert linesearch_cert_shifted(const FbState& state, const SeparableNonsmooth& g,
                                       const Vec& r, const Vec& dir, const PrimalPoint& hom_r,
                                       const PrimalPoint& hom_dir, const ProblemInstance& prob,
                                       OracleStats* stats) {
  const double lambda = state.lambda;
  LineSearchCert cert;
  cert.anchor = lincomb(state.y, 1.0, r);
  cert.dir = sub(dir, r);
  cert.lambda = lambda;
  const Vec Hr = apply_H(prob, hom_r);
  cert.Hx_anchor = lincomb(state.Hx, 1.0, Hr);
  cert.Hx_dir = sub(apply_H(prob, hom_dir), Hr);
  cert.fhat_anchor = state.fhat - dot(state.Hx, r) - 0.5 * dot(r, Hr);
  Vec v(cert.anchor.size());
  for (size_t i = 0; i < v.size(); ++i) v[i] = cert.anchor[i] / lambda + cert.Hx_anchor[i];
  const Vec z_anchor = prox_g(g, v, 1.0 / lambda);
  if (stats) ++stats->prox_calls;
  const Vec res_anchor = sub(z_anchor, cert.Hx_anchor);
  cert.conj_anchor = conj_value_g(g, lincomb(cert.anchor, -lambda, res_anchor));
  if (stats) ++stats->conj_calls;
  cert.znorm_sq_anchor = sqnorm(z_anchor);
  cert.value_anchor = cert.fhat_anchor + cert.conj_anchor + lambda * dot(cert.Hx_anchor, res_anchor) +
                      0.5 * lambda * sqnorm(res_anchor);
  fill_cert_coefficients(cert);
  return cert;
}

// fbe.hpp:207-210
double cert_fhat(const LineSearchCert& cert, double tau) {
  return cert.fhat_anchor - tau * dot(cert.Hx_anchor, cert.dir) -
         0.5 * tau * tau * dot(cert.dir, cert.Hx_dir);
}

// fbe.hpp:214-231
CertEval evaluate_cert(const LineSearchCert& cert, const SeparableNonsmooth& g, double tau,
                       OracleStats* stats) {
  CertEval ev;
  ev.tau = tau;
  ev.w = lincomb(cert.anchor, tau, cert.dir);
  ev.Hx_w = lincomb(cert.Hx_anchor, tau, cert.Hx_dir);
  ev.z = prox_g(g, lincomb(cert.prox_base, tau, cert.prox_slope), 1.0 / cert.lambda);
  if (stats) ++stats->prox_calls;
  ev.R = sub(ev.z, ev.Hx_w);
  ev.T = lincomb(ev.w, -cert.lambda, ev.R);
  const double conj = conj_value_g(g, ev.T);
  if (stats) ++stats->conj_calls;
  ev.delta = cert.alpha2 * tau * tau + cert.alpha1 * tau + conj - cert.conj_anchor +
             0.5 * cert.lambda * (sqnorm(ev.z) - cert.znorm_sq_anchor);
  return ev;
}

// ============================================================ lbfgs
// lbfgs.hpp:30-84
LbfgsBuffer::LbfgsBuffer(int memory, double eps_curv) : memory_(memory), eps_curv_(eps_curv) {
  if (memory < 1) ORC_THROW(kInvalidParams, "LbfgsBuffer: memory must be >= 1");
  if (!(eps_curv > 0.0)) ORC_THROW(kInvalidParams, "LbfgsBuffer: eps_curv must be > 0");
}
bool LbfgsBuffer::push(const Vec& step, const Vec& change, double scale_ref) {
  const double curvature = dot(step, change);
  if (!(curvature > eps_curv_ * sqnorm(step) * scale_ref)) return false;
  const double change_sq = sqnorm(change);
  if (!(change_sq > 0.0)) return false;
  if (static_cast<int>(pairs_.size()) == memory_) pairs_.pop_front();
  pairs_.push_back(Pair{step, change, curvature});
  gamma0_ = curvature / change_sq;
  return true;
}
Vec LbfgsBuffer::apply_direction(const Vec& grad) const {
  Vec work = grad;
  const int count = static_cast<int>(pairs_.size());
  std::vector<double> alpha(static_cast<size_t>(count));
  for (int i = count - 1; i >= 0; --i) {
    const auto& p = pairs_[static_cast<size_t>(i)];
    alpha[static_cast<size_t>(i)] = dot(p.step, work) / p.curvature;
    axpy(-alpha[static_cast<size_t>(i)], p.change, work);
  }
  for (auto& v : work) v *= gamma0_;
  for (int i = 0; i < count; ++i) {
    const auto& p = pairs_[static_cast<size_t>(i)];
    const double beta = dot(p.change, work) / p.curvature;
    axpy(alpha[static_cast<size_t>(i)] - beta, p.step, work);
  }
  return scaled(work, -1.0);
}
void LbfgsBuffer::clear() {
  pairs_.clear();
  gamma0_ = 1.0;
}

// ============================================================ solvers
// solvers.hpp:48-60
void validate_config(const SolverConfig& cfg) {
  if (cfg.lambda0 < 0.0) ORC_THROW(kInvalidParams, "lambda0 must be >= 0");
  if (!(cfg.eps > 0.0)) ORC_THROW(kInvalidParams, "eps must be > 0");
  if (!(cfg.eps_curv > 0.0)) ORC_THROW(kInvalidParams, "eps_curv must be > 0");
  if (!(cfg.eps_bt > 0.0 && cfg.eps_bt < 0.5)) ORC_THROW(kInvalidParams, "eps_bt must lie in (0, 1/2)");
  if (cfg.beta_bt < 0.0 || cfg.beta_bt >= 1.0) ORC_THROW(kInvalidParams, "beta_bt must lie in [0, 1)");
  if (cfg.memory < 1) ORC_THROW(kInvalidParams, "memory must be >= 1");
  if (cfg.max_iters < 1) ORC_THROW(kInvalidParams, "max_iters must be >= 1");
  if (cfg.warm_start_iters < 0) ORC_THROW(kInvalidParams, "warm_start_iters must be >= 0");
}

// solvers.hpp:89-113
double estimate_dual_lipschitz(const FactorCache& cache, const ProblemInstance& prob,
                               std::uint64_t* calls, double rel_tol, int max_rounds) {
  std::mt19937_64 gen(0x5eed5eed5eed5eedULL);
  Vec v(static_cast<size_t>(prob.dual_dim));
  for (int i = 0; i < prob.dual_dim; ++i)
    v[static_cast<size_t>(i)] = 2.0 * (static_cast<double>(gen() >> 11) * 0x1.0p-53) - 1.0;
  {
    const double nv = std::sqrt(sqnorm(v));
    for (auto& e : v) e /= nv;
  }
  double rayleigh = 0.0;
  for (int round = 0; round < max_rounds; ++round) {
    const Vec image = scaled(apply_H(prob, hessian_vec(cache, prob, v)), -1.0);
    if (calls) ++*calls;
    const double next = dot(v, image);
    const double magnitude = std::sqrt(sqnorm(image));
    if (!(magnitude > 0.0)) return 1e-12;
    const bool settled = std::abs(next - rayleigh) <= rel_tol * std::abs(next);
    rayleigh = next;
    if (settled) break;
    v = scaled(image, 1.0 / magnitude);
  }
  return std::max(rayleigh, 1e-12);
}

namespace {
// solvers.hpp:117-120
double weighted_inf(const Vec& res, const Vec* weight) {
  if (weight == nullptr) return inf_norm(res);
  double m = 0.0;
  for (size_t i = 0; i < res.size(); ++i) m = std::max(m, std::abs(res[i] * (*weight)[i]));
  return m;
}
// solvers.hpp:122-127
double halve_lambda(double lambda) {
  const double next = 0.5 * lambda;
  if (next < 1e-14) ORC_THROW(kStepUnderflow, "backtracking drove lambda below 1e-14");
  return next;
}
// solvers.hpp:129-138
double resolve_lambda0(const SolverConfig& cfg, SolverKind kind, const FactorCache& cache,
                       const ProblemInstance& prob, SolverReport& rep) {
  if (cfg.lambda0 > 0.0) return cfg.lambda0;
  rep.lipschitz_estimate = estimate_dual_lipschitz(cache, prob, &rep.lipschitz_calls);
  const bool fixed_step = kind == SolverKind::Gpad || cfg.backtracking_rule == BacktrackingRule::None;
  return (fixed_step ? 0.95 : 0.9) / rep.lipschitz_estimate;
}
void merge_stats(OracleStats& into, const OracleStats& from) {  // :140-145
  into.dual_grad_calls += from.dual_grad_calls;
  into.hessian_vec_calls += from.hessian_vec_calls;
  into.prox_calls += from.prox_calls;
  into.conj_calls += from.conj_calls;
}
void refresh_trace_tail(SolverReport& rep, const FbState& state, const Vec* w) {  // :151-155
  rep.residual_trace.back() = weighted_inf(state.R, w);
  rep.fbe_trace.back() = state.value;
}
void finish_report(SolverReport& rep, SolverStatus status, const FbState& state, double residual,
                   std::chrono::steady_clock::time_point start) {  // :157-169
  rep.status = status;
  rep.x = state.x;
  rep.y = state.y;
  rep.z = state.z;
  rep.residual_inf = residual;
  rep.lambda_final = state.lambda;
  rep.wall_ms =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - start).count();
}
struct BacktrackProbe {  // :180-186
  double candidate_fhat = 0.0, anchor_fhat = 0.0, anchor_inner = 0.0, anchor_res_sq = 0.0;
  const Vec* curvature_image = nullptr;
};
struct BacktrackDecision {
  double lambda;
  bool restarted;
};
// solvers.hpp:195-227
BacktrackDecision backtrack_lambda(const FbState& state, BacktrackingRule rule,
                                   const SolverConfig& cfg, const BacktrackProbe& probe) {
  const double lambda = state.lambda;
  bool trigger = false;
  switch (rule) {
    case BacktrackingRule::None:
      break;
    case BacktrackingRule::Original: {
      const double model = probe.anchor_fhat + lambda * probe.anchor_inner +
                           0.5 * (1.0 - cfg.beta_bt) * lambda * probe.anchor_res_sq;
      trigger = probe.candidate_fhat > model;
      break;
    }
    case BacktrackingRule::Simple: {
      if (probe.curvature_image == nullptr)
        ORC_THROW(kInvalidParams, "simple rule needs the curvature image");
      trigger = lambda * std::sqrt(sqnorm(*probe.curvature_image)) >
                cfg.eps_bt * std::sqrt(sqnorm(state.R));
      break;
    }
  }
  if (!trigger) return {lambda, false};
  return {halve_lambda(lambda), true};
}
}  // namespace

// solvers.hpp:234-356
SolverReport solve_minfbe(const ProblemInstance& prob, const FactorCache& cache,
                          const SeparableNonsmooth& g, const SolverConfig& cfg, const Vec& y0,
                          const Vec* residual_weight) {
  validate_config(cfg);
  const auto start = std::chrono::steady_clock::now();
  SolverReport rep;
  rep.eps = cfg.eps;
  double lambda = resolve_lambda0(cfg, SolverKind::Minfbe, cache, prob, rep);
  LbfgsBuffer buffer(cfg.memory, cfg.eps_curv);
  FbState state = fb_step(cache, prob, g, y0, lambda, &rep.stats);
  Vec grad, prev_y, prev_grad;
  bool grad_valid = false, have_pair = false, fresh_iterate = true;
  int iter = 0;
  for (;;) {
    const double residual = weighted_inf(state.R, residual_weight);
    if (fresh_iterate) {
      rep.residual_trace.push_back(residual);
      rep.fbe_trace.push_back(state.value);
      fresh_iterate = false;
    }
    if (residual <= cfg.eps) {
      rep.iterations = iter;
      finish_report(rep, SolverStatus::Converged, state, residual, start);
      return rep;
    }
    if (iter >= cfg.max_iters) {
      rep.iterations = iter;
      finish_report(rep, SolverStatus::MaxItersExceeded, state, residual, start);
      return rep;
    }
    if (!grad_valid) {
      grad = fbe_grad(state, cache, prob, &rep.stats);
      grad_valid = true;
    }
    if (cfg.backtracking_rule == BacktrackingRule::Simple) {
      bool halved = false;
      for (;;) {
        Vec image = sub(grad, state.R);
        for (auto& e : image) e /= lambda;
        BacktrackProbe probe;
        probe.curvature_image = &image;
        const auto decision = backtrack_lambda(state, BacktrackingRule::Simple, cfg, probe);
        if (!decision.restarted) break;
        lambda = decision.lambda;
        buffer.clear();
        have_pair = false;
        rescale_state(state, g, lambda, &rep.stats);
        grad = fbe_grad(state, cache, prob, &rep.stats);
        halved = true;
      }
      if (halved) {
        refresh_trace_tail(rep, state, residual_weight);
        continue;
      }
    }
    if (have_pair) {
      buffer.push(sub(state.y, prev_y), sub(grad, prev_grad), sqnorm(prev_grad));
      have_pair = false;
    }
    const Vec dir = buffer.apply_direction(grad);
    const PrimalPoint hom_dir = hessian_vec(cache, prob, dir, &rep.stats);
    const LineSearchCert cert = linesearch_cert(state, dir, hom_dir, prob);
    const double slack = 1e-12 * (1.0 + std::abs(state.value));
    CertEval accepted;
    bool found = false;
    double tau = 1.0;
    for (int halving = 0; halving <= 60; ++halving, tau *= 0.5) {
      accepted = evaluate_cert(cert, g, tau, &rep.stats);
      if (accepted.delta <= slack) {
        found = true;
        break;
      }
    }
    if (!found) ORC_THROW(kLineSearchStalled, "no step in {2^-nu, nu <= 60} decreases the envelope");
    FbState next = fb_step(cache, prob, g, accepted.T, lambda, &rep.stats);
    if (cfg.backtracking_rule == BacktrackingRule::Original) {
      BacktrackProbe probe;
      probe.candidate_fhat = next.fhat;
      probe.anchor_fhat = cert_fhat(cert, accepted.tau);
      probe.anchor_inner = dot(accepted.Hx_w, accepted.R);
      probe.anchor_res_sq = sqnorm(accepted.R);
      const auto decision = backtrack_lambda(state, BacktrackingRule::Original, cfg, probe);
      if (decision.restarted) {
        lambda = decision.lambda;
        buffer.clear();
        have_pair = false;
        rescale_state(state, g, lambda, &rep.stats);
        refresh_trace_tail(rep, state, residual_weight);
        grad_valid = false;
        continue;
      }
    }
    prev_y = state.y;
    prev_grad = std::move(grad);
    grad_valid = false;
    have_pair = true;
    state = std::move(next);
    ++iter;
    fresh_iterate = true;
  }
}

// solvers.hpp:362-492
SolverReport solve_nama(const ProblemInstance& prob, const FactorCache& cache,
                        const SeparableNonsmooth& g, const SolverConfig& cfg, const Vec& y0,
                        const Vec* residual_weight) {
  validate_config(cfg);
  const auto start = std::chrono::steady_clock::now();
  SolverReport rep;
  rep.eps = cfg.eps;
  double lambda = resolve_lambda0(cfg, SolverKind::Nama, cache, prob, rep);
  LbfgsBuffer buffer(cfg.memory, cfg.eps_curv);
  FbState state = fb_step(cache, prob, g, y0, lambda, &rep.stats);
  Vec prev_y, prev_res;
  bool have_pair = false, fresh_iterate = true;
  int iter = 0;
  for (;;) {
    const double residual = weighted_inf(state.R, residual_weight);
    if (fresh_iterate) {
      rep.residual_trace.push_back(residual);
      rep.fbe_trace.push_back(state.value);
      fresh_iterate = false;
    }
    if (residual <= cfg.eps) {
      rep.iterations = iter;
      finish_report(rep, SolverStatus::Converged, state, residual, start);
      return rep;
    }
    if (iter >= cfg.max_iters) {
      rep.iterations = iter;
      finish_report(rep, SolverStatus::MaxItersExceeded, state, residual, start);
      return rep;
    }
    if (have_pair) {
      buffer.push(sub(state.y, prev_y), sub(state.R, prev_res), sqnorm(prev_res));
      have_pair = false;
    }
    const Vec res = state.R;
    const Vec dir = buffer.apply_direction(res);
    PrimalPoint hom_res, hom_dir;
    if (cfg.nama_parallel_linesearch && std::thread::hardware_concurrency() >= 2) {
      OracleStats side;
      std::thread worker([&] { hom_res = hessian_vec(cache, prob, res, &side); });
      hom_dir = hessian_vec(cache, prob, dir, &rep.stats);
      worker.join();
      merge_stats(rep.stats, side);
    } else {
      hom_res = hessian_vec(cache, prob, res, &rep.stats);
      hom_dir = hessian_vec(cache, prob, dir, &rep.stats);
    }
    if (cfg.backtracking_rule == BacktrackingRule::Simple) {
      const Vec image = apply_H(prob, hom_res);
      BacktrackProbe probe;
      probe.curvature_image = &image;
      const auto decision = backtrack_lambda(state, BacktrackingRule::Simple, cfg, probe);
      if (decision.restarted) {
        lambda = decision.lambda;
        buffer.clear();
        have_pair = false;
        rescale_state(state, g, lambda, &rep.stats);
        refresh_trace_tail(rep, state, residual_weight);
        continue;
      }
    }
    const Vec shift = scaled(res, -lambda);
    const PrimalPoint hom_shift{scaled(hom_res.x, -lambda), scaled(hom_res.u, -lambda)};
    const LineSearchCert cert =
        linesearch_cert_shifted(state, g, shift, dir, hom_shift, hom_dir, prob, &rep.stats);
    const double slack = 1e-12 * (1.0 + std::abs(state.value));
    CertEval accepted;
    bool found = false;
    double tau = 1.0;
    for (int halving = 0; halving <= 60; ++halving, tau *= 0.5) {
      accepted = evaluate_cert(cert, g, tau, &rep.stats);
      if (cert.value_anchor + accepted.delta <= state.value + slack) {
        found = true;
        break;
      }
    }
    if (!found) ORC_THROW(kLineSearchStalled, "no step in {2^-nu, nu <= 60} decreases the envelope");
    const Vec y_next = cfg.nama_update_tlambda ? accepted.T : lincomb(state.y, -lambda, accepted.R);
    FbState next = fb_step(cache, prob, g, y_next, lambda, &rep.stats);
    if (cfg.backtracking_rule == BacktrackingRule::Original) {
      BacktrackProbe probe;
      probe.candidate_fhat = next.fhat;
      probe.anchor_fhat = cert_fhat(cert, accepted.tau);
      probe.anchor_inner = dot(accepted.Hx_w, accepted.R);
      probe.anchor_res_sq = sqnorm(accepted.R);
      const auto decision = backtrack_lambda(state, BacktrackingRule::Original, cfg, probe);
      if (decision.restarted) {
        lambda = decision.lambda;
        buffer.clear();
        have_pair = false;
        rescale_state(state, g, lambda, &rep.stats);
        refresh_trace_tail(rep, state, residual_weight);
        continue;
      }
    }
    prev_y = state.y;
    prev_res = state.R;
    have_pair = true;
    state = std::move(next);
    ++iter;
    fresh_iterate = true;
  }
}

// solvers.hpp:498-540
SolverReport solve_gpad(const ProblemInstance& prob, const FactorCache& cache,
                        const SeparableNonsmooth& g, const SolverConfig& cfg, const Vec& y0,
                        const Vec* residual_weight) {
  validate_config(cfg);
  const auto start = std::chrono::steady_clock::now();
  SolverReport rep;
  rep.eps = cfg.eps;
  const double lambda = resolve_lambda0(cfg, SolverKind::Gpad, cache, prob, rep);
  Vec y_prev = y0;
  double t = 1.0;
  FbState state = fb_step(cache, prob, g, y0, lambda, &rep.stats);
  int iter = 0;
  for (;;) {
    const double residual = weighted_inf(state.R, residual_weight);
    rep.residual_trace.push_back(residual);
    rep.fbe_trace.push_back(state.value);
    if (residual <= cfg.eps) {
      rep.iterations = iter;
      finish_report(rep, SolverStatus::Converged, state, residual, start);
      return rep;
    }
    if (iter >= cfg.max_iters) {
      rep.iterations = iter;
      finish_report(rep, SolverStatus::MaxItersExceeded, state, residual, start);
      return rep;
    }
    const Vec y_next = state.T;
    const double t_next = 0.5 * (1.0 + std::sqrt(1.0 + 4.0 * t * t));
    Vec w(y_next.size());
    const double mom = (t - 1.0) / t_next;
    for (size_t i = 0; i < w.size(); ++i) w[i] = y_next[i] + mom * (y_next[i] - y_prev[i]);
    y_prev = y_next;
    t = t_next;
    state = fb_step(cache, prob, g, w, lambda, &rep.stats);
    ++iter;
  }
}

// solvers.hpp:545-564
Vec warm_start(const ProblemInstance& prob, const FactorCache& cache, const SeparableNonsmooth& g,
               const SolverConfig& cfg, double lambda, OracleStats* stats) {
  Vec y(static_cast<size_t>(prob.dual_dim), 0.0);
  if (cfg.warm_start_iters <= 0) return y;
  if (!(lambda > 0.0)) ORC_THROW(kInvalidParams, "warm_start: lambda must be > 0");
  Vec w = y;
  double t = 1.0;
  for (int k = 0; k < cfg.warm_start_iters; ++k) {
    const FbState state = fb_step(cache, prob, g, w, lambda, stats);
    const Vec y_next = state.T;
    const double t_next = 0.5 * (1.0 + std::sqrt(1.0 + 4.0 * t * t));
    const double mom = (t - 1.0) / t_next;
    for (size_t i = 0; i < w.size(); ++i) w[i] = y_next[i] + mom * (y_next[i] - y[i]);
    y = y_next;
    t = t_next;
  }
  return y;
}

// solvers.hpp:569-602
ProblemInstance precondition(const ProblemInstance& prob) {
  ProblemInstance scaled_prob = prob;
  auto scale_spec = [](NonsmoothSpec& spec, double root) {
    switch (spec.kind) {
      case NonsmoothKind::None:
        break;
      case NonsmoothKind::Box:
        for (auto& v : spec.zmin) v *= root;
        for (auto& v : spec.zmax) v *= root;
        break;
      case NonsmoothKind::ScaledL1:
        spec.gamma /= root;
        break;
    }
  };
  for (int i = 1; i < prob.num_nodes(); ++i) {
    const auto si = static_cast<size_t>(i);
    const double pi = prob.tree.probability[si];
    if (!(pi > 0.0)) ORC_THROW(kZeroProbability, "precondition: node probability");
    const double root = std::sqrt(pi);
    for (auto& v : scaled_prob.con[si].F.d) v *= root;
    for (auto& v : scaled_prob.con[si].G.d) v *= root;
    scale_spec(scaled_prob.con[si].g, root);
  }
  for (int i = prob.tree.first_leaf(); i < prob.num_nodes(); ++i) {
    const auto li = static_cast<size_t>(prob.leaf_ordinal(i));
    const double pi = prob.tree.probability[static_cast<size_t>(i)];
    if (!(pi > 0.0)) ORC_THROW(kZeroProbability, "precondition: leaf probability");
    const double root = std::sqrt(pi);
    for (auto& v : scaled_prob.tcon[li].F.d) v *= root;
    scale_spec(scaled_prob.tcon[li].g, root);
  }
  return scaled_prob;
}

// solvers.hpp:608-623
Vec probability_roots(const ProblemInstance& prob) {
  Vec roots(static_cast<size_t>(prob.dual_dim), 0.0);
  for (int i = 1; i < prob.num_nodes(); ++i) {
    const auto si = static_cast<size_t>(i);
    const double r = std::sqrt(prob.tree.probability[si]);
    for (int k = 0; k < prob.stage_rows(i); ++k) roots[static_cast<size_t>(prob.dual_offset[si] + k)] = r;
  }
  for (int i = prob.tree.first_leaf(); i < prob.num_nodes(); ++i) {
    const int l = prob.leaf_ordinal(i);
    const double r = std::sqrt(prob.tree.probability[static_cast<size_t>(i)]);
    for (int k = 0; k < prob.terminal_rows(l); ++k)
      roots[static_cast<size_t>(prob.tdual_offset[static_cast<size_t>(l)] + k)] = r;
  }
  return roots;
}

// solvers.hpp:630-639
void verify_report(const ProblemInstance& prob, const SeparableNonsmooth& g, SolverReport& rep) {
  const Vec Hx = apply_H(prob, rep.x);
  rep.verify_residual_inf = inf_norm(sub(rep.z, Hx));
  rep.verify_subdiff_dist = dist_subdiff_inf(g, rep.y, rep.z);
  const double slop = 1.0 + 1e-9;
  rep.verified = rep.status == SolverStatus::Converged && rep.verify_residual_inf <= rep.eps * slop &&
                 rep.verify_subdiff_dist <= rep.lambda_final * rep.eps * slop;
}

// solvers.hpp:645-720. Note the reference's `dispatch` forwards the caller's
// cfg (not run_cfg), so the solver re-runs the power iteration itself; the
// returned lipschitz fields are then overwritten by the driver's estimate.
// Both estimates are identical (deterministic), so we follow that exactly.
SolverReport solve(const ProblemInstance& prob, const SolverConfig& cfg, SolverKind kind,
                   const FactorCache* shared_cache) {
  validate_config(cfg);
  const auto start = std::chrono::steady_clock::now();
  auto dispatch = [&](const ProblemInstance& inst, const FactorCache& cache,
                      const SeparableNonsmooth& g, const Vec& y0, const Vec* weight) {
    switch (kind) {
      case SolverKind::Minfbe:
        return solve_minfbe(inst, cache, g, cfg, y0, weight);
      case SolverKind::Nama:
        return solve_nama(inst, cache, g, cfg, y0, weight);
      case SolverKind::Gpad:
        return solve_gpad(inst, cache, g, cfg, y0, weight);
    }
    ORC_THROW(kInvalidParams, "unknown solver kind");
  };
  auto run = [&](const ProblemInstance& inst, const FactorCache& cache, const SeparableNonsmooth& g,
                 const Vec* weight) {
    double lhat = 0.0;
    std::uint64_t lhat_calls = 0;
    if (!(cfg.lambda0 > 0.0)) lhat = estimate_dual_lipschitz(cache, inst, &lhat_calls);
    OracleStats warm_stats;
    Vec y0(static_cast<size_t>(inst.dual_dim), 0.0);
    if (cfg.warm_start) {
      const double lambda_ws = cfg.lambda0 > 0.0 ? cfg.lambda0 : 0.95 / lhat;
      y0 = warm_start(inst, cache, g, cfg, lambda_ws, &warm_stats);
    }
    SolverReport out = dispatch(inst, cache, g, y0, weight);
    merge_stats(out.stats, warm_stats);
    out.lipschitz_estimate = lhat;
    out.lipschitz_calls = lhat_calls;
    return out;
  };
  SolverReport rep;
  if (!cfg.precondition) {
    FactorCache local;
    const FactorCache* cache = shared_cache;
    if (cache == nullptr) {
      local = factor(prob);
      cache = &local;
    }
    const SeparableNonsmooth g = make_nonsmooth(prob);
    rep = run(prob, *cache, g, nullptr);
    verify_report(prob, g, rep);
  } else {
    const ProblemInstance scaled_prob = precondition(prob);
    const FactorCache cache = factor(scaled_prob);
    const SeparableNonsmooth g_scaled = make_nonsmooth(scaled_prob);
    const Vec roots = probability_roots(prob);
    Vec weight(roots.size());
    for (size_t i = 0; i < roots.size(); ++i) weight[i] = 1.0 / roots[i];
    rep = run(scaled_prob, cache, g_scaled, &weight);
    for (size_t i = 0; i < rep.y.size(); ++i) rep.y[i] = rep.y[i] * roots[i];
    for (size_t i = 0; i < rep.z.size(); ++i) rep.z[i] = rep.z[i] * weight[i];
    verify_report(prob, make_nonsmooth(prob), rep);
  }
  rep.wall_ms =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - start).count();
  return rep;
}

// ============================================================ generators
namespace {
double unit_draw(std::mt19937_64& gen) {  // generators.hpp:20-22
  return static_cast<double>(gen() >> 11) * 0x1.0p-53;
}
double sym_draw(std::mt19937_64& gen) { return 2.0 * unit_draw(gen) - 1.0; }  // :25-27
Mat random_mat(std::mt19937_64& gen, int rows, int cols, double scale = 1.0) {  // :29-35 (row-major draws)
  Mat out(rows, cols);
  for (int i = 0; i < rows; ++i)
    for (int j = 0; j < cols; ++j) out(i, j) = scale * sym_draw(gen);
  return out;
}
Mat gram_plus_ridge(const Mat& root, double ridge) {  // root root' + ridge I
  const int n = root.r;
  Mat out(n, n);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) {
      double s = 0.0;
      for (int k = 0; k < root.c; ++k) s += root(i, k) * root(j, k);
      out(i, j) = s + (i == j ? ridge : 0.0);
    }
  return out;
}
}  // namespace

// generators.hpp:255-328. The reference builds the full `branching`-ary tree
// via build_from_markov with a uniform chain (:264-269); the extension takes
// a per-stage branching list br[t] (1 after the listed stages) and builds the
// same BFS-ordered tree with uniform conditional probabilities 1/br[t]. With
// a single-entry list repeated over the horizon it is the reference exactly.
ProblemInstance gen_random_instance(std::uint64_t seed, int nx, int nu, int horizon,
                                    const std::vector<int>& branching) {
  if (nx < 1 || nu < 1) ORC_THROW(kInvalidParams, "gen_random_instance: dims must be positive");
  if (horizon < 1) ORC_THROW(kInvalidParams, "gen_random_instance: tree shape must be positive");
  for (int b : branching)
    if (b < 1) ORC_THROW(kInvalidParams, "gen_random_instance: tree shape must be positive");
  std::mt19937_64 gen(seed);
  ProblemInstance prob;
  {
    ScenarioTree& tree = prob.tree;
    tree.num_stages = horizon;
    tree.node_stage = {0};
    tree.ancestor = {-1};
    tree.children = {{}};
    tree.probability = {1.0};
    tree.mode = {-1};
    tree.stage_offsets = {0, 1};
    int begin = 0, end = 1;
    for (int t = 0; t < horizon; ++t) {
      const int nb = t < static_cast<int>(branching.size()) ? branching[static_cast<size_t>(t)] : 1;
      const double branch = 1.0 / nb;
      for (int i = begin; i < end; ++i)
        for (int w = 0; w < nb; ++w) {
          const int id = tree.num_nodes();
          tree.node_stage.push_back(t + 1);
          tree.ancestor.push_back(i);
          tree.children.emplace_back();
          tree.probability.push_back(tree.probability[static_cast<size_t>(i)] * branch);
          tree.mode.push_back(w);
          tree.children[static_cast<size_t>(i)].push_back(id);
        }
      begin = end;
      end = tree.num_nodes();
      tree.stage_offsets.push_back(end);
    }
  }
  prob.nx = nx;
  prob.nu = nu;
  prob.root_state.assign(static_cast<size_t>(nx), 0.0);
  const int n = prob.num_nodes();
  prob.dyn.resize(static_cast<size_t>(n));
  prob.cost.resize(static_cast<size_t>(n));
  prob.con.resize(static_cast<size_t>(n));
  prob.dyn[0] = NodeDynamics{Mat(nx, nx), Mat(nx, nu), Vec(static_cast<size_t>(nx), 0.0)};
  prob.cost[0] = NodeCost{Mat(nx, nx), Mat(nu, nu), Mat(nu, nx), Vec(static_cast<size_t>(nx), 0.0),
                          Vec(static_cast<size_t>(nu), 0.0)};
  prob.con[0] = ConstraintBlock{Mat(0, nx), Mat(0, nu), NonsmoothSpec{}};
  for (int i = 1; i < n; ++i) {
    const auto si = static_cast<size_t>(i);
    Mat A = random_mat(gen, nx, nx);
    const double radius = spectral_radius(A);
    if (radius > 0.0) {
      const double s = 0.95 / radius;
      for (auto& v : A.d) v *= s;
    }
    prob.dyn[si].A = A;
    prob.dyn[si].B = random_mat(gen, nx, nu);
    prob.dyn[si].c.assign(static_cast<size_t>(nx), 0.0);
    const int nw = nx + nu;
    const Mat root = random_mat(gen, nw, nw);
    const Mat block = gram_plus_ridge(root, 0.1);
    Mat Q(nx, nx), S(nu, nx), R(nu, nu);
    for (int j = 0; j < nx; ++j)
      for (int k = 0; k < nx; ++k) Q(k, j) = block(k, j);
    for (int j = 0; j < nx; ++j)
      for (int k = 0; k < nu; ++k) S(k, j) = block(nx + k, j);
    for (int j = 0; j < nu; ++j)
      for (int k = 0; k < nu; ++k) R(k, j) = block(nx + k, nx + j);
    prob.cost[si].Q = Q;
    prob.cost[si].S = S;
    prob.cost[si].R = R;
    prob.cost[si].q = random_mat(gen, nx, 1, 1.5).d;
    prob.cost[si].r = random_mat(gen, nu, 1, 1.5).d;
    const int rows = 2;
    prob.con[si].F = random_mat(gen, rows, nx);
    prob.con[si].G = random_mat(gen, rows, nu);
    prob.con[si].g.kind = NonsmoothKind::Box;
    prob.con[si].g.zmin.assign(static_cast<size_t>(rows), 0.0);
    prob.con[si].g.zmax.assign(static_cast<size_t>(rows), 0.0);
    for (int k = 0; k < rows; ++k) {
      prob.con[si].g.zmin[static_cast<size_t>(k)] = -(0.05 + 0.3 * unit_draw(gen));
      prob.con[si].g.zmax[static_cast<size_t>(k)] = 0.05 + 0.3 * unit_draw(gen);
    }
  }
  const int leaves = prob.tree.num_leaves();
  prob.tcost.resize(static_cast<size_t>(leaves));
  prob.tcon.resize(static_cast<size_t>(leaves));
  for (int l = 0; l < leaves; ++l) {
    const auto sl = static_cast<size_t>(l);
    const Mat root = random_mat(gen, nx, nx);
    prob.tcost[sl].P = gram_plus_ridge(root, 0.1);
    prob.tcost[sl].p = random_mat(gen, nx, 1, 1.5).d;
    prob.tcon[sl].F = random_mat(gen, 1, nx);
    prob.tcon[sl].g.kind = NonsmoothKind::Box;
    prob.tcon[sl].g.zmin = {-(0.05 + 0.3 * unit_draw(gen))};
    prob.tcon[sl].g.zmax = {0.05 + 0.3 * unit_draw(gen)};
  }
  prob.finalize_layout();
  return prob;
}

// ============================================================ spring-mass
// generators.hpp:66-91: d/dt [p; v] = [[0, I], [-(k/m) T, -(b/m) T]] [p; v] + [[0], [D/m]] u
// with T the tridiagonal (2, -1) coupling and D the signed actuator incidence.
void spring_mass_continuous(int masses, const SpringMassParams& par, Mat& A, Mat& B) {
  const int n = masses;
  Mat T(n, n), D(n, n - 1);
  for (int j = 0; j < n; ++j) {
    T(j, j) = 2.0;
    if (j > 0) T(j, j - 1) = -1.0;
    if (j + 1 < n) T(j, j + 1) = -1.0;
  }
  for (int a = 0; a + 1 < n; ++a) {
    D(a, a) = -1.0;
    D(a + 1, a) = 1.0;
  }
  A = Mat(2 * n, 2 * n);
  for (int j = 0; j < n; ++j) A(j, n + j) = 1.0;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      A(n + i, j) = -(par.stiffness / par.mass_kg) * T(i, j);
      A(n + i, n + j) = -(par.damping / par.mass_kg) * T(i, j);
    }
  B = Mat(2 * n, n - 1);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j + 1 < n; ++j) B(n + i, j) = D(i, j) / par.mass_kg;
}

namespace {
double fro(const Mat& X) {
  double s = 0.0;
  for (double v : X.d) s += v * v;
  return std::sqrt(s);
}
}  // namespace

// test_generators.cpp:23-38: halve into ||X||_F <= 0.25, sum the series to
// 1e-20 relative (at most 60 terms), square back.
Mat expm_series(Mat X) {
  int squarings = 0;
  while (fro(X) > 0.25) {
    for (double& v : X.d) v *= 0.5;
    ++squarings;
  }
  Mat sum = Mat::identity(X.r);
  Mat term = sum;
  for (int k = 1; k <= 60; ++k) {
    term = matmul(term, X);
    for (double& v : term.d) v /= static_cast<double>(k);
    for (size_t t = 0; t < sum.d.size(); ++t) sum.d[t] += term.d[t];
    if (fro(term) <= 1e-20 * fro(sum)) break;
  }
  for (int s = 0; s < squarings; ++s) sum = matmul(sum, sum);
  return sum;
}

// generators.hpp:97-112: exp([[A, B], [0, 0]] period) holds A_d | B_d in its top rows.
void discretize_zoh(const Mat& A, const Mat& B, double period, Mat& Ad, Mat& Bd) {
  if (A.r != A.c || B.r != A.r) ORC_THROW(kDimensionMismatch, "discretize_zoh: A must be square and match B");
  if (!(period > 0.0)) ORC_THROW(kInvalidParams, "discretize_zoh: period must be > 0");
  const int n = A.r, m = B.c;
  Mat aug(n + m, n + m);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) aug(i, j) = A(i, j) * period;
  for (int j = 0; j < m; ++j)
    for (int i = 0; i < n; ++i) aug(i, n + j) = B(i, j) * period;
  const Mat big = expm_series(aug);
  Ad = Mat(n, n);
  Bd = Mat(n, m);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) Ad(i, j) = big(i, j);
  for (int j = 0; j < m; ++j)
    for (int i = 0; i < n; ++i) Bd(i, j) = big(i, n + j);
}

// generators.hpp:119-218
ProblemInstance gen_spring_mass(int masses, const SpringMassParams& params) {
  if (masses < 2) ORC_THROW(kInvalidParams, "gen_spring_mass: masses must be >= 2");
  if (!(params.mass_kg > 0.0)) ORC_THROW(kInvalidParams, "gen_spring_mass: mass_kg must be > 0");
  if (!(params.input_bound > 0.0) || !(params.velocity_bound > 0.0))
    ORC_THROW(kInvalidParams, "gen_spring_mass: bounds must be > 0");
  if (!(params.input_weight > 0.0) || !(params.terminal_weight > 0.0))
    ORC_THROW(kInvalidParams, "gen_spring_mass: input and terminal weights must be > 0");
  if (params.state_weight < 0.0) ORC_THROW(kInvalidParams, "gen_spring_mass: state_weight must be >= 0");
  SpringMassParams par = params;
  if (par.initial_probs.empty()) par.initial_probs = {0.5, 0.5};
  if (par.transition.d.empty()) {
    par.transition = Mat(2, 2);
    par.transition(0, 0) = 0.1;
    par.transition(0, 1) = 0.9;
    par.transition(1, 0) = 0.9;
    par.transition(1, 1) = 0.1;
  }
  if (par.mode_values.empty()) {
    par.mode_values.assign(par.initial_probs.size(), 0.0);
    if (par.mode_values.size() > 1) par.mode_values[1] = 0.1;
  }
  if (par.mode_values.size() != par.initial_probs.size())
    ORC_THROW(kDimensionMismatch, "gen_spring_mass: one mode value per Markov mode required");
  const int nx = 2 * masses, nu = masses - 1;
  Mat Ac, Bc, Ad, Bd;
  spring_mass_continuous(masses, par, Ac, Bc);
  discretize_zoh(Ac, Bc, par.sampling, Ad, Bd);
  ProblemInstance prob;
  prob.tree = build_from_markov(par.transition, par.initial_probs, par.horizon);
  prob.nx = nx;
  prob.nu = nu;
  prob.root_state = par.root_state.empty() ? Vec(static_cast<size_t>(nx), 0.0) : par.root_state;
  if (static_cast<int>(prob.root_state.size()) != nx)
    ORC_THROW(kDimensionMismatch, "gen_spring_mass: root_state must have length 2M");
  const int rows = masses + nu;
  NodeCost cost{Mat(nx, nx), Mat(nu, nu), Mat(nu, nx), Vec(static_cast<size_t>(nx), 0.0),
                Vec(static_cast<size_t>(nu), 0.0)};
  for (int i = 0; i < nx; ++i) cost.Q(i, i) = par.state_weight;
  for (int i = 0; i < nu; ++i) cost.R(i, i) = par.input_weight;
  ConstraintBlock con{Mat(rows, nx), Mat(rows, nu), NonsmoothSpec{}};
  for (int k = 0; k < masses; ++k) con.F(k, masses + k) = 1.0;  // velocity rows
  for (int k = 0; k < nu; ++k) con.G(masses + k, k) = 1.0;      // input rows
  con.g.kind = NonsmoothKind::Box;
  con.g.zmin.assign(static_cast<size_t>(rows), 0.0);
  for (int k = 0; k < rows; ++k) con.g.zmin[static_cast<size_t>(k)] = k < masses ? -par.velocity_bound : -par.input_bound;
  con.g.zmax.resize(static_cast<size_t>(rows));
  for (int k = 0; k < rows; ++k) con.g.zmax[static_cast<size_t>(k)] = -con.g.zmin[static_cast<size_t>(k)];
  const int n = prob.num_nodes();
  prob.dyn.resize(static_cast<size_t>(n));
  prob.cost.resize(static_cast<size_t>(n));
  prob.con.resize(static_cast<size_t>(n));
  prob.dyn[0] = NodeDynamics{Mat(nx, nx), Mat(nx, nu), Vec(static_cast<size_t>(nx), 0.0)};
  prob.cost[0] = NodeCost{Mat(nx, nx), Mat(nu, nu), Mat(nu, nx), Vec(static_cast<size_t>(nx), 0.0),
                          Vec(static_cast<size_t>(nu), 0.0)};
  prob.con[0] = ConstraintBlock{Mat(0, nx), Mat(0, nu), NonsmoothSpec{}};
  for (int i = 1; i < n; ++i) {
    const auto si = static_cast<size_t>(i);
    prob.dyn[si] = NodeDynamics{Ad, Bd, Vec(static_cast<size_t>(nx), par.mode_values[static_cast<size_t>(prob.tree.mode[si])])};
    prob.cost[si] = cost;
    prob.con[si] = con;
  }
  const int leaves = prob.tree.num_leaves();
  TerminalCost tc{Mat(nx, nx), Vec(static_cast<size_t>(nx), 0.0)};
  for (int i = 0; i < nx; ++i) tc.P(i, i) = par.terminal_weight;
  TerminalBlock tb{Mat(masses, nx), NonsmoothSpec{}};
  for (int k = 0; k < masses; ++k) tb.F(k, masses + k) = 1.0;
  tb.g.kind = NonsmoothKind::Box;
  tb.g.zmin.assign(static_cast<size_t>(masses), -par.velocity_bound);
  tb.g.zmax.assign(static_cast<size_t>(masses), par.velocity_bound);
  prob.tcost.assign(static_cast<size_t>(leaves), tc);
  prob.tcon.assign(static_cast<size_t>(leaves), tb);
  prob.finalize_layout();
  return prob;
}

// generators.hpp:223-234: positions in +-velocity_bound, velocities in +-velocity_bound / 2
Vec sample_initial_state(int masses, const SpringMassParams& params, std::mt19937_64& gen) {
  if (masses < 2) ORC_THROW(kInvalidParams, "sample_initial_state: masses must be >= 2");
  const double half = 0.5 * params.velocity_bound, pos_box = params.velocity_bound;
  Vec state(static_cast<size_t>(2 * masses));
  for (int i = 0; i < masses; ++i) state[static_cast<size_t>(i)] = pos_box * (2.0 * unit_draw(gen) - 1.0);
  for (int i = masses; i < 2 * masses; ++i) state[static_cast<size_t>(i)] = half * (2.0 * unit_draw(gen) - 1.0);
  return state;
}

// ============================================================ test support
// tests/support.hpp:33-43 (column-major draws)
Mat Rng::matrix(int rows, int cols, double scale) {
  Mat m(rows, cols);
  for (int j = 0; j < cols; ++j)
    for (int i = 0; i < rows; ++i) m(i, j) = scale * uniform(-1.0, 1.0);
  return m;
}
Vec Rng::vector(int size, double scale) {
  Vec v(static_cast<size_t>(size));
  for (int i = 0; i < size; ++i) v[static_cast<size_t>(i)] = scale * uniform(-1.0, 1.0);
  return v;
}

// tests/support.hpp:49-88
ScenarioTree random_tree(Rng& rng, int stages, int max_nodes, int max_children) {
  ScenarioTree tree;
  tree.num_stages = stages;
  tree.node_stage = {0};
  tree.ancestor = {-1};
  tree.children = {{}};
  tree.probability = {1.0};
  tree.stage_offsets = {0, 1};
  int begin = 0, end = 1;
  for (int t = 0; t < stages; ++t) {
    const int stages_left = stages - t;
    for (int i = begin; i < end; ++i) {
      const int created = tree.num_nodes() - end;
      const int budget = (max_nodes - tree.num_nodes() - created * (stages_left - 1) -
                          (end - i - 1) * stages_left) /
                         stages_left;
      int kids = std::min(max_children, std::max(1, budget));
      kids = rng.integer(1, kids);
      Vec w(static_cast<size_t>(kids));
      double wsum = 0.0;
      for (int k = 0; k < kids; ++k) {
        w[static_cast<size_t>(k)] = rng.uniform(0.2, 1.0);
      }
      for (double v : w) wsum += v;
      const double scale = tree.probability[static_cast<size_t>(i)] / wsum;
      for (auto& v : w) v *= scale;
      for (int k = 0; k < kids; ++k) {
        const int id = tree.num_nodes();
        tree.node_stage.push_back(t + 1);
        tree.ancestor.push_back(i);
        tree.children.emplace_back();
        tree.probability.push_back(w[static_cast<size_t>(k)]);
        tree.children[static_cast<size_t>(i)].push_back(id);
      }
    }
    begin = end;
    end = tree.num_nodes();
    tree.stage_offsets.push_back(end);
  }
  return tree;
}

// tests/support.hpp:104-203
ProblemInstance random_instance(Rng& rng, ScenarioTree tree, int nx, int nu,
                                const InstanceOptions& opt) {
  ProblemInstance prob;
  prob.tree = std::move(tree);
  prob.nx = nx;
  prob.nu = nu;
  prob.root_state = rng.vector(nx);
  const int n = prob.num_nodes();
  prob.dyn.resize(static_cast<size_t>(n));
  prob.cost.resize(static_cast<size_t>(n));
  prob.con.resize(static_cast<size_t>(n));
  prob.tcost.resize(static_cast<size_t>(prob.tree.num_leaves()));
  prob.tcon.resize(static_cast<size_t>(prob.tree.num_leaves()));
  prob.dyn[0] = NodeDynamics{Mat(nx, nx), Mat(nx, nu), Vec(static_cast<size_t>(nx), 0.0)};
  prob.cost[0] = NodeCost{Mat(nx, nx), Mat(nu, nu), Mat(nu, nx), Vec(static_cast<size_t>(nx), 0.0),
                          Vec(static_cast<size_t>(nu), 0.0)};
  prob.con[0] = ConstraintBlock{Mat(0, nx), Mat(0, nu), NonsmoothSpec{}};
  std::vector<NonsmoothKind> kinds;
  if (opt.with_box) kinds.push_back(NonsmoothKind::Box);
  if (opt.with_l1) kinds.push_back(NonsmoothKind::ScaledL1);
  if (opt.with_none) kinds.push_back(NonsmoothKind::None);
  if (kinds.empty()) kinds.push_back(NonsmoothKind::Box);
  auto spec_for = [&](int rows) {
    NonsmoothSpec g;
    g.kind = kinds[static_cast<size_t>(rng.integer(0, static_cast<int>(kinds.size()) - 1))];
    if (g.kind == NonsmoothKind::Box) {
      g.zmin.assign(static_cast<size_t>(rows), 0.0);
      g.zmax.assign(static_cast<size_t>(rows), 0.0);
      for (int j = 0; j < rows; ++j) {
        g.zmin[static_cast<size_t>(j)] = rng.uniform(-2.0, -0.1);
        g.zmax[static_cast<size_t>(j)] = rng.uniform(0.1, 2.0);
      }
    } else if (g.kind == NonsmoothKind::ScaledL1) {
      g.gamma = rng.uniform(0.2, 2.0);
    }
    return g;
  };
  for (int i = 1; i < n; ++i) {
    const auto si = static_cast<size_t>(i);
    auto& d = prob.dyn[si];
    d.A = rng.matrix(nx, nx, 0.6);
    d.B = rng.matrix(nx, nu, 0.8);
    d.c = opt.affine ? rng.vector(nx, 0.3) : Vec(static_cast<size_t>(nx), 0.0);
    auto& c = prob.cost[si];
    const Mat m = rng.matrix(nx + nu, nx + nu, 0.7);
    Mat blk = matmul_nt(m, m);
    for (int k = 0; k < nu; ++k) blk(nx + k, nx + k) += 0.5;
    c.Q = Mat(nx, nx);
    c.R = Mat(nu, nu);
    c.S = Mat(nu, nx);
    for (int j = 0; j < nx; ++j)
      for (int k = 0; k < nx; ++k) c.Q(k, j) = blk(k, j);
    for (int j = 0; j < nu; ++j)
      for (int k = 0; k < nu; ++k) c.R(k, j) = blk(nx + k, nx + j);
    for (int j = 0; j < nx; ++j)
      for (int k = 0; k < nu; ++k) c.S(k, j) = blk(nx + k, j);
    c.q = opt.affine ? rng.vector(nx, 0.5) : Vec(static_cast<size_t>(nx), 0.0);
    c.r = opt.affine ? rng.vector(nu, 0.5) : Vec(static_cast<size_t>(nu), 0.0);
    auto& b = prob.con[si];
    const int rows = rng.integer(opt.stage_rows_lo, opt.stage_rows_hi);
    b.F = rng.matrix(rows, nx);
    b.G = rng.matrix(rows, nu);
    b.g = spec_for(rows);
  }
  for (int l = 0; l < prob.tree.num_leaves(); ++l) {
    const auto sl = static_cast<size_t>(l);
    const Mat m = rng.matrix(nx, nx, 0.7);
    Mat P = matmul_nt(m, m);
    for (int k = 0; k < nx; ++k) P(k, k) += 0.3;
    prob.tcost[sl].P = P;
    prob.tcost[sl].p = opt.affine ? rng.vector(nx, 0.5) : Vec(static_cast<size_t>(nx), 0.0);
    const int rows = rng.integer(opt.stage_rows_lo, opt.stage_rows_hi);
    prob.tcon[sl].F = rng.matrix(rows, nx);
    prob.tcon[sl].g = spec_for(rows);
  }
  prob.finalize_layout();
  if (opt.feasible_boxes) {
    PrimalPoint pt;
    pt.u = rng.matrix(nu, prob.tree.first_leaf(), 0.5);
    pt.x = Mat(nx, n);
    for (int k = 0; k < nx; ++k) pt.x(k, 0) = prob.root_state[static_cast<size_t>(k)];
    for (int i = 1; i < n; ++i) {
      const int a = prob.tree.ancestor[static_cast<size_t>(i)];
      const auto& d = prob.dyn[static_cast<size_t>(i)];
      gemv(d.A, pt.x.col(a), pt.x.col(i), false);
      gemv(d.B, pt.u.col(a), pt.x.col(i), true);
      for (int k = 0; k < nx; ++k) pt.x(k, i) += d.c[static_cast<size_t>(k)];
    }
    const Vec z = apply_H(prob, pt);
    auto recenter = [&](NonsmoothSpec& g, int off, int rows) {
      if (g.kind != NonsmoothKind::Box) return;
      for (int j = 0; j < rows; ++j) {
        g.zmin[static_cast<size_t>(j)] = z[static_cast<size_t>(off + j)] - rng.uniform(0.3, 1.2);
        g.zmax[static_cast<size_t>(j)] = z[static_cast<size_t>(off + j)] + rng.uniform(0.3, 1.2);
      }
    };
    for (int i = 1; i < n; ++i)
      recenter(prob.con[static_cast<size_t>(i)].g, prob.dual_offset[static_cast<size_t>(i)],
               prob.stage_rows(i));
    for (int l = 0; l < prob.tree.num_leaves(); ++l)
      recenter(prob.tcon[static_cast<size_t>(l)].g, prob.tdual_offset[static_cast<size_t>(l)],
               prob.terminal_rows(l));
  }
  return prob;
}

}  // namespace orc
