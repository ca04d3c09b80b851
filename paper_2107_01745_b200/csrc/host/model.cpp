// SPDX-License-Identifier: MIT
// Problem model, validation, preconditioning and the seeded generator.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <functional>
#include <random>
#include <thread>

#include "model.hpp"

namespace scn {

void parallel_for(int count, int grain, const std::function<void(int, int)>& body) {
  if (count <= 0) return;
  unsigned hw = std::thread::hardware_concurrency();
  if (hw == 0) hw = 1;
  const int chunks = std::max(1, std::min<int>(static_cast<int>(hw), (count + grain - 1) / grain));
  if (chunks == 1) {
    body(0, count);
    return;
  }
  std::vector<std::thread> pool;
  const int per = (count + chunks - 1) / chunks;
  for (int c = 0; c < chunks; ++c) {
    const int b = c * per, e = std::min(count, b + per);
    if (b >= e) break;
    pool.emplace_back([&body, b, e] { body(b, e); });
  }
  for (auto& t : pool) t.join();
}

// problem_data.hpp:126-140 plus the BFS child ranges (scenario_tree.hpp:228-238)
void Problem::finalize() {
  node_stage.assign(static_cast<size_t>(n), 0);
  for (int s = 0; s <= N; ++s)
    for (int i = stage_offsets[s]; i < stage_offsets[s + 1]; ++i) node_stage[i] = s;
  first_leaf = stage_offsets[N];
  L = n - first_leaf;
  child_begin.assign(static_cast<size_t>(n), 0);
  child_count.assign(static_cast<size_t>(n), 0);
  for (int i = n - 1; i >= 1; --i) {
    const int a = ancestor[i];
    if (a < 0 || a >= n) continue;
    child_begin[a] = i;
    ++child_count[a];
  }
  dual_offset.assign(static_cast<size_t>(n), -1);
  int off = 0;
  for (int i = 1; i < n; ++i) {
    dual_offset[i] = off;
    off += stage_rows[i];
  }
  stage_total = off;
  tdual_offset.assign(static_cast<size_t>(L), 0);
  for (int l = 0; l < L; ++l) {
    tdual_offset[l] = off;
    off += terminal_rows[l];
  }
  dual_dim = off;
}

template <class T, class V = std::vector<T>>
static V take(const T* src, size_t n) {
  if (n == 0) return {};
  if (!src) fail(SCENOPT_E_DIMENSION_MISMATCH, "problem view: missing array");
  return V(src, src + n);
}

Problem problem_from_view(const scenopt_problem_view& v) {
  if (v.nx <= 0 || v.nu <= 0 || v.num_nodes <= 0 || v.num_stages < 1)
    fail(SCENOPT_E_INVALID_PARAMS, "problem view: nx, nu, num_nodes and num_stages must be positive");
  Problem p;
  p.nx = v.nx;
  p.nu = v.nu;
  p.N = v.num_stages;
  p.n = v.num_nodes;
  const size_t n = static_cast<size_t>(p.n);
  p.stage_offsets = take(v.stage_offsets, static_cast<size_t>(p.N) + 2);
  if (p.stage_offsets.back() != p.n || p.stage_offsets.front() != 0)
    fail(SCENOPT_E_DIMENSION_MISMATCH, "problem view: stage_offsets must span [0, num_nodes]");
  p.ancestor = take(v.ancestor, n);
  p.probability = take(v.probability, n);
  p.root_state = take(v.root_state, static_cast<size_t>(p.nx));
  p.A = take<double, BigVec>(v.A, n * p.sxx());
  p.B = take<double, BigVec>(v.B, n * p.sxu());
  p.c = take(v.c, n * p.nx);
  p.Q = take<double, BigVec>(v.Q, n * p.sxx());
  p.R = take<double, BigVec>(v.R, n * p.suu());
  p.S = take<double, BigVec>(v.S, n * p.sxu());
  p.q = take(v.q, n * p.nx);
  p.r = take(v.r, n * p.nu);
  p.stage_rows = take(v.stage_rows, n);
  p.stage_rows[0] = 0;
  p.g_kind = take(v.g_kind, n);
  p.g_gamma = take(v.g_gamma, n);
  const int L = p.n - p.stage_offsets[p.N];
  p.terminal_rows = take(v.terminal_rows, static_cast<size_t>(L));
  p.tg_kind = take(v.tg_kind, static_cast<size_t>(L));
  p.tg_gamma = take(v.tg_gamma, static_cast<size_t>(L));
  for (int i = 1; i < p.n; ++i)
    if (p.stage_rows[i] < 0) fail(SCENOPT_E_DIMENSION_MISMATCH, "problem view: negative stage rows");
  for (int l = 0; l < L; ++l)
    if (p.terminal_rows[l] < 0) fail(SCENOPT_E_DIMENSION_MISMATCH, "problem view: negative terminal rows");
  p.finalize();
  p.P = take<double, BigVec>(v.P, static_cast<size_t>(L) * p.sxx());
  p.p = take(v.p, static_cast<size_t>(L) * p.nx);
  p.F = take(v.F, static_cast<size_t>(p.stage_total) * p.nx);
  p.G = take(v.G, static_cast<size_t>(p.stage_total) * p.nu);
  p.FN = take(v.FN, static_cast<size_t>(p.dual_dim - p.stage_total) * p.nx);
  p.zmin = take(v.zmin, static_cast<size_t>(p.dual_dim));
  p.zmax = take(v.zmax, static_cast<size_t>(p.dual_dim));
  for (int k = 0; k < p.dual_dim; ++k)
    if (!std::isfinite(p.zmin[k]) && p.zmin[k] > 0) p.zmin[k] = 0.0;  // unused rows
  return p;
}

void problem_to_view(const Problem& p, scenopt_problem_view* v) {
  v->nx = p.nx;
  v->nu = p.nu;
  v->num_stages = p.N;
  v->num_nodes = p.n;
  v->ancestor = p.ancestor.data();
  v->probability = p.probability.data();
  v->stage_offsets = p.stage_offsets.data();
  v->root_state = p.root_state.data();
  v->A = p.A.data();
  v->B = p.B.data();
  v->c = p.c.data();
  v->Q = p.Q.data();
  v->R = p.R.data();
  v->S = p.S.data();
  v->q = p.q.data();
  v->r = p.r.data();
  v->stage_rows = p.stage_rows.data();
  v->F = p.F.data();
  v->G = p.G.data();
  v->g_kind = p.g_kind.data();
  v->g_gamma = p.g_gamma.data();
  v->P = p.P.data();
  v->p = p.p.data();
  v->terminal_rows = p.terminal_rows.data();
  v->FN = p.FN.data();
  v->tg_kind = p.tg_kind.data();
  v->tg_gamma = p.tg_gamma.data();
  v->zmin = p.zmin.data();
  v->zmax = p.zmax.data();
}

// scenario_tree.hpp:128-240 and problem_data.hpp:233-314, over the flat model.
std::vector<std::string> validate_tree(const Problem& p) {
  std::vector<std::string> bad;
  auto complain = [&bad](const std::string& m) { bad.push_back(m); };
  constexpr double kTol = 1e-9;
  const int n = p.n, N = p.N;
  if (N < 1) complain("tree: num_stages must be >= 1");
  for (int t = 0; t <= N; ++t)
    if (p.stage_offsets[t] >= p.stage_offsets[t + 1])
      complain("stage " + std::to_string(t) + ": empty stage");
  if (p.ancestor[0] != -1) complain("node 0: root must have ancestor -1");
  if (std::abs(p.probability[0] - 1.0) > kTol) complain("node 0: root probability must be 1");
  std::vector<double> mass(static_cast<size_t>(n), 0.0);
  for (int i = 0; i < n; ++i) {
    const int t = p.node_stage[i];
    if (!(p.probability[i] > 0.0) || p.probability[i] > 1.0 + kTol)
      complain("node " + std::to_string(i) + ": probability not in (0, 1]");
    if (i > 0) {
      const int a = p.ancestor[i];
      if (a < 0 || a >= i) {
        complain("node " + std::to_string(i) + ": ancestor id must be smaller than the node's own id");
      } else {
        if (p.node_stage[a] != t - 1)
          complain("node " + std::to_string(i) + ": ancestor is not one stage earlier");
        mass[a] += p.probability[i];
      }
    }
  }
  for (int i = 0; i < n; ++i) {
    if (p.node_stage[i] == N) continue;
    if (p.child_count[i] == 0)
      complain("node " + std::to_string(i) +
               ": interior node without children (leaves must sit at the final stage)");
    else if (std::abs(mass[i] - p.probability[i]) > kTol)
      complain("node " + std::to_string(i) + ": children probabilities do not sum to the node's own");
  }
  for (int t = 0; t <= N; ++t) {
    double m = 0.0;
    for (int i = p.stage_offsets[t]; i < p.stage_offsets[t + 1]; ++i) m += p.probability[i];
    if (std::abs(m - 1.0) > kTol) complain("stage " + std::to_string(t) + ": probabilities do not sum to 1");
  }
  for (int i = 1; i + 1 < n; ++i)
    if (p.node_stage[i] == p.node_stage[i + 1] && p.ancestor[i] > p.ancestor[i + 1])
      complain("node " + std::to_string(i + 1) +
               ": siblings out of BFS order (ancestor ids must be nondecreasing within a stage)");
  return bad;
}

std::vector<std::string> validate(const Problem& p) {
  std::vector<std::string> bad = validate_tree(p);
  auto complain = [&bad](const std::string& m) { bad.push_back(m); };
  const int n = p.n;
  const int nx = p.nx, nu = p.nu;
  auto check_spec = [&](int kind, double gamma, int off, int rows, const std::string& where) {
    if (kind < 0 || kind > 2) {
      complain(where + ": unknown nonsmooth kind");
      return;
    }
    if (kind == 1) {
      for (int j = 0; j < rows; ++j)
        if (p.zmax[off + j] - p.zmin[off + j] < 0.0) {
          complain(where + ": box needs zmin <= zmax");
          break;
        }
    } else if (kind == 2 && !(gamma > 0.0)) {
      complain(where + ": scaled_l1 needs gamma > 0");
    }
  };
  std::vector<double> blk(static_cast<size_t>((nx + nu) * (nx + nu)));
  for (int i = 1; i < n; ++i) {
    const std::string where = "node " + std::to_string(i);
    if (sym_min_eig(p.Ri(i), nu) < 1e-10) complain(where + ": R must be positive definite");
    const double* Q = p.Qi(i);
    const double* S = p.Si(i);
    const double* R = p.Ri(i);
    const int w = nx + nu;
    for (int j = 0; j < nx; ++j)
      for (int k = 0; k < nx; ++k) blk[k + j * w] = Q[k + j * nx];
    for (int j = 0; j < nu; ++j)
      for (int k = 0; k < nx; ++k) blk[k + (nx + j) * w] = S[j + k * nu];
    for (int j = 0; j < nx; ++j)
      for (int k = 0; k < nu; ++k) blk[nx + k + j * w] = S[k + j * nu];
    for (int j = 0; j < nu; ++j)
      for (int k = 0; k < nu; ++k) blk[nx + k + (nx + j) * w] = R[k + j * nu];
    if (sym_min_eig(blk.data(), w) < -1e-10)
      complain(where + ": cost block [[Q, S'], [S, R]] must be positive semidefinite");
    check_spec(p.g_kind[i], p.g_gamma[i], p.dual_offset[i], p.stage_rows[i], where + " stage block");
  }
  for (int l = 0; l < p.L; ++l) {
    const std::string where = "leaf " + std::to_string(l);
    if (sym_min_eig(p.Pl(l), nx) < 1e-10) complain(where + ": P_N must be positive definite");
    check_spec(p.tg_kind[l], p.tg_gamma[l], p.tdual_offset[l], p.terminal_rows[l],
               where + " terminal block");
  }
  return bad;
}

void require_valid(const Problem& p) {
  // Only the structural rules the device layout depends on are enforced here;
  // full validation is scenopt_problem_validate.
  for (int i = 1; i < p.n; ++i) {
    const int a = p.ancestor[i];
    if (a < 0 || a >= i || p.node_stage[a] != p.node_stage[i] - 1)
      fail(SCENOPT_E_DIMENSION_MISMATCH, "problem: node " + std::to_string(i) + " has an invalid ancestor");
    if (i + 1 < p.n && p.node_stage[i] == p.node_stage[i + 1] && p.ancestor[i] > p.ancestor[i + 1])
      fail(SCENOPT_E_DIMENSION_MISMATCH, "problem: tree is not in BFS order");
  }
  for (int i = 0; i < p.first_leaf; ++i)
    if (p.child_count[i] == 0)
      fail(SCENOPT_E_DIMENSION_MISMATCH, "problem: interior node " + std::to_string(i) + " has no children");
}

// solvers.hpp:569-602
Problem precondition(const Problem& src) {
  Problem p = src;
  auto scale_block = [&](int kind, double& gamma, int off, int rows, double root) {
    if (kind == 1) {
      for (int j = 0; j < rows; ++j) {
        p.zmin[off + j] *= root;
        p.zmax[off + j] *= root;
      }
    } else if (kind == 2) {
      gamma /= root;
    }
  };
  for (int i = 1; i < p.n; ++i) {
    const double pi = p.probability[i];
    if (!(pi > 0.0)) fail(SCENOPT_E_ZERO_PROBABILITY, "precondition: node probability");
    const double root = std::sqrt(pi);
    const int m = p.stage_rows[i], off = p.dual_offset[i];
    for (size_t k = 0; k < static_cast<size_t>(m) * p.nx; ++k) p.F[off * static_cast<size_t>(p.nx) + k] *= root;
    for (size_t k = 0; k < static_cast<size_t>(m) * p.nu; ++k) p.G[off * static_cast<size_t>(p.nu) + k] *= root;
    scale_block(p.g_kind[i], p.g_gamma[i], off, m, root);
  }
  for (int l = 0; l < p.L; ++l) {
    const int i = p.first_leaf + l;
    const double pi = p.probability[i];
    if (!(pi > 0.0)) fail(SCENOPT_E_ZERO_PROBABILITY, "precondition: leaf probability");
    const double root = std::sqrt(pi);
    const int m = p.terminal_rows[l], off = p.tdual_offset[l];
    for (size_t k = 0; k < static_cast<size_t>(m) * p.nx; ++k)
      p.FN[static_cast<size_t>(off - p.stage_total) * p.nx + k] *= root;
    scale_block(p.tg_kind[l], p.tg_gamma[l], off, m, root);
  }
  return p;
}

// solvers.hpp:608-623
std::vector<double> probability_roots(const Problem& p) {
  std::vector<double> roots(static_cast<size_t>(p.dual_dim), 0.0);
  for (int i = 1; i < p.n; ++i)
    std::fill(roots.begin() + p.dual_offset[i], roots.begin() + p.dual_offset[i] + p.stage_rows[i],
              std::sqrt(p.probability[i]));
  for (int l = 0; l < p.L; ++l)
    std::fill(roots.begin() + p.tdual_offset[l],
              roots.begin() + p.tdual_offset[l] + p.terminal_rows[l],
              std::sqrt(p.probability[p.first_leaf + l]));
  return roots;
}

// ---------------------------------------------------------------- generator
// generators.hpp:255-328 extended with per-stage branching. The draw stream
// is consumed strictly in the reference's order (A row-major, B, W, q, r, F,
// G, box pairs; leaves W_P, p, F_N, box), so it is drawn sequentially into
// the node arrays first; the spectral rescaling of A and the W W' + 0.1 I
// blocks consume no draws and run on the worker pool afterwards.
Problem gen_random_tree(int nx, int nu, int horizon, const std::vector<int>& br) {
  if (nx < 1 || nu < 1) fail(SCENOPT_E_INVALID_PARAMS, "gen_random_instance: dims must be positive");
  if (horizon < 1) fail(SCENOPT_E_INVALID_PARAMS, "gen_random_instance: tree shape must be positive");
  for (int b : br)
    if (b < 1) fail(SCENOPT_E_INVALID_PARAMS, "gen_random_instance: tree shape must be positive");
  Problem p;
  p.nx = nx;
  p.nu = nu;
  p.N = horizon;
  p.ancestor = {-1};
  p.probability = {1.0};
  p.stage_offsets = {0, 1};
  p.mode = {-1};
  {
    int begin = 0, end = 1;
    for (int t = 0; t < horizon; ++t) {
      const int nb = t < static_cast<int>(br.size()) ? br[t] : 1;
      const double branch = 1.0 / nb;
      for (int i = begin; i < end; ++i)
        for (int w = 0; w < nb; ++w) {
          p.ancestor.push_back(i);
          p.probability.push_back(p.probability[i] * branch);
          p.mode.push_back(w);
        }
      begin = end;
      end = static_cast<int>(p.ancestor.size());
      p.stage_offsets.push_back(end);
    }
  }
  p.n = static_cast<int>(p.ancestor.size());
  const int n = p.n;
  const int L = n - p.stage_offsets[horizon];
  p.stage_rows.assign(static_cast<size_t>(n), 2);
  p.stage_rows[0] = 0;
  p.terminal_rows.assign(static_cast<size_t>(L), 1);
  p.finalize();
  return p;
}

void require_full(const Problem& p, const char* who) {
  if (!p.held.empty())
    fail(SCENOPT_E_INVALID_PARAMS, std::string(who) + ": the instance holds only one shard's nodes");
}

Problem gen_random(uint64_t seed, int nx, int nu, int horizon, const std::vector<int>& br,
                   const std::vector<char>* keep) {
  Problem p = gen_random_tree(nx, nu, horizon, br);
  const int n = p.n;
  const int L = p.L;
  if (keep) {
    if (static_cast<int>(keep->size()) != n) fail(SCENOPT_E_INVALID_PARAMS, "gen_random_instance: keep mask size");
    if (std::find(keep->begin(), keep->end(), 0) != keep->end()) p.held = *keep;  // else: the full instance
  }
  auto kept = [&](int i) { return !keep || (*keep)[i]; };
  p.root_state.assign(static_cast<size_t>(nx), 0.0);
  const size_t sxx = p.sxx(), sxu = p.sxu(), suu = p.suu();
  const int nw = nx + nu;
  const size_t sww = static_cast<size_t>(nw) * nw;
  zeros(p.A, n * sxx);
  zeros(p.B, n * sxu);
  p.c.assign(static_cast<size_t>(n) * nx, 0.0);
  zeros(p.Q, n * sxx);
  zeros(p.R, n * suu);
  zeros(p.S, n * sxu);
  p.q.assign(static_cast<size_t>(n) * nx, 0.0);
  p.r.assign(static_cast<size_t>(n) * nu, 0.0);
  p.F.assign(static_cast<size_t>(p.stage_total) * nx, 0.0);
  p.G.assign(static_cast<size_t>(p.stage_total) * nu, 0.0);
  p.g_kind.assign(static_cast<size_t>(n), 1);
  p.g_kind[0] = 0;
  p.g_gamma.assign(static_cast<size_t>(n), 0.0);
  p.zmin.assign(static_cast<size_t>(p.dual_dim), 0.0);
  p.zmax.assign(static_cast<size_t>(p.dual_dim), 0.0);
  zeros(p.P, static_cast<size_t>(L) * sxx);
  p.p.assign(static_cast<size_t>(L) * nx, 0.0);
  p.FN.assign(static_cast<size_t>(L) * nx, 0.0);
  p.tg_kind.assign(static_cast<size_t>(L), 1);
  p.tg_gamma.assign(static_cast<size_t>(L), 0.0);

  std::mt19937_64 gen(seed);
  auto unit = [&gen]() { return static_cast<double>(gen() >> 11) * 0x1.0p-53; };
  auto sym = [&unit]() { return 2.0 * unit() - 1.0; };
  // raw W roots of the kept nodes (consumed by the parallel pass); the
  // draws of other nodes go to scratch
  std::vector<int> wslot(static_cast<size_t>(n), -1), knodes;
  for (int i = 1; i < n; ++i)
    if (kept(i)) {
      wslot[i] = static_cast<int>(knodes.size());
      knodes.push_back(i);
    }
  std::vector<double> wroot(std::max<size_t>(knodes.size(), 1) * sww), scratch(sxx + sxu + sww);
  for (int i = 1; i < n; ++i) {
    const bool k = kept(i);
    double* A = k ? p.A.data() + i * sxx : scratch.data();
    for (int a = 0; a < nx; ++a)
      for (int b = 0; b < nx; ++b) A[a + b * nx] = sym();  // row-major draw order
    double* B = k ? p.B.data() + i * sxu : scratch.data() + sxx;
    for (int a = 0; a < nx; ++a)
      for (int b = 0; b < nu; ++b) B[a + b * nx] = sym();
    double* W = k ? wroot.data() + static_cast<size_t>(wslot[i]) * sww : scratch.data() + sxx + sxu;
    for (int a = 0; a < nw; ++a)
      for (int b = 0; b < nw; ++b) W[a + b * nw] = sym();
    for (int a = 0; a < nx; ++a) p.q[static_cast<size_t>(i) * nx + a] = 1.5 * sym();
    for (int a = 0; a < nu; ++a) p.r[static_cast<size_t>(i) * nu + a] = 1.5 * sym();
    const int off = p.dual_offset[i];
    double* F = p.F.data() + static_cast<size_t>(off) * nx;
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < nx; ++b) F[a + b * 2] = sym();
    double* G = p.G.data() + static_cast<size_t>(off) * nu;
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < nu; ++b) G[a + b * 2] = sym();
    for (int k = 0; k < 2; ++k) {
      p.zmin[off + k] = -(0.05 + 0.3 * unit());
      p.zmax[off + k] = 0.05 + 0.3 * unit();
    }
  }
  BigVec proot;
  zeros(proot, static_cast<size_t>(L) * sxx);
  for (int l = 0; l < L; ++l) {
    double* W = kept(p.first_leaf + l) ? proot.data() + l * sxx : scratch.data();
    for (int a = 0; a < nx; ++a)
      for (int b = 0; b < nx; ++b) W[a + b * nx] = sym();
    for (int a = 0; a < nx; ++a) p.p[static_cast<size_t>(l) * nx + a] = 1.5 * sym();
    for (int b = 0; b < nx; ++b) p.FN[static_cast<size_t>(l) * nx + b] = sym();
    const int off = p.tdual_offset[l];
    p.zmin[off] = -(0.05 + 0.3 * unit());
    p.zmax[off] = 0.05 + 0.3 * unit();
  }
  parallel_for(static_cast<int>(knodes.size()), 64, [&](int b, int e) {
    std::vector<double> blk(sww);
    for (int k = b; k < e; ++k) {
      const int i = knodes[k];
      double* A = p.A.data() + i * sxx;
      const double radius = spectral_radius(A, nx);
      if (radius > 0.0) {
        const double s = 0.95 / radius;
        for (size_t t = 0; t < sxx; ++t) A[t] *= s;
      }
      const double* W = wroot.data() + k * sww;
      for (int cidx = 0; cidx < nw; ++cidx)
        for (int ridx = 0; ridx < nw; ++ridx) {
          double s = 0.0;
          for (int t = 0; t < nw; ++t) s += W[ridx + t * nw] * W[cidx + t * nw];
          blk[ridx + cidx * nw] = s + (ridx == cidx ? 0.1 : 0.0);
        }
      double* Q = p.Q.data() + i * sxx;
      double* S = p.S.data() + i * sxu;
      double* R = p.R.data() + i * suu;
      for (int a = 0; a < nx; ++a)
        for (int b2 = 0; b2 < nx; ++b2) Q[b2 + a * nx] = blk[b2 + a * nw];
      for (int a = 0; a < nx; ++a)
        for (int b2 = 0; b2 < nu; ++b2) S[b2 + a * nu] = blk[nx + b2 + a * nw];
      for (int a = 0; a < nu; ++a)
        for (int b2 = 0; b2 < nu; ++b2) R[b2 + a * nu] = blk[nx + b2 + (nx + a) * nw];
    }
  });
  parallel_for(L, 64, [&](int b, int e) {
    for (int l = b; l < e; ++l) {
      if (!kept(p.first_leaf + l)) continue;
      const double* W = proot.data() + l * sxx;
      double* P = p.P.data() + l * sxx;
      for (int cidx = 0; cidx < nx; ++cidx)
        for (int ridx = 0; ridx < nx; ++ridx) {
          double s = 0.0;
          for (int t = 0; t < nx; ++t) s += W[ridx + t * nx] * W[cidx + t * nx];
          P[ridx + cidx * nx] = s + (ridx == cidx ? 0.1 : 0.0);
        }
    }
  });
  return p;
}

}  // namespace scn

namespace scn {
// ---------------------------------------------------------------- spring-mass
// generators.hpp:66-91 (column-major 2M x 2M and 2M x (M-1))
void spring_mass_continuous(int masses, const SpringMass& par, std::vector<double>& A, std::vector<double>& B) {
  const int M = masses, nx = 2 * M, nu = M - 1;
  A.assign(static_cast<size_t>(nx) * nx, 0.0);
  B.assign(static_cast<size_t>(nx) * nu, 0.0);
  const double ks = par.stiffness / par.mass_kg, bs = par.damping / par.mass_kg;
  auto a = [&](int i, int j) -> double& { return A[i + static_cast<size_t>(j) * nx]; };
  for (int j = 0; j < M; ++j) {
    a(j, M + j) = 1.0;                         // dp/dt = v
    a(M + j, j) = -ks * 2.0;                   // -(k/m) T, T = tridiag(-1, 2, -1)
    a(M + j, M + j) = -bs * 2.0;               // -(b/m) T
    if (j > 0) {
      a(M + j, j - 1) = -ks * -1.0;
      a(M + j, M + j - 1) = -bs * -1.0;
    }
    if (j + 1 < M) {
      a(M + j, j + 1) = -ks * -1.0;
      a(M + j, M + j + 1) = -bs * -1.0;
    }
  }
  for (int u = 0; u < nu; ++u) {  // actuator u: -u on mass u, +u on mass u+1
    B[(M + u) + static_cast<size_t>(u) * nx] = -1.0 / par.mass_kg;
    B[(M + u + 1) + static_cast<size_t>(u) * nx] = 1.0 / par.mass_kg;
  }
}

// generators.hpp:97-112
void discretize_zoh(const double* A, const double* B, int n, int m, double period, double* Ad, double* Bd) {
  if (!(period > 0.0)) fail(SCENOPT_E_INVALID_PARAMS, "discretize_zoh: period must be > 0");
  const int k = n + m;
  std::vector<double> aug(static_cast<size_t>(k) * k, 0.0);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) aug[i + static_cast<size_t>(j) * k] = A[i + static_cast<size_t>(j) * n] * period;
  for (int j = 0; j < m; ++j)
    for (int i = 0; i < n; ++i) aug[i + static_cast<size_t>(n + j) * k] = B[i + static_cast<size_t>(j) * n] * period;
  const std::vector<double> E = expm(aug, k);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) Ad[i + static_cast<size_t>(j) * n] = E[i + static_cast<size_t>(j) * k];
  for (int j = 0; j < m; ++j)
    for (int i = 0; i < n; ++i) Bd[i + static_cast<size_t>(j) * n] = E[i + static_cast<size_t>(n + j) * k];
}

// build_from_markov, scenario_tree.hpp:72-126: all positive-probability mode
// paths in BFS order, children in mode order (fills the tree members of p)
void markov_tree(const std::vector<double>& T, int rows, int cols, const std::vector<double>& initial, int horizon,
                 Problem& p) {
  const int modes = static_cast<int>(initial.size());
  if (horizon < 1) fail(SCENOPT_E_INVALID_PARAMS, "build_from_markov: horizon must be >= 1");
  if (rows != modes || cols != modes)
    fail(SCENOPT_E_DIMENSION_MISMATCH,
         "build_from_markov: transition must be square and match the initial distribution size");
  double sum = 0.0, mn = 0.0;
  for (double v : initial) {
    sum += v;
    mn = std::min(mn, v);
  }
  if (modes == 0 || mn < 0.0 || std::fabs(sum - 1.0) > 1e-9)
    fail(SCENOPT_E_NON_STOCHASTIC_MATRIX, "build_from_markov: initial distribution");
  for (int w = 0; w < modes; ++w) {
    double rs = 0.0, rm = 0.0;
    for (int j = 0; j < modes; ++j) {
      rs += T[static_cast<size_t>(w) * modes + j];
      rm = std::min(rm, T[static_cast<size_t>(w) * modes + j]);
    }
    if (rm < 0.0 || std::fabs(rs - 1.0) > 1e-9)
      fail(SCENOPT_E_NON_STOCHASTIC_MATRIX, "build_from_markov: transition row " + std::to_string(w));
  }
  p.N = horizon;
  p.ancestor = {-1};
  p.probability = {1.0};
  p.stage_offsets = {0, 1};
  p.mode = {-1};
  for (int t = 0, begin = 0, end = 1; t < horizon; ++t) {
    for (int i = begin; i < end; ++i)
      for (int w = 0; w < modes; ++w) {
        const double branch = t == 0 ? initial[static_cast<size_t>(w)]
                                     : T[static_cast<size_t>(p.mode[static_cast<size_t>(i)]) * modes + w];
        if (branch <= 0.0) continue;
        p.ancestor.push_back(i);
        p.probability.push_back(p.probability[static_cast<size_t>(i)] * branch);
        p.mode.push_back(w);
      }
    begin = end;
    end = static_cast<int>(p.ancestor.size());
    p.stage_offsets.push_back(end);
  }
  p.n = static_cast<int>(p.ancestor.size());
}

// generators.hpp:119-218 on the tree of scenario_tree.hpp:72-126 (positive-probability
// mode paths, BFS order, children in mode order)
Problem gen_spring_mass(int masses, const SpringMass& params) {
  if (masses < 2) fail(SCENOPT_E_INVALID_PARAMS, "gen_spring_mass: masses must be >= 2");
  if (!(params.mass_kg > 0.0)) fail(SCENOPT_E_INVALID_PARAMS, "gen_spring_mass: mass_kg must be > 0");
  if (!(params.input_bound > 0.0) || !(params.velocity_bound > 0.0))
    fail(SCENOPT_E_INVALID_PARAMS, "gen_spring_mass: bounds must be > 0");
  if (!(params.input_weight > 0.0) || !(params.terminal_weight > 0.0))
    fail(SCENOPT_E_INVALID_PARAMS, "gen_spring_mass: input and terminal weights must be > 0");
  if (params.state_weight < 0.0) fail(SCENOPT_E_INVALID_PARAMS, "gen_spring_mass: state_weight must be >= 0");
  SpringMass par = params;
  if (par.initial_probs.empty()) par.initial_probs = {0.5, 0.5};
  if (par.transition.empty()) {
    par.transition = {0.1, 0.9, 0.9, 0.1};
    par.transition_rows = par.transition_cols = 2;
  }
  if (par.mode_values.empty()) {
    par.mode_values.assign(par.initial_probs.size(), 0.0);
    if (par.mode_values.size() > 1) par.mode_values[1] = 0.1;
  }
  if (par.mode_values.size() != par.initial_probs.size())
    fail(SCENOPT_E_DIMENSION_MISMATCH, "gen_spring_mass: one mode value per Markov mode required");
  const int M = masses, nx = 2 * M, nu = M - 1;
  std::vector<double> Ac, Bc, Ad(static_cast<size_t>(nx) * nx), Bd(static_cast<size_t>(nx) * nu);
  spring_mass_continuous(M, par, Ac, Bc);
  discretize_zoh(Ac.data(), Bc.data(), nx, nu, par.sampling, Ad.data(), Bd.data());
  Problem p;
  markov_tree(par.transition, par.transition_rows, par.transition_cols, par.initial_probs, par.horizon, p);
  if (!par.root_state.empty() && static_cast<int>(par.root_state.size()) != nx)
    fail(SCENOPT_E_DIMENSION_MISMATCH, "gen_spring_mass: root_state must have length 2M");

  p.nx = nx;
  p.nu = nu;
  const std::vector<int32_t>& mode = p.mode;
  const int n = p.n, L = n - p.stage_offsets[static_cast<size_t>(par.horizon)], rows = M + nu;
  p.stage_rows.assign(static_cast<size_t>(n), rows);
  p.stage_rows[0] = 0;
  p.terminal_rows.assign(static_cast<size_t>(L), M);
  p.finalize();
  p.root_state = par.root_state.empty() ? std::vector<double>(static_cast<size_t>(nx), 0.0) : par.root_state;
  const size_t sxx = p.sxx(), sxu = p.sxu(), suu = p.suu();
  zeros(p.A, n * sxx);
  zeros(p.B, n * sxu);
  p.c.assign(static_cast<size_t>(n) * nx, 0.0);
  zeros(p.Q, n * sxx);
  zeros(p.R, n * suu);
  zeros(p.S, n * sxu);
  p.q.assign(static_cast<size_t>(n) * nx, 0.0);
  p.r.assign(static_cast<size_t>(n) * nu, 0.0);
  p.F.assign(static_cast<size_t>(p.stage_total) * nx, 0.0);
  p.G.assign(static_cast<size_t>(p.stage_total) * nu, 0.0);
  p.g_kind.assign(static_cast<size_t>(n), 1);
  p.g_kind[0] = 0;
  p.g_gamma.assign(static_cast<size_t>(n), 0.0);
  p.zmin.assign(static_cast<size_t>(p.dual_dim), 0.0);
  p.zmax.assign(static_cast<size_t>(p.dual_dim), 0.0);
  zeros(p.P, static_cast<size_t>(L) * sxx);
  p.p.assign(static_cast<size_t>(L) * nx, 0.0);
  p.FN.assign(static_cast<size_t>(L) * M * nx, 0.0);
  p.tg_kind.assign(static_cast<size_t>(L), 1);
  p.tg_gamma.assign(static_cast<size_t>(L), 0.0);
  for (int i = 1; i < n; ++i) {
    std::copy(Ad.begin(), Ad.end(), p.A.begin() + static_cast<std::ptrdiff_t>(i * sxx));
    std::copy(Bd.begin(), Bd.end(), p.B.begin() + static_cast<std::ptrdiff_t>(i * sxu));
    std::fill_n(p.c.begin() + static_cast<std::ptrdiff_t>(i) * nx, nx, par.mode_values[static_cast<size_t>(mode[static_cast<size_t>(i)])]);
    for (int k = 0; k < nx; ++k) p.Q[i * sxx + k + static_cast<size_t>(k) * nx] = par.state_weight;
    for (int k = 0; k < nu; ++k) p.R[i * suu + k + static_cast<size_t>(k) * nu] = par.input_weight;
    const int off = p.dual_offset[i];
    double* F = p.F.data() + static_cast<size_t>(off) * nx;  // rows x nx column-major
    double* G = p.G.data() + static_cast<size_t>(off) * nu;
    for (int k = 0; k < M; ++k) F[k + static_cast<size_t>(M + k) * rows] = 1.0;  // velocity rows
    for (int k = 0; k < nu; ++k) G[(M + k) + static_cast<size_t>(k) * rows] = 1.0;  // input rows
    for (int k = 0; k < rows; ++k) {
      const double bnd = k < M ? par.velocity_bound : par.input_bound;
      p.zmin[static_cast<size_t>(off + k)] = -bnd;
      p.zmax[static_cast<size_t>(off + k)] = bnd;
    }
  }
  for (int l = 0; l < L; ++l) {
    for (int k = 0; k < nx; ++k) p.P[l * sxx + k + static_cast<size_t>(k) * nx] = par.terminal_weight;
    const int off = p.tdual_offset[l];
    double* FN = p.FN.data() + static_cast<size_t>(off - p.stage_total) * nx;
    for (int k = 0; k < M; ++k) {
      FN[k + static_cast<size_t>(M + k) * M] = 1.0;
      p.zmin[static_cast<size_t>(off + k)] = -par.velocity_bound;
      p.zmax[static_cast<size_t>(off + k)] = par.velocity_bound;
    }
  }
  return p;
}
}  // namespace scn
