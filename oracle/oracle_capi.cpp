// SPDX-License-Identifier: MIT
// TEST INFRASTRUCTURE ONLY — C-ABI wrapper of the CPU parity oracle.
#include "oracle_capi.h"

#include <chrono>
#include <cstring>
#include <memory>
#include <string>

#include "oracle_core.hpp"

using namespace orc;

struct orc_problem {
  ProblemInstance prob;
  // flat export storage
  std::vector<int32_t> anc, soff, srows, gkind, trows, tgkind;
  std::vector<double> A, B, c, Q, R, S, q, r, F, G, ggam, P, p, FN, tggam, zmin, zmax;
};
struct orc_factor { FactorCache cache; };
struct orc_g { SeparableNonsmooth g; };
struct orc_rng { Rng rng; explicit orc_rng(uint64_t s) : rng(s) {} };
struct orc_lbfgs { LbfgsBuffer buf; orc_lbfgs(int m, double e) : buf(m, e) {} };
struct orc_report { SolverReport rep; };

static thread_local std::string g_err;

#define ORC_GUARD(...)                        \
  try {                                        \
    __VA_ARGS__;                               \
    return 0;                                  \
  } catch (const orc::Error& e) {              \
    g_err = e.what();                          \
    return e.code;                             \
  } catch (const std::exception& e) {          \
    g_err = e.what();                          \
    return kError;                             \
  }

extern "C" const char* orc_last_error(void) { return g_err.c_str(); }

namespace {
Mat mat_from(const double* src, int r, int c) {
  Mat m(r, c);
  if (r > 0 && c > 0) std::memcpy(m.d.data(), src, sizeof(double) * static_cast<size_t>(r) * c);
  return m;
}
Vec vec_from(const double* src, int n) { return Vec(src, src + n); }

NonsmoothSpec spec_from(int kind, double gamma, const double* zmin, const double* zmax, int rows) {
  NonsmoothSpec s;
  s.kind = static_cast<NonsmoothKind>(kind);
  s.gamma = gamma;
  if (s.kind == NonsmoothKind::Box) {
    s.zmin = vec_from(zmin, rows);
    s.zmax = vec_from(zmax, rows);
  }
  return s;
}

ProblemInstance from_view(const orc_problem_view& v) {
  ProblemInstance prob;
  const int n = v.num_nodes, nx = v.nx, nu = v.nu;
  ScenarioTree& t = prob.tree;
  t.num_stages = v.num_stages;
  t.stage_offsets.assign(v.stage_offsets, v.stage_offsets + v.num_stages + 2);
  t.ancestor.assign(v.ancestor, v.ancestor + n);
  t.probability.assign(v.probability, v.probability + n);
  t.node_stage.assign(static_cast<size_t>(n), 0);
  t.children.assign(static_cast<size_t>(n), {});
  for (int s = 0; s <= v.num_stages; ++s)
    for (int i = v.stage_offsets[s]; i < v.stage_offsets[s + 1]; ++i) t.node_stage[static_cast<size_t>(i)] = s;
  for (int i = 1; i < n; ++i) t.children[static_cast<size_t>(v.ancestor[i])].push_back(i);
  prob.nx = nx;
  prob.nu = nu;
  prob.root_state = vec_from(v.root_state, nx);
  prob.dyn.resize(static_cast<size_t>(n));
  prob.cost.resize(static_cast<size_t>(n));
  prob.con.resize(static_cast<size_t>(n));
  const size_t sxx = static_cast<size_t>(nx) * nx, sxu = static_cast<size_t>(nx) * nu,
               suu = static_cast<size_t>(nu) * nu;
  int off = 0;
  for (int i = 0; i < n; ++i) {
    const auto si = static_cast<size_t>(i);
    prob.dyn[si] = NodeDynamics{mat_from(v.A + si * sxx, nx, nx), mat_from(v.B + si * sxu, nx, nu),
                                vec_from(v.c + si * nx, nx)};
    prob.cost[si] = NodeCost{mat_from(v.Q + si * sxx, nx, nx), mat_from(v.R + si * suu, nu, nu),
                             mat_from(v.S + si * sxu, nu, nx), vec_from(v.q + si * nx, nx),
                             vec_from(v.r + si * nu, nu)};
    const int m = i == 0 ? 0 : v.stage_rows[i];
    prob.con[si].F = mat_from(v.F + static_cast<size_t>(off) * nx, m, nx);
    prob.con[si].G = mat_from(v.G + static_cast<size_t>(off) * nu, m, nu);
    prob.con[si].g = i == 0 ? NonsmoothSpec{}
                            : spec_from(v.g_kind[i], v.g_gamma[i], v.zmin + off, v.zmax + off, m);
    off += m;
  }
  const int stage_total = off;
  const int L = n - v.stage_offsets[v.num_stages];
  prob.tcost.resize(static_cast<size_t>(L));
  prob.tcon.resize(static_cast<size_t>(L));
  for (int l = 0; l < L; ++l) {
    const auto sl = static_cast<size_t>(l);
    prob.tcost[sl] = TerminalCost{mat_from(v.P + sl * sxx, nx, nx), vec_from(v.p + sl * nx, nx)};
    const int m = v.terminal_rows[l];
    prob.tcon[sl].F = mat_from(v.FN + static_cast<size_t>(off - stage_total) * nx, m, nx);
    prob.tcon[sl].g = spec_from(v.tg_kind[l], v.tg_gamma[l], v.zmin + off, v.zmax + off, m);
    off += m;
  }
  prob.finalize_layout();
  return prob;
}

void export_flat(orc_problem* h, orc_problem_view* v, int32_t* dual_dim) {
  const ProblemInstance& pr = h->prob;
  const int n = pr.num_nodes(), nx = pr.nx, nu = pr.nu, L = pr.tree.num_leaves();
  h->anc.assign(pr.tree.ancestor.begin(), pr.tree.ancestor.end());
  h->soff.assign(pr.tree.stage_offsets.begin(), pr.tree.stage_offsets.end());
  h->srows.assign(static_cast<size_t>(n), 0);
  h->gkind.assign(static_cast<size_t>(n), 0);
  h->ggam.assign(static_cast<size_t>(n), 0.0);
  const size_t sxx = static_cast<size_t>(nx) * nx, sxu = static_cast<size_t>(nx) * nu,
               suu = static_cast<size_t>(nu) * nu;
  h->A.assign(n * sxx, 0.0);
  h->B.assign(n * sxu, 0.0);
  h->c.assign(static_cast<size_t>(n) * nx, 0.0);
  h->Q.assign(n * sxx, 0.0);
  h->R.assign(n * suu, 0.0);
  h->S.assign(n * sxu, 0.0);
  h->q.assign(static_cast<size_t>(n) * nx, 0.0);
  h->r.assign(static_cast<size_t>(n) * nu, 0.0);
  const int D = pr.dual_dim;
  int stage_total = 0;
  for (int i = 1; i < n; ++i) stage_total += pr.stage_rows(i);
  h->F.assign(static_cast<size_t>(stage_total) * nx, 0.0);
  h->G.assign(static_cast<size_t>(stage_total) * nu, 0.0);
  h->FN.assign(static_cast<size_t>(D - stage_total) * nx, 0.0);
  h->zmin.assign(static_cast<size_t>(D), 0.0);
  h->zmax.assign(static_cast<size_t>(D), 0.0);
  for (int i = 1; i < n; ++i) {
    const auto si = static_cast<size_t>(i);
    auto cp = [](const Mat& m, double* dst) { std::copy(m.d.begin(), m.d.end(), dst); };
    cp(pr.dyn[si].A, h->A.data() + si * sxx);
    cp(pr.dyn[si].B, h->B.data() + si * sxu);
    std::copy(pr.dyn[si].c.begin(), pr.dyn[si].c.end(), h->c.data() + si * nx);
    cp(pr.cost[si].Q, h->Q.data() + si * sxx);
    cp(pr.cost[si].R, h->R.data() + si * suu);
    cp(pr.cost[si].S, h->S.data() + si * sxu);
    std::copy(pr.cost[si].q.begin(), pr.cost[si].q.end(), h->q.data() + si * nx);
    std::copy(pr.cost[si].r.begin(), pr.cost[si].r.end(), h->r.data() + si * nu);
    const int m = pr.stage_rows(i), off = pr.dual_offset[si];
    h->srows[si] = m;
    cp(pr.con[si].F, h->F.data() + static_cast<size_t>(off) * nx);
    cp(pr.con[si].G, h->G.data() + static_cast<size_t>(off) * nu);
    h->gkind[si] = static_cast<int32_t>(pr.con[si].g.kind);
    h->ggam[si] = pr.con[si].g.gamma;
    if (pr.con[si].g.kind == NonsmoothKind::Box)
      for (int k = 0; k < m; ++k) {
        h->zmin[static_cast<size_t>(off + k)] = pr.con[si].g.zmin[static_cast<size_t>(k)];
        h->zmax[static_cast<size_t>(off + k)] = pr.con[si].g.zmax[static_cast<size_t>(k)];
      }
  }
  h->P.assign(static_cast<size_t>(L) * sxx, 0.0);
  h->p.assign(static_cast<size_t>(L) * nx, 0.0);
  h->trows.assign(static_cast<size_t>(L), 0);
  h->tgkind.assign(static_cast<size_t>(L), 0);
  h->tggam.assign(static_cast<size_t>(L), 0.0);
  for (int l = 0; l < L; ++l) {
    const auto sl = static_cast<size_t>(l);
    std::copy(pr.tcost[sl].P.d.begin(), pr.tcost[sl].P.d.end(), h->P.data() + sl * sxx);
    std::copy(pr.tcost[sl].p.begin(), pr.tcost[sl].p.end(), h->p.data() + sl * nx);
    const int m = pr.terminal_rows(l), off = pr.tdual_offset[sl];
    h->trows[sl] = m;
    std::copy(pr.tcon[sl].F.d.begin(), pr.tcon[sl].F.d.end(),
              h->FN.data() + static_cast<size_t>(off - stage_total) * nx);
    h->tgkind[sl] = static_cast<int32_t>(pr.tcon[sl].g.kind);
    h->tggam[sl] = pr.tcon[sl].g.gamma;
    if (pr.tcon[sl].g.kind == NonsmoothKind::Box)
      for (int k = 0; k < m; ++k) {
        h->zmin[static_cast<size_t>(off + k)] = pr.tcon[sl].g.zmin[static_cast<size_t>(k)];
        h->zmax[static_cast<size_t>(off + k)] = pr.tcon[sl].g.zmax[static_cast<size_t>(k)];
      }
  }
  v->nx = nx;
  v->nu = nu;
  v->num_stages = pr.tree.num_stages;
  v->num_nodes = n;
  v->ancestor = h->anc.data();
  v->probability = pr.tree.probability.data();
  v->stage_offsets = h->soff.data();
  v->root_state = pr.root_state.data();
  v->A = h->A.data();
  v->B = h->B.data();
  v->c = h->c.data();
  v->Q = h->Q.data();
  v->R = h->R.data();
  v->S = h->S.data();
  v->q = h->q.data();
  v->r = h->r.data();
  v->stage_rows = h->srows.data();
  v->F = h->F.data();
  v->G = h->G.data();
  v->g_kind = h->gkind.data();
  v->g_gamma = h->ggam.data();
  v->P = h->P.data();
  v->p = h->p.data();
  v->terminal_rows = h->trows.data();
  v->FN = h->FN.data();
  v->tg_kind = h->tgkind.data();
  v->tg_gamma = h->tggam.data();
  v->zmin = h->zmin.data();
  v->zmax = h->zmax.data();
  if (dual_dim) *dual_dim = D;
}

SolverConfig cfg_from(const orc_solver_config* c) {
  SolverConfig s;
  s.lambda0 = c->lambda0;
  s.eps = c->eps;
  s.eps_curv = c->eps_curv;
  s.eps_bt = c->eps_bt;
  s.beta_bt = c->beta_bt;
  s.memory = c->memory;
  s.max_iters = c->max_iters;
  s.backtracking_rule = static_cast<BacktrackingRule>(c->backtracking_rule);
  s.warm_start = c->warm_start != 0;
  s.warm_start_iters = c->warm_start_iters;
  s.precondition = c->precondition != 0;
  s.nama_parallel_linesearch = c->nama_parallel_linesearch != 0;
  s.nama_update_tlambda = c->nama_update_tlambda != 0;
  return s;
}

PrimalPoint primal_from(const ProblemInstance& p, const double* x, const double* u) {
  PrimalPoint pt = zero_primal(p.nx, p.nu, p.tree);
  std::memcpy(pt.x.d.data(), x, sizeof(double) * pt.x.d.size());
  std::memcpy(pt.u.d.data(), u, sizeof(double) * pt.u.d.size());
  return pt;
}
void primal_to(const PrimalPoint& pt, double* x, double* u) {
  if (x) std::memcpy(x, pt.x.d.data(), sizeof(double) * pt.x.d.size());
  if (u) std::memcpy(u, pt.u.d.data(), sizeof(double) * pt.u.d.size());
}
void vec_to(const Vec& v, double* dst) {
  if (dst) std::memcpy(dst, v.data(), sizeof(double) * v.size());
}
}  // namespace

extern "C" {

int orc_problem_from_view(const orc_problem_view* v, orc_problem** out) {
  ORC_GUARD({
    auto h = std::make_unique<orc_problem>();
    h->prob = from_view(*v);
    *out = h.release();
  })
}
int orc_problem_view_get(orc_problem* p, orc_problem_view* v, int32_t* dual_dim) {
  ORC_GUARD(export_flat(p, v, dual_dim))
}
void orc_problem_free(orc_problem* p) { delete p; }

int orc_gen_random(uint64_t seed, int nx, int nu, int horizon, const int32_t* br, int nbr,
                   orc_problem** out) {
  ORC_GUARD({
    auto h = std::make_unique<orc_problem>();
    h->prob = gen_random_instance(seed, nx, nu, horizon, std::vector<int>(br, br + nbr));
    *out = h.release();
  })
}

namespace {
SpringMassParams sm_from(const orc_spring_mass_params* c) {
  SpringMassParams p;
  if (!c) return p;
  p.mass_kg = c->mass_kg;
  p.stiffness = c->stiffness;
  p.damping = c->damping;
  p.input_bound = c->input_bound;
  p.velocity_bound = c->velocity_bound;
  p.horizon = c->horizon;
  p.sampling = c->sampling;
  p.state_weight = c->state_weight;
  p.input_weight = c->input_weight;
  p.terminal_weight = c->terminal_weight;
  if (c->initial_len > 0) p.initial_probs.assign(c->initial_probs, c->initial_probs + c->initial_len);
  if (c->transition_rows > 0 && c->transition_cols > 0) {
    p.transition = Mat(c->transition_rows, c->transition_cols);
    for (int i = 0; i < c->transition_rows; ++i)
      for (int j = 0; j < c->transition_cols; ++j) p.transition(i, j) = c->transition[i * c->transition_cols + j];
  }
  if (c->mode_values_len > 0) p.mode_values.assign(c->mode_values, c->mode_values + c->mode_values_len);
  if (c->root_state_len > 0) p.root_state.assign(c->root_state, c->root_state + c->root_state_len);
  return p;
}
}  // namespace

int orc_gen_spring_mass(int masses, const orc_spring_mass_params* par, orc_problem** out) {
  ORC_GUARD({
    auto h = std::make_unique<orc_problem>();
    h->prob = gen_spring_mass(masses, sm_from(par));
    *out = h.release();
  })
}
int orc_expm_series(const double* X, int n, double* out) {
  ORC_GUARD({
    Mat M(n, n);
    std::copy(X, X + static_cast<size_t>(n) * n, M.d.begin());
    const Mat E = expm_series(M);
    std::copy(E.d.begin(), E.d.end(), out);
  })
}
int orc_spring_mass_continuous(int masses, const orc_spring_mass_params* par, double* A, double* B) {
  ORC_GUARD({
    Mat Ac, Bc;
    spring_mass_continuous(masses, sm_from(par), Ac, Bc);
    std::copy(Ac.d.begin(), Ac.d.end(), A);
    std::copy(Bc.d.begin(), Bc.d.end(), B);
  })
}
int orc_sample_initial_states(int masses, const orc_spring_mass_params* par, uint64_t seed, int count,
                              double* out) {
  ORC_GUARD({
    std::mt19937_64 gen(seed);
    const SpringMassParams p = sm_from(par);
    for (int k = 0; k < count; ++k) {
      const Vec s = sample_initial_state(masses, p, gen);
      std::copy(s.begin(), s.end(), out + static_cast<size_t>(k) * s.size());
    }
  })
}

int orc_problem_validate(const orc_problem* p, char* buf, int buflen) {
  try {
    const auto bad = validate_problem(p->prob);
    std::string all;
    for (const auto& b : bad) all += b + "\n";
    if (buf && buflen > 0) {
      std::strncpy(buf, all.c_str(), static_cast<size_t>(buflen - 1));
      buf[buflen - 1] = 0;
    }
    return static_cast<int>(bad.size());
  } catch (const orc::Error& e) {
    g_err = e.what();
    return e.code;
  }
}

int orc_problem_layout(const orc_problem* p, int32_t* dual_offset, int32_t* tdual_offset) {
  ORC_GUARD({
    std::copy(p->prob.dual_offset.begin(), p->prob.dual_offset.end(), dual_offset);
    std::copy(p->prob.tdual_offset.begin(), p->prob.tdual_offset.end(), tdual_offset);
  })
}
int orc_precondition(const orc_problem* p, orc_problem** out) {
  ORC_GUARD({
    auto h = std::make_unique<orc_problem>();
    h->prob = precondition(p->prob);
    *out = h.release();
  })
}
int orc_probability_roots(const orc_problem* p, double* out) {
  ORC_GUARD(vec_to(probability_roots(p->prob), out))
}

int orc_rng_new(uint64_t seed, orc_rng** out) {
  *out = new orc_rng(seed);
  return 0;
}
void orc_rng_free(orc_rng* r) { delete r; }
double orc_rng_uniform(orc_rng* r, double lo, double hi) { return r->rng.uniform(lo, hi); }
int orc_rng_integer(orc_rng* r, int lo, int hi) { return r->rng.integer(lo, hi); }
void orc_rng_vector(orc_rng* r, int n, double scale, double* out) {
  const Vec v = r->rng.vector(n, scale);
  std::copy(v.begin(), v.end(), out);
}
void orc_rng_matrix(orc_rng* r, int rows, int cols, double scale, double* out) {
  const Mat m = r->rng.matrix(rows, cols, scale);
  std::copy(m.d.begin(), m.d.end(), out);
}

static InstanceOptions opts_from(const orc_instance_options* o) {
  InstanceOptions opt;
  if (o) {
    opt.with_box = o->with_box != 0;
    opt.with_l1 = o->with_l1 != 0;
    opt.with_none = o->with_none != 0;
    opt.affine = o->affine != 0;
    opt.stage_rows_lo = o->stage_rows_lo;
    opt.stage_rows_hi = o->stage_rows_hi;
    opt.feasible_boxes = o->feasible_boxes != 0;
  }
  return opt;
}

int orc_random_instance(orc_rng* r, int stages, int max_nodes, int nx, int nu,
                        const orc_instance_options* o, orc_problem** out) {
  ORC_GUARD({
    auto h = std::make_unique<orc_problem>();
    ScenarioTree tree = random_tree(r->rng, stages, max_nodes);
    h->prob = random_instance(r->rng, std::move(tree), nx, nu, opts_from(o));
    *out = h.release();
  })
}

int orc_markov_instance(orc_rng* r, const double* transition, const double* initial, int modes,
                        int horizon, int nx, int nu, const orc_instance_options* o,
                        orc_problem** out) {
  ORC_GUARD({
    Mat T(modes, modes);
    for (int i = 0; i < modes; ++i)
      for (int j = 0; j < modes; ++j) T(i, j) = transition[i * modes + j];  // row-major input
    ScenarioTree tree = build_from_markov(T, Vec(initial, initial + modes), horizon);
    auto h = std::make_unique<orc_problem>();
    h->prob = random_instance(r->rng, std::move(tree), nx, nu, opts_from(o));
    *out = h.release();
  })
}

int orc_tree_from_markov(const double* transition, const double* initial, int modes, int horizon,
                         int32_t* num_nodes, int32_t* ancestor, double* probability,
                         int32_t* stage_offsets, int32_t* mode, int cap) {
  ORC_GUARD({
    Mat T(modes, modes);
    for (int i = 0; i < modes; ++i)
      for (int j = 0; j < modes; ++j) T(i, j) = transition[i * modes + j];
    const ScenarioTree tree = build_from_markov(T, Vec(initial, initial + modes), horizon);
    *num_nodes = tree.num_nodes();
    if (tree.num_nodes() <= cap) {
      for (int i = 0; i < tree.num_nodes(); ++i) {
        ancestor[i] = tree.ancestor[static_cast<size_t>(i)];
        probability[i] = tree.probability[static_cast<size_t>(i)];
        mode[i] = tree.mode[static_cast<size_t>(i)];
      }
      for (size_t t = 0; t < tree.stage_offsets.size(); ++t) stage_offsets[t] = tree.stage_offsets[t];
    }
  })
}

int orc_factor_create(const orc_problem* p, orc_factor** out) {
  ORC_GUARD({
    auto f = std::make_unique<orc_factor>();
    f->cache = factor(p->prob);
    *out = f.release();
  })
}
void orc_factor_free(orc_factor* f) { delete f; }
int orc_refactor_affine(orc_factor* f, const orc_problem* p) { ORC_GUARD(refactor_affine(f->cache, p->prob)) }

int orc_factor_export(const orc_factor* f, double* gain, double* c2i, double* cl, double* d2i,
                      double* d2c, double* ia, double* ca, double* vq, double* lca) {
  ORC_GUARD({
    const FactorCache& c = f->cache;
    const size_t nx = static_cast<size_t>(c.nx), nu = static_cast<size_t>(c.nu);
    for (int i = 0; i < c.first_leaf; ++i) {
      const auto si = static_cast<size_t>(i);
      std::copy(c.gain[si].d.begin(), c.gain[si].d.end(), gain + si * nu * nx);
      const size_t off = static_cast<size_t>(c.child_dual_offset[si]);
      std::copy(c.dual_to_input[si].d.begin(), c.dual_to_input[si].d.end(), d2i + off * nu);
      std::copy(c.dual_to_costate[si].d.begin(), c.dual_to_costate[si].d.end(), d2c + off * nx);
      std::copy(c.input_affine[si].begin(), c.input_affine[si].end(), ia + si * nu);
      std::copy(c.costate_affine[si].begin(), c.costate_affine[si].end(), ca + si * nx);
    }
    for (int i = 0; i < c.num_nodes; ++i) {
      const auto si = static_cast<size_t>(i);
      if (i > 0) {
        std::copy(c.child_to_input[si].d.begin(), c.child_to_input[si].d.end(), c2i + si * nu * nx);
        std::copy(c.closed_loop[si].d.begin(), c.closed_loop[si].d.end(), cl + si * nx * nx);
      }
      std::copy(c.value_quad[si].d.begin(), c.value_quad[si].d.end(), vq + si * nx * nx);
    }
    for (size_t l = 0; l < c.leaf_costate_affine.size(); ++l)
      std::copy(c.leaf_costate_affine[l].begin(), c.leaf_costate_affine[l].end(), lca + l * nx);
  })
}

int orc_sweep(const orc_factor* f, const orc_problem* p, const double* y, int affine, double* x,
              double* u) {
  ORC_GUARD({
    const Vec yv(y, y + p->prob.dual_dim);
    const PrimalPoint pt = affine ? dual_grad(f->cache, p->prob, yv) : hessian_vec(f->cache, p->prob, yv);
    primal_to(pt, x, u);
  })
}
int orc_apply_H(const orc_problem* p, const double* x, const double* u, double* z) {
  ORC_GUARD(vec_to(apply_H(p->prob, primal_from(p->prob, x, u)), z))
}
int orc_apply_H_adjoint(const orc_problem* p, const double* y, double* x, double* u) {
  ORC_GUARD(primal_to(apply_H_adjoint(p->prob, Vec(y, y + p->prob.dual_dim)), x, u))
}
int orc_eval_f(const orc_problem* p, const double* x, const double* u, double* out) {
  ORC_GUARD(*out = eval_f(p->prob, primal_from(p->prob, x, u)))
}
int orc_fhat_value(const orc_factor* f, const orc_problem* p, const double* y, double* out) {
  ORC_GUARD(*out = fhat_value(f->cache, p->prob, Vec(y, y + p->prob.dual_dim)))
}

int orc_g_from_problem(const orc_problem* p, orc_g** out) {
  ORC_GUARD({
    auto g = std::make_unique<orc_g>();
    g->g = make_nonsmooth(p->prob);
    *out = g.release();
  })
}
int orc_g_create(int dim, int nblocks, const int32_t* offset, const int32_t* size,
                 const double* weight, const int32_t* kind, const double* gamma, const double* zmin,
                 const double* zmax, orc_g** out) {
  ORC_GUARD({
    auto g = std::make_unique<orc_g>();
    g->g.dim = dim;
    for (int b = 0; b < nblocks; ++b) {
      GBlock blk;
      blk.offset = offset[b];
      blk.size = size[b];
      blk.weight = weight[b];
      blk.kind = static_cast<NonsmoothKind>(kind[b]);
      blk.gamma = gamma[b];
      if (blk.kind == NonsmoothKind::Box) {
        blk.zmin = Vec(zmin + blk.offset, zmin + blk.offset + blk.size);
        blk.zmax = Vec(zmax + blk.offset, zmax + blk.offset + blk.size);
      }
      g->g.blocks.push_back(blk);
    }
    *out = g.release();
  })
}
void orc_g_free(orc_g* g) { delete g; }
int orc_prox_g(const orc_g* g, const double* v, double gamma_prox, double* out) {
  ORC_GUARD(vec_to(prox_g(g->g, Vec(v, v + g->g.dim), gamma_prox), out))
}
int orc_conj_value_g(const orc_g* g, const double* w, double* out) {
  ORC_GUARD(*out = conj_value_g(g->g, Vec(w, w + g->g.dim)))
}
int orc_prox_g_conj(const orc_g* g, const double* v, double lambda, double* out) {
  ORC_GUARD(vec_to(prox_g_conj(g->g, Vec(v, v + g->g.dim), lambda), out))
}
int orc_dist_subdiff_inf(const orc_g* g, const double* y, const double* z, double* out) {
  ORC_GUARD(*out = dist_subdiff_inf(g->g, Vec(y, y + g->g.dim), Vec(z, z + g->g.dim)))
}

int orc_fb_step(const orc_factor* f, const orc_problem* p, const orc_g* g, const double* y,
                double lambda, double* x, double* u, double* Hx, double* z, double* R, double* T,
                double* scalars) {
  ORC_GUARD({
    const FbState s = fb_step(f->cache, p->prob, g->g, Vec(y, y + p->prob.dual_dim), lambda);
    primal_to(s.x, x, u);
    vec_to(s.Hx, Hx);
    vec_to(s.z, z);
    vec_to(s.R, R);
    vec_to(s.T, T);
    if (scalars) {
      scalars[0] = s.fhat;
      scalars[1] = s.conj_T;
      scalars[2] = s.znorm_sq;
      scalars[3] = s.value;
    }
  })
}

int orc_fbe_grad(const orc_factor* f, const orc_problem* p, const double* R, double lambda,
                 double* grad) {
  ORC_GUARD({
    FbState s;
    s.R = Vec(R, R + p->prob.dual_dim);
    s.lambda = lambda;
    vec_to(fbe_grad(s, f->cache, p->prob), grad);
  })
}

int orc_linesearch_cert(const orc_factor* f, const orc_problem* p, const orc_g* g, const double* y,
                        const double* Hx, double lambda, const double* ss, const double* shift,
                        const double* dir, int ntau, const double* taus, double* deltas,
                        double* cs, double* cfh, double* w, double* Hx_w, double* z, double* R,
                        double* T) {
  ORC_GUARD({
    const int D = p->prob.dual_dim;
    FbState s;
    s.y = Vec(y, y + D);
    s.Hx = Vec(Hx, Hx + D);
    s.lambda = lambda;
    s.fhat = ss[0];
    s.conj_T = ss[1];
    s.znorm_sq = ss[2];
    s.value = ss[3];
    const Vec d(dir, dir + D);
    const PrimalPoint hom_dir = hessian_vec(f->cache, p->prob, d);
    LineSearchCert cert;
    if (shift) {
      const Vec r(shift, shift + D);
      const PrimalPoint hom_r = hessian_vec(f->cache, p->prob, r);
      cert = linesearch_cert_shifted(s, g->g, r, d, hom_r, hom_dir, p->prob);
    } else {
      cert = linesearch_cert(s, d, hom_dir, p->prob);
    }
    if (cs) {
      cs[0] = cert.alpha1;
      cs[1] = cert.alpha2;
      cs[2] = cert.conj_anchor;
      cs[3] = cert.znorm_sq_anchor;
      cs[4] = cert.value_anchor;
      cs[5] = cert.fhat_anchor;
    }
    CertEval ev;
    for (int k = 0; k < ntau; ++k) {
      ev = evaluate_cert(cert, g->g, taus[k]);
      deltas[k] = ev.delta;
      if (cfh) cfh[k] = cert_fhat(cert, taus[k]);
    }
    if (ntau > 0) {
      vec_to(ev.w, w);
      vec_to(ev.Hx_w, Hx_w);
      vec_to(ev.z, z);
      vec_to(ev.R, R);
      vec_to(ev.T, T);
    }
  })
}

int orc_lbfgs_new(int memory, double eps_curv, orc_lbfgs** out) {
  ORC_GUARD(*out = new orc_lbfgs(memory, eps_curv))
}
void orc_lbfgs_free(orc_lbfgs* b) { delete b; }
int orc_lbfgs_push(orc_lbfgs* b, int n, const double* step, const double* change, double scale_ref) {
  return b->buf.push(Vec(step, step + n), Vec(change, change + n), scale_ref) ? 1 : 0;
}
int orc_lbfgs_apply(const orc_lbfgs* b, int n, const double* grad, double* out) {
  ORC_GUARD(vec_to(b->buf.apply_direction(Vec(grad, grad + n)), out))
}
void orc_lbfgs_clear(orc_lbfgs* b) { b->buf.clear(); }
int orc_lbfgs_size(const orc_lbfgs* b) { return b->buf.size(); }
double orc_lbfgs_gamma0(const orc_lbfgs* b) { return b->buf.gamma0(); }

int orc_estimate_lipschitz(const orc_factor* f, const orc_problem* p, uint64_t* calls, double* out) {
  ORC_GUARD(*out = estimate_dual_lipschitz(f->cache, p->prob, calls))
}
int orc_estimate_lipschitz_ex(const orc_factor* f, const orc_problem* p, double rel_tol, int max_rounds,
                              uint64_t* calls, double* out) {
  ORC_GUARD(*out = estimate_dual_lipschitz(f->cache, p->prob, calls, rel_tol, max_rounds))
}

int orc_solve(const orc_problem* p, const orc_solver_config* cfg, int kind, const orc_factor* shared,
              orc_report** out) {
  ORC_GUARD({
    auto r = std::make_unique<orc_report>();
    r->rep = solve(p->prob, cfg_from(cfg), static_cast<SolverKind>(kind),
                   shared ? &shared->cache : nullptr);
    *out = r.release();
  })
}

int orc_solve_direct(const orc_problem* p, const orc_factor* f, const orc_solver_config* cfg,
                     int kind, const double* y0, const double* weight, orc_report** out) {
  ORC_GUARD({
    const int D = p->prob.dual_dim;
    const SeparableNonsmooth g = make_nonsmooth(p->prob);
    const Vec y(y0, y0 + D);
    Vec wv;
    if (weight) wv = Vec(weight, weight + D);
    const Vec* wp = weight ? &wv : nullptr;
    const SolverConfig c = cfg_from(cfg);
    auto r = std::make_unique<orc_report>();
    switch (kind) {
      case 0: r->rep = solve_minfbe(p->prob, f->cache, g, c, y, wp); break;
      case 1: r->rep = solve_nama(p->prob, f->cache, g, c, y, wp); break;
      case 2: r->rep = solve_gpad(p->prob, f->cache, g, c, y, wp); break;
      default: ORC_THROW(kInvalidParams, "unknown solver kind");
    }
    *out = r.release();
  })
}

int orc_warm_start(const orc_problem* p, const orc_factor* f, const orc_solver_config* cfg,
                   double lambda, double* y_out, uint64_t* dg) {
  ORC_GUARD({
    OracleStats st;
    const Vec y = warm_start(p->prob, f->cache, make_nonsmooth(p->prob), cfg_from(cfg), lambda, &st);
    vec_to(y, y_out);
    if (dg) *dg = st.dual_grad_calls;
  })
}

void orc_report_free(orc_report* r) { delete r; }
int orc_report_summary_get(const orc_report* r, orc_report_summary* s) {
  const SolverReport& p = r->rep;
  s->status = static_cast<int32_t>(p.status);
  s->iterations = p.iterations;
  s->verified = p.verified ? 1 : 0;
  s->trace_len = static_cast<int32_t>(p.residual_trace.size());
  s->dual_grad_calls = p.stats.dual_grad_calls;
  s->hessian_vec_calls = p.stats.hessian_vec_calls;
  s->prox_calls = p.stats.prox_calls;
  s->conj_calls = p.stats.conj_calls;
  s->lipschitz_calls = p.lipschitz_calls;
  s->lipschitz_estimate = p.lipschitz_estimate;
  s->lambda_final = p.lambda_final;
  s->eps = p.eps;
  s->residual_inf = p.residual_inf;
  s->wall_ms = p.wall_ms;
  s->verify_residual_inf = p.verify_residual_inf;
  s->verify_subdiff_dist = p.verify_subdiff_dist;
  return 0;
}
int orc_report_arrays(const orc_report* r, double* x, double* u, double* y, double* z, double* rt,
                      double* ft) {
  const SolverReport& p = r->rep;
  primal_to(p.x, x, u);
  vec_to(p.y, y);
  vec_to(p.z, z);
  vec_to(p.residual_trace, rt);
  vec_to(p.fbe_trace, ft);
  return 0;
}
int orc_verify_report(const orc_problem* p, orc_report* r, const double* z_override) {
  ORC_GUARD({
    if (z_override) r->rep.z = Vec(z_override, z_override + p->prob.dual_dim);
    verify_report(p->prob, make_nonsmooth(p->prob), r->rep);
  })
}

int orc_time_sweeps(const orc_factor* f, const orc_problem* p, int nsweeps, int affine,
                    double* seconds) {
  ORC_GUARD({
    Vec y(static_cast<size_t>(p->prob.dual_dim));
    for (size_t i = 0; i < y.size(); ++i) y[i] = 0.001 * static_cast<double>(i % 17);
    volatile double sink = 0.0;
    const auto t0 = std::chrono::steady_clock::now();
    for (int k = 0; k < nsweeps; ++k) {
      const PrimalPoint pt = affine ? dual_grad(f->cache, p->prob, y) : hessian_vec(f->cache, p->prob, y);
      sink = sink + pt.x.d.back();
    }
    const auto t1 = std::chrono::steady_clock::now();
    *seconds = std::chrono::duration<double>(t1 - t0).count() / nsweeps;
  })
}

}  // extern "C"
