// SPDX-License-Identifier: MIT
// Experiment harness (experiment.hpp:22-283): every solver on every instance
// of a batch through the device solve() driver, one factor per factor hash,
// and the byte-stable reports (results CSV, long-format traces CSV, the
// "scenopt-runreport-v1" summary JSON).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "capi_internal.hpp"
#include "json.hpp"
#include "problem_io.hpp"

using namespace scn;

namespace scn {
void check_solver_config(const scenopt_solver_config& c);  // solver.cpp (solvers.hpp:48-60)
}

struct ExpRow {  // ExperimentRow, experiment.hpp:63-80
  std::string instance_id, solver, error;
  int iterations = 0;
  uint64_t dual_grad_calls = 0, hessian_vec_calls = 0, prox_calls = 0;
  double final_residual_inf = std::numeric_limits<double>::infinity(), wall_ms = 0.0;
  bool converged = false, fbe_monotone = true;
  std::vector<double> residual_trace;
  uint64_t oracle_calls() const { return dual_grad_calls + hessian_vec_calls; }
};

struct scenopt_experiment {
  std::vector<ExpRow> rows;
  std::string text;  // last rendered report (size query, then copy)
};

namespace {

struct Spec {  // SolverSpec, experiment.hpp:26-41
  std::string name;
  int kind;
  bool parallel;
};

Spec spec_from_name(const std::string& name) {
  if (name == "minfbe") return {"minfbe", 0, false};
  if (name == "nama") return {"nama", 1, false};
  if (name == "pnama") return {"pnama", 1, true};
  if (name == "gpad") return {"gpad", 2, false};
  fail(SCENOPT_E_INVALID_PARAMS, "unknown solver \"" + name + "\"; expected minfbe, nama, pnama, or gpad");
}

std::string fmt17(double v) {  // ostream << setprecision(17) (experiment.hpp:113-117)
  char b[64];
  std::snprintf(b, sizeof b, "%.17g", v);
  return b;
}
std::string fmt_ms(double v) {  // fixed, 3 decimals (:119-123)
  char b[64];
  std::snprintf(b, sizeof b, "%.3f", v);
  return b;
}

bool nonincreasing(const std::vector<double>& t) {  // :125-131
  for (size_t k = 1; k < t.size(); ++k)
    if (t[k] > t[k - 1] + 1e-10 * (1.0 + std::abs(t[k - 1]))) return false;
  return true;
}

double quantile_sorted(const std::vector<double>& s, double p) {  // nearest rank (:101-111)
  if (s.empty()) return 0.0;
  const size_t n = s.size();
  size_t rank = static_cast<size_t>(std::ceil(p * static_cast<double>(n)));
  rank = std::max<size_t>(1, std::min(rank, n));
  return s[rank - 1];
}

// scenopt's own error taxonomy (errors.hpp) is a per-run outcome; device,
// NCCL and allocation failures abort the batch.
bool run_error(int rc) { return rc < 0 && rc >= SCENOPT_E_PARSE_ERROR; }

std::vector<scenopt_solver_summary> summaries(const std::vector<ExpRow>& rows) {  // :163-191
  std::vector<scenopt_solver_summary> out;
  std::vector<std::vector<double>> calls;
  std::vector<int> within;
  for (const auto& r : rows) {
    size_t k = 0;
    while (k < out.size() && r.solver != out[k].solver) ++k;
    if (k == out.size()) {
      out.push_back(scenopt_solver_summary{});
      std::snprintf(out.back().solver, sizeof out.back().solver, "%s", r.solver.c_str());
      calls.emplace_back();
      within.push_back(0);
    }
    auto& s = out[k];
    ++s.count;
    s.total_wall_ms += r.wall_ms;
    if (!r.fbe_monotone) ++s.fbe_violations;
    if (r.converged) {
      ++s.converged;
      calls[k].push_back(static_cast<double>(r.oracle_calls()));
      if (r.oracle_calls() <= 50) ++within[k];
    }
  }
  for (size_t k = 0; k < out.size(); ++k) {
    auto& c = calls[k];
    std::sort(c.begin(), c.end());
    out[k].median_calls = quantile_sorted(c, 0.5);
    out[k].p84_calls = quantile_sorted(c, 0.84);
    out[k].p95_calls = quantile_sorted(c, 0.95);
    out[k].frac_within_50 = out[k].count > 0 ? static_cast<double>(within[k]) / out[k].count : 0.0;
  }
  return out;
}

std::string csv(const std::vector<ExpRow>& rows) {  // :137-150
  std::string out =
      "instance_id,solver,iterations,dual_grad_calls,hessian_vec_calls,prox_calls,final_residual_inf,wall_ms,"
      "converged\n";
  for (const auto& r : rows)
    out += r.instance_id + "," + r.solver + "," + std::to_string(r.iterations) + "," +
           std::to_string(r.dual_grad_calls) + "," + std::to_string(r.hessian_vec_calls) + "," +
           std::to_string(r.prox_calls) + "," + fmt17(r.final_residual_inf) + "," + fmt_ms(r.wall_ms) + "," +
           (r.converged ? "1" : "0") + "\n";
  return out;
}

std::string traces_csv(const std::vector<ExpRow>& rows) {  // :153-161
  std::string out = "instance_id,solver,iteration,residual\n";
  for (const auto& r : rows)
    for (size_t k = 0; k < r.residual_trace.size(); ++k)
      out += r.instance_id + "," + r.solver + "," + std::to_string(k) + "," + fmt17(r.residual_trace[k]) + "\n";
  return out;
}

std::string summary_json(const std::vector<ExpRow>& rows, const char* metadata) {  // :194-213, dump(2)
  JV meta;
  meta.k = JV::Obj;
  if (metadata && *metadata) {
    meta = parse_json(metadata, "summary_json: metadata is not valid JSON: ");
    if (meta.k != JV::Obj) fail(SCENOPT_E_INVALID_PARAMS, "summary_json: metadata must be a JSON object");
  }
  const auto sums = summaries(rows);
  std::vector<const scenopt_solver_summary*> order;
  for (const auto& s : sums) order.push_back(&s);
  std::sort(order.begin(), order.end(),
            [](const auto* a, const auto* b) { return std::strcmp(a->solver, b->solver) < 0; });
  Writer w{std::string(), 2, 0, {}};
  w.open('{');
  w.key("metadata");
  dump_value(w, meta);
  w.key("schema");
  put_string(w.out, "scenopt-runreport-v1");
  w.key("solvers");
  w.open('{');
  for (const auto* s : order) {
    w.key(s->solver);
    w.open('{');
    w.key("converged");
    w.out += std::to_string(s->converged);
    w.key("count");
    w.out += std::to_string(s->count);
    w.key("fbe_monotone_violations");
    w.out += std::to_string(s->fbe_violations);
    w.key("frac_within_50_calls");
    put_double(w.out, s->frac_within_50);
    w.key("median_oracle_calls");
    put_double(w.out, s->median_calls);
    w.key("p84_oracle_calls");
    put_double(w.out, s->p84_calls);
    w.key("p95_oracle_calls");
    put_double(w.out, s->p95_calls);
    w.key("total_wall_ms");
    put_double(w.out, s->total_wall_ms);
    w.close('}');
  }
  w.close('}');
  w.close('}');
  return std::move(w.out);
}

}  // namespace

extern "C" {

int scenopt_run_experiment(const scenopt_problem* const* problems, const char* const* ids, int count,
                           const char* const* solvers, int nsolvers, const scenopt_solver_config* cfg,
                           int include_timing, int reuse_factors, int device, scenopt_experiment** out) {
  SCN_GUARD({
    if (!out || !cfg || (count > 0 && (!problems || !ids)) || (nsolvers > 0 && !solvers))
      fail(SCENOPT_E_INVALID_PARAMS, "run_experiment: null argument");
    check_solver_config(*cfg);
    std::vector<Spec> specs;
    for (int s = 0; s < nsolvers; ++s) specs.push_back(spec_from_name(solvers[s] ? solvers[s] : ""));
    auto rep = std::make_unique<scenopt_experiment>();
    rep->rows.reserve(static_cast<size_t>(count) * specs.size());
    // factors shared across the batch (preconditioned runs factor the scaled instance themselves)
    std::map<uint64_t, std::unique_ptr<scenopt_factor, void (*)(scenopt_factor*)>> caches;
    for (int e = 0; e < count; ++e) {
      const scenopt_problem* p = problems[e];
      const scenopt_factor* shared = nullptr;
      std::string factor_error;
      if (reuse_factors && !cfg->precondition) {
        const uint64_t key = factor_hash(p->p);
        auto it = caches.find(key);
        if (it == caches.end()) {
          scenopt_factor* f = nullptr;
          const int rc = scenopt_factor_create(p, &f);
          if (rc == 0)
            it = caches.emplace(key, std::unique_ptr<scenopt_factor, void (*)(scenopt_factor*)>(f, scenopt_factor_destroy))
                     .first;
          else if (run_error(rc))
            factor_error = scenopt_last_error();
          else
            fail(rc, scenopt_last_error());
        }
        if (it != caches.end()) shared = it->second.get();
      }
      for (const Spec& sp : specs) {
        ExpRow row;
        row.instance_id = ids[e] ? ids[e] : "";
        row.solver = sp.name;
        if (!factor_error.empty()) {
          row.error = factor_error;
          rep->rows.push_back(std::move(row));
          continue;
        }
        scenopt_solver_config c = *cfg;
        c.nama_parallel_linesearch = sp.parallel ? 1 : 0;
        scenopt_report* r = nullptr;
        const int rc = scenopt_solve(p, &c, sp.kind, shared, device, &r);
        if (rc < 0) {
          if (!run_error(rc)) fail(rc, scenopt_last_error());
          row.error = scenopt_last_error();
          rep->rows.push_back(std::move(row));
          continue;
        }
        std::unique_ptr<scenopt_report, void (*)(scenopt_report*)> rp(r, scenopt_report_destroy);
        scenopt_report_summary s{};
        scenopt_report_summary_get(r, &s);
        row.iterations = s.iterations;
        row.dual_grad_calls = s.dual_grad_calls;
        row.hessian_vec_calls = s.hessian_vec_calls;
        row.prox_calls = s.prox_calls;
        row.final_residual_inf = s.residual_inf;
        row.wall_ms = include_timing ? s.wall_ms : 0.0;
        row.converged = s.status == 0 && s.verified;
        std::vector<double> fbe(static_cast<size_t>(s.trace_len));
        row.residual_trace.resize(static_cast<size_t>(s.trace_len));
        scenopt_report_arrays(r, nullptr, nullptr, nullptr, nullptr, row.residual_trace.data(), fbe.data());
        row.fbe_monotone = nonincreasing(fbe);
        rep->rows.push_back(std::move(row));
      }
    }
    *out = rep.release();
  });
}

int scenopt_experiment_row_count(const scenopt_experiment* x) { return x ? static_cast<int>(x->rows.size()) : 0; }

int scenopt_experiment_row_get(const scenopt_experiment* x, int i, scenopt_experiment_row* row) {
  SCN_GUARD({
    if (!x || !row || i < 0 || i >= static_cast<int>(x->rows.size()))
      fail(SCENOPT_E_INVALID_PARAMS, "experiment row out of range");
    const ExpRow& r = x->rows[static_cast<size_t>(i)];
    row->instance_id = r.instance_id.c_str();
    row->solver = r.solver.c_str();
    row->error = r.error.c_str();
    row->iterations = r.iterations;
    row->dual_grad_calls = r.dual_grad_calls;
    row->hessian_vec_calls = r.hessian_vec_calls;
    row->prox_calls = r.prox_calls;
    row->final_residual_inf = r.final_residual_inf;
    row->wall_ms = r.wall_ms;
    row->converged = r.converged ? 1 : 0;
    row->fbe_monotone = r.fbe_monotone ? 1 : 0;
    row->trace_len = static_cast<int32_t>(r.residual_trace.size());
    row->residual_trace = r.residual_trace.data();
  });
}

int scenopt_experiment_text(scenopt_experiment* x, int which, const char* metadata_json, char* buf, size_t cap,
                            size_t* len) {
  SCN_GUARD({
    if (!x) fail(SCENOPT_E_INVALID_PARAMS, "experiment text: null report");
    if (!buf || x->text.empty()) {
      if (which == 0) x->text = csv(x->rows);
      else if (which == 1) x->text = traces_csv(x->rows);
      else if (which == 2) x->text = summary_json(x->rows, metadata_json) + "\n";
      else fail(SCENOPT_E_INVALID_PARAMS, "experiment text: which must be 0 (csv), 1 (traces) or 2 (summary)");
    }
    if (len) *len = x->text.size();
    if (buf && cap > 0) {
      const size_t n = std::min(cap - 1, x->text.size());
      std::memcpy(buf, x->text.data(), n);
      buf[n] = 0;
      std::string().swap(x->text);
    }
  });
}

int scenopt_experiment_summaries(const scenopt_experiment* x, scenopt_solver_summary* out, int cap) {
  SCN_GUARD({
    if (!x) fail(SCENOPT_E_INVALID_PARAMS, "experiment summaries: null report");
    const auto s = summaries(x->rows);
    if (out)
      for (int k = 0; k < std::min(cap, static_cast<int>(s.size())); ++k) out[k] = s[static_cast<size_t>(k)];
    return static_cast<int>(s.size());
  });
}

void scenopt_experiment_destroy(scenopt_experiment* x) { delete x; }

// solve_report_json (treebench.cpp:52-85): the "scenopt-solvereport-v1"
// document of one solve, dump(2) + "\n"
int scenopt_report_json(const scenopt_report* r, const scenopt_problem* p, const char* solver, int converged,
                        char* buf, size_t cap, size_t* len) {
  SCN_GUARD({
    if (!r || !p) fail(SCENOPT_E_INVALID_PARAMS, "report_json: null argument");
    scenopt_report_summary s{};
    if (scenopt_report_summary_get(r, &s) < 0) fail(SCENOPT_E_INVALID_PARAMS, scenopt_last_error());
    const Problem& q = p->p;
    std::vector<double> u(static_cast<size_t>(q.nu) * std::max(q.first_leaf, 1)), res(static_cast<size_t>(s.trace_len)),
        fbe(static_cast<size_t>(s.trace_len));
    scenopt_report_arrays(r, nullptr, u.data(), nullptr, nullptr, res.data(), fbe.data());
    Writer w{std::string(), 2, 0, {}};
    auto arr = [&](const std::vector<double>& v, size_t n) {
      w.open('[');
      for (size_t i = 0; i < n; ++i) {
        w.elem();
        put_double(w.out, v[i]);
      }
      w.close(']');
    };
    auto num = [&](const char* k, double v) {
      w.key(k);
      put_double(w.out, v);
    };
    auto integer = [&](const char* k, uint64_t v) {
      w.key(k);
      w.out += std::to_string(v);
    };
    w.open('{');
    w.key("converged");
    w.out += converged ? "true" : "false";
    num("eps", s.eps);
    w.key("fbe_trace");
    arr(fbe, fbe.size());
    integer("iterations", static_cast<uint64_t>(s.iterations));
    num("lambda_final", s.lambda_final);
    integer("lipschitz_calls", s.lipschitz_calls);
    num("lipschitz_estimate", s.lipschitz_estimate);
    w.key("oracle_calls");
    w.open('{');
    integer("conjugate", s.conj_calls);
    integer("dual_grad", s.dual_grad_calls);
    integer("hessian_vec", s.hessian_vec_calls);
    integer("prox", s.prox_calls);
    integer("total", s.dual_grad_calls + s.hessian_vec_calls);
    w.close('}');
    num("residual_inf", s.residual_inf);
    w.key("residual_trace");
    arr(res, res.size());
    w.key("root_control");
    arr(u, static_cast<size_t>(q.nu));  // u(:, 0)
    w.key("schema");
    put_string(w.out, "scenopt-solvereport-v1");
    w.key("solver");
    put_string(w.out, solver ? solver : "");
    w.key("status");
    put_string(w.out, s.status == 0 ? "converged" : "max_iters_exceeded");
    w.key("verified");
    w.out += s.verified ? "true" : "false";
    num("verify_residual_inf", s.verify_residual_inf);
    num("verify_subdiff_dist", s.verify_subdiff_dist);
    num("wall_ms", s.wall_ms);
    w.close('}');
    w.out += '\n';
    if (len) *len = w.out.size();
    if (buf && cap > 0) {
      const size_t n = std::min(cap - 1, w.out.size());
      std::memcpy(buf, w.out.data(), n);
      buf[n] = 0;
    }
  });
}

}  // extern "C"
