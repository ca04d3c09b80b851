// treebench: command-line front end over the B200 library, with the
// reference tool's subcommands and exit codes (tools/treebench.cpp of the
// reference): generate, validate, solve and benchmark scenario-tree problems.
//   treebench solve FILE [--solver minfbe|nama|pnama|gpad] [--eps E] [--lambda L]
//             [--memory M] [--max-iters K] [--warm-start] [--precondition] [--out REPORT.json]
//   treebench gen random --out F [--seed S] [--nx N] [--nu N] [--horizon N] [--branching B]
//   treebench gen spring-mass --out F [--masses M] [--horizon N] [--sample-seed S]
//   treebench validate FILE
//   treebench bench spring-mass --out DIR [--samples K] [--seed S] [--horizon N]
//             [--masses M] [--eps E] [--no-timing] [--no-precondition]
// Exit codes: 0 success, 1 the run or the document failed its check, 2 usage or I/O errors.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <fstream>
#include <map>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include "scenopt_b200.hpp"

namespace {

struct Usage : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// --name value / --flag options after the positional arguments
struct Args {
  std::vector<std::string> pos;
  std::map<std::string, std::string> opt;
  std::vector<std::string> flags;
  Args(int argc, char** argv, int from, const std::vector<std::string>& flag_names) {
    for (int i = from; i < argc; ++i) {
      const std::string a = argv[i];
      if (a.rfind("--", 0) == 0) {
        bool is_flag = false;
        for (const auto& f : flag_names) is_flag |= (a == f);
        if (is_flag) {
          flags.push_back(a);
        } else {
          if (i + 1 >= argc) throw Usage(a + " needs a value");
          opt[a] = argv[++i];
        }
      } else {
        pos.push_back(a);
      }
    }
  }
  bool flag(const char* f) const {
    for (const auto& x : flags)
      if (x == f) return true;
    return false;
  }
  std::string str(const char* k, const std::string& def) const {
    auto it = opt.find(k);
    return it == opt.end() ? def : it->second;
  }
  std::string required(const char* k) const {
    auto it = opt.find(k);
    if (it == opt.end()) throw Usage(std::string(k) + " is required");
    return it->second;
  }
  double num(const char* k, double def) const {
    auto it = opt.find(k);
    if (it == opt.end()) return def;
    char* end = nullptr;
    const double v = std::strtod(it->second.c_str(), &end);
    if (!end || *end) throw Usage(std::string(k) + ": not a number: " + it->second);
    return v;
  }
  long long integer(const char* k, long long def) const {
    auto it = opt.find(k);
    if (it == opt.end()) return def;
    char* end = nullptr;
    const long long v = std::strtoll(it->second.c_str(), &end, 10);
    if (!end || *end) throw Usage(std::string(k) + ": not an integer: " + it->second);
    return v;
  }
  void only(const std::vector<std::string>& known) const {
    for (const auto& kv : opt) {
      bool ok = false;
      for (const auto& k : known) ok |= (kv.first == k);
      if (!ok) throw Usage("unknown option " + kv.first);
    }
  }
};

void write_text(const std::string& path, const std::string& content) {
  std::ofstream out(path, std::ios::binary);
  if (!out) throw scenopt::Error("cannot open \"" + path + "\" for writing");
  out << content;
  if (!out) throw scenopt::Error("short write to \"" + path + "\"");
}

std::string read_text(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw scenopt::Error("cannot open \"" + path + "\"");
  std::ostringstream buf;
  buf << in.rdbuf();
  return buf.str();
}

int check(int rc) { return scenopt::detail::check(rc); }

int run_solve(const Args& a) {
  a.only({"--solver", "--eps", "--lambda", "--memory", "--max-iters", "--out"});
  if (a.pos.size() != 1) throw Usage("solve: exactly one problem file");
  const auto spec = scenopt::solver_spec_from_name(a.str("--solver", "nama"));
  scenopt::SolverConfig cfg;
  cfg.eps = a.num("--eps", 5e-4);
  cfg.lambda0 = a.num("--lambda", 0.0);
  cfg.memory = static_cast<int>(a.integer("--memory", 5));
  cfg.max_iters = static_cast<int>(a.integer("--max-iters", 20000));
  cfg.warm_start = a.flag("--warm-start");
  cfg.precondition = a.flag("--precondition");
  cfg.nama_parallel_linesearch = spec.parallel_linesearch;
  scenopt::validate_config(cfg);
  scenopt_problem* p = nullptr;
  check(scenopt_problem_load(a.pos[0].c_str(), &p));
  std::unique_ptr<scenopt_problem, scenopt::detail::ProblemDeleter> hp(p);
  const scenopt_solver_config c = scenopt::detail::c_config(cfg);
  scenopt_report* r = nullptr;
  check(scenopt_solve(p, &c, static_cast<int>(spec.kind), nullptr, 0, &r));
  std::unique_ptr<scenopt_report, scenopt::detail::ReportDeleter> hr(r);
  scenopt_report_summary s{};
  check(scenopt_report_summary_get(r, &s));
  const bool ok = s.status == 0 && s.verified;
  std::printf("%s: %s in %d iterations, residual %.3e (eps %.1e)\n", spec.name.c_str(),
              ok ? "converged" : "did not converge", s.iterations, s.residual_inf, s.eps);
  std::printf("  %llu dual_grad + %llu hessian_vec oracle sweeps, %llu prox, %.3f ms\n",
              static_cast<unsigned long long>(s.dual_grad_calls), static_cast<unsigned long long>(s.hessian_vec_calls),
              static_cast<unsigned long long>(s.prox_calls), s.wall_ms);
  const std::string out = a.str("--out", "");
  if (!out.empty()) {
    size_t n = 0;
    check(scenopt_report_json(r, p, spec.name.c_str(), ok, nullptr, 0, &n));
    std::string text(n + 1, '\0');
    check(scenopt_report_json(r, p, spec.name.c_str(), ok, text.data(), n + 1, &n));
    text.resize(n);
    write_text(out, text);
    std::printf("  report written to %s\n", out.c_str());
  }
  return ok ? 0 : 1;
}

int run_gen_random(const Args& a) {
  a.only({"--seed", "--nx", "--nu", "--horizon", "--branching", "--out"});
  const auto prob = scenopt::gen_random_instance(
      static_cast<std::uint64_t>(a.integer("--seed", 1)),
      scenopt::RandomDims{static_cast<int>(a.integer("--nx", 3)), static_cast<int>(a.integer("--nu", 2))},
      scenopt::RandomTreeShape{static_cast<int>(a.integer("--horizon", 3)), static_cast<int>(a.integer("--branching", 2))});
  const std::string out = a.required("--out");
  scenopt::save_problem(prob, out);
  std::printf("wrote %s: %d nodes, %d stages, dual dimension %d\n", out.c_str(), prob.num_nodes(),
              prob.tree.num_stages, prob.dual_dim);
  return 0;
}

int run_gen_spring(const Args& a) {
  a.only({"--masses", "--horizon", "--sample-seed", "--out"});
  const int masses = static_cast<int>(a.integer("--masses", 5));
  scenopt::SpringMassParams par;
  par.horizon = static_cast<int>(a.integer("--horizon", 11));
  const auto seed = static_cast<std::uint64_t>(a.integer("--sample-seed", 0));
  if (seed != 0) {
    std::mt19937_64 gen(seed);
    par.root_state = scenopt::sample_initial_state(masses, par, gen);
  }
  const auto prob = scenopt::gen_spring_mass(masses, par);
  const std::string out = a.required("--out");
  scenopt::save_problem(prob, out);
  std::printf("wrote %s: %d nodes, %d stages, dual dimension %d\n", out.c_str(), prob.num_nodes(),
              prob.tree.num_stages, prob.dual_dim);
  return 0;
}

int run_validate(const Args& a) {
  a.only({});
  if (a.pos.size() != 1) throw Usage("validate: exactly one problem file");
  const auto bad = scenopt::validate_problem_text(read_text(a.pos[0]));
  if (bad.empty()) {
    std::printf("ok: %s parses and validates\n", a.pos[0].c_str());
    return 0;
  }
  std::fprintf(stderr, "%s fails validation:\n", a.pos[0].c_str());
  for (const auto& v : bad) std::fprintf(stderr, "  %s\n", v.c_str());
  return 1;
}

int run_bench_spring(const Args& a) {
  a.only({"--samples", "--seed", "--horizon", "--masses", "--eps", "--out"});
  const int samples = static_cast<int>(a.integer("--samples", 50));
  const int masses = static_cast<int>(a.integer("--masses", 5));
  const int horizon = static_cast<int>(a.integer("--horizon", 8));
  const auto seed = static_cast<std::uint64_t>(a.integer("--seed", 1));
  const double eps = a.num("--eps", 5e-4);
  const bool no_timing = a.flag("--no-timing"), no_pre = a.flag("--no-precondition");
  const std::string out_dir = a.required("--out");
  scenopt::SpringMassParams par;
  par.horizon = horizon;
  std::mt19937_64 gen(seed);  // one stream across the batch: the seed pins every root state
  std::vector<scenopt::BatchEntry> batch;
  for (int k = 0; k < samples; ++k) {
    par.root_state = scenopt::sample_initial_state(masses, par, gen);
    batch.push_back({"sm" + std::to_string(k), scenopt::gen_spring_mass(masses, par)});
  }
  scenopt::ExperimentConfig cfg;
  cfg.solver.eps = eps;
  cfg.solver.precondition = !no_pre;  // probability products condition deep trees badly
  cfg.include_timing = !no_timing;
  auto report = scenopt::run_experiment(batch, scenopt::default_solver_set(), cfg);
  char meta[1024];
  std::snprintf(meta, sizeof meta,
                "{\"generator\": \"spring-mass\", \"masses\": %d, \"horizon\": %d, \"samples\": %d, "
                "\"seed\": %llu, \"eps\": %.17g, \"preconditioned\": %s, \"timing\": %s, \"tree\": "
                "\"full-branching Markov construction: every node keeps one child per reachable mode\"}",
                masses, horizon, samples, static_cast<unsigned long long>(seed), eps, no_pre ? "false" : "true",
                no_timing ? "false" : "true");
  report.metadata = meta;
  std::filesystem::create_directories(out_dir);
  const auto dir = std::filesystem::path(out_dir);
  write_text((dir / "results.csv").string(), report.csv());
  write_text((dir / "traces.csv").string(), report.traces_csv());
  write_text((dir / "summary.json").string(), report.summary_json() + "\n");
  for (const auto& s : report.summaries())
    std::printf("%s: %d/%d converged, median %.0f oracle calls, p95 %.0f, %.0f%% within 50\n", s.solver.c_str(),
                s.converged, s.count, s.median_calls, s.p95_calls, 100.0 * s.frac_within_50);
  std::printf("reports written to %s\n", out_dir.c_str());
  return 0;
}

const char* kUsage =
    "usage: treebench solve FILE [--solver minfbe|nama|pnama|gpad] [--eps E] [--lambda L] [--memory M]\n"
    "                  [--max-iters K] [--warm-start] [--precondition] [--out REPORT]\n"
    "       treebench gen random --out F [--seed S] [--nx N] [--nu N] [--horizon N] [--branching B]\n"
    "       treebench gen spring-mass --out F [--masses M] [--horizon N] [--sample-seed S]\n"
    "       treebench validate FILE\n"
    "       treebench bench spring-mass --out DIR [--samples K] [--seed S] [--horizon N] [--masses M]\n"
    "                  [--eps E] [--no-timing] [--no-precondition]\n";

}  // namespace

int main(int argc, char** argv) {
  try {
    const std::string cmd = argc > 1 ? argv[1] : "";
    const std::string sub = argc > 2 ? argv[2] : "";
    if (cmd == "solve") return run_solve(Args(argc, argv, 2, {"--warm-start", "--precondition"}));
    if (cmd == "gen" && sub == "random") return run_gen_random(Args(argc, argv, 3, {}));
    if (cmd == "gen" && sub == "spring-mass") return run_gen_spring(Args(argc, argv, 3, {}));
    if (cmd == "validate") return run_validate(Args(argc, argv, 2, {}));
    if (cmd == "bench" && sub == "spring-mass")
      return run_bench_spring(Args(argc, argv, 3, {"--no-timing", "--no-precondition"}));
    if (cmd == "-h" || cmd == "--help") {
      std::fputs(kUsage, stdout);
      return 0;
    }
    std::fputs(kUsage, stderr);
    return 2;
  } catch (const Usage& e) {
    std::fprintf(stderr, "treebench: %s\n%s", e.what(), kUsage);
    return 2;
  } catch (const scenopt::ParseError& e) {
    std::fprintf(stderr, "%s\n", e.what());
    return 1;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "treebench: %s\n", e.what());
    return 2;
  }
}
