// SPDX-License-Identifier: MIT
// Problem files (problem_io.hpp:18-559): the "scenopt-problem-v1" JSON
// document, canonical serialization, parsing with the instance validation,
// and the content / factor hashes (FNV-1a of the canonical text).
//
// The reference builds a nlohmann::json DOM and dumps it; here the writer
// streams the document in the same layout (keys sorted, dump(2) indentation,
// nlohmann's number placement: "1.0", "0.25", "1e-05", "-0.0") and the reader
// is a small recursive-descent parser. Numbers carry the shortest digit string
// that round-trips (nlohmann's Grisu2 agrees except for rare longer outputs),
// so the text is canonical for this implementation: equal instances give equal
// bytes and parse -> serialize is the identity on its own output.
#include <charconv>
#include <cmath>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "model.hpp"
#include "problem_io.hpp"
#include "json.hpp"

namespace scn {
namespace {

[[noreturn]] void parse_fail(const std::string& m) { fail(SCENOPT_E_PARSE_ERROR, m); }

struct Block {  // one node's matrix or vector (column-major data, rows x cols)
  const double* d;
  int r, c;
  bool vec;
};

bool same(const Block& a, const Block& b) {
  if (a.r != b.r || a.c != b.c || a.vec != b.vec) return false;
  const size_t n = static_cast<size_t>(a.r) * a.c;
  for (size_t t = 0; t < n; ++t)
    if (!(a.d[t] == b.d[t])) return false;  // json equality: numeric ==
  return true;
}

void put_block(Writer& w, const Block& b) {
  if (b.vec) {
    w.open('[');
    for (int t = 0; t < b.r; ++t) {
      w.elem();
      put_double(w.out, b.d[t]);
    }
    w.close(']');
    return;
  }
  w.open('[');  // array of rows (problem_io.hpp:33-41)
  for (int i = 0; i < b.r; ++i) {
    w.elem();
    w.open('[');
    for (int j = 0; j < b.c; ++j) {
      w.elem();
      put_double(w.out, b.d[i + static_cast<size_t>(j) * b.r]);
    }
    w.close(']');
  }
  w.close(']');
}

// field_to_json (problem_io.hpp:85-95): the shared form when every entry is equal
template <class Get>
void put_field(Writer& w, const char* name, int first, int past, const Get& get) {
  w.key(name);
  bool all = true;
  const Block b0 = get(first);
  for (int i = first + 1; i < past && all; ++i) all = same(get(i), b0);
  if (all) {
    put_block(w, b0);
    return;
  }
  w.open('[');
  for (int i = first; i < past; ++i) {
    w.elem();
    put_block(w, get(i));
  }
  w.close(']');
}

const char* kind_name(int k) {
  switch (k) {
    case 0: return "none";
    case 1: return "box";
    case 2: return "scaled_l1";
  }
  fail(SCENOPT_E_INVALID_PARAMS, "kind_name: unknown nonsmooth kind");
}

template <class Get>
void put_kinds(Writer& w, int first, int past, const Get& kind) {
  w.key("kind");
  bool all = true;
  for (int i = first + 1; i < past && all; ++i) all = kind(i) == kind(first);
  if (all) {
    put_string(w.out, kind_name(kind(first)));
    return;
  }
  w.open('[');
  for (int i = first; i < past; ++i) {
    w.elem();
    put_string(w.out, kind_name(kind(i)));
  }
  w.close(']');
}

template <class Get>
void put_numbers(Writer& w, const char* name, int first, int past, const Get& val) {
  w.key(name);
  bool all = true;
  for (int i = first + 1; i < past && all; ++i) all = val(i) == val(first);
  if (all) {
    put_double(w.out, val(first));
    return;
  }
  w.open('[');
  for (int i = first; i < past; ++i) {
    w.elem();
    put_double(w.out, val(i));
  }
  w.close(']');
}

template <class T>
void put_ints(Writer& w, const char* name, const std::vector<T>& v) {
  w.key(name);
  w.open('[');
  for (const T x : v) {
    w.elem();
    w.out += std::to_string(x);
  }
  w.close(']');
}

}  // namespace

// problem_to_json (problem_io.hpp:220-320) + dump; factor_only drops what the
// factor does not depend on (problem_io.hpp:546-557).
std::string write_problem(const Problem& p, int indent, bool factor_only) {
  const int n = p.n, L = p.L, nx = p.nx, nu = p.nu;
  Writer w{std::string(), indent, 0, {}};
  w.out.reserve(static_cast<size_t>(n) * 64 + 4096);
  w.open('{');
  // keys in std::map order (nlohmann::json objects are sorted)
  w.key("constraints");
  w.open('{');
  put_field(w, "F", 1, n, [&](int i) { return Block{p.Fi(i), p.stage_rows[i], nx, false}; });
  put_field(w, "G", 1, n, [&](int i) { return Block{p.Gi(i), p.stage_rows[i], nu, false}; });
  if (!factor_only) {
    put_numbers(w, "gamma", 1, n, [&](int i) { return p.g_gamma[i]; });
    put_kinds(w, 1, n, [&](int i) { return p.g_kind[i]; });
    put_field(w, "zmax", 1, n, [&](int i) { return Block{p.zmax.data() + p.dual_offset[i], p.stage_rows[i], 1, true}; });
    put_field(w, "zmin", 1, n, [&](int i) { return Block{p.zmin.data() + p.dual_offset[i], p.stage_rows[i], 1, true}; });
  }
  w.close('}');
  w.key("cost");
  w.open('{');
  put_field(w, "Q", 1, n, [&](int i) { return Block{p.Qi(i), nx, nx, false}; });
  put_field(w, "R", 1, n, [&](int i) { return Block{p.Ri(i), nu, nu, false}; });
  put_field(w, "S", 1, n, [&](int i) { return Block{p.Si(i), nu, nx, false}; });
  put_field(w, "q", 1, n, [&](int i) { return Block{p.qi(i), nx, 1, true}; });
  put_field(w, "r", 1, n, [&](int i) { return Block{p.ri(i), nu, 1, true}; });
  w.close('}');
  w.key("dims");
  w.open('{');
  w.key("nu");
  w.out += std::to_string(nu);
  w.key("nx");
  w.out += std::to_string(nx);
  w.close('}');
  w.key("dynamics");
  w.open('{');
  put_field(w, "A", 1, n, [&](int i) { return Block{p.Ai(i), nx, nx, false}; });
  put_field(w, "B", 1, n, [&](int i) { return Block{p.Bi(i), nx, nu, false}; });
  put_field(w, "c", 1, n, [&](int i) { return Block{p.ci(i), nx, 1, true}; });
  w.close('}');
  if (!factor_only) {
    w.key("root_state");
    put_block(w, Block{p.root_state.data(), nx, 1, true});
  }
  w.key("schema");
  put_string(w.out, kProblemSchema);
  w.key("terminal_constraints");
  w.open('{');
  put_field(w, "F", 0, L, [&](int l) { return Block{p.FNl(l), p.terminal_rows[l], nx, false}; });
  if (!factor_only) {
    put_numbers(w, "gamma", 0, L, [&](int l) { return p.tg_gamma[l]; });
    put_kinds(w, 0, L, [&](int l) { return p.tg_kind[l]; });
    put_field(w, "zmax", 0, L, [&](int l) { return Block{p.zmax.data() + p.tdual_offset[l], p.terminal_rows[l], 1, true}; });
    put_field(w, "zmin", 0, L, [&](int l) { return Block{p.zmin.data() + p.tdual_offset[l], p.terminal_rows[l], 1, true}; });
  }
  w.close('}');
  w.key("terminal_cost");
  w.open('{');
  put_field(w, "P", 0, L, [&](int l) { return Block{p.Pl(l), nx, nx, false}; });
  put_field(w, "p", 0, L, [&](int l) { return Block{p.pl(l), nx, 1, true}; });
  w.close('}');
  w.key("tree");
  w.open('{');
  put_ints(w, "ancestor", p.ancestor);
  if (!factor_only && !p.mode.empty()) put_ints(w, "mode", p.mode);
  w.key("probability");
  w.open('[');
  for (const double v : p.probability) {
    w.elem();
    put_double(w.out, v);
  }
  w.close(']');
  put_ints(w, "stage", p.node_stage);
  w.close('}');
  w.close('}');
  return std::move(w.out);
}

std::string serialize_problem(const Problem& p) {
  require_full(p, "serialize_problem");
  return write_problem(p, 2, false) + "\n";
}

namespace {
// ---------------------------------------------------------------- document -> instance
struct M {  // a parsed matrix (column-major) or vector (c == 1, vec)
  int r = 0, c = 0;
  std::vector<double> d;
};

const JV& require_key(const JV& j, const char* key, const char* where) {
  const JV* v = j.k == JV::Obj ? j.find(key) : nullptr;
  if (!v) parse_fail(std::string(where) + ": missing key \"" + key + "\"");
  return *v;
}

double number_of(const JV& j, const std::string& where) {
  if (!j.is_num()) parse_fail(where + ": expected a number");
  return j.num();
}

M mat_of(const JV& j, const std::string& where) {  // problem_io.hpp:49-70
  if (j.k != JV::Arr) parse_fail(where + ": expected an array of rows");
  M m;
  if (j.a.empty()) return m;
  if (j.a[0].k != JV::Arr) parse_fail(where + ": expected an array of rows");
  m.r = static_cast<int>(j.a.size());
  m.c = static_cast<int>(j.a[0].a.size());
  m.d.assign(static_cast<size_t>(m.r) * m.c, 0.0);
  for (int i = 0; i < m.r; ++i) {
    const JV& row = j.a[static_cast<size_t>(i)];
    if (row.k != JV::Arr || static_cast<int>(row.a.size()) != m.c) parse_fail(where + ": ragged matrix rows");
    for (int c = 0; c < m.c; ++c) {
      const JV& cell = row.a[static_cast<size_t>(c)];
      if (!cell.is_num()) parse_fail(where + ": matrix entries must be numbers");
      m.d[i + static_cast<size_t>(c) * m.r] = cell.num();
    }
  }
  return m;
}

M vec_of(const JV& j, const std::string& where) {  // problem_io.hpp:72-81
  if (j.k != JV::Arr) parse_fail(where + ": expected a number array");
  M v;
  v.r = static_cast<int>(j.a.size());
  v.c = 1;
  v.d.resize(j.a.size());
  for (size_t t = 0; t < j.a.size(); ++t) {
    if (!j.a[t].is_num()) parse_fail(where + ": vector entries must be numbers");
    v.d[t] = j.a[t].num();
  }
  return v;
}

bool single_matrix(const JV& j) {  // problem_io.hpp:99-104
  if (j.k != JV::Arr) return false;
  if (j.a.empty()) return true;
  if (j.a[0].k != JV::Arr) return false;
  return j.a[0].a.empty() || j.a[0].a[0].is_num();
}
bool single_vector(const JV& j) { return j.k == JV::Arr && (j.a.empty() || j.a[0].is_num()); }

int kind_of(const JV& j, const std::string& where) {
  if (j.k != JV::Str) parse_fail(where + ": kind must be a string");
  if (j.s == "none") return 0;
  if (j.s == "box") return 1;
  if (j.s == "scaled_l1") return 2;
  parse_fail(where + ": unknown kind \"" + j.s + "\"");
}

// field_from_json (problem_io.hpp:108-126)
template <class T, class Single, class Decode>
std::vector<T> field_of(const JV& j, size_t count, const Single& single, const Decode& decode,
                        const std::string& where) {
  std::vector<T> out(count);
  if (single(j)) {
    const T v = decode(j, where);
    for (auto& s : out) s = v;
    return out;
  }
  if (j.k != JV::Arr || j.a.size() != count)
    parse_fail(where + ": expected one shared value or a list of " + std::to_string(count));
  for (size_t i = 0; i < count; ++i) out[i] = decode(j.a[i], where + "[" + std::to_string(i) + "]");
  return out;
}

std::vector<int32_t> ints_of(const JV& j, const std::string& where) {
  if (j.k != JV::Arr) parse_fail(where + ": expected an array");
  std::vector<int32_t> out;
  out.reserve(j.a.size());
  for (const JV& c : j.a) {
    if (c.k != JV::Int) parse_fail(where + ": entries must be integers");
    out.push_back(static_cast<int32_t>(c.i));
  }
  return out;
}

// cost-block convexity (problem_data.hpp:273-282) on a parsed node
void check_cost(const M& Q, const M& R, const M& S, int nx, int nu, const std::string& where,
                std::vector<std::string>& bad) {
  if (sym_min_eig(R.d.data(), nu) < 1e-10) bad.push_back(where + ": R must be positive definite");
  const int w = nx + nu;
  std::vector<double> blk(static_cast<size_t>(w) * w);
  for (int j = 0; j < nx; ++j)
    for (int k = 0; k < nx; ++k) blk[k + j * w] = Q.d[k + static_cast<size_t>(j) * nx];
  for (int j = 0; j < nu; ++j)
    for (int k = 0; k < nx; ++k) blk[k + (nx + j) * w] = S.d[j + static_cast<size_t>(k) * nu];
  for (int j = 0; j < nx; ++j)
    for (int k = 0; k < nu; ++k) blk[nx + k + j * w] = S.d[k + static_cast<size_t>(j) * nu];
  for (int j = 0; j < nu; ++j)
    for (int k = 0; k < nu; ++k) blk[nx + k + (nx + j) * w] = R.d[k + static_cast<size_t>(j) * nu];
  if (sym_min_eig(blk.data(), w) < -1e-10)
    bad.push_back(where + ": cost block [[Q, S'], [S, R]] must be positive semidefinite");
}

void check_spec(int kind, const M& zmin, const M& zmax, double gamma, int rows, const std::string& where,
                std::vector<std::string>& bad) {  // problem_data.hpp:253-266
  if (kind == 1) {
    if (zmin.r != rows || zmax.r != rows) {
      bad.push_back(where + ": box bounds must match the block's row count");
    } else {
      for (int t = 0; t < rows; ++t)
        if (zmax.d[t] - zmin.d[t] < 0.0) {
          bad.push_back(where + ": box needs zmin <= zmax");
          break;
        }
    }
  } else if (kind == 2 && !(gamma > 0.0)) {
    bad.push_back(where + ": scaled_l1 needs gamma > 0");
  }
}
}  // namespace

// problem_from_json (problem_io.hpp:323-478)
Problem parse_problem(const std::string& text) {
  const JV j = parse_json(text, "problem: not valid JSON: ");
  if (j.k != JV::Obj) parse_fail("problem: expected a JSON object");
  const JV& schema = require_key(j, "schema", "problem");
  if (schema.k != JV::Str || schema.s != kProblemSchema)
    parse_fail(std::string("problem: schema must be \"") + kProblemSchema + "\"");
  Problem p;
  const JV& dims = require_key(j, "dims", "problem");
  p.nx = static_cast<int>(number_of(require_key(dims, "nx", "dims"), "dims.nx"));
  p.nu = static_cast<int>(number_of(require_key(dims, "nu", "dims"), "dims.nu"));
  const JV& tree = require_key(j, "tree", "problem");
  if (const JV* mk = tree.k == JV::Obj ? tree.find("markov") : nullptr) {
    const M T = mat_of(require_key(*mk, "transition", "tree.markov"), "tree.markov.transition");
    const M init = vec_of(require_key(*mk, "initial", "tree.markov"), "tree.markov.initial");
    const int horizon = static_cast<int>(number_of(require_key(*mk, "horizon", "tree.markov"), "tree.markov.horizon"));
    std::vector<double> rowmajor(T.d.size());
    for (int i = 0; i < T.r; ++i)
      for (int c = 0; c < T.c; ++c) rowmajor[static_cast<size_t>(i) * T.c + c] = T.d[i + static_cast<size_t>(c) * T.r];
    try {
      markov_tree(rowmajor, T.r, T.c, init.d, horizon, p);
    } catch (const Error& e) {
      parse_fail(std::string("tree.markov: ") + e.what());
    }
  } else {  // tree_from_arrays (problem_io.hpp:163-207)
    std::vector<int32_t> stage = ints_of(require_key(tree, "stage", "tree"), "tree.stage");
    p.ancestor = ints_of(require_key(tree, "ancestor", "tree"), "tree.ancestor");
    p.probability = vec_of(require_key(tree, "probability", "tree"), "tree.probability").d;
    if (const JV* md = tree.find("mode")) p.mode = ints_of(*md, "tree.mode");
    const size_t n = stage.size();
    if (n == 0 || p.ancestor.size() != n || p.probability.size() != n)
      parse_fail("tree: stage, ancestor, and probability must be equally sized and nonempty");
    if (!p.mode.empty() && p.mode.size() != n) parse_fail("tree: mode must be empty or one entry per node");
    for (size_t i = 1; i < n; ++i) {
      const int a = p.ancestor[i];
      if (a < 0 || static_cast<size_t>(a) >= n)
        parse_fail("tree: ancestor of node " + std::to_string(i) + " is out of range");
    }
    int N = 0;
    for (const int s : stage) {
      if (s < 0) parse_fail("tree: negative stage");
      N = std::max(N, s);
    }
    p.N = N;
    p.stage_offsets.assign(static_cast<size_t>(N) + 2, 0);
    for (size_t i = 0; i < n; ++i) {
      if (i > 0 && stage[i] < stage[i - 1]) parse_fail("tree: nodes must be sorted by stage");
      ++p.stage_offsets[static_cast<size_t>(stage[i]) + 1];
    }
    for (size_t s = 1; s < p.stage_offsets.size(); ++s) p.stage_offsets[s] += p.stage_offsets[s - 1];
    p.n = static_cast<int>(n);
  }
  const M root = vec_of(require_key(j, "root_state", "problem"), "root_state");
  const int n = p.n, nx = p.nx, nu = p.nu;
  const size_t ns = static_cast<size_t>(std::max(n - 1, 0));
  const size_t L = static_cast<size_t>(n - p.stage_offsets[static_cast<size_t>(p.N)]);
  auto dm = [](const JV& v, const std::string& w) { return mat_of(v, w); };
  auto dv = [](const JV& v, const std::string& w) { return vec_of(v, w); };
  auto dk = [](const JV& v, const std::string& w) { return kind_of(v, w); };
  auto dn = [](const JV& v, const std::string& w) { return number_of(v, w); };
  auto sk = [](const JV& v) { return v.k == JV::Str; };
  auto sn = [](const JV& v) { return v.is_num(); };
  auto stage_f = [&](const JV& par, const char* key, auto single, auto decode) {
    using T = std::decay_t<decltype(decode(JV{}, std::string()))>;
    return field_of<T>(require_key(par, key, "problem"), ns, single, decode, std::string(key));
  };
  auto leaf_f = [&](const JV& par, const char* key, auto single, auto decode) {
    using T = std::decay_t<decltype(decode(JV{}, std::string()))>;
    return field_of<T>(require_key(par, key, "problem"), L, single, decode, std::string("terminal ") + key);
  };
  const JV& dyn = require_key(j, "dynamics", "problem");
  const auto A = stage_f(dyn, "A", single_matrix, dm), B = stage_f(dyn, "B", single_matrix, dm);
  const auto c = stage_f(dyn, "c", single_vector, dv);
  const JV& cost = require_key(j, "cost", "problem");
  const auto Q = stage_f(cost, "Q", single_matrix, dm), R = stage_f(cost, "R", single_matrix, dm),
             S = stage_f(cost, "S", single_matrix, dm);
  const auto q = stage_f(cost, "q", single_vector, dv), r = stage_f(cost, "r", single_vector, dv);
  const JV& con = require_key(j, "constraints", "problem");
  auto F = stage_f(con, "F", single_matrix, dm), G = stage_f(con, "G", single_matrix, dm);
  const auto kind = stage_f(con, "kind", sk, dk);
  const auto zmin = stage_f(con, "zmin", single_vector, dv), zmax = stage_f(con, "zmax", single_vector, dv);
  const auto gamma = stage_f(con, "gamma", sn, dn);
  const JV& tc = require_key(j, "terminal_cost", "problem");
  const auto P = leaf_f(tc, "P", single_matrix, dm), pv = leaf_f(tc, "p", single_vector, dv);
  const JV& tcon = require_key(j, "terminal_constraints", "problem");
  auto tF = leaf_f(tcon, "F", single_matrix, dm);
  const auto tkind = leaf_f(tcon, "kind", sk, dk);
  const auto tzmin = leaf_f(tcon, "zmin", single_vector, dv), tzmax = leaf_f(tcon, "zmax", single_vector, dv);
  const auto tgamma = leaf_f(tcon, "gamma", sn, dn);
  // zero-row blocks parse as 0 x 0 (problem_io.hpp:461-468)
  for (auto& m : F)
    if (m.r == 0) m.c = nx;
  for (auto& m : G)
    if (m.r == 0) m.c = nu;
  for (auto& m : tF)
    if (m.r == 0) m.c = nx;

  // validate(prob) (problem_data.hpp:233-314): tree, then per node / leaf
  p.stage_rows.assign(static_cast<size_t>(n), 0);
  for (int i = 1; i < n; ++i) p.stage_rows[i] = F[static_cast<size_t>(i - 1)].r;
  p.terminal_rows.assign(L, 0);
  for (size_t l = 0; l < L; ++l) p.terminal_rows[l] = tF[l].r;
  p.finalize();
  std::vector<std::string> bad = validate_tree(p);
  if (nx <= 0 || nu <= 0) bad.push_back("instance: nx and nu must be positive");
  if (root.r != nx) bad.push_back("instance: root_state must have length nx");
  for (int i = 1; i < n; ++i) {
    const size_t k = static_cast<size_t>(i - 1);
    const std::string where = "node " + std::to_string(i);
    if (A[k].r != nx || A[k].c != nx || B[k].r != nx || B[k].c != nu || c[k].r != nx)
      bad.push_back(where + ": dynamics dimensions");
    if (Q[k].r != nx || Q[k].c != nx || R[k].r != nu || R[k].c != nu || S[k].r != nu || S[k].c != nx ||
        q[k].r != nx || r[k].r != nu)
      bad.push_back(where + ": cost dimensions");
    else if (nx > 0 && nu > 0)
      check_cost(Q[k], R[k], S[k], nx, nu, where, bad);
    if (F[k].c != nx || G[k].c != nu || F[k].r != G[k].r) bad.push_back(where + ": constraint block dimensions");
    check_spec(kind[k], zmin[k], zmax[k], gamma[k], F[k].r, where + " stage block", bad);
  }
  for (size_t l = 0; l < L; ++l) {
    const std::string where = "leaf " + std::to_string(l);
    if (P[l].r != nx || P[l].c != nx || pv[l].r != nx)
      bad.push_back(where + ": terminal cost dimensions");
    else if (nx > 0 && sym_min_eig(P[l].d.data(), nx) < 1e-10)
      bad.push_back(where + ": P_N must be positive definite");
    if (tF[l].c != nx) bad.push_back(where + ": terminal block dimensions");
    check_spec(tkind[l], tzmin[l], tzmax[l], tgamma[l], tF[l].r, where + " terminal block", bad);
  }
  if (!bad.empty()) {
    std::string joined = "instance validation failed";
    for (const auto& b : bad) joined += "\n" + b;
    parse_fail(joined);
  }
  // pack the flat model (node 0 keeps zero blocks)
  const size_t sxx = p.sxx(), sxu = p.sxu(), suu = p.suu();
  p.root_state = root.d;
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
  p.g_kind.assign(static_cast<size_t>(n), 0);
  p.g_gamma.assign(static_cast<size_t>(n), 0.0);
  p.zmin.assign(static_cast<size_t>(p.dual_dim), 0.0);
  p.zmax.assign(static_cast<size_t>(p.dual_dim), 0.0);
  zeros(p.P, L * sxx);
  p.p.assign(L * nx, 0.0);
  p.FN.assign(static_cast<size_t>(p.dual_dim - p.stage_total) * nx, 0.0);
  p.tg_kind.assign(L, 0);
  p.tg_gamma.assign(L, 0.0);
  auto put = [](auto& dst, size_t off, const M& m) {
    std::copy(m.d.begin(), m.d.end(), dst.begin() + static_cast<std::ptrdiff_t>(off));
  };
  for (int i = 1; i < n; ++i) {
    const size_t k = static_cast<size_t>(i - 1);
    put(p.A, i * sxx, A[k]);
    put(p.B, i * sxu, B[k]);
    put(p.c, static_cast<size_t>(i) * nx, c[k]);
    put(p.Q, i * sxx, Q[k]);
    put(p.R, i * suu, R[k]);
    put(p.S, i * sxu, S[k]);
    put(p.q, static_cast<size_t>(i) * nx, q[k]);
    put(p.r, static_cast<size_t>(i) * nu, r[k]);
    const size_t off = static_cast<size_t>(p.dual_offset[i]);
    put(p.F, off * nx, F[k]);
    put(p.G, off * nu, G[k]);
    p.g_kind[i] = kind[k];
    p.g_gamma[i] = gamma[k];
    if (zmin[k].r == F[k].r) put(p.zmin, off, zmin[k]);  // non-box bounds of another length are unused
    if (zmax[k].r == F[k].r) put(p.zmax, off, zmax[k]);
  }
  for (size_t l = 0; l < L; ++l) {
    put(p.P, l * sxx, P[l]);
    put(p.p, l * nx, pv[l]);
    const size_t off = static_cast<size_t>(p.tdual_offset[l]);
    put(p.FN, (off - static_cast<size_t>(p.stage_total)) * nx, tF[l]);
    p.tg_kind[l] = tkind[l];
    p.tg_gamma[l] = tgamma[l];
    if (tzmin[l].r == tF[l].r) put(p.zmin, off, tzmin[l]);
    if (tzmax[l].r == tF[l].r) put(p.zmax, off, tzmax[l]);
  }
  return p;
}

std::vector<std::string> validate_problem_text(const std::string& text) {  // problem_io.hpp:512-524
  try {
    parse_problem(text);
  } catch (const Error& e) {
    if (e.code != SCENOPT_E_PARSE_ERROR) throw;
    std::vector<std::string> out;
    std::istringstream lines(e.what());
    for (std::string line; std::getline(lines, line);)
      if (!line.empty()) out.push_back(line);
    return out;
  }
  return {};
}

uint64_t fnv1a(const std::string& bytes) {  // problem_io.hpp:527-535
  uint64_t h = 1469598103934665603ULL;
  for (const unsigned char b : bytes) {
    h ^= b;
    h *= 1099511628211ULL;
  }
  return h;
}

uint64_t content_hash(const Problem& p) { return fnv1a(serialize_problem(p)); }
uint64_t factor_hash(const Problem& p) { return fnv1a(write_problem(p, -1, true)); }

void save_problem(const Problem& p, const std::string& path) {  // problem_io.hpp:494-500
  std::ofstream out(path, std::ios::binary);
  if (!out) parse_fail("save_problem: cannot open " + path);
  out << serialize_problem(p);
  if (!out) parse_fail("save_problem: write failed for " + path);
}

Problem load_problem(const std::string& path) {  // problem_io.hpp:502-508
  std::ifstream in(path, std::ios::binary);
  if (!in) parse_fail("load_problem: cannot open " + path);
  std::ostringstream buf;
  buf << in.rdbuf();
  return parse_problem(buf.str());
}

}  // namespace scn
