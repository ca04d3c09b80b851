// SPDX-License-Identifier: MIT
// extern "C" boundary (include/scenopt_b200.h). Every entry point converts
// scn::Error (the errors.hpp taxonomy) into its status code and records the
// message for scenopt_last_error().
#include <cstring>
#include <memory>
#include <random>
#include <string>

#include "capi_internal.hpp"
#include "problem_io.hpp"

using namespace scn;

namespace scn {
thread_local std::string g_last_error;
}


extern "C" {

const char* scenopt_last_error(void) { return g_last_error.c_str(); }
int scenopt_abi_version(void) { return SCENOPT_ABI_VERSION; }
int scenopt_device_count(void) { return device_count_sm100(); }

// ---------------------------------------------------------------- problem
int scenopt_problem_create(const scenopt_problem_view* v, scenopt_problem** out) {
  SCN_GUARD({
    if (!v || !out) fail(SCENOPT_E_INVALID_PARAMS, "scenopt_problem_create: null argument");
    auto h = std::make_unique<scenopt_problem>();
    h->p = problem_from_view(*v);
    *out = h.release();
  });
}

int scenopt_problem_gen_random(uint64_t seed, int nx, int nu, int horizon, const int32_t* branching,
                               int nbranch, scenopt_problem** out) {
  SCN_GUARD({
    std::vector<int> br(branching, branching + (nbranch > 0 ? nbranch : 0));
    auto h = std::make_unique<scenopt_problem>();
    h->p = gen_random(seed, nx, nu, horizon, br);
    *out = h.release();
  });
}

int scenopt_problem_gen_random_shard(uint64_t seed, int nx, int nu, int horizon, const int32_t* branching,
                                     int nbranch, int world, int rank, int shard_stage, scenopt_problem** out) {
  SCN_GUARD({
    if (world < 1 || rank < 0 || rank >= world) fail(SCENOPT_E_INVALID_PARAMS, "gen_random_instance: bad rank/world");
    std::vector<int> br(branching, branching + (nbranch > 0 ? nbranch : 0));
    const Problem tree = gen_random_tree(nx, nu, horizon, br);
    int s = shard_stage;
    const std::vector<int> b = shard_plan(tree, world, &s);
    std::vector<char> keep = shard_nodes(tree, s, b[rank], b[rank + 1], rank);
    for (int c = 0; c < tree.stage_offsets[s + 1]; ++c) keep[c] = 1;  // the top and every shard-stage node
    auto h = std::make_unique<scenopt_problem>();
    h->p = gen_random(seed, nx, nu, horizon, br, &keep);
    *out = h.release();
  });
}

namespace {
SpringMass spring_from(const scenopt_spring_mass_params* c) {
  SpringMass p;
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
    p.transition.assign(c->transition, c->transition + static_cast<size_t>(c->transition_rows) * c->transition_cols);
    p.transition_rows = c->transition_rows;
    p.transition_cols = c->transition_cols;
  }
  if (c->mode_values_len > 0) p.mode_values.assign(c->mode_values, c->mode_values + c->mode_values_len);
  if (c->root_state_len > 0) p.root_state.assign(c->root_state, c->root_state + c->root_state_len);
  return p;
}
}  // namespace

void scenopt_spring_mass_defaults(scenopt_spring_mass_params* par) {
  if (!par) return;
  const SpringMass d;
  *par = scenopt_spring_mass_params{};
  par->mass_kg = d.mass_kg;
  par->stiffness = d.stiffness;
  par->damping = d.damping;
  par->input_bound = d.input_bound;
  par->velocity_bound = d.velocity_bound;
  par->horizon = d.horizon;
  par->sampling = d.sampling;
  par->state_weight = d.state_weight;
  par->input_weight = d.input_weight;
  par->terminal_weight = d.terminal_weight;
}

int scenopt_problem_gen_spring_mass(int masses, const scenopt_spring_mass_params* par, scenopt_problem** out) {
  SCN_GUARD({
    if (!out) fail(SCENOPT_E_INVALID_PARAMS, "gen_spring_mass: null output");
    auto h = std::make_unique<scenopt_problem>();
    h->p = gen_spring_mass(masses, spring_from(par));
    *out = h.release();
  });
}

int scenopt_spring_mass_continuous(int masses, const scenopt_spring_mass_params* par, double* A, double* B) {
  SCN_GUARD({
    if (masses < 2) fail(SCENOPT_E_INVALID_PARAMS, "spring_mass_continuous: masses must be >= 2");
    std::vector<double> a, b;
    spring_mass_continuous(masses, spring_from(par), a, b);
    std::copy(a.begin(), a.end(), A);
    std::copy(b.begin(), b.end(), B);
  });
}

int scenopt_discretize_zoh(const double* A, const double* B, int n, int m, double period, double* Ad, double* Bd) {
  SCN_GUARD({
    if (n < 1 || m < 0) fail(SCENOPT_E_DIMENSION_MISMATCH, "discretize_zoh: A must be square and match B");
    discretize_zoh(A, B, n, m, period, Ad, Bd);
  });
}

int scenopt_expm(const double* X, int n, double* out) {
  SCN_GUARD({
    if (n < 1) fail(SCENOPT_E_DIMENSION_MISMATCH, "expm: matrix must be square and non-empty");
    const std::vector<double> E = expm(std::vector<double>(X, X + static_cast<size_t>(n) * n), n);
    std::copy(E.begin(), E.end(), out);
  });
}

int scenopt_sample_initial_states(int masses, const scenopt_spring_mass_params* par, uint64_t seed, int count,
                                  double* out) {
  SCN_GUARD({
    if (masses < 2) fail(SCENOPT_E_INVALID_PARAMS, "sample_initial_state: masses must be >= 2");
    const SpringMass p = spring_from(par);
    const double half = 0.5 * p.velocity_bound, pos_box = 1.0 * p.velocity_bound;
    std::mt19937_64 gen(seed);
    auto sym = [&gen]() { return 2.0 * (static_cast<double>(gen() >> 11) * 0x1.0p-53) - 1.0; };
    for (int k = 0; k < count; ++k) {
      double* s = out + static_cast<size_t>(k) * 2 * masses;
      for (int i = 0; i < masses; ++i) s[i] = pos_box * sym();
      for (int i = masses; i < 2 * masses; ++i) s[i] = half * sym();
    }
  });
}

int scenopt_problem_get_view(scenopt_problem* p, scenopt_problem_view* v, int32_t* dual_dim) {
  SCN_GUARD({
    problem_to_view(p->p, v);
    if (dual_dim) *dual_dim = p->p.dual_dim;
  });
}

int scenopt_problem_dims(const scenopt_problem* p, int32_t* dims) {
  SCN_GUARD({
    const Problem& q = p->p;
    dims[0] = q.nx;
    dims[1] = q.nu;
    dims[2] = q.N;
    dims[3] = q.n;
    dims[4] = q.L;
    dims[5] = q.first_leaf;
    dims[6] = q.dual_dim;
    dims[7] = q.primal_dim();
  });
}

int scenopt_problem_validate(const scenopt_problem* p, char* buf, int buflen) {
  try {
    const auto bad = validate(p->p);
    std::string all;
    for (const auto& b : bad) all += b + "\n";
    if (buf && buflen > 0) {
      std::strncpy(buf, all.c_str(), static_cast<size_t>(buflen) - 1);
      buf[buflen - 1] = 0;
    }
    return static_cast<int>(bad.size());
  } catch (const Error& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return SCENOPT_E_ERROR;
  }
}

int scenopt_problem_precondition(const scenopt_problem* p, scenopt_problem** out) {
  SCN_GUARD({
    auto h = std::make_unique<scenopt_problem>();
    h->p = precondition(p->p);
    *out = h.release();
  });
}

void scenopt_problem_destroy(scenopt_problem* p) { delete p; }

// ---------------------------------------------------------------- factor
int scenopt_factor_create(const scenopt_problem* p, scenopt_factor** out) {
  SCN_GUARD({
    auto h = std::make_unique<scenopt_factor>();
    h->f = factor(p->p);
    *out = h.release();
  });
}

int scenopt_refactor_affine(scenopt_factor* f, const scenopt_problem* p) {
  SCN_GUARD(refactor_affine(f->f, p->p));
}

int scenopt_factor_export(const scenopt_factor* h, double* gain, double* c2i, double* cl, double* d2i,
                          double* d2c, double* ia, double* ca, double* vq, double* lca) {
  SCN_GUARD({
    const Factor& f = h->f;
    auto cp = [](const std::vector<double>& v, double* dst) {
      if (dst && !v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(double));
    };
    cp(f.gain, gain);
    cp(f.child_to_input, c2i);
    cp(f.closed_loop, cl);
    cp(f.dual_to_input, d2i);
    cp(f.dual_to_costate, d2c);
    cp(f.input_affine, ia);
    cp(f.costate_affine, ca);
    cp(f.value_quad, vq);
    cp(f.leaf_costate_affine, lca);
  });
}

void scenopt_factor_destroy(scenopt_factor* f) { delete f; }

// ---------------------------------------------------------------- device
int scenopt_dev_create(const scenopt_problem* p, const scenopt_factor* f, int device, scenopt_dev** out) {
  SCN_GUARD({
    auto h = std::make_unique<scenopt_dev>();
    h->d = dev_create(p->p, f ? &f->f : nullptr, device);
    h->init_solver_buffers();
    *out = h.release();
  });
}

int scenopt_nccl_unique_id(void* out128) { SCN_GUARD(nccl_unique_id(out128)); }

int scenopt_shard_plan(const scenopt_problem* p, int world, int shard_stage, int32_t* stage_out,
                       int32_t* bounds) {
  SCN_GUARD({
    int s = shard_stage;
    const std::vector<int> b = shard_plan(p->p, world, &s);
    *stage_out = s;
    for (size_t i = 0; i < b.size(); ++i) bounds[i] = b[i];
  });
}

int scenopt_shard_rows(const scenopt_problem* p, int world, int shard_stage, int rank, uint8_t* counted) {
  SCN_GUARD({
    if (world < 1 || rank < 0 || rank >= world) fail(SCENOPT_E_INVALID_PARAMS, "shard rows: bad rank/world");
    int s = shard_stage;
    const std::vector<int> b = shard_plan(p->p, world, &s);
    const std::vector<uint8_t> cnt = shard_rows(p->p, shard_nodes(p->p, s, b[rank], b[rank + 1], rank));
    std::copy(cnt.begin(), cnt.end(), counted);
  });
}

int scenopt_dev_create_sharded(const scenopt_problem* p, const scenopt_factor* f, int device, int rank,
                               int world, int shard_stage, const void* nccl_id, scenopt_dev** out) {
  SCN_GUARD({
    if (world < 1 || rank < 0 || rank >= world) fail(SCENOPT_E_INVALID_PARAMS, "dev_create_sharded: bad rank/world");
    ShardSpec spec;
    spec.rank = rank;
    spec.world = world;
    spec.stage = shard_stage;
    spec.nccl_id = nccl_id;
    auto h = std::make_unique<scenopt_dev>();
    h->d = f ? dev_create(p->p, &f->f, device, &spec) : dev_create_device_factor(p->p, device, &spec);
    h->init_solver_buffers();
    *out = h.release();
  });
}

struct scenopt_shard_group {
  std::shared_ptr<EmuGroup> g;
};

int scenopt_shard_group_create(int world, scenopt_shard_group** out) {
  SCN_GUARD({
    auto g = std::make_unique<scenopt_shard_group>();
    g->g = emu_group_create(world);
    *out = g.release();
  });
}

void scenopt_shard_group_destroy(scenopt_shard_group* g) { delete g; }

int scenopt_dev_create_sharded_group(const scenopt_problem* p, const scenopt_factor* f, int device, int rank,
                                     scenopt_shard_group* g, int shard_stage, scenopt_dev** out) {
  SCN_GUARD({
    if (!g) fail(SCENOPT_E_INVALID_PARAMS, "dev_create_sharded: null shard group");
    ShardSpec spec;
    spec.rank = rank;
    spec.world = emu_group_world(*g->g);
    spec.stage = shard_stage;
    spec.emu = g->g;
    if (rank < 0 || rank >= spec.world) fail(SCENOPT_E_INVALID_PARAMS, "dev_create_sharded: bad rank/world");
    auto h = std::make_unique<scenopt_dev>();
    h->d = f ? dev_create(p->p, &f->f, device, &spec) : dev_create_device_factor(p->p, device, &spec);
    h->init_solver_buffers();
    *out = h.release();
  });
}

int scenopt_shard_sweep_phase(scenopt_dev* h, int phase, int nrhs, int affine, const double* const* y,
                              double* const* Hx) {
  SCN_GUARD({
    SCN_CUDA(cudaSetDevice(h->d->device));
    dev_sweep_phase(*h->d, phase, nrhs, affine != 0, y, Hx);
  });
}

int scenopt_shard_exchange_buffer(scenopt_dev* h, double** buf, size_t* doubles_per_rhs) {
  SCN_GUARD({
    const DevState& d = *h->d;
    if (!d.sharded()) fail(SCENOPT_E_INVALID_PARAMS, "exchange buffer: handle is not sharded");
    *buf = d.xbuf;
    *doubles_per_rhs = static_cast<size_t>(d.xbuf_rhs);
  });
}

int scenopt_dev_create_device_factor(const scenopt_problem* p, int device, scenopt_dev** out) {
  SCN_GUARD({
    auto h = std::make_unique<scenopt_dev>();
    h->d = dev_create_device_factor(p->p, device);
    h->init_solver_buffers();
    *out = h.release();
  });
}

int scenopt_dev_factor_export(scenopt_dev* h, const scenopt_problem* p, double* gain, double* c2i, double* cl,
                              double* d2i, double* d2c, double* ia, double* ca, double* vq, double* lca) {
  SCN_GUARD({
    const Factor f = dev_factor_export(*h->d, p->p);
    auto cp = [](const std::vector<double>& v, double* dst) {
      if (dst && !v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(double));
    };
    cp(f.gain, gain);
    cp(f.child_to_input, c2i);
    cp(f.closed_loop, cl);
    cp(f.dual_to_input, d2i);
    cp(f.dual_to_costate, d2c);
    cp(f.input_affine, ia);
    cp(f.costate_affine, ca);
    cp(f.value_quad, vq);
    cp(f.leaf_costate_affine, lca);
  });
}

int scenopt_dev_info_get(const scenopt_dev* h, scenopt_dev_info* info) {
  SCN_GUARD({
    const DevState& d = *h->d;
    *info = scenopt_dev_info{};
    info->device = d.device;
    info->sm_count = d.sm_count;
    info->grid_ctas = d.grid;
    info->ctas_per_sm = d.ctas_per_sm;
    info->slots = d.nslot;
    info->items_bw = d.items_bw;
    info->items_fw = d.items_fw;
    info->nodes_per_item_max = d.max_count;
    info->slot_bytes = static_cast<int64_t>(d.slot_doubles) * 8;
    info->matrix_bytes_bw = d.bw_doubles * 8;
    info->matrix_bytes_fw = d.fw_doubles * 8;
    info->device_bytes = static_cast<int64_t>(d.bytes_allocated);
    info->sweep_bytes_hom = d.bytes_hom;
    info->sweep_bytes_aff = d.bytes_aff;
    info->sweep_bytes_hom2 = d.bytes_hom2;
    info->cut_stage = d.cut_stage;
    info->shard_stage = d.shard_stage;
    info->rank = d.rank;
    info->world = d.world;
    info->shard_first = d.shard_lo;
    info->shard_past = d.shard_hi;
    info->exchange_doubles = d.sharded() ? d.xbuf_rhs : 0;
    info->items_global = d.items_global;
    info->consumer_stage = d.consumer_stage ? 1 : 0;
    info->flat_top = d.flat_top ? 1 : 0;
    info->device_factor = d.device_factor ? 1 : 0;
    info->producer_warps = d.sweep->producers;
  });
}

int scenopt_dev_stream(scenopt_dev* h, void** stream) {
  SCN_GUARD(*stream = static_cast<void*>(h->d->stream));
}

int scenopt_dev_synchronize(scenopt_dev* h) {
  SCN_GUARD({
    SCN_CUDA(cudaSetDevice(h->d->device));
    SCN_CUDA(cudaStreamSynchronize(h->d->stream));
  });
}

void scenopt_dev_destroy(scenopt_dev* h) { delete h; }

int scenopt_dev_alloc(scenopt_dev* h, size_t bytes, void** out) {
  SCN_GUARD({
    SCN_CUDA(cudaSetDevice(h->d->device));
    *out = h->d->alloc<char>(bytes);
  });
}

int scenopt_dev_free(scenopt_dev* h, void* ptr) {
  SCN_GUARD({
    SCN_CUDA(cudaSetDevice(h->d->device));
    h->d->free_owned(ptr);
  });
}

int scenopt_dev_memcpy(scenopt_dev* h, void* dst, const void* src, size_t bytes, int kind) {
  SCN_GUARD({
    SCN_CUDA(cudaSetDevice(h->d->device));
    SCN_CUDA(cudaMemcpyAsync(dst, src, bytes, static_cast<cudaMemcpyKind>(kind), h->d->stream));
    SCN_CUDA(cudaStreamSynchronize(h->d->stream));
  });
}

// ---------------------------------------------------------------- oracles
int scenopt_dev_sweep(scenopt_dev* h, int nrhs, int affine, const double* const* y, double* const* x,
                      double* const* u, double* const* Hx, int flags) {
  SCN_GUARD(h->sweep(nrhs, affine != 0, y, x, u, Hx, flags, true));
}

int scenopt_dev_sweep_async(scenopt_dev* h, int nrhs, int affine, const double* const* y,
                            double* const* x, double* const* u, double* const* Hx) {
  SCN_GUARD(h->sweep(nrhs, affine != 0, y, x, u, Hx, 0, false));
}

int scenopt_dual_grad(scenopt_dev* h, const double* y, double* x, double* u, int flags) {
  SCN_GUARD({
    ++h->stats.dual_grad_calls;
    h->sweep(1, true, &y, &x, &u, nullptr, flags, true);
  });
}

int scenopt_hessian_vec(scenopt_dev* h, const double* r, double* x, double* u, int flags) {
  SCN_GUARD({
    ++h->stats.hessian_vec_calls;
    h->sweep(1, false, &r, &x, &u, nullptr, flags, true);
  });
}

/* Development hook: per-role cycle counters of a -DSCN_SWEEP_PROFILE build
 * (all zero in the production library). */
int scenopt_debug_sweep_profile(unsigned long long* out16, int reset) {
  SCN_GUARD(SCN_CUDA(sweep_profile_read(out16, reset != 0)));
}

// Profiling build only: per-item retirement timestamps into dev_buf (one
// u64 per item in handle order; NULL switches the timeline off).
int scenopt_debug_sweep_timeline(void* dev_buf) {
  SCN_GUARD(SCN_CUDA(sweep_timeline(static_cast<unsigned long long*>(dev_buf))));
}

int scenopt_debug_sweep_trace(void* dev_buf) {
  SCN_GUARD(SCN_CUDA(sweep_trace(static_cast<long long*>(dev_buf))));
}

// Items in handle order: {launch, cta, pass, first, count, ldep, publish} x n.
int scenopt_debug_items(scenopt_dev* h, int32_t* out, int cap) {
  int total = 0;
  try {
    const DevState& d = *h->d;
    int li = 0;
    for (const auto& ln : d.launches) {
      std::vector<Item> it(static_cast<size_t>(ln.count));
      std::vector<int32_t> off(static_cast<size_t>(d.grid) + 1);
      SCN_CUDA(cudaMemcpy(it.data(), ln.items, it.size() * sizeof(Item), cudaMemcpyDeviceToHost));
      SCN_CUDA(cudaMemcpy(off.data(), ln.cta_off, off.size() * sizeof(int32_t), cudaMemcpyDeviceToHost));
      for (int b = 0; b < d.grid; ++b)
        for (int k = off[b]; k < off[b + 1]; ++k, ++total)
          if (out && total < cap) {
            int32_t* o = out + 7 * total;
            o[0] = li, o[1] = b, o[2] = it[k].pass, o[3] = it[k].first, o[4] = it[k].count, o[5] = it[k].ldep,
            o[6] = it[k].publish;
          }
      ++li;
    }
    return total;
  } catch (const Error& e) {
    g_last_error = e.what();
    return e.code;
  }
}

}  // extern "C"

// ---------------------------------------------------------------- problem files (problem_io.hpp)
namespace {
int copy_out(const std::string& s, char* buf, size_t cap, size_t* len) {
  if (len) *len = s.size();
  if (buf && cap > 0) {
    const size_t n = std::min(cap - 1, s.size());
    std::memcpy(buf, s.data(), n);
    buf[n] = 0;
  }
  return 0;
}
}  // namespace

int scenopt_problem_serialize(scenopt_problem* p, char* buf, size_t cap, size_t* len) {
  SCN_GUARD({
    if (!p) fail(SCENOPT_E_INVALID_PARAMS, "serialize_problem: null problem");
    if (!buf || p->text.empty()) p->text = serialize_problem(p->p);
    copy_out(p->text, buf, cap, len);
    if (buf) std::string().swap(p->text);
  });
}

int scenopt_problem_parse(const char* text, size_t len, scenopt_problem** out) {
  SCN_GUARD({
    if (!text || !out) fail(SCENOPT_E_INVALID_PARAMS, "parse_problem: null argument");
    auto h = std::make_unique<scenopt_problem>();
    h->p = parse_problem(std::string(text, len));
    *out = h.release();
  });
}

int scenopt_problem_validate_text(const char* text, size_t len, char* buf, int buflen) {
  try {
    const auto bad = validate_problem_text(std::string(text ? text : "", text ? len : 0));
    std::string all;
    for (const auto& b : bad) all += b + "\n";
    if (buf && buflen > 0) {
      std::strncpy(buf, all.c_str(), static_cast<size_t>(buflen) - 1);
      buf[buflen - 1] = 0;
    }
    return static_cast<int>(bad.size());
  } catch (const Error& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return SCENOPT_E_ERROR;
  }
}

int scenopt_problem_save(const scenopt_problem* p, const char* path) {
  SCN_GUARD({
    if (!p || !path) fail(SCENOPT_E_INVALID_PARAMS, "save_problem: null argument");
    save_problem(p->p, path);
  });
}

int scenopt_problem_load(const char* path, scenopt_problem** out) {
  SCN_GUARD({
    if (!path || !out) fail(SCENOPT_E_INVALID_PARAMS, "load_problem: null argument");
    auto h = std::make_unique<scenopt_problem>();
    h->p = load_problem(path);
    *out = h.release();
  });
}

int scenopt_problem_hashes(const scenopt_problem* p, uint64_t* content, uint64_t* factor) {
  SCN_GUARD({
    if (!p) fail(SCENOPT_E_INVALID_PARAMS, "problem hashes: null problem");
    if (content) *content = content_hash(p->p);
    if (factor) *factor = factor_hash(p->p);
  });
}

int scenopt_problem_set_mode(scenopt_problem* p, const int32_t* mode, int n) {
  SCN_GUARD({
    if (!p) fail(SCENOPT_E_INVALID_PARAMS, "set_mode: null problem");
    if (n != 0 && n != p->p.n) fail(SCENOPT_E_DIMENSION_MISMATCH, "tree: mode must be empty or one entry per node");
    p->p.mode.assign(mode, mode + n);
  });
}

int scenopt_problem_get_mode(const scenopt_problem* p, int32_t* out, int cap) {
  SCN_GUARD({
    if (!p) fail(SCENOPT_E_INVALID_PARAMS, "get_mode: null problem");
    const int n = static_cast<int>(p->p.mode.size());
    if (out)
      for (int i = 0; i < std::min(n, cap); ++i) out[i] = p->p.mode[static_cast<size_t>(i)];
    return n;
  });
}
