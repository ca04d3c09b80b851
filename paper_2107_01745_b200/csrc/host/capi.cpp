// SPDX-License-Identifier: MIT
// extern "C" boundary (include/scenopt_b200.h). Every entry point converts
// scn::Error (the errors.hpp taxonomy) into its status code and records the
// message for scenopt_last_error().
#include <cstring>
#include <memory>
#include <string>

#include "capi_internal.hpp"

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

int scenopt_dev_create_sharded(const scenopt_problem* p, const scenopt_factor* f, int device, int rank,
                               int world, int shard_stage, const void* nccl_id, scenopt_dev** out) {
  SCN_GUARD({
    if (!f) fail(SCENOPT_E_INVALID_PARAMS, "dev_create_sharded: a factor cache is required");
    if (world < 1 || rank < 0 || rank >= world) fail(SCENOPT_E_INVALID_PARAMS, "dev_create_sharded: bad rank/world");
    ShardSpec spec;
    spec.rank = rank;
    spec.world = world;
    spec.stage = shard_stage;
    spec.nccl_id = nccl_id;
    auto h = std::make_unique<scenopt_dev>();
    h->d = dev_create(p->p, &f->f, device, &spec);
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
    *doubles_per_rhs = static_cast<size_t>(d.sstage_hi - d.sstage_lo) * (d.lay.nx + d.lay.nu);
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
    info->items_global = d.items_global;
    info->consumer_stage = d.consumer_stage ? 1 : 0;
    info->flat_top = d.flat_top ? 1 : 0;
    info->device_factor = d.device_factor ? 1 : 0;
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
