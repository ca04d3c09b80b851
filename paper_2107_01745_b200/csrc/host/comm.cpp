// SPDX-License-Identifier: MIT
// NCCL plumbing of a subtree-sharded handle:
// one communicator per handle, sum-allreduces enqueued on the handle's
// stream. The exchange of a sweep is the shard-stage contributions (one
// allreduce between the two sweep launches) and Hx assembled from disjoint
// row sets (exact: every row is nonzero on exactly one rank).
//
// NCCL is loaded on first use (dlopen), not linked: a process that loads this
// library and later imports a framework with its own NCCL build (PyTorch
// bundles a newer one) must not find an older libnccl.so.2 already bound.
// Resolution order: an libnccl.so.2 already in the process, then
// $SCENOPT_NCCL_LIBRARY (the Python package points it at the framework's
// copy when present), then the loader's search path.
#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <cstring>
#include <mutex>

#include "device.hpp"

namespace scn {

namespace {
struct Nccl {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  std::string load_error;
};

const Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h)
      if (const char* p = std::getenv("SCENOPT_NCCL_LIBRARY"); p && *p) h = dlopen(p, RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      const char* e = dlerror();
      n.load_error = e ? e : "libnccl.so.2 not found";
      return;
    }
    auto sym = [&](const char* name) { return dlsym(h, name); };
    n.get_unique_id = reinterpret_cast<decltype(n.get_unique_id)>(sym("ncclGetUniqueId"));
    n.comm_init_rank = reinterpret_cast<decltype(n.comm_init_rank)>(sym("ncclCommInitRank"));
    n.comm_destroy = reinterpret_cast<decltype(n.comm_destroy)>(sym("ncclCommDestroy"));
    n.all_reduce = reinterpret_cast<decltype(n.all_reduce)>(sym("ncclAllReduce"));
    n.error_string = reinterpret_cast<decltype(n.error_string)>(sym("ncclGetErrorString"));
    if (!n.get_unique_id || !n.comm_init_rank || !n.comm_destroy || !n.all_reduce || !n.error_string) {
      n.load_error = "libnccl.so.2 lacks an expected entry point";
      n.get_unique_id = nullptr;
    }
  });
  if (!n.get_unique_id) fail(SCENOPT_E_NCCL, "NCCL unavailable: " + n.load_error);
  return n;
}

void check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) fail(SCENOPT_E_NCCL, std::string(what) + ": " + nccl().error_string(r));
}
}  // namespace

void nccl_unique_id(void* out128) {
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  ncclUniqueId id;
  check(nccl().get_unique_id(&id), "ncclGetUniqueId");
  std::memcpy(out128, &id, sizeof(id));
}

void nccl_comm_init(DevState& d, const void* id128) {
  if (!id128) fail(SCENOPT_E_INVALID_PARAMS, "dev_create_sharded: missing NCCL unique id");
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof(id));
  SCN_CUDA(cudaSetDevice(d.device));
  ncclComm_t c = nullptr;
  check(nccl().comm_init_rank(&c, d.world, id, d.rank), "ncclCommInitRank");
  d.comm = c;
}

void nccl_comm_destroy(void* comm) {
  if (comm) nccl().comm_destroy(static_cast<ncclComm_t>(comm));
}

void dev_allreduce(DevState& d, double* buf, size_t n) {
  if (!d.sharded() || d.world == 1 || n == 0) return;
  if (!d.comm)
    fail(SCENOPT_E_INVALID_PARAMS, "sharded handle without a communicator: use the phase API (scenopt_shard_sweep_phase)");
  check(nccl().all_reduce(buf, buf, n, ncclDouble, ncclSum, static_cast<ncclComm_t>(d.comm), d.stream),
        "ncclAllReduce");
}

}  // namespace scn
