// SPDX-License-Identifier: MIT
// NCCL plumbing of a subtree-sharded handle:
// one communicator per handle, sum-allreduces enqueued on the handle's
// stream. The exchange of a sweep is the shard-stage contributions (one
// allreduce between the two sweep launches) and Hx assembled from disjoint
// row sets (exact: every row is nonzero on exactly one rank).
#include <nccl.h>

#include <cstring>

#include "device.hpp"

namespace scn {

#define SCN_NCCL(expr)                                                                    \
  do {                                                                                    \
    ncclResult_t _r = (expr);                                                             \
    if (_r != ncclSuccess) fail(SCENOPT_E_NCCL, std::string(#expr) + ": " + ncclGetErrorString(_r)); \
  } while (0)

void nccl_unique_id(void* out128) {
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  ncclUniqueId id;
  SCN_NCCL(ncclGetUniqueId(&id));
  std::memcpy(out128, &id, sizeof(id));
}

void nccl_comm_init(DevState& d, const void* id128) {
  if (!id128) fail(SCENOPT_E_INVALID_PARAMS, "dev_create_sharded: missing NCCL unique id");
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof(id));
  SCN_CUDA(cudaSetDevice(d.device));
  ncclComm_t c = nullptr;
  SCN_NCCL(ncclCommInitRank(&c, d.world, id, d.rank));
  d.comm = c;
}

void nccl_comm_destroy(void* comm) {
  if (comm) ncclCommDestroy(static_cast<ncclComm_t>(comm));
}

void dev_allreduce(DevState& d, double* buf, size_t n) {
  if (!d.sharded() || d.world == 1 || n == 0) return;
  if (!d.comm)
    fail(SCENOPT_E_INVALID_PARAMS, "sharded handle without a communicator: use the phase API (scenopt_shard_sweep_phase)");
  SCN_NCCL(ncclAllReduce(buf, buf, n, ncclDouble, ncclSum, static_cast<ncclComm_t>(d.comm), d.stream));
}

}  // namespace scn
