// SPDX-License-Identifier: MIT
// Collectives of a subtree-sharded handle,
// enqueued on the handle's stream:
//   - allreduce_sum: the shard-stage exchange of every sweep (the partial
//     [u_off; w] contributions of the shard-stage nodes to their parents,
//     plus those nodes' own dual rows, which the replicated top backward
//     reads) -- the one vector collective of the path;
//   - allgather: the per-rank partial sums of the dual-space kernels (a few
//     dozen doubles), combined on the device in rank order, so every rank
//     holds bitwise-identical scalars and takes identical decisions.
// Two implementations: NCCL (one communicator per handle), and an emulated
// group of handles in ONE process (one host thread per rank) that exchanges
// through host memory after a stream synchronisation -- kernels of different
// ranks never wait on one another, so W ranks can share one GPU in tests.
//
// NCCL is loaded on first use (dlopen), not linked: a process that loads this
// library and later imports a framework with its own NCCL build (PyTorch
// bundles a newer one) must not find an older libnccl.so.2 already bound.
// Resolution order: an libnccl.so.2 already in the process, then
// $SCENOPT_NCCL_LIBRARY (the Python package points it at the framework's
// copy when present), then the loader's search path.
#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
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
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
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
    n.all_gather = reinterpret_cast<decltype(n.all_gather)>(sym("ncclAllGather"));
    n.error_string = reinterpret_cast<decltype(n.error_string)>(sym("ncclGetErrorString"));
    if (!n.get_unique_id || !n.comm_init_rank || !n.comm_destroy || !n.all_reduce || !n.all_gather ||
        !n.error_string) {
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

struct NcclComm final : Comm {
  ncclComm_t c = nullptr;
  ~NcclComm() override {
    if (c) nccl().comm_destroy(c);
  }
  void allreduce_sum(double* buf, size_t n, cudaStream_t st) override {
    if (n) check(nccl().all_reduce(buf, buf, n, ncclDouble, ncclSum, c, st), "ncclAllReduce");
  }
  void allgather(const double* send, double* recv, size_t n, cudaStream_t st) override {
    if (n) check(nccl().all_gather(send, recv, n, ncclDouble, c, st), "ncclAllGather");
  }
};
}  // namespace

// ---------------------------------------------------------------- emulated group
struct EmuGroup {
  int world = 1;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  unsigned long long gen = 0;
  bool broken = false;  // a rank failed: the others must not wait forever
  std::vector<std::vector<double>> slot;
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const unsigned long long g = gen;
    if (++arrived == world) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g || broken; });
    }
    if (broken) fail(SCENOPT_E_ERROR, "emulated shard group: another rank failed");
  }
  void abort() {
    std::lock_guard<std::mutex> lk(mu);
    broken = true;
    cv.notify_all();
  }
};

namespace {
struct EmuComm final : Comm {
  std::shared_ptr<EmuGroup> g;
  int rank = 0;
  template <class F>
  void guarded(F&& f) {
    try {
      f();
    } catch (...) {
      g->abort();
      throw;
    }
  }
  void allreduce_sum(double* buf, size_t n, cudaStream_t st) override {
    if (!n) return;
    guarded([&] {
      std::vector<double>& mine = g->slot[rank];
      mine.resize(n);
      SCN_CUDA(cudaMemcpyAsync(mine.data(), buf, n * sizeof(double), cudaMemcpyDeviceToHost, st));
      SCN_CUDA(cudaStreamSynchronize(st));
      g->barrier();
      std::vector<double> sum(g->slot[0]);  // rank order, as every rank computes it
      for (int q = 1; q < g->world; ++q)
        for (size_t i = 0; i < n; ++i) sum[i] += g->slot[q][i];
      SCN_CUDA(cudaMemcpyAsync(buf, sum.data(), n * sizeof(double), cudaMemcpyHostToDevice, st));
      SCN_CUDA(cudaStreamSynchronize(st));
      g->barrier();  // every rank has read every slot
    });
  }
  void allgather(const double* send, double* recv, size_t n, cudaStream_t st) override {
    if (!n) return;
    guarded([&] {
      std::vector<double>& mine = g->slot[rank];
      mine.resize(n);
      SCN_CUDA(cudaMemcpyAsync(mine.data(), send, n * sizeof(double), cudaMemcpyDeviceToHost, st));
      SCN_CUDA(cudaStreamSynchronize(st));
      g->barrier();
      for (int q = 0; q < g->world; ++q)
        SCN_CUDA(cudaMemcpyAsync(recv + static_cast<size_t>(q) * n, g->slot[q].data(), n * sizeof(double),
                                 cudaMemcpyHostToDevice, st));
      SCN_CUDA(cudaStreamSynchronize(st));
      g->barrier();
    });
  }
};
}  // namespace

std::shared_ptr<EmuGroup> emu_group_create(int world) {
  if (world < 1) fail(SCENOPT_E_INVALID_PARAMS, "emulated shard group: world must be >= 1");
  auto g = std::make_shared<EmuGroup>();
  g->world = world;
  g->slot.resize(static_cast<size_t>(world));
  return g;
}

int emu_group_world(const EmuGroup& g) { return g.world; }

std::unique_ptr<Comm> emu_comm(const std::shared_ptr<EmuGroup>& g, int rank) {
  if (!g || rank < 0 || rank >= g->world) fail(SCENOPT_E_INVALID_PARAMS, "emulated shard group: bad rank");
  auto c = std::make_unique<EmuComm>();
  c->g = g;
  c->rank = rank;
  return c;
}

void nccl_unique_id(void* out128) {
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  ncclUniqueId id;
  check(nccl().get_unique_id(&id), "ncclGetUniqueId");
  std::memcpy(out128, &id, sizeof(id));
}

std::unique_ptr<Comm> nccl_comm(int device, int rank, int world, const void* id128) {
  if (!id128) fail(SCENOPT_E_INVALID_PARAMS, "dev_create_sharded: missing NCCL unique id");
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof(id));
  SCN_CUDA(cudaSetDevice(device));
  auto c = std::make_unique<NcclComm>();
  check(nccl().comm_init_rank(&c->c, world, id, rank), "ncclCommInitRank");
  return c;
}

void dev_allreduce(DevState& d, double* buf, size_t n) {
  if (!d.sharded() || n == 0 || (d.world == 1 && !d.comm)) return;
  if (!d.comm)
    fail(SCENOPT_E_INVALID_PARAMS, "sharded handle without a communicator: use the phase API (scenopt_shard_sweep_phase)");
  d.comm->allreduce_sum(buf, n, d.stream);
}

// dualops.cu's phase launchers reach the communicator through DualCtx::xc
void dual_allgather(void* xc, const double* send, double* recv, size_t n, cudaStream_t st) {
  static_cast<Comm*>(xc)->allgather(send, recv, n, st);
}

}  // namespace scn
