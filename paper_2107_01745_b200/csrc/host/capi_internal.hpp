// SPDX-License-Identifier: MIT
// Internals shared by the C-ABI translation units.
#pragma once

#include <cstdint>
#include <memory>
#include <string>

#include "device.hpp"
#include "model.hpp"

namespace scn {
extern thread_local std::string g_last_error;

struct Stats {  // OracleStats, tree_oracles.hpp:14-21
  uint64_t dual_grad_calls = 0, hessian_vec_calls = 0, prox_calls = 0, conj_calls = 0;
};
}  // namespace scn

#define SCN_GUARD(...)                   \
  do {                                   \
    try {                                \
      __VA_ARGS__;                       \
      return SCENOPT_OK;                 \
    } catch (const ::scn::Error& e) {    \
      ::scn::g_last_error = e.what();    \
      return e.code;                     \
    } catch (const std::bad_alloc&) {    \
      ::scn::g_last_error = "out of host memory"; \
      return SCENOPT_E_NOMEM;            \
    } catch (const std::exception& e) {  \
      ::scn::g_last_error = e.what();    \
      return SCENOPT_E_ERROR;            \
    }                                    \
  } while (0)

struct scenopt_problem {
  scn::Problem p;
  std::string text;  // last serialization (size query, then copy)
};
struct scenopt_factor {
  scn::Factor f;
};

struct scenopt_dev {
  std::unique_ptr<scn::DevState> d;
  scn::Stats stats;
  // solver workspace (device): dual vectors and scalar block, see solver.cpp
  struct Work;
  std::unique_ptr<Work> w;

  scenopt_dev();
  ~scenopt_dev();
  void init_solver_buffers();

  // sweep with optional host I/O (flags & SCENOPT_HOST_IO)
  void sweep(int nrhs, bool affine, const double* const* y, double* const* x, double* const* u,
             double* const* Hx, int flags, bool sync);
  // helpers for host/device I/O of dual and primal vectors
  const double* in_dual(const double* src, int flags, int slot);
  void out_copy(double* dst, const double* dev_src, size_t count, int flags);
  void sync();
  static double* mapped(double* p);  // device address of a pinned host buffer, or nullptr
};
