// SPDX-License-Identifier: MIT
#include "capi_internal.hpp"
struct scenopt_dev::Work {};
void scenopt_dev::init_solver_buffers() {}
scenopt_dev::scenopt_dev() = default;
scenopt_dev::~scenopt_dev() = default;
