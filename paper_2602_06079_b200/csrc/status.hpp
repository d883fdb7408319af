// Thread-local error channel behind osh_last_error() and the helpers that
// turn CUDA / NCCL / C++ failures into osh_status codes at the C ABI.
#pragma once

#include <string>

#include "osh.h"

namespace osh {

void set_error(const std::string& msg);
osh_status fail(osh_status code, const std::string& msg);

}  // namespace osh

#define OSH_CUDA_TRY(expr)                                                          \
  do {                                                                              \
    cudaError_t e_ = (expr);                                                        \
    if (e_ != cudaSuccess)                                                          \
      return ::osh::fail(e_ == cudaErrorMemoryAllocation ? OSH_ERR_OOM : OSH_ERR_CUDA, \
                         std::string(#expr) + ": " + cudaGetErrorString(e_));       \
  } while (0)
