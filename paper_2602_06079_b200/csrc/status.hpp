// Thread-local error channel behind osh_last_error() and the helpers that
// turn CUDA / NCCL / C++ failures into osh_status codes at the C ABI.
#pragma once

#include <string>

#include <cuda_runtime.h>

#include "osh.h"

namespace osh {

void set_error(const std::string& msg);
osh_status fail(osh_status code, const std::string& msg);

// cudaMalloc that, when OSH_DEBUG_POISON is set in the environment, fills the
// new buffer with 0xFF bytes (NaN in bf16/fp32/fp64) so reads-before-writes
// show up; the explicit zeroing of buffers that must start at 0 is kept.
cudaError_t dev_alloc(void** p, size_t bytes);
bool debug_poison();

// cudaFuncAttributeMaxDynamicSharedMemorySize of `kernel` on the CURRENT
// device, set once per (kernel, device); thread-safe (contexts on several GPUs
// may share one process).
cudaError_t set_max_dynamic_smem(const void* kernel, int bytes);
// Multiprocessor count of the current device (cached per device).
int device_sm_count();

}  // namespace osh

#define OSH_CUDA_TRY(expr)                                                          \
  do {                                                                              \
    cudaError_t e_ = (expr);                                                        \
    if (e_ != cudaSuccess)                                                          \
      return ::osh::fail(e_ == cudaErrorMemoryAllocation ? OSH_ERR_OOM : OSH_ERR_CUDA, \
                         std::string(#expr) + ": " + cudaGetErrorString(e_));       \
  } while (0)
