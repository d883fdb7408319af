#include "status.hpp"

#include <cstdlib>

namespace osh {
namespace {
thread_local std::string g_last_error;
}

void set_error(const std::string& msg) { g_last_error = msg; }

osh_status fail(osh_status code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

bool debug_poison() {
  static const bool on = [] {
    const char* v = std::getenv("OSH_DEBUG_POISON");
    return v != nullptr && v[0] != '\0' && v[0] != '0';
  }();
  return on;
}

cudaError_t dev_alloc(void** p, size_t bytes) {
  cudaError_t e = cudaMalloc(p, bytes);
  if (e == cudaSuccess && debug_poison()) {
    e = cudaMemset(*p, 0xFF, bytes);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
  }
  return e;
}

}  // namespace osh

extern "C" const char* osh_last_error(void) { return osh::g_last_error.c_str(); }
extern "C" int osh_abi_version(void) { return OSH_ABI_VERSION; }
