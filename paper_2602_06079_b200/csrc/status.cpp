#include "status.hpp"

#include <cstdlib>
#include <map>
#include <mutex>
#include <set>
#include <utility>

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

cudaError_t set_max_dynamic_smem(const void* kernel, int bytes) {
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;
  int dev = 0;
  if (cudaError_t e = cudaGetDevice(&dev); e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  if (done.count({kernel, dev}) != 0) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.insert({kernel, dev});
  return e;
}

int device_sm_count() {
  static std::mutex mu;
  static std::map<int, int> counts;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  auto it = counts.find(dev);
  if (it != counts.end()) return it->second;
  int n = 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
  counts[dev] = n;
  return n;
}

}  // namespace osh

extern "C" const char* osh_last_error(void) { return osh::g_last_error.c_str(); }
extern "C" int osh_abi_version(void) { return OSH_ABI_VERSION; }
