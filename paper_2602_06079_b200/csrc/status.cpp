#include "status.hpp"

namespace osh {
namespace {
thread_local std::string g_last_error;
}

void set_error(const std::string& msg) { g_last_error = msg; }

osh_status fail(osh_status code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

}  // namespace osh

extern "C" const char* osh_last_error(void) { return osh::g_last_error.c_str(); }
extern "C" int osh_abi_version(void) { return OSH_ABI_VERSION; }
