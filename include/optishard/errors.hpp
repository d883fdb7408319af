// optishard (B200 build) — integer cost type and the error taxonomy.
//
// Drop-in for the reference's proj/include/optishard/common.hpp:12-60: the
// same seven exception classes, so callers' catch clauses keep working. The
// C ABI (include/osh.h) maps each class to an osh_status code and back.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>

namespace optishard {

// Planning costs are exact integers (elements, bytes, polynomial flops).
using Cost = std::uint64_t;

#define OPTISHARD_DECLARE_ERROR(Name)                                  \
  class Name : public std::runtime_error {                             \
   public:                                                             \
    explicit Name(const std::string& msg) : std::runtime_error(msg) {} \
  }

OPTISHARD_DECLARE_ERROR(ConfigError);         // bad model / run configuration
OPTISHARD_DECLARE_ERROR(LayoutError);         // bucket packing impossible
OPTISHARD_DECLARE_ERROR(ShardError);          // tensor-parallel split impossible
OPTISHARD_DECLARE_ERROR(UnsupportedError);    // operation not defined for the input
OPTISHARD_DECLARE_ERROR(PlanError);           // malformed or mismatched plan
OPTISHARD_DECLARE_ERROR(UnschedulableError);  // capacity cannot be met
OPTISHARD_DECLARE_ERROR(FormatError);         // plan / config text malformed

#undef OPTISHARD_DECLARE_ERROR

}  // namespace optishard
