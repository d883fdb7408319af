// optishard (B200 build) — umbrella header, drop-in for the reference's
// proj/include/optishard/optishard.hpp. The planner half is header-only host
// C++ (bit-exact with the reference); the optimizer half (muon.hpp) runs on
// sm_100a through the C ABI of include/osh.h (libosh.so).
#pragma once

#define OPTISHARD_VERSION_MAJOR 0
#define OPTISHARD_VERSION_MINOR 1
#define OPTISHARD_VERSION_PATCH 0
#define OPTISHARD_B200 1

#include "optishard/balance.hpp"
#include "optishard/costing.hpp"
#include "optishard/errors.hpp"
#include "optishard/microgroup.hpp"
#include "optishard/model.hpp"
#include "optishard/partition.hpp"
#include "optishard/planfile.hpp"
#include "optishard/runconfig.hpp"
