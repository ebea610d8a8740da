// C-ABI: thread-local error channel and version.
#include <string>

#include "capi_common.hpp"
#include "foundry_b200.h"

namespace foundry {
namespace {
thread_local std::string g_last_error;
}
void fdy_set_last_error(const std::string& msg) { g_last_error = msg; }
}  // namespace foundry

extern "C" const char* fdy_last_error(void) { return foundry::g_last_error.c_str(); }

extern "C" const char* fdy_version(void) { return "foundry-b200 0.1.0 (sm_100a)"; }
