// C-ABI plumbing shared by every entry point: thread-local last error, version.
#include <string>

#include "common.hpp"

namespace ps {
namespace {
thread_local std::string g_last_error;
}
void set_last_error(const std::string& msg) { g_last_error = msg; }
}  // namespace ps

extern "C" {
const char* ps_last_error(void) { return ps::g_last_error.c_str(); }
const char* ps_version(void) { return "prescope-b200 0.1 (sm_100a)"; }
}
