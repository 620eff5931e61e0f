// Library identity and error reporting for the C ABI (include/pearl_b200.h).
#include <string>

#include "common.h"

namespace pearl {
thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }
}  // namespace pearl

extern "C" int pearl_version(void) { return 1; }

extern "C" const char* pearl_last_error(void) { return pearl::g_last_error.c_str(); }
