// Library identity and error reporting for the C ABI (include/pearl_b200.h).
#include <atomic>
#include <cstdlib>
#include <string>

#include "common.h"

namespace pearl {
thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }
static std::atomic<unsigned long long> g_launches{0};
bool pdl_enabled() {
  static const bool on = [] {
    const char* v = std::getenv("PEARL_PDL");
    return !(v && v[0] == '0');
  }();
  return on;
}
void count_launch(int n) { g_launches.fetch_add(static_cast<unsigned long long>(n), std::memory_order_relaxed); }
}  // namespace pearl

extern "C" int pearl_version(void) { return 1; }

extern "C" const char* pearl_last_error(void) { return pearl::g_last_error.c_str(); }

extern "C" unsigned long long pearl_launch_count(void) { return pearl::g_launches.load(); }
