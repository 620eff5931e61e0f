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

#ifdef PEARL_TIMELINE
// Diagnostic builds: per-CTA globaltimer stamps of GEMM / attention launches.
namespace pearl {
Timeline& timeline() {
  static Timeline t;
  return t;
}
}  // namespace pearl

extern "C" int pearl_tl_enable(int max_launches) {
  pearl::Timeline& t = pearl::timeline();
  if (t.buf) cudaFree(t.buf);
  t.buf = nullptr;
  t.seq = 0;
  t.max_launches = max_launches;
  if (max_launches <= 0) return PEARL_OK;
  const size_t n = static_cast<size_t>(max_launches) * pearl::kTlCtas * pearl::kTlSlots;
  PEARL_CUDA_TRY(cudaMalloc(&t.buf, n * sizeof(unsigned long long)));
  PEARL_CUDA_TRY(cudaMemset(t.buf, 0, n * sizeof(unsigned long long)));
  return PEARL_OK;
}

// copies the stamps of the launches so far; returns their count
extern "C" int pearl_tl_read(unsigned long long* dst, int max_launches) {
  pearl::Timeline& t = pearl::timeline();
  const int n = t.seq < max_launches ? t.seq : max_launches;
  if (!t.buf || n <= 0) return 0;
  if (cudaMemcpy(dst, t.buf, static_cast<size_t>(n) * pearl::kTlCtas * pearl::kTlSlots * 8, cudaMemcpyDeviceToHost))
    return -1;
  return n;
}
#endif
