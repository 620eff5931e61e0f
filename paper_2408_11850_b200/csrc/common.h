// Shared host-side helpers for libpearl_b200: error reporting and launch checks.
#pragma once

#include <cuda_runtime.h>

#include <cstdio>
#include <string>

#include "../../include/pearl_b200.h"

namespace pearl {

void set_error(const std::string& msg);
// Every kernel launch issued by the library bumps this counter (read with
// pearl_launch_count); during graph capture it counts captured nodes.
void count_launch(int n = 1);
// Programmatic dependent launch on/off (env PEARL_PDL=0 disables; diagnostics).
bool pdl_enabled();

#define PEARL_CUDA_TRY(expr)                                                              \
  do {                                                                                    \
    cudaError_t _e = (expr);                                                              \
    if (_e != cudaSuccess) {                                                              \
      ::pearl::set_error(std::string(#expr) + ": " + cudaGetErrorString(_e) + " @" +     \
                         __FILE__ + ":" + std::to_string(__LINE__));                      \
      return PEARL_ERR_CUDA;                                                              \
    }                                                                                     \
  } while (0)

#define PEARL_ARG_CHECK(cond, msg)          \
  do {                                      \
    if (!(cond)) {                          \
      ::pearl::set_error(std::string(msg)); \
      return PEARL_ERR_ARG;                 \
    }                                       \
  } while (0)

// Diagnostic builds only (-DPEARL_TIMELINE, tools/timeline.py): per-CTA
// globaltimer stamps of every GEMM / attention launch, kTlSlots u64 per CTA.
#ifdef PEARL_TIMELINE
constexpr int kTlSlots = 16;
constexpr int kTlCtas = 160;
struct Timeline {
  unsigned long long* buf = nullptr;  // [max_launches][kTlCtas][kTlSlots]
  int max_launches = 0;
  int seq = 0;                        // next launch index (host)
};
Timeline& timeline();
// device-side stamp target of one launch (nullptr when disabled / full)
inline unsigned long long* timeline_next(int kind) {
  Timeline& t = timeline();
  if (!t.buf || t.seq >= t.max_launches) return nullptr;
  unsigned long long* p = t.buf + static_cast<size_t>(t.seq++) * kTlCtas * kTlSlots;
  (void)kind;
  return p;
}
#endif

// Pairwise-sum plan for a vocabulary size (plan.cpp).
struct VocabPlan {
  int V = 0;
  int C = 1;        // CTAs per row (thread-block cluster size)
  int cap = 0;      // largest per-CTA slice length
  int* d_plan = nullptr;  // C * kPlanStride ints on device
};

// Returns nullptr (and sets the error) if V was never prepared.
const VocabPlan* get_plan(int V);
int prepare_plan(int V);

}  // namespace pearl
