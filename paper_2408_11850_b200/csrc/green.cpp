// SM partitions for concurrently running models (green contexts).
//
// PEARL runs the draft and the target at the same time.  Sharing every SM,
// the draft's short latency-bound kernels interleave with the target's
// persistent stream-K GEMM grid and delay it (a late CTA holds up every
// tile it contributes to).  A green context gives each model its own SMs:
// the draft gets a small partition, the target the rest, and the target's
// stream-K grid is sized to its partition (pearl_llama_config.sm_count), so
// both streams run undisturbed.  Driver entry points are resolved at run
// time (no libcuda link dependency).
#include <cuda.h>
#include <cuda_runtime.h>

#include <mutex>
#include <string>

#include "common.h"

namespace pearl {
namespace {

template <class F>
F driver_fn(const char* name) {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &fn, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
    return nullptr;
  return reinterpret_cast<F>(fn);
}

struct Partition {
  int want = -1;
  CUstream first = nullptr, rest = nullptr;
  int first_sms = 0, rest_sms = 0;
};
std::mutex g_mu;
Partition g_part;

#define PEARL_CU_TRY(call, what)                                                  \
  do {                                                                            \
    CUresult r_ = (call);                                                         \
    if (r_ != CUDA_SUCCESS) {                                                     \
      set_error(std::string(what) + " failed: CUresult " + std::to_string(r_));  \
      return PEARL_ERR_CUDA;                                                      \
    }                                                                             \
  } while (0)

}  // namespace
}  // namespace pearl

using namespace pearl;

extern "C" int pearl_green_streams(int first_sms, void** first_stream, void** rest_stream, int* first_count,
                                   int* rest_count) {
  PEARL_ARG_CHECK(first_sms > 0 && first_stream && rest_stream, "bad green-stream arguments");
  std::lock_guard<std::mutex> lk(g_mu);
  if (g_part.want != first_sms) {
    PEARL_ARG_CHECK(g_part.want < 0, "SM partition already created with a different size");
    auto getres = driver_fn<decltype(&cuDeviceGetDevResource)>("cuDeviceGetDevResource");
    auto split = driver_fn<decltype(&cuDevSmResourceSplitByCount)>("cuDevSmResourceSplitByCount");
    auto gendesc = driver_fn<decltype(&cuDevResourceGenerateDesc)>("cuDevResourceGenerateDesc");
    auto gcreate = driver_fn<decltype(&cuGreenCtxCreate)>("cuGreenCtxCreate");
    auto gstream = driver_fn<decltype(&cuGreenCtxStreamCreate)>("cuGreenCtxStreamCreate");
    if (!getres || !split || !gendesc || !gcreate || !gstream) {
      set_error("green contexts unavailable in this driver");
      return PEARL_ERR_CUDA;
    }
    int dev = 0;
    PEARL_CUDA_TRY(cudaGetDevice(&dev));
    PEARL_CUDA_TRY(cudaFree(nullptr));  // primary context exists
    CUdevResource all{}, part{}, rest{};
    PEARL_CU_TRY(getres(static_cast<CUdevice>(dev), &all, CU_DEV_RESOURCE_TYPE_SM), "cuDeviceGetDevResource");
    unsigned int n = 1;
    PEARL_CU_TRY(split(&part, &n, &all, &rest, 0, static_cast<unsigned>(first_sms)), "cuDevSmResourceSplitByCount");
    PEARL_ARG_CHECK(n == 1 && rest.sm.smCount > 0, "SM split left no SMs");
    CUstream streams[2];
    CUdevResource* rs[2] = {&part, &rest};
    for (int i = 0; i < 2; ++i) {
      CUdevResourceDesc desc;
      PEARL_CU_TRY(gendesc(&desc, rs[i], 1), "cuDevResourceGenerateDesc");
      CUgreenCtx g;
      PEARL_CU_TRY(gcreate(&g, desc, static_cast<CUdevice>(dev), CU_GREEN_CTX_DEFAULT_STREAM), "cuGreenCtxCreate");
      PEARL_CU_TRY(gstream(&streams[i], g, CU_STREAM_NON_BLOCKING, 0), "cuGreenCtxStreamCreate");
    }
    g_part.want = first_sms;
    g_part.first = streams[0];
    g_part.rest = streams[1];
    g_part.first_sms = static_cast<int>(part.sm.smCount);
    g_part.rest_sms = static_cast<int>(rest.sm.smCount);
  }
  *first_stream = g_part.first;
  *rest_stream = g_part.rest;
  if (first_count) *first_count = g_part.first_sms;
  if (rest_count) *rest_count = g_part.rest_sms;
  return PEARL_OK;
}
