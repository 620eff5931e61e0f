// K3: tcgen05 + TMA small-M contraction for the target's window forward.
// (Declarations; the implementation lives in gemm_tc.cu.)
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "common.h"

namespace pearl {

struct EpiArgs;

struct TcGemmCtx {
  void* splitk_ws = nullptr;   // fp32 split-K partial tiles
  int* tile_flags = nullptr;   // arrival counters (self-resetting)
  size_t ws_bytes = 0;
  int max_tokens = 0;
};

int tc_init(TcGemmCtx& ctx, const pearl_llama_config& cfg);
void tc_free(TcGemmCtx& ctx);
int tc_gemm(TcGemmCtx& ctx, const __nv_bfloat16* W, const __nv_bfloat16* X, int M, int N, int K,
            const EpiArgs& e, cudaStream_t st);

}  // namespace pearl
