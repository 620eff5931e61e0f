// K3: tcgen05 + TMA small-M contraction for the target's window forward.
//
// Y[t, n] = sum_k W[n, k] X[t, k] with W bf16 [N, K] (K-major) streamed by
// TMA in 128 x 64 tiles (SWIZZLE_128B) and the window's tokens X bf16
// [M <= 64, K] as up to four 16-token tiles.  Swap-AB: weight rows sit on
// MMA-M = 128, tokens on MMA-N = 16, accumulators in TMEM.  Split-K over a
// fixed number of CTAs per row tile (a function of (N, K) only) with the
// last-arriving CTA summing the fp32 partials in split order, so results
// are bitwise independent of M (batch invariance).
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <map>
#include <tuple>

#include "common.h"

namespace pearl {

struct EpiArgs;

struct TcWeightMap {
  alignas(64) CUtensorMap map;
};

struct TcGemmCtx {
  float* partials = nullptr;   // fp32 split-K partial tiles
  int* tile_flags = nullptr;   // arrival counters (self-resetting)
  size_t partial_floats = 0;
  int n_flags = 0;
  int max_tokens = 0;
  int num_sms = 148;
  int min_plan_splits = 1;  // workspace sized for at least this many splits (microbenchmarks)
  // per weight matrix, keyed by (address, N, K): a map encodes the shape too
  std::map<std::tuple<const void*, int, int>, TcWeightMap> wmaps;
};

int tc_init(TcGemmCtx& ctx, const pearl_llama_config& cfg);
void tc_free(TcGemmCtx& ctx);
int tc_gemm(TcGemmCtx& ctx, const __nv_bfloat16* W, const __nv_bfloat16* X, int M, int N, int K,
            const EpiArgs& e, cudaStream_t st, int force_grid = 0, bool w_tiled = false);
// number of K splits the (legacy round-robin) planner picks for an (N, K) GEMM
int tc_splits(int N, int K, int num_sms);
// most stream-K segments any tile of an (tiles x KB) GEMM is cut into over G CTAs
int tc_seg_max(int tiles, int KB, int G);
// bf16 [rows, inner] row-major tensor map, box kTileK x box_rows, 128B swizzle
int tc_encode_2d(CUtensorMap* map, const void* base, int inner, int rows, int box_rows);

}  // namespace pearl
