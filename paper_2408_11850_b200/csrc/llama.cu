// Llama decoder runtime for GPU SequenceModels (draft and target).
//
// Replaces SequenceModel.next_dist (pearl_lab/models.py:58-71) for the
// transformer models the B200 build serves: the draft's per-token forward
// inside _draft_block (engines.py:277-282) and the target's window forward
// (engines.py:302, 373, 425, 492).  A forward processes n tokens at device
// positions *pos..*pos+n-1 against the per-layer KV cache.
//
// Layer = RMSNorm -> QKV GEMM (+RoPE, +K/V append) -> causal attention over
// the cache (K4, attention.cu) -> O GEMM (+residual) -> RMSNorm -> gate/up
// GEMM (+SwiGLU) -> down GEMM (+residual).  The residual stream is fp32;
// GEMM operands bf16.
//
// RMSNorm has no kernel of its own:
//  * tcgen05 models (K3) fold it into the GEMMs.  The producer of the
//    residual (embedding, O and down epilogues) also writes the next GEMM's
//    operand x = bf16(h * gain) and per-128-row-tile sums of h^2; the
//    consumer (QKV / gate-up / lm_head) scales its fp32 outputs by
//    rs = 1/sqrt(mean(h^2) + eps) in its epilogue:
//        y = rs * (W . bf16(h * g))        (== W . (h * rs * g) up to rounding)
//  * CUDA-core models (K2) fuse it into the consuming GEMV's operand load:
//        y = W . bf16(h * rs * g).
// Every kernel is launched with programmatic dependent launch (PDL): it may
// start while its predecessor drains and calls griddepcontrol.wait before
// touching the predecessor's outputs (the tcgen05 GEMM prefetches weights
// before that wait).
//
// Batch invariance: every per-token value is computed by the same sequence
// of fp32 operations whatever the number of tokens in the launch (fixed
// K-order FMA chains, fixed reduction trees, attention over fixed position
// segments folded in a fixed order), so a position's logits are bitwise the
// same in an M=1 AR step, an M=gamma PEARL window or an M=gamma+1 SD window
// -- which makes GPU greedy PEARL/SD token-identical to AR.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "attention.cuh"
#include "common.h"
#include "epilogue.cuh"
#include "gemm_tc.cuh"
#include "tc_common.cuh"

namespace pearl {

struct LayerW {
  const float* attn_norm;
  const bf16* wqkv;
  const bf16* wo;
  const float* mlp_norm;
  const bf16* wgu;
  const bf16* wdown;
};


struct L2Window {
  const void* base = nullptr;
  size_t bytes = 0;
  float hit_ratio = 0.f;
};

struct Llama {
  pearl_llama_config cfg;
  const bf16* embed;
  const float* final_norm;
  const bf16* lm_head;
  const float* rope_cos;
  const float* rope_sin;
  bf16* kcache;
  bf16* vcache;
  std::vector<LayerW> layers;
  L2Window l2win;         // optional persisting-L2 window over the streamed weights
  // workspace
  float* h = nullptr;     // [T, d]
  bf16* x = nullptr;      // [T, max(d, ffn, H hd)]
  bf16* q = nullptr;      // [T, H hd]
  bf16* o = nullptr;      // [T, H hd]
  bf16* act = nullptr;    // [T, ffn]
  float* ss = nullptr;    // [ceil(d / 128), T] per-tile sums of h^2 (folded RMSNorm)
  int num_sms = 148;
  TcGemmCtx tc;           // tcgen05 path state (split-K scratch, descriptors)
};

// Optional per-op timing of an eager forward (pearl_llama_profile): an event
// is recorded after every launch; deltas are attributed to the op label.
struct OpProfiler {
  bool on = false;
  std::vector<std::pair<int, cudaEvent_t>> marks;
  cudaEvent_t start = nullptr;
  void mark(int op, cudaStream_t st) {
    if (!on) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, st);
    marks.emplace_back(op, e);
  }
};
OpProfiler g_prof;
enum ProfOp { OP_EMBED = 0, OP_NORM, OP_QKV, OP_ATTN, OP_O, OP_GU, OP_DOWN, OP_HEAD, OP_OTHER, OP_COUNT };

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// L2 access-policy window attached to every launch of the model currently
// running a forward (pearl_llama_set_l2_window): its streamed weights are
// kept L2-resident (persisting lines), so a draft's per-token weight reads
// are served from L2 instead of competing with the target for HBM.
L2Window g_l2win;  // set for the duration of pearl_llama_forward

template <typename... KArgs, typename... Args>
int launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  int na = 0;
  if (pdl_enabled()) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (g_l2win.bytes > 0) {
    at[na].id = cudaLaunchAttributeAccessPolicyWindow;
    at[na].val.accessPolicyWindow.base_ptr = const_cast<void*>(g_l2win.base);
    at[na].val.accessPolicyWindow.num_bytes = g_l2win.bytes;
    at[na].val.accessPolicyWindow.hitRatio = g_l2win.hit_ratio;
    at[na].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    at[na].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    ++na;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  PEARL_CUDA_TRY(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
  count_launch();
  return PEARL_OK;
}

// ---------------------------------------------------------------------------
// small kernels
// ---------------------------------------------------------------------------
// h[t] = embed[token t] (fp32).  Folded-norm models (nx != nullptr) also get
// the first QKV GEMM's operand x[t] = bf16(h[t] * g) and the per-tile sums of
// h^2 (warp w: 128-row tiles w, w + 4, ...; the same tile_sumsq order as the
// residual epilogue).
constexpr int kEmbedThreads = 128;
__global__ void __launch_bounds__(kEmbedThreads) embed_kernel(const int32_t* __restrict__ tokens,
                                                              const bf16* __restrict__ emb, float* __restrict__ h,
                                                              int d, int V, const float* __restrict__ g,
                                                              bf16* __restrict__ nx, float* __restrict__ ss, int ss_ld) {
  pdl_wait();
  pdl_trigger();
  const int t = blockIdx.x;
  int tok = tokens[t];
  tok = tok < 0 ? 0 : (tok >= V ? V - 1 : tok);
  const bf16* row = emb + static_cast<size_t>(tok) * d;
  float* hr = h + static_cast<size_t>(t) * d;
  if (nx == nullptr) {
    for (int i = threadIdx.x; i < d; i += blockDim.x) hr[i] = __bfloat162float(row[i]);
    return;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tiles = (d + 127) / 128;
  for (int k = warp; k < tiles; k += kEmbedThreads / 32) {
    const int n0 = k * 128 + lane * 4;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (n0 < d) {  // d % 8 == 0
      const uint2 u = *reinterpret_cast<const uint2*>(row + n0);
      v = make_float4(__uint_as_float(u.x << 16), __uint_as_float(u.x & 0xffff0000u), __uint_as_float(u.y << 16),
                      __uint_as_float(u.y & 0xffff0000u));
      *reinterpret_cast<float4*>(hr + n0) = v;
      const float4 gg = *reinterpret_cast<const float4*>(g + n0);
      const __nv_bfloat162 lo = __floats2bfloat162_rn(v.x * gg.x, v.y * gg.y);
      const __nv_bfloat162 hi = __floats2bfloat162_rn(v.z * gg.z, v.w * gg.w);
      *reinterpret_cast<uint2*>(nx + static_cast<size_t>(t) * d + n0) =
          make_uint2(*reinterpret_cast<const uint32_t*>(&lo), *reinterpret_cast<const uint32_t*>(&hi));
    }
    const float sq = tile_sumsq(v);
    if (lane == 0) ss[static_cast<size_t>(k) * ss_ld + t] = sq;
  }
}

__global__ void advance_kernel(int32_t* pos, int n) {
  pdl_wait();
  *pos += n;
}

// ---------------------------------------------------------------------------
// K2: batch-invariant CUDA-core GEMV / skinny GEMM
//   Y[t, n] = sum_k W[n, k] X[t, k]; W bf16 [N, K] row-major, X bf16 [M, K]
// Each warp owns 4 consecutive rows; lane l streams 16-byte (8 x bf16)
// chunks k = 256 c + 8 l with 128-bit non-allocating loads, FMA-accumulates
// per (row, token) in fp32, then a fixed xor-shuffle tree reduces the lanes.
// ---------------------------------------------------------------------------
constexpr int kGemvRows = 4;
constexpr int kGemvWarps = 8;

__device__ __forceinline__ uint4 ld_nc_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ void bf16x8_to_f32(const uint4& u, float* f) {
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    f[2 * i] = __uint_as_float(w[i] << 16);
    f[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
  }
}

// Optional fused RMSNorm of the input: when xh != nullptr the operand is
// x[t] = bf16(xh[t] * rs[t] * ng), rs[t] = 1/sqrt(mean(xh[t]^2) + eps), with
// rs computed by every block in the same fixed order (warp t%8 strides the
// row with float4 loads, xor tree) -- identical in every block and for any M.
struct GemvNorm {
  const float* xh;  // [M, K] fp32 residual stream, or nullptr (X is bf16 input)
  const float* g;   // [K] gain
  float eps;
  // gemv1_kernel only (single token, layer 0 of a CUDA-core model): the row
  // is the embedding of *tok (bf16 -> fp32 is exact, so rs and the operand are
  // bitwise those of the embed kernel's h), and block 0 also writes it to
  // h_out -- the embedding kernel folded into the first QKV GEMV.
  const bf16* emb = nullptr;
  const int32_t* tok = nullptr;
  int V = 0;
  float* h_out = nullptr;
};

constexpr int kGemvMaxNormTok = 64;

// TOK: tokens accumulated per pass (1 for single-token decode: fewer live
// registers, more loads in flight; 8 otherwise).  RPW: weight rows per warp --
// 4 for wide layers, 1 for narrow ones (N < ~9.5k: the draft's o / down /
// qkv / gate_up), which gives 4x the warps so the per-SM load queue stays
// full; the 4 rows an epilogue needs (SwiGLU / RoPE pairs) are then gathered
// from 4 warps through shared memory.  Per-row arithmetic (chunk order, FMA
// order, xor tree) is identical for every TOK and RPW (batch invariance).
// The block-level body: block `bid` of a GEMV grid.  Needs 8 warps; s_rs /
// s_out are the block's smem.
// Barrier of a GEMV block's 256 threads: the whole CTA (bar = 0) or named
// barrier `bar` of one 256-thread group of a larger CTA.
__device__ __forceinline__ void grp_sync(int bar) {
  if (bar == 0) __syncthreads();
  else asm volatile("bar.sync %0, 256;" ::"r"(bar) : "memory");
}

// 16-byte load through L2 (no non-coherent path), for an X written earlier
// in the same kernel (COH = true), which must not be read with ld.global.nc.
__device__ __forceinline__ uint4 ld_cg_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

template <int TOK, int RPW, bool COH = false>
__device__ __forceinline__ void gemv_block(const bf16* __restrict__ W, const bf16* __restrict__ X, int M, int N, int K,
                                           const EpiArgs& e, const GemvNorm& nrm, int bid, float* s_rs, float* s_out,
                                           int tid = threadIdx.x, int bar = 0) {
  const int warp = tid >> 5, lane = tid & 31;
  if (nrm.xh != nullptr) {
    for (int t = warp; t < M; t += kGemvWarps) {
      const float4* hr = reinterpret_cast<const float4*>(nrm.xh + static_cast<size_t>(t) * K);
      float ss = 0.f;
      // 8 float4 loads in flight per lane, then summed in j order
      for (int j0 = lane; j0 < K / 4; j0 += 32 * 8) {
        float4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int j = j0 + 32 * u;
          v[u] = j < K / 4 ? hr[j] : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (j0 + 32 * u < K / 4) {
            ss = fmaf(v[u].x, v[u].x, ss);
            ss = fmaf(v[u].y, v[u].y, ss);
            ss = fmaf(v[u].z, v[u].z, ss);
            ss = fmaf(v[u].w, v[u].w, ss);
          }
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
      if (lane == 0) s_rs[t] = 1.0f / sqrtf(ss / static_cast<float>(K) + nrm.eps);
    }
    grp_sync(bar);
  }
  const int n0 = (bid * kGemvWarps + warp) * RPW;
  const bool active = n0 < N;
  if (RPW > 1 && !active) return;
  const int nchunk = (K + 255) / 256;
  for (int t0 = 0; t0 < M; t0 += TOK) {
    const int mt = min(TOK, M - t0);
    float acc[RPW][TOK];
#pragma unroll
    for (int r = 0; r < RPW; ++r)
#pragma unroll
      for (int t = 0; t < TOK; ++t) acc[r][t] = 0.f;
#pragma unroll(TOK == 1 ? (RPW == 1 ? 8 : 4) : 2)
    for (int c = 0; c < nchunk; ++c) {
      const int k = c * 256 + lane * 8;
      if (active && k < K) {
        float w[RPW][8];
#pragma unroll
        for (int r = 0; r < RPW; ++r) {
          const int n = min(n0 + r, N - 1);
          bf16x8_to_f32(ld_nc_v4(W + static_cast<size_t>(n) * K + k), w[r]);
        }
        float gk[8];
        if (nrm.xh != nullptr) {
          const float4 g0 = *reinterpret_cast<const float4*>(nrm.g + k);
          const float4 g1 = *reinterpret_cast<const float4*>(nrm.g + k + 4);
          gk[0] = g0.x; gk[1] = g0.y; gk[2] = g0.z; gk[3] = g0.w;
          gk[4] = g1.x; gk[5] = g1.y; gk[6] = g1.z; gk[7] = g1.w;
        }
#pragma unroll
        for (int t = 0; t < TOK; ++t) {
          if (t < mt) {
            float xv[8];
            if (nrm.xh != nullptr) {
              const float* hr = nrm.xh + static_cast<size_t>(t0 + t) * K + k;
              const float4 h0 = *reinterpret_cast<const float4*>(hr);
              const float4 h1 = *reinterpret_cast<const float4*>(hr + 4);
              const float hv[8] = {h0.x, h0.y, h0.z, h0.w, h1.x, h1.y, h1.z, h1.w};
              const float rs = s_rs[t0 + t];
#pragma unroll
              for (int j = 0; j < 8; ++j) xv[j] = __bfloat162float(__float2bfloat16(hv[j] * rs * gk[j]));
            } else {
              const bf16* xp = X + static_cast<size_t>(t0 + t) * K + k;
              bf16x8_to_f32(COH ? ld_cg_v4(xp) : __ldg(reinterpret_cast<const uint4*>(xp)), xv);
            }
#pragma unroll
            for (int r = 0; r < RPW; ++r)
#pragma unroll
              for (int j = 0; j < 8; ++j) acc[r][t] = fmaf(w[r][j], xv[j], acc[r][t]);
          }
        }
      }
    }
#pragma unroll
    for (int r = 0; r < RPW; ++r)
#pragma unroll
      for (int t = 0; t < TOK; ++t)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc[r][t] += __shfl_xor_sync(0xffffffffu, acc[r][t], o);
    if (RPW == 4) {
      if (lane == 0) {
        for (int t = 0; t < mt; ++t) {
          float v[4] = {acc[0][t], acc[1 % RPW][t], acc[2 % RPW][t], acc[3 % RPW][t]};
          epilogue4(e, t0 + t, n0, v, N);
        }
      }
    } else {
      // gather rows 4g..4g+3 (warps 4g'..4g'+3 of this block) for the epilogue
      if (lane == 0)
        for (int t = 0; t < TOK; ++t) s_out[warp * TOK + t] = acc[0][t];
      grp_sync(bar);
      const int grp = tid / TOK, t = tid % TOK;  // (row quad, token)
      const int nq = bid * kGemvWarps + 4 * grp;
      if (grp < kGemvWarps / 4 && t < mt && nq < N) {
        float v[4] = {s_out[(4 * grp) * TOK + t], s_out[(4 * grp + 1) * TOK + t], s_out[(4 * grp + 2) * TOK + t],
                      s_out[(4 * grp + 3) * TOK + t]};
        epilogue4(e, t0 + t, nq, v, N);
      }
      grp_sync(bar);
    }
  }
}

template <int TOK, int RPW>
__global__ void __launch_bounds__(kGemvWarps * 32) gemv_kernel(const bf16* __restrict__ W, const bf16* __restrict__ X,
                                                               int M, int N, int K, EpiArgs e, GemvNorm nrm) {
  __shared__ float s_rs[kGemvMaxNormTok];
  __shared__ float s_out[RPW == 1 ? kGemvWarps * TOK : 1];
  pdl_wait();
  pdl_trigger();
  if (e.adv_pos != nullptr && blockIdx.x == 0 && threadIdx.x == 0) *e.adv_pos += e.adv_n;
  gemv_block<TOK, RPW>(W, X, M, N, K, e, nrm, blockIdx.x, s_rs, s_out);
}

// Single-token K2 (M = 1, K <= kGemv1MaxK): gemv_block<1, RPW>'s per-row
// arithmetic exactly (chunk k = 256 c + 8 lane, FMA order, xor tree, operand
// rounding), restructured for memory-level parallelism.  gemv_block's chunk
// loop issues one chunk's loads, branches, and FMAs them before the next
// chunk's loads (one DRAM round trip per chunk: 12 for the 68M down
// projection); here a warp requests CB chunks of all its rows before using
// any -- the first batch BEFORE the PDL wait, since weights never depend on
// the previous kernel -- and the operand row (bf16 X, or the fused-norm
// bf16(h * rs * g)) is staged once per block in shared memory.
constexpr int kGemv1MaxK = 4096;

// Four consecutive row values as fp32: the fp32 residual row, or (bf16 row)
// the embedding row widened exactly.
__device__ __forceinline__ float4 row4(const float* xh, const bf16* eb, int j4) {
  if (eb == nullptr) return reinterpret_cast<const float4*>(xh)[j4];
  const uint2 u = *reinterpret_cast<const uint2*>(eb + 4 * j4);
  return make_float4(__uint_as_float(u.x << 16), __uint_as_float(u.x & 0xffff0000u), __uint_as_float(u.y << 16),
                     __uint_as_float(u.y & 0xffff0000u));
}

// rs = 1 / sqrt(mean(row^2) + eps) of one row, in gemv_block's order
// (lane l: float4 elements l + 32 u, 8 in flight per pass; xor tree)
__device__ __forceinline__ float gemv_row_rs(const float* xh, const bf16* eb, int K, float eps, int lane) {
  float ss = 0.f;
  for (int j0 = lane; j0 < K / 4; j0 += 32 * 8) {
    float4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int j = j0 + 32 * u;
      v[u] = j < K / 4 ? row4(xh, eb, j) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (j0 + 32 * u < K / 4) {
        ss = fmaf(v[u].x, v[u].x, ss);
        ss = fmaf(v[u].y, v[u].y, ss);
        ss = fmaf(v[u].z, v[u].z, ss);
        ss = fmaf(v[u].w, v[u].w, ss);
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  return 1.0f / sqrtf(ss / static_cast<float>(K) + eps);
}

// Single-token fused-norm GEMV with the RMS scale in registers (K = 128 NV:
// the 68M draft's QKV / gate-up, d = 768).  gemv1_kernel stages the operand
// through smem: warp 0 computes rs (one L2 round trip), block barrier, every
// thread builds bf16(h * rs * g) (a second round trip), block barrier.  Here
// every warp loads the whole row once in gemv_row_rs's own layout (lane l:
// float4 elements l + 32 u), computes rs itself in that order, and gathers the
// h values of its lanes' chunks with shuffles -- one round trip after the PDL
// wait and no block barrier; g is staged in smem before the wait.  4 rows per
// warp, every chunk of a row in flight at once.  Bitwise gemv_block's rows.
template <int NV, bool EMB>
__global__ void __launch_bounds__(kGemvWarps * 32, 2) gemv1n_kernel(const bf16* __restrict__ W, int N, EpiArgs e,
                                                                    GemvNorm nrm) {
  constexpr int K = 128 * NV;
  constexpr int NC = NV / 2;  // 256-element chunks
  __shared__ __align__(16) float s_g[K];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n0 = (blockIdx.x * kGemvWarps + warp) * 4;
  const bool active = n0 < N;
  uint4 wr[NC][4];
#pragma unroll
  for (int c = 0; c < NC; ++c)
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int n = min(n0 + r, N - 1);
      wr[c][r] = active ? ld_nc_v4(W + static_cast<size_t>(n) * K + c * 256 + lane * 8) : make_uint4(0, 0, 0, 0);
    }
  for (int k = tid * 4; k < K; k += kGemvWarps * 32 * 4)
    *reinterpret_cast<float4*>(s_g + k) = *reinterpret_cast<const float4*>(nrm.g + k);
  __syncthreads();
  pdl_wait();
  pdl_trigger();
  if (e.adv_pos != nullptr && blockIdx.x == 0 && tid == 0) *e.adv_pos += e.adv_n;
  const bf16* eb = nullptr;
  if (EMB) {
    int tok = *nrm.tok;
    tok = tok < 0 ? 0 : (tok >= nrm.V ? nrm.V - 1 : tok);
    eb = nrm.emb + static_cast<size_t>(tok) * K;
  }
  float4 v[NV];
#pragma unroll
  for (int u = 0; u < NV; ++u) v[u] = row4(nrm.xh, eb, lane + 32 * u);
  if (EMB && blockIdx.x == 0 && warp == 0)
#pragma unroll
    for (int u = 0; u < NV; ++u) *reinterpret_cast<float4*>(nrm.h_out + 4 * (lane + 32 * u)) = v[u];
  float ss = 0.f;  // gemv_row_rs: one pass of K / 4 <= 256 float4s, u order
#pragma unroll
  for (int u = 0; u < NV; ++u) {
    ss = fmaf(v[u].x, v[u].x, ss);
    ss = fmaf(v[u].y, v[u].y, ss);
    ss = fmaf(v[u].z, v[u].z, ss);
    ss = fmaf(v[u].w, v[u].w, ss);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  const float rs = 1.0f / sqrtf(ss / static_cast<float>(K) + nrm.eps);
  // chunk c of lane l covers float4 elements 64 c + 2 l and + 1: held by lanes
  // (2 l) % 32 and (2 l + 1) % 32 in slot 2 c + (l >= 16)
  const int srcA = (2 * lane) & 31, srcB = srcA + 1;
  const bool hi = lane >= 16;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    float hv[8];
    {
      const float4 p = v[2 * c], q = v[2 * c + 1];
      const float a0 = __shfl_sync(0xffffffffu, p.x, srcA), a1 = __shfl_sync(0xffffffffu, q.x, srcA);
      const float b0 = __shfl_sync(0xffffffffu, p.y, srcA), b1 = __shfl_sync(0xffffffffu, q.y, srcA);
      const float c0 = __shfl_sync(0xffffffffu, p.z, srcA), c1 = __shfl_sync(0xffffffffu, q.z, srcA);
      const float d0 = __shfl_sync(0xffffffffu, p.w, srcA), d1 = __shfl_sync(0xffffffffu, q.w, srcA);
      const float e0 = __shfl_sync(0xffffffffu, p.x, srcB), e1 = __shfl_sync(0xffffffffu, q.x, srcB);
      const float f0 = __shfl_sync(0xffffffffu, p.y, srcB), f1 = __shfl_sync(0xffffffffu, q.y, srcB);
      const float g0 = __shfl_sync(0xffffffffu, p.z, srcB), g1 = __shfl_sync(0xffffffffu, q.z, srcB);
      const float h0 = __shfl_sync(0xffffffffu, p.w, srcB), h1 = __shfl_sync(0xffffffffu, q.w, srcB);
      hv[0] = hi ? a1 : a0; hv[1] = hi ? b1 : b0; hv[2] = hi ? c1 : c0; hv[3] = hi ? d1 : d0;
      hv[4] = hi ? e1 : e0; hv[5] = hi ? f1 : f0; hv[6] = hi ? g1 : g0; hv[7] = hi ? h1 : h0;
    }
    const int k = c * 256 + lane * 8;
    const float4 g0 = *reinterpret_cast<const float4*>(s_g + k);
    const float4 g1 = *reinterpret_cast<const float4*>(s_g + k + 4);
    const float gk[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
    float xv[8];
#pragma unroll
    for (int j = 0; j < 8; j += 2) {
      const __nv_bfloat162 b2 = __floats2bfloat162_rn(hv[j] * rs * gk[j], hv[j + 1] * rs * gk[j + 1]);
      xv[j] = __low2float(b2);
      xv[j + 1] = __high2float(b2);
    }
    if (active) {
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        float w[8];
        bf16x8_to_f32(wr[c][r], w);
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[r] = fmaf(w[j], xv[j], acc[r]);
      }
    }
  }
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc[r] += __shfl_xor_sync(0xffffffffu, acc[r], o);
  if (active && lane == 0) epilogue4(e, 0, n0, acc, N);
}

// Single-token GEMV with a bf16 operand (no fused norm: the 68M o / down
// projections), one row per warp, all of a lane's CB weight AND operand chunks
// requested before any is used -- no smem staging, no block barrier before
// the FMAs.  Bitwise gemv_block's rows.
template <int CB>
__global__ void __launch_bounds__(kGemvWarps * 32, 2) gemv1x_kernel(const bf16* __restrict__ W,
                                                                   const bf16* __restrict__ X, int N, int K, EpiArgs e) {
  __shared__ float s_out[kGemvWarps];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n0 = blockIdx.x * kGemvWarps + warp;
  const bool active = n0 < N;
  uint4 wr[CB], xr[CB];
#pragma unroll
  for (int u = 0; u < CB; ++u) {
    const int k = u * 256 + lane * 8;
    wr[u] = (active && k < K) ? ld_nc_v4(W + static_cast<size_t>(n0) * K + k) : make_uint4(0, 0, 0, 0);
  }
  pdl_wait();
  pdl_trigger();
  if (e.adv_pos != nullptr && blockIdx.x == 0 && tid == 0) *e.adv_pos += e.adv_n;
#pragma unroll
  for (int u = 0; u < CB; ++u) {
    const int k = u * 256 + lane * 8;
    xr[u] = k < K ? __ldg(reinterpret_cast<const uint4*>(X + k)) : make_uint4(0, 0, 0, 0);
  }
  float acc = 0.f;
#pragma unroll
  for (int u = 0; u < CB; ++u) {
    const int k = u * 256 + lane * 8;
    if (active && k < K) {
      float xv[8], w[8];
      bf16x8_to_f32(xr[u], xv);
      bf16x8_to_f32(wr[u], w);
#pragma unroll
      for (int j = 0; j < 8; ++j) acc = fmaf(w[j], xv[j], acc);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) s_out[warp] = acc;
  __syncthreads();
  const int nq = blockIdx.x * kGemvWarps + 4 * tid;
  if (tid < kGemvWarps / 4 && nq < N) {
    float v[4] = {s_out[4 * tid], s_out[4 * tid + 1], s_out[4 * tid + 2], s_out[4 * tid + 3]};
    epilogue4(e, 0, nq, v, N);
  }
}

// residency: at least 6 blocks per SM for the short single-batch rows (the
// 68M draft's qkv / gate_up grids in one wave), 3 for 4-row warps, 2 for CB = 12
// and the embedding-fold variants (one launch per token: no spills)
template <int RPW, int CB, bool EMB>
constexpr int gemv1_min_blocks() { return (EMB || CB >= 12) ? 2 : (RPW == 4 ? 3 : 6); }

template <int RPW, int CB, bool EMB = false>
__global__ void __launch_bounds__(kGemvWarps * 32, gemv1_min_blocks<RPW, CB, EMB>()) gemv1_kernel(const bf16* __restrict__ W,
                                                                const bf16* __restrict__ X, int N, int K, EpiArgs e,
                                                                GemvNorm nrm) {
  __shared__ __align__(16) bf16 s_x[kGemv1MaxK];
  __shared__ float s_rs;
  __shared__ float s_out[RPW == 1 ? kGemvWarps : 1];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n0 = (blockIdx.x * kGemvWarps + warp) * RPW;
  const bool active = n0 < N;
  const int nchunk = (K + 255) / 256;
  uint4 wr[CB][RPW];
  auto issue = [&](int c0) {
#pragma unroll
    for (int u = 0; u < CB; ++u) {
      const int k = (c0 + u) * 256 + lane * 8;
#pragma unroll
      for (int r = 0; r < RPW; ++r) {
        const int n = min(n0 + r, N - 1);
        wr[u][r] = (active && k < K) ? ld_nc_v4(W + static_cast<size_t>(n) * K + k) : make_uint4(0, 0, 0, 0);
      }
    }
  };
  issue(0);
  pdl_wait();
  pdl_trigger();
  if (e.adv_pos != nullptr && blockIdx.x == 0 && tid == 0) *e.adv_pos += e.adv_n;
  if (EMB || nrm.xh != nullptr) {
    const bf16* eb = nullptr;
    if (EMB) {
      int tok = *nrm.tok;
      tok = tok < 0 ? 0 : (tok >= nrm.V ? nrm.V - 1 : tok);
      eb = nrm.emb + static_cast<size_t>(tok) * K;
    }
    if (warp == 0) {
      const float rs = gemv_row_rs(nrm.xh, eb, K, nrm.eps, lane);
      if (lane == 0) s_rs = rs;
    }
    __syncthreads();
    const float rs = s_rs;
    for (int k = tid * 4; k < K; k += kGemvWarps * 32 * 4) {
      const float4 h4 = row4(nrm.xh, eb, k / 4);
      if (EMB && blockIdx.x == 0) *reinterpret_cast<float4*>(nrm.h_out + k) = h4;
      const float4 g4 = *reinterpret_cast<const float4*>(nrm.g + k);
      const __nv_bfloat162 lo = __floats2bfloat162_rn(h4.x * rs * g4.x, h4.y * rs * g4.y);
      const __nv_bfloat162 hi = __floats2bfloat162_rn(h4.z * rs * g4.z, h4.w * rs * g4.w);
      *reinterpret_cast<uint2*>(s_x + k) =
          make_uint2(*reinterpret_cast<const uint32_t*>(&lo), *reinterpret_cast<const uint32_t*>(&hi));
    }
  } else {
    for (int k = tid * 8; k < K; k += kGemvWarps * 32 * 8)
      *reinterpret_cast<uint4*>(s_x + k) = __ldg(reinterpret_cast<const uint4*>(X + k));
  }
  __syncthreads();
  float acc[RPW];
#pragma unroll
  for (int r = 0; r < RPW; ++r) acc[r] = 0.f;
  for (int c0 = 0; c0 < nchunk; c0 += CB) {
    if (c0 > 0) issue(c0);
#pragma unroll
    for (int u = 0; u < CB; ++u) {
      const int k = (c0 + u) * 256 + lane * 8;
      if (active && k < K) {
        float xv[8];
        bf16x8_to_f32(*reinterpret_cast<const uint4*>(s_x + k), xv);
#pragma unroll
        for (int r = 0; r < RPW; ++r) {
          float w[8];
          bf16x8_to_f32(wr[u][r], w);
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[r] = fmaf(w[j], xv[j], acc[r]);
        }
      }
    }
  }
#pragma unroll
  for (int r = 0; r < RPW; ++r)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc[r] += __shfl_xor_sync(0xffffffffu, acc[r], o);
  if (RPW == 4) {
    if (active && lane == 0) {
      float v[4] = {acc[0], acc[1 % RPW], acc[2 % RPW], acc[3 % RPW]};
      epilogue4(e, 0, n0, v, N);
    }
  } else {
    if (lane == 0) s_out[warp] = acc[0];
    __syncthreads();
    const int nq = blockIdx.x * kGemvWarps + 4 * tid;
    if (tid < kGemvWarps / 4 && nq < N) {
      float v[4] = {s_out[4 * tid], s_out[4 * tid + 1], s_out[4 * tid + 2], s_out[4 * tid + 3]};
      epilogue4(e, 0, nq, v, N);
    }
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
namespace {

// PEARL_GEMV1=0 restores gemv_kernel<1, RPW> for single tokens (A/B diagnostics;
// bitwise the same results)
static bool gemv1_enabled() {
  static const bool on = [] {
    const char* v = std::getenv("PEARL_GEMV1");
    return !(v && std::atoi(v) == 0);
  }();
  return on;
}

// PEARL_GEMV1N=0: fused-norm single-token GEMVs stage the operand through smem
// (gemv1_kernel) instead of the register-norm gemv1n_kernel (A/B; bitwise equal)
static bool gemv1n_enabled() {
  static const bool on = [] {
    const char* v = std::getenv("PEARL_GEMV1N");
    return !(v && std::atoi(v) == 0);
  }();
  return on;
}

// PEARL_GEMV1X=0: bf16-operand single-token GEMVs stage the operand in smem
// (gemv1_kernel) instead of holding it in registers (gemv1x_kernel; A/B)
static bool gemv1x_enabled() {
  static const bool on = [] {
    const char* v = std::getenv("PEARL_GEMV1X");
    return !(v && std::atoi(v) == 0);
  }();
  return on;
}

template <int NV>
int launch_gemv1n(const bf16* W, int N, const EpiArgs& e, cudaStream_t st, const GemvNorm& nrm) {
  const dim3 grid((N + kGemvWarps * 4 - 1) / (kGemvWarps * 4)), block(kGemvWarps * 32);
  if (nrm.emb != nullptr) return launch_pdl(gemv1n_kernel<NV, true>, grid, block, 0, st, W, N, e, nrm);
  return launch_pdl(gemv1n_kernel<NV, false>, grid, block, 0, st, W, N, e, nrm);
}

int launch_gemv(const bf16* W, const bf16* X, int M, int N, int K, const EpiArgs& e, cudaStream_t st,
                GemvNorm nrm = GemvNorm{nullptr, nullptr, 0.f}) {
  // single token, fused norm, d = 512 / 768 / 1024, not the lm_head (its 1000
  // blocks want gemv1_kernel's 3 per SM: gemv1n there measured 48.7 vs 49.2 us
  // per 68M token on the whole GPU, and would run ~50 % more waves on a partition)
  if (M == 1 && (nrm.xh != nullptr || nrm.emb != nullptr) && N <= 8192 && gemv1_enabled() && gemv1n_enabled()) {
    if (K == 512) return launch_gemv1n<4>(W, N, e, st, nrm);
    if (K == 768) return launch_gemv1n<6>(W, N, e, st, nrm);
    if (K == 1024) return launch_gemv1n<8>(W, N, e, st, nrm);
  }
  // narrow layers: one row per warp (4x the warps; same per-row arithmetic)
  const bool narrow = (N + kGemvWarps * kGemvRows - 1) / (kGemvWarps * kGemvRows) < 296;
  const dim3 block(kGemvWarps * 32);
  const bool m1 = M == 1 && K <= kGemv1MaxK && gemv1_enabled();
  const int nchunk = (K + 255) / 256;
  if (narrow) {
    const dim3 grid((N + kGemvWarps - 1) / kGemvWarps);
    if (m1 && nrm.xh == nullptr && nrm.emb == nullptr && gemv1x_enabled()) {
      if (nchunk <= 4) return launch_pdl(gemv1x_kernel<4>, grid, block, 0, st, W, X, N, K, e);
      if (nchunk <= 12) return launch_pdl(gemv1x_kernel<12>, grid, block, 0, st, W, X, N, K, e);
    }
    if (m1 && nrm.emb != nullptr && nchunk <= 4)
      return launch_pdl(gemv1_kernel<1, 4, true>, grid, block, 0, st, W, X, N, K, e, nrm);
    if (m1 && nrm.emb != nullptr) return launch_pdl(gemv1_kernel<1, 12, true>, grid, block, 0, st, W, X, N, K, e, nrm);
    if (m1 && nchunk <= 4) return launch_pdl(gemv1_kernel<1, 4>, grid, block, 0, st, W, X, N, K, e, nrm);
    if (m1) return launch_pdl(gemv1_kernel<1, 12>, grid, block, 0, st, W, X, N, K, e, nrm);
    if (M == 1) return launch_pdl(gemv_kernel<1, 1>, grid, block, 0, st, W, X, M, N, K, e, nrm);
    return launch_pdl(gemv_kernel<8, 1>, grid, block, 0, st, W, X, M, N, K, e, nrm);
  }
  const dim3 grid((N + kGemvWarps * kGemvRows - 1) / (kGemvWarps * kGemvRows));
  if (m1 && nrm.emb != nullptr) return launch_pdl(gemv1_kernel<4, 3, true>, grid, block, 0, st, W, X, N, K, e, nrm);
  if (m1) return launch_pdl(gemv1_kernel<4, 3>, grid, block, 0, st, W, X, N, K, e, nrm);
  if (M == 1) return launch_pdl(gemv_kernel<1, 4>, grid, block, 0, st, W, X, M, N, K, e, nrm);
  return launch_pdl(gemv_kernel<8, 4>, grid, block, 0, st, W, X, M, N, K, e, nrm);
}

static int ablate_mask();
int launch_gemm(Llama& m, const bf16* W, const bf16* X, int M, int N, int K, const EpiArgs& e, cudaStream_t st,
                GemvNorm nrm = GemvNorm{nullptr, nullptr, 0.f}) {
  if (ablate_mask() & 4) return PEARL_OK;
  if (m.cfg.gemm_kind == PEARL_GEMM_TCGEN05) return tc_gemm(m.tc, W, X, M, N, K, e, st, 0);
  return launch_gemv(W, X, M, N, K, e, st, nrm);
}

// Diagnostics only (PEARL_ABLATE=attn|gemm): skip a kernel class to
// measure its in-graph cost.  Results are wrong while set.
static int ablate_mask() {
  static const int m = [] {
    const char* v = std::getenv("PEARL_ABLATE");
    if (!v) return 0;
    std::string s(v);
    return (s.find("attn") != std::string::npos ? 1 : 0) | (s.find("norm") != std::string::npos ? 2 : 0) |
           (s.find("gemm") != std::string::npos ? 4 : 0);
  }();
  return m;
}

// Diagnostics only (PEARL_STOP=k): run only the first k ops of a forward
// (embed, then per layer qkv, attn, o, gate_up, down, then lm_head), so the
// intermediate buffers can be compared with the oracle
// (pearl_llama_debug_buffer).
static int stop_after() {
  const char* v = std::getenv("PEARL_STOP");
  return v ? std::atoi(v) : -1;
}

int forward_chunk(Llama& m, const int32_t* tokens, int M, int32_t* pos, int pos_add, bool logits_all,
                  bool want_logits, float* logits, cudaStream_t st, int adv_n = 0, bool* advanced = nullptr,
                  const int32_t* tok_slot = nullptr, const int32_t* tok_pos = nullptr) {
  const int abl = ablate_mask();
  const int stop = stop_after();
  int n_ops = 0;
  auto halt = [&]() { return stop >= 0 && ++n_ops >= stop; };
  const auto& c = m.cfg;
  const int d = c.d_model, hd = c.head_dim, H = c.n_heads, KV = c.n_kv_heads, L = c.n_layers;
  const int nq = H * hd, nkv = KV * hd;
  const int T = c.max_tokens;
  // tcgen05 models fold every RMSNorm into their GEMMs; CUDA-core models
  // fuse it into the consuming GEMV's operand load
  const bool fold = c.gemm_kind == PEARL_GEMM_TCGEN05;
  const bool fuse_norm = !fold;
  // producer-side / consumer-side halves of a folded norm
  auto produce = [&](EpiArgs& e, const float* gain) {
    if (!fold) return;
    e.x_out = m.x;
    e.gain = gain;
    e.ss_out = m.ss;
    e.ss_ld = T;
  };
  auto consume = [&](EpiArgs& e, int row0) {
    if (!fold) return;
    e.ss_in = m.ss + row0;
    e.ss_ld = T;
    e.ss_tiles = (d + 127) / 128;
    e.norm_d = d;
    e.norm_eps = c.norm_eps;
  };
  // single-token CUDA-core forwards fold the embedding into layer 0's QKV
  // GEMV (gemv1_kernel reads the embedding row and writes h)
  const bool embed_fold = fuse_norm && M == 1 && d <= kGemv1MaxK && gemv1_enabled() && stop < 0 && abl == 0;
  int rc = PEARL_OK;
  if (!embed_fold) {
    rc = launch_pdl(embed_kernel, dim3(M), dim3(kEmbedThreads), 0, st, tokens, m.embed, m.h, d, c.vocab,
                    fold ? m.layers[0].attn_norm : static_cast<const float*>(nullptr),
                    fold ? m.x : static_cast<bf16*>(nullptr), m.ss, T);
    if (rc) return rc;
  }
  g_prof.mark(OP_EMBED, st);
  if (halt()) return PEARL_OK;
  const size_t slot_kv = static_cast<size_t>(c.max_seq) * nkv;
  const size_t layer_kv = static_cast<size_t>(std::max(1, c.n_slots)) * slot_kv;
  int tpb = 1, spw = 1, agrid = 1;
  attn_plan(AttnShape{M, H, KV, hd, c.max_seq, m.num_sms, tok_pos != nullptr}, &tpb, &spw, &agrid);
  for (int l = 0; l < L; ++l) {
    const LayerW& Lw = m.layers[l];
    EpiArgs e{};
    e.kind = EPI_QKV;
    e.out_bf16 = m.q;
    e.kc = m.kcache + l * layer_kv;
    e.vc = m.vcache + l * layer_kv;
    e.cos_t = m.rope_cos;
    e.sin_t = m.rope_sin;
    e.pos = pos;
    e.pos_add = pos_add;
    e.tok_pos = tok_pos;
    e.tok_slot = tok_slot;
    e.slot_stride = static_cast<long long>(slot_kv);
    e.n_q = nq;
    e.n_kv = nkv;
    e.hd = hd;
    consume(e, 0);
    GemvNorm qn = fuse_norm ? GemvNorm{m.h, Lw.attn_norm, c.norm_eps} : GemvNorm{nullptr, nullptr, 0.f};
    if (embed_fold && l == 0) {
      qn.xh = nullptr;
      qn.emb = m.embed;
      qn.tok = tokens;
      qn.V = c.vocab;
      qn.h_out = m.h;
    }
    rc = launch_gemm(m, Lw.wqkv, m.x, M, nq + 2 * nkv, d, e, st, qn);
    if (rc) return rc;
    g_prof.mark(OP_QKV, st);
    if (halt()) return PEARL_OK;
    if (!(abl & 1)) {
      AttnArgs aa{};
      aa.q = m.q;
      aa.kc = e.kc;
      aa.vc = e.vc;
      aa.o = m.o;
      aa.pos = pos;
      aa.pos_add = pos_add;
      aa.tok_pos = tok_pos;
      aa.tok_slot = tok_slot;
      aa.slot_stride = static_cast<long long>(slot_kv);
      aa.M = M;
      aa.H = H;
      aa.KV = KV;
      aa.scale = 1.0f / sqrtf(static_cast<float>(hd));
      aa.tpb = tpb;
      aa.spw = spw;
      rc = attn_launch(aa, hd, agrid, st);
      if (rc) return rc;
    }
    g_prof.mark(OP_ATTN, st);
    if (halt()) return PEARL_OK;
    EpiArgs r{};
    r.kind = EPI_RESID;
    r.out_f32 = m.h;
    r.ld = d;
    produce(r, Lw.mlp_norm);
    rc = launch_gemm(m, Lw.wo, m.o, M, d, nq, r, st);
    if (rc) return rc;
    g_prof.mark(OP_O, st);
    if (halt()) return PEARL_OK;
    EpiArgs g{};
    g.kind = EPI_SWIGLU;
    g.out_bf16 = m.act;
    g.ld = c.ffn;
    consume(g, 0);
    rc = launch_gemm(m, Lw.wgu, m.x, M, 2 * c.ffn, d, g, st,
                     fuse_norm ? GemvNorm{m.h, Lw.mlp_norm, c.norm_eps} : GemvNorm{nullptr, nullptr, 0.f});
    if (rc) return rc;
    g_prof.mark(OP_GU, st);
    if (halt()) return PEARL_OK;
    EpiArgs dn{};
    dn.kind = EPI_RESID;
    dn.out_f32 = m.h;
    dn.ld = d;
    // the next consumer: layer l + 1's QKV, or the lm_head
    if (l + 1 < L) produce(dn, m.layers[l + 1].attn_norm);
    else if (want_logits) produce(dn, m.final_norm);
    rc = launch_gemm(m, Lw.wdown, m.act, M, d, c.ffn, dn, st);
    if (rc) return rc;
    g_prof.mark(OP_DOWN, st);
    if (halt()) return PEARL_OK;
  }
  if (!want_logits) return PEARL_OK;
  const int first = logits_all ? 0 : M - 1;
  const int rows = M - first;
  EpiArgs s{};
  s.kind = EPI_STORE_F32;
  s.out_f32 = logits;
  s.ld = c.vocab;
  consume(s, first);
  if (adv_n > 0 && stop < 0 && !abl) {
    s.adv_pos = pos;  // the lm_head GEMM advances pos (no separate advance kernel)
    s.adv_n = adv_n;
    if (advanced) *advanced = true;
  }
  rc = launch_gemm(m, m.lm_head, fuse_norm ? m.x : m.x + static_cast<size_t>(first) * d, rows, c.vocab, d, s, st,
                   fuse_norm ? GemvNorm{m.h + static_cast<size_t>(first) * d, m.final_norm, c.norm_eps}
                             : GemvNorm{nullptr, nullptr, 0.f});
  g_prof.mark(OP_HEAD, st);
  return rc;
}

}  // namespace
}  // namespace pearl

using namespace pearl;

extern "C" int pearl_llama_create(const pearl_llama_config* cfg, const void* const* ptrs, int n_ptrs, void** handle) {
  PEARL_ARG_CHECK(cfg && ptrs && handle, "null argument");
  const auto& c = *cfg;
  PEARL_ARG_CHECK(n_ptrs == PEARL_LLAMA_FIXED_PTRS + PEARL_LLAMA_PTRS_PER_LAYER * c.n_layers, "pointer table size");
  PEARL_ARG_CHECK(c.head_dim == 64 || c.head_dim == 128, "head_dim must be 64 or 128");
  PEARL_ARG_CHECK(c.n_heads % c.n_kv_heads == 0, "n_heads % n_kv_heads");
  PEARL_ARG_CHECK(c.d_model % 8 == 0 && c.ffn % 8 == 0, "d_model and ffn must be multiples of 8");
  PEARL_ARG_CHECK(c.d_model <= 16384, "d_model <= 16384");
  PEARL_ARG_CHECK(c.gemm_kind != PEARL_GEMM_CUDACORE || (c.max_tokens <= kGemvMaxNormTok && c.d_model % 256 == 0),
                  "CUDA-core models need max_tokens <= 64 and d_model % 256 == 0 (fused norm)");
  PEARL_ARG_CHECK(c.max_tokens >= 1 && c.max_tokens <= (c.gemm_kind == PEARL_GEMM_TCGEN05 ? 128 : 64),
                  "max_tokens in [1, 128] (tcgen05) / [1, 64] (CUDA-core)");
  PEARL_ARG_CHECK(c.max_seq >= 1 && c.max_seq <= 4096, "max_seq in [1, 4096]");
  // logits / q rows are read and written with 16-byte vectors (GEMM epilogue,
  // commit, K6): every row must start 16-byte aligned
  PEARL_ARG_CHECK(c.vocab >= 2 && c.vocab % 4 == 0, "vocab must be a multiple of 4 (16-byte aligned logits rows)");
  Llama* m = new Llama();
  m->cfg = c;
  m->embed = static_cast<const bf16*>(ptrs[0]);
  m->final_norm = static_cast<const float*>(ptrs[1]);
  m->lm_head = static_cast<const bf16*>(ptrs[2]);
  m->rope_cos = static_cast<const float*>(ptrs[3]);
  m->rope_sin = static_cast<const float*>(ptrs[4]);
  m->kcache = static_cast<bf16*>(const_cast<void*>(ptrs[5]));
  m->vcache = static_cast<bf16*>(const_cast<void*>(ptrs[6]));
  for (int l = 0; l < c.n_layers; ++l) {
    const void* const* p = ptrs + PEARL_LLAMA_FIXED_PTRS + PEARL_LLAMA_PTRS_PER_LAYER * l;
    m->layers.push_back(LayerW{static_cast<const float*>(p[0]), static_cast<const bf16*>(p[1]),
                               static_cast<const bf16*>(p[2]), static_cast<const float*>(p[3]),
                               static_cast<const bf16*>(p[4]), static_cast<const bf16*>(p[5])});
  }
  const size_t T = static_cast<size_t>(c.max_tokens);
  const size_t wide = std::max<size_t>(std::max<size_t>(c.d_model, c.ffn), static_cast<size_t>(c.n_heads) * c.head_dim);
  auto fail = [&](cudaError_t e) {
    set_error(std::string("pearl_llama_create: ") + cudaGetErrorString(e));
    delete m;
    return PEARL_ERR_CUDA;
  };
  cudaError_t e;
  if ((e = cudaMalloc(&m->h, T * c.d_model * sizeof(float)))) return fail(e);
  if ((e = cudaMalloc(&m->x, T * wide * sizeof(bf16)))) return fail(e);
  if ((e = cudaMalloc(&m->q, T * c.n_heads * c.head_dim * sizeof(bf16)))) return fail(e);
  if ((e = cudaMalloc(&m->o, T * c.n_heads * c.head_dim * sizeof(bf16)))) return fail(e);
  if ((e = cudaMalloc(&m->act, T * c.ffn * sizeof(bf16)))) return fail(e);
  {
    int dev = 0;
    if ((e = cudaGetDevice(&dev))) return fail(e);
    if ((e = cudaDeviceGetAttribute(&m->num_sms, cudaDevAttrMultiProcessorCount, dev))) return fail(e);
    if (c.sm_count > 0) m->num_sms = std::min(m->num_sms, static_cast<int>(c.sm_count));
  }
  const size_t ss_floats = static_cast<size_t>((c.d_model + 127) / 128) * T;
  if ((e = cudaMalloc(&m->ss, ss_floats * sizeof(float)))) return fail(e);
  if ((e = cudaMemset(m->ss, 0, ss_floats * sizeof(float)))) return fail(e);
  {
    int rc = attn_init();
    if (rc) {
      delete m;
      return rc;
    }
  }
  if (c.gemm_kind == PEARL_GEMM_TCGEN05) {
    int rc = tc_init(m->tc, c);
    if (rc) {
      delete m;
      return rc;
    }
  }
  *handle = m;
  return PEARL_OK;
}

extern "C" int pearl_llama_destroy(void* handle) {
  Llama* m = static_cast<Llama*>(handle);
  if (!m) return PEARL_OK;
  cudaFree(m->h);
  cudaFree(m->x);
  cudaFree(m->q);
  cudaFree(m->o);
  cudaFree(m->act);
  cudaFree(m->ss);
  tc_free(m->tc);
  delete m;
  return PEARL_OK;
}

namespace {
std::mutex g_gemm_mu;
TcGemmCtx g_gemm_ctx;  // standalone pearl_gemm (tests / microbenchmarks)
}  // namespace

extern "C" int pearl_gemm(int kind, const void* W, const void* X, float* Y, int M, int N, int K, int splits,
                          void* stream) {
  PEARL_ARG_CHECK(W && X && Y && M >= 1 && N >= 1 && K >= 8, "bad gemm arguments");
  EpiArgs e{};
  e.kind = EPI_STORE_F32;
  e.out_f32 = Y;
  e.ld = N;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool w_tiled = (kind & PEARL_GEMM_W_TILED) != 0;
  kind &= ~PEARL_GEMM_W_TILED;
  if (kind == PEARL_GEMM_CUDACORE) {
    PEARL_ARG_CHECK(!w_tiled, "the CUDA-core GEMV takes row-major weights");
    return launch_gemv(static_cast<const bf16*>(W), static_cast<const bf16*>(X), M, N, K, e, st);
  }
  std::lock_guard<std::mutex> lk(g_gemm_mu);
  if (!g_gemm_ctx.partials) {
    pearl_llama_config c{};
    c.n_layers = 1;
    c.d_model = 8192;
    c.n_heads = 64;
    c.n_kv_heads = 8;
    c.head_dim = 128;
    c.ffn = 28672;
    c.vocab = 131072;
    c.max_tokens = 128;
    g_gemm_ctx.min_plan_splits = 16;
    int rc = tc_init(g_gemm_ctx, c);
    if (rc) return rc;
  }
  return tc_gemm(g_gemm_ctx, static_cast<const bf16*>(W), static_cast<const bf16*>(X), M, N, K, e, st, splits,
                 w_tiled);
}

extern "C" int pearl_gemm_splits(int N, int K) {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return tc_splits(N, K, sms);
}

extern "C" size_t pearl_llama_workspace_bytes(void* handle, int n_tokens) {
  (void)handle;
  (void)n_tokens;
  return 0;
}

extern "C" int pearl_llama_forward(void* handle, const int32_t* tokens, int n_tokens, int32_t* pos, int flags,
                                   float* logits, void* stream) {
  Llama* m = static_cast<Llama*>(handle);
  PEARL_ARG_CHECK(m && tokens && pos && n_tokens >= 1, "bad forward arguments");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int T = m->cfg.max_tokens;
  const bool last_only = (flags & PEARL_FWD_LAST_LOGITS) != 0;
  PEARL_ARG_CHECK(last_only || n_tokens <= T || logits == nullptr,
                  "windows longer than max_tokens need PEARL_FWD_LAST_LOGITS");
  struct WindowScope {
    explicit WindowScope(const L2Window& w) { g_l2win = w; }
    ~WindowScope() { g_l2win = L2Window{}; }
  } window_scope(m->l2win);
  bool advanced = false;
  for (int c0 = 0; c0 < n_tokens; c0 += T) {
    const int mt = std::min(T, n_tokens - c0);
    const bool last_chunk = c0 + mt == n_tokens;
    int rc = forward_chunk(*m, tokens + c0, mt, pos, c0, !last_only, last_chunk && logits != nullptr, logits, st,
                           last_chunk && (flags & PEARL_FWD_ADVANCE) ? n_tokens : 0, &advanced);
    if (rc) return rc;
  }
  if ((flags & PEARL_FWD_ADVANCE) && !advanced) {
    int rc = launch_pdl(advance_kernel, dim3(1), dim3(1), 0, st, pos, n_tokens);
    if (rc) return rc;
  }
  return PEARL_OK;
}

extern "C" int pearl_llama_forward_slots(void* handle, const int32_t* tokens, int n_tokens, const int32_t* tok_slot,
                                         const int32_t* tok_pos, float* logits, void* stream) {
  Llama* m = static_cast<Llama*>(handle);
  PEARL_ARG_CHECK(m && tokens && tok_slot && tok_pos && n_tokens >= 1, "bad forward_slots arguments");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int T = m->cfg.max_tokens;
  int32_t* pos_dummy = const_cast<int32_t*>(tok_pos);  // unread in slot mode
  struct WindowScope {
    explicit WindowScope(const L2Window& w) { g_l2win = w; }
    ~WindowScope() { g_l2win = L2Window{}; }
  } window_scope(m->l2win);
  for (int c0 = 0; c0 < n_tokens; c0 += T) {
    const int mt = std::min(T, n_tokens - c0);
    int rc = forward_chunk(*m, tokens + c0, mt, pos_dummy, 0, true, logits != nullptr,
                           logits ? logits + static_cast<size_t>(c0) * m->cfg.vocab : nullptr, st, 0, nullptr,
                           tok_slot + c0, tok_pos + c0);
    if (rc) return rc;
  }
  return PEARL_OK;
}

extern "C" int pearl_llama_set_l2_window(void* handle, const void* base, size_t bytes, size_t* granted) {
  Llama* m = static_cast<Llama*>(handle);
  PEARL_ARG_CHECK(m != nullptr, "null handle");
  if (base == nullptr || bytes == 0) {
    m->l2win = L2Window{};
    if (granted) *granted = 0;
    return PEARL_OK;
  }
  int dev = 0, max_persist = 0, max_window = 0;
  PEARL_CUDA_TRY(cudaGetDevice(&dev));
  PEARL_CUDA_TRY(cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, dev));
  PEARL_CUDA_TRY(cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, dev));
  if (max_persist <= 0 || max_window <= 0) {
    m->l2win = L2Window{};
    if (granted) *granted = 0;
    return PEARL_OK;
  }
  size_t cur = 0;
  PEARL_CUDA_TRY(cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize));
  const size_t want = std::min(bytes, static_cast<size_t>(max_persist));
  if (want > cur) PEARL_CUDA_TRY(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want));
  PEARL_CUDA_TRY(cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize));
  m->l2win.base = base;
  m->l2win.bytes = std::min(bytes, static_cast<size_t>(max_window));
  m->l2win.hit_ratio = std::min(1.0f, static_cast<float>(cur) / static_cast<float>(m->l2win.bytes));
  if (granted) *granted = cur;
  return PEARL_OK;
}

// Diagnostic: copy an internal activation buffer (0 h fp32 [T, d], 1 x, 2 q,
// 3 o, 4 act; bf16) to dst.
extern "C" int pearl_llama_debug_buffer(void* handle, int which, void* dst, size_t bytes, void* stream) {
  Llama* m = static_cast<Llama*>(handle);
  PEARL_ARG_CHECK(m && dst && which >= 0 && which <= 6, "bad debug_buffer arguments");
  const void* src[7] = {m->h, m->x, m->q, m->o, m->act, m->tc.tile_flags, m->ss};
  PEARL_CUDA_TRY(cudaMemcpyAsync(dst, src[which], bytes, cudaMemcpyDeviceToDevice, static_cast<cudaStream_t>(stream)));
  return PEARL_OK;
}

// Per-op device time (ms) of one eager forward: out[op] for op in
// {embed, norm, qkv, attn, o, gate_up, down, lm_head, other}; out[9] = total.
extern "C" int pearl_llama_profile(void* handle, const int32_t* tokens, int n_tokens, int32_t* pos, float* logits,
                                   float* out_ms, void* stream) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  PEARL_CUDA_TRY(cudaStreamSynchronize(st));
  g_prof.on = true;
  g_prof.marks.clear();
  cudaEventCreate(&g_prof.start);
  cudaEventRecord(g_prof.start, st);
  int rc = pearl_llama_forward(handle, tokens, n_tokens, pos, 0, logits, stream);
  g_prof.on = false;
  PEARL_CUDA_TRY(cudaStreamSynchronize(st));
  for (int i = 0; i <= OP_COUNT; ++i) out_ms[i] = 0.f;
  cudaEvent_t prev = g_prof.start;
  for (auto& mk : g_prof.marks) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, prev, mk.second);
    out_ms[mk.first] += ms;
    out_ms[OP_COUNT] += ms;
    prev = mk.second;
  }
  for (auto& mk : g_prof.marks) cudaEventDestroy(mk.second);
  cudaEventDestroy(g_prof.start);
  g_prof.marks.clear();
  return rc;
}
