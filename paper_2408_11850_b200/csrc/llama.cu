// Llama decoder runtime for GPU SequenceModels (draft and target).
//
// Replaces SequenceModel.next_dist (pearl_lab/models.py:58-71) for the
// transformer models the B200 build serves: the draft's per-token forward
// inside _draft_block (engines.py:277-282) and the target's window forward
// (engines.py:302, 373, 425, 492).  A forward processes n tokens at device
// positions *pos..*pos+n-1 against the per-layer KV cache.
//
// Layer = RMSNorm -> QKV GEMM (+RoPE, +K/V append) -> causal attention over
// the cache -> O GEMM (+residual) -> RMSNorm -> gate/up GEMM (+SwiGLU) ->
// down GEMM (+residual).  The residual stream is fp32; GEMM operands bf16.
//
// Batch invariance: every per-token value is computed by the same sequence
// of fp32 operations whatever the number of tokens in the launch (fixed
// K-order FMA chains, fixed shuffle trees, per-(token, head) attention with
// a sequential softmax-weighted sum), so a position's logits are bitwise the
// same in an M=1 AR step, an M=gamma PEARL window or an M=gamma+1 SD window.
// That property is what makes GPU greedy PEARL/SD token-identical to GPU AR.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "common.h"
#include "epilogue.cuh"
#include "gemm_tc.cuh"

namespace pearl {

using bf16 = __nv_bfloat16;

struct LayerW {
  const float* attn_norm;
  const bf16* wqkv;
  const bf16* wo;
  const float* mlp_norm;
  const bf16* wgu;
  const bf16* wdown;
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
  // workspace
  float* h = nullptr;     // [T, d]
  bf16* x = nullptr;      // [T, max(d, ffn, H hd)]
  bf16* q = nullptr;      // [T, H hd]
  bf16* o = nullptr;      // [T, H hd]
  bf16* act = nullptr;    // [T, ffn]
  TcGemmCtx tc;           // tcgen05 path state (split-K scratch, descriptors)
};

// ---------------------------------------------------------------------------
// small kernels
// ---------------------------------------------------------------------------
__global__ void embed_kernel(const int32_t* __restrict__ tokens, const bf16* __restrict__ emb, float* __restrict__ h,
                             int d, int V) {
  const int t = blockIdx.x;
  int tok = tokens[t];
  tok = tok < 0 ? 0 : (tok >= V ? V - 1 : tok);
  const bf16* row = emb + static_cast<size_t>(tok) * d;
  for (int i = threadIdx.x; i < d; i += blockDim.x) h[static_cast<size_t>(t) * d + i] = __bfloat162float(row[i]);
}

// x[t] = bf16(h[t] * rsqrt(mean(h[t]^2) + eps) * g); one block per token,
// fixed reduction order.
__global__ void rmsnorm_kernel(const float* __restrict__ h, const float* __restrict__ g, bf16* __restrict__ x,
                               int d, float eps, int row_off) {
  const int t = blockIdx.x + row_off;
  const float* hr = h + static_cast<size_t>(t) * d;
  float ss = 0.f;
  for (int i = threadIdx.x; i < d; i += blockDim.x) ss = fmaf(hr[i], hr[i], ss);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  __shared__ float ws[32];
  __shared__ float s_rs;
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x == 0) {
    float tot = 0.f;
    for (int w = 0; w < (blockDim.x >> 5); ++w) tot += ws[w];
    s_rs = 1.0f / sqrtf(tot / static_cast<float>(d) + eps);
  }
  __syncthreads();
  const float rs = s_rs;
  bf16* xr = x + static_cast<size_t>(blockIdx.x) * d;
  for (int i = threadIdx.x; i < d; i += blockDim.x) xr[i] = __float2bfloat16(hr[i] * rs * g[i]);
}

__global__ void advance_kernel(int32_t* pos, int n) { *pos += n; }

// ---------------------------------------------------------------------------
// K2: batch-invariant CUDA-core GEMV / skinny GEMM
//   Y[t, n] = sum_k W[n, k] X[t, k]; W bf16 [N, K] row-major, X bf16 [M, K]
// Each warp owns 4 consecutive rows; lane l streams 16-byte (8 x bf16)
// chunks k = 256 c + 8 l with 128-bit non-allocating loads, FMA-accumulates
// per (row, token) in fp32, then a fixed xor-shuffle tree reduces the lanes.
// ---------------------------------------------------------------------------
constexpr int kGemvRows = 4;
constexpr int kGemvTok = 8;
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

__global__ void __launch_bounds__(kGemvWarps * 32) gemv_kernel(const bf16* __restrict__ W, const bf16* __restrict__ X,
                                                               int M, int N, int K, EpiArgs e) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n0 = (blockIdx.x * kGemvWarps + warp) * kGemvRows;
  if (n0 >= N) return;
  const int nchunk = (K + 255) / 256;
  for (int t0 = 0; t0 < M; t0 += kGemvTok) {
    const int mt = min(kGemvTok, M - t0);
    float acc[kGemvRows][kGemvTok];
#pragma unroll
    for (int r = 0; r < kGemvRows; ++r)
#pragma unroll
      for (int t = 0; t < kGemvTok; ++t) acc[r][t] = 0.f;
#pragma unroll 2
    for (int c = 0; c < nchunk; ++c) {
      const int k = c * 256 + lane * 8;
      if (k < K) {
        float w[kGemvRows][8];
#pragma unroll
        for (int r = 0; r < kGemvRows; ++r) {
          const int n = min(n0 + r, N - 1);
          bf16x8_to_f32(ld_nc_v4(W + static_cast<size_t>(n) * K + k), w[r]);
        }
#pragma unroll
        for (int t = 0; t < kGemvTok; ++t) {
          if (t < mt) {
            float xv[8];
            bf16x8_to_f32(__ldg(reinterpret_cast<const uint4*>(X + static_cast<size_t>(t0 + t) * K + k)), xv);
#pragma unroll
            for (int r = 0; r < kGemvRows; ++r)
#pragma unroll
              for (int j = 0; j < 8; ++j) acc[r][t] = fmaf(w[r][j], xv[j], acc[r][t]);
          }
        }
      }
    }
#pragma unroll
    for (int r = 0; r < kGemvRows; ++r)
#pragma unroll
      for (int t = 0; t < kGemvTok; ++t)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc[r][t] += __shfl_xor_sync(0xffffffffu, acc[r][t], o);
    if (lane == 0) {
      for (int t = 0; t < mt; ++t) {
        float v[4] = {acc[0][t], acc[1][t], acc[2][t], acc[3][t]};
        epilogue4(e, t0 + t, n0, v, N);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// K4: causal attention of the window's queries over the cache
//   one block per (head, token); scores in smem; softmax and the weighted
//   value sum in a fixed order, so the result depends only on the token's
//   own position and the cache contents.
// ---------------------------------------------------------------------------
__global__ void attention_kernel(const bf16* __restrict__ q, const bf16* __restrict__ kc, const bf16* __restrict__ vc,
                                 bf16* __restrict__ o, const int32_t* pos, int pos_add, int H, int KV, int hd,
                                 float scale) {
  extern __shared__ float sc[];
  __shared__ float red[32];
  const int h = blockIdx.x, t = blockIdx.y;
  const int kvh = h / (H / KV);
  const int ctx = *pos + pos_add + t + 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int per = hd / 32;  // 2 or 4
  float qv[4];
  const bf16* qr = q + (static_cast<size_t>(t) * H + h) * hd;
  for (int i = 0; i < per; ++i) qv[i] = __bfloat162float(qr[lane * per + i]);
  const size_t kstride = static_cast<size_t>(KV) * hd;
  for (int j = warp; j < ctx; j += nw) {
    const bf16* kr = kc + j * kstride + kvh * hd + lane * per;
    float s = 0.f;
    for (int i = 0; i < per; ++i) s = fmaf(qv[i], __bfloat162float(kr[i]), s);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (lane == 0) sc[j] = s * scale;
  }
  __syncthreads();
  // max
  float m = -INFINITY;
  for (int j = threadIdx.x; j < ctx; j += blockDim.x) m = fmaxf(m, sc[j]);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
  if (lane == 0) red[warp] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    float mm = -INFINITY;
    for (int w = 0; w < nw; ++w) mm = fmaxf(mm, red[w]);
    red[31] = mm;
  }
  __syncthreads();
  m = red[31];
  __syncthreads();
  float sum = 0.f;
  for (int j = threadIdx.x; j < ctx; j += blockDim.x) {
    const float p = expf(sc[j] - m);
    sc[j] = p;
    sum += p;
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
  if (lane == 0) red[warp] = sum;
  __syncthreads();
  if (threadIdx.x == 0) {
    float ss = 0.f;
    for (int w = 0; w < nw; ++w) ss += red[w];
    red[30] = ss;
  }
  __syncthreads();
  const float inv = 1.0f / red[30];
  for (int d = threadIdx.x; d < hd; d += blockDim.x) {
    const bf16* vr = vc + kvh * hd + d;
    float acc = 0.f;
#pragma unroll 8
    for (int j = 0; j < ctx; ++j) acc = fmaf(sc[j], __bfloat162float(vr[j * kstride]), acc);
    o[(static_cast<size_t>(t) * H + h) * hd + d] = __float2bfloat16(acc * inv);
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
namespace {

int launch_gemm(Llama& m, const bf16* W, const bf16* X, int M, int N, int K, const EpiArgs& e, cudaStream_t st) {
  if (m.cfg.gemm_kind == PEARL_GEMM_TCGEN05) return tc_gemm(m.tc, W, X, M, N, K, e, st);
  const int rows_per_block = kGemvWarps * kGemvRows;
  gemv_kernel<<<(N + rows_per_block - 1) / rows_per_block, kGemvWarps * 32, 0, st>>>(W, X, M, N, K, e);
  PEARL_CUDA_TRY(cudaGetLastError());
  count_launch();
  return PEARL_OK;
}

int forward_chunk(Llama& m, const int32_t* tokens, int M, int32_t* pos, int pos_add, bool logits_all,
                  bool want_logits, float* logits, cudaStream_t st) {
  const auto& c = m.cfg;
  const int d = c.d_model, hd = c.head_dim, H = c.n_heads, KV = c.n_kv_heads;
  const int nq = H * hd, nkv = KV * hd;
  embed_kernel<<<M, 256, 0, st>>>(tokens, m.embed, m.h, d, c.vocab);
  PEARL_CUDA_TRY(cudaGetLastError());
  count_launch();
  const size_t layer_kv = static_cast<size_t>(c.max_seq) * nkv;
  const float scale = 1.0f / sqrtf(static_cast<float>(hd));
  const int attn_threads = 128;
  const size_t attn_smem = static_cast<size_t>(c.max_seq) * sizeof(float);
  for (int l = 0; l < c.n_layers; ++l) {
    const LayerW& L = m.layers[l];
    rmsnorm_kernel<<<M, 256, 0, st>>>(m.h, L.attn_norm, m.x, d, c.norm_eps, 0);
    PEARL_CUDA_TRY(cudaGetLastError());
    count_launch();
    EpiArgs e{};
    e.kind = EPI_QKV;
    e.out_bf16 = m.q;
    e.kc = m.kcache + l * layer_kv;
    e.vc = m.vcache + l * layer_kv;
    e.cos_t = m.rope_cos;
    e.sin_t = m.rope_sin;
    e.pos = pos;
    e.pos_add = pos_add;
    e.n_q = nq;
    e.n_kv = nkv;
    e.hd = hd;
    int rc = launch_gemm(m, L.wqkv, m.x, M, nq + 2 * nkv, d, e, st);
    if (rc) return rc;
    attention_kernel<<<dim3(H, M), attn_threads, attn_smem, st>>>(m.q, e.kc, e.vc, m.o, pos, pos_add, H, KV, hd,
                                                                  scale);
    PEARL_CUDA_TRY(cudaGetLastError());
    count_launch();
    EpiArgs r{};
    r.kind = EPI_RESID;
    r.out_f32 = m.h;
    r.ld = d;
    rc = launch_gemm(m, L.wo, m.o, M, d, nq, r, st);
    if (rc) return rc;
    rmsnorm_kernel<<<M, 256, 0, st>>>(m.h, L.mlp_norm, m.x, d, c.norm_eps, 0);
    PEARL_CUDA_TRY(cudaGetLastError());
    count_launch();
    EpiArgs g{};
    g.kind = EPI_SWIGLU;
    g.out_bf16 = m.act;
    g.ld = c.ffn;
    rc = launch_gemm(m, L.wgu, m.x, M, 2 * c.ffn, d, g, st);
    if (rc) return rc;
    rc = launch_gemm(m, L.wdown, m.act, M, d, c.ffn, r, st);
    if (rc) return rc;
  }
  if (!want_logits) return PEARL_OK;
  const int first = logits_all ? 0 : M - 1;
  const int rows = M - first;
  rmsnorm_kernel<<<rows, 256, 0, st>>>(m.h, m.final_norm, m.x, d, c.norm_eps, first);
  PEARL_CUDA_TRY(cudaGetLastError());
  count_launch();
  EpiArgs s{};
  s.kind = EPI_STORE_F32;
  s.out_f32 = logits;
  s.ld = c.vocab;
  return launch_gemm(m, m.lm_head, m.x, rows, c.vocab, d, s, st);
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
  PEARL_ARG_CHECK(c.max_tokens >= 1 && c.max_tokens <= 256, "max_tokens in [1, 256]");
  PEARL_ARG_CHECK(static_cast<size_t>(c.max_seq) * 4 <= 200 * 1024, "max_seq too large for attention smem");
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
  const size_t attn_smem = static_cast<size_t>(c.max_seq) * sizeof(float);
  if (attn_smem > 48 * 1024) {
    if ((e = cudaFuncSetAttribute(attention_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(attn_smem))))
      return fail(e);
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
  if (kind == PEARL_GEMM_CUDACORE) {
    const int rows_per_block = kGemvWarps * kGemvRows;
    gemv_kernel<<<(N + rows_per_block - 1) / rows_per_block, kGemvWarps * 32, 0, st>>>(
        static_cast<const bf16*>(W), static_cast<const bf16*>(X), M, N, K, e);
    PEARL_CUDA_TRY(cudaGetLastError());
    count_launch();
    return PEARL_OK;
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
    c.max_tokens = 64;
    int rc = tc_init(g_gemm_ctx, c);
    if (rc) return rc;
  }
  return tc_gemm(g_gemm_ctx, static_cast<const bf16*>(W), static_cast<const bf16*>(X), M, N, K, e, st, splits);
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
  for (int c0 = 0; c0 < n_tokens; c0 += T) {
    const int mt = std::min(T, n_tokens - c0);
    const bool last_chunk = c0 + mt == n_tokens;
    int rc = forward_chunk(*m, tokens + c0, mt, pos, c0, !last_only, last_chunk && logits != nullptr, logits, st);
    if (rc) return rc;
  }
  if (flags & PEARL_FWD_ADVANCE) {
    advance_kernel<<<1, 1, 0, st>>>(pos, n_tokens);
    PEARL_CUDA_TRY(cudaGetLastError());
    count_launch();
  }
  return PEARL_OK;
}
