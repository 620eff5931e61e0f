// Llama decoder runtime for GPU SequenceModels (draft and target).
//
// Replaces SequenceModel.next_dist (pearl_lab/models.py:58-71) for the
// transformer models the B200 build serves: the draft's per-token forward
// inside _draft_block (engines.py:277-282) and the target's window forward
// (engines.py:302, 373, 425, 492).  A forward processes n tokens at device
// positions *pos..*pos+n-1 against the per-layer KV cache.
//
// Layer = RMSNorm -> QKV GEMM (+RoPE, +K/V append) -> causal attention over
// the cache (K4) -> O GEMM (+residual) -> RMSNorm -> gate/up GEMM (+SwiGLU)
// -> down GEMM (+residual).  The residual stream is fp32; GEMM operands bf16.
// Every kernel is launched with programmatic dependent launch (PDL): it may
// start while its predecessor drains and calls griddepcontrol.wait before
// touching the predecessor's outputs (the tcgen05 GEMM prefetches weights
// before that wait).
//
// Batch invariance: every per-token value is computed by the same sequence
// of fp32 operations whatever the number of tokens in the launch (fixed
// K-order FMA chains, fixed reduction trees, per-(token, head) attention with
// fixed 64-position chunks combined in chunk order), so a position's logits
// are bitwise the same in an M=1 AR step, an M=gamma PEARL window or an
// M=gamma+1 SD window -- which makes GPU greedy PEARL/SD token-identical to AR.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "common.h"
#include "epilogue.cuh"
#include "fwd_mega.cuh"
#include "gemm_tc.cuh"

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
  TcGemmCtx tc;           // tcgen05 path state (split-K scratch, descriptors)
  // persistent forward (fwd_mega.cu): phase lists per (window M, logits mode),
  // built once at create time, device resident
  bool mega_ok = false;
  int mega_grid = 0;
  MegaMap* mg_maps = nullptr;       // [4 L + 1 weight maps | 4 x 16 activation maps]
  MegaPhase* mg_phases = nullptr;   // every list, concatenated
  unsigned* mg_counter = nullptr;
  unsigned long long* mg_trace = nullptr;  // set only inside pearl_llama_mega_trace
  int mg_off[17][3] = {};           // list offset / length per (M, mode)
  int mg_len[17][3] = {};
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
__global__ void embed_kernel(const int32_t* __restrict__ tokens, const bf16* __restrict__ emb, float* __restrict__ h,
                             int d, int V) {
  pdl_wait();
  pdl_trigger();
  const int t = blockIdx.x;
  int tok = tokens[t];
  tok = tok < 0 ? 0 : (tok >= V ? V - 1 : tok);
  const bf16* row = emb + static_cast<size_t>(tok) * d;
  for (int i = threadIdx.x; i < d; i += blockDim.x) h[static_cast<size_t>(t) * d + i] = __bfloat162float(row[i]);
}

// x[t] = bf16(h[t] * rsqrt(mean(h[t]^2) + eps) * g); one 128-thread block per
// token.  Fixed order: thread-strided float4 sums in k order, warp xor tree,
// (w0 + w1) + (w2 + w3) -- exactly mg_norm_row of the persistent forward
// kernel, so both paths produce identical bits.
constexpr int kNormThreads = 128;
constexpr int kNormVec = 16;  // d <= 4 * 128 * 16 = 8192
__global__ void __launch_bounds__(kNormThreads) rmsnorm_kernel(const float* __restrict__ h, const float* __restrict__ g,
                                                               bf16* __restrict__ x, int d, float eps, int row_off) {
  pdl_wait();
  pdl_trigger();
  __shared__ float red[4];
  const int t = blockIdx.x + row_off;
  const float4* hr = reinterpret_cast<const float4*>(h + static_cast<size_t>(t) * d);
  const int nv = d / 4;
  float4 v[kNormVec];
#pragma unroll
  for (int i = 0; i < kNormVec; ++i) {
    const int j = threadIdx.x + i * kNormThreads;
    v[i] = j < nv ? hr[j] : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < kNormVec; ++i) {
    if (threadIdx.x + i * kNormThreads < nv) {
      ss = fmaf(v[i].x, v[i].x, ss);
      ss = fmaf(v[i].y, v[i].y, ss);
      ss = fmaf(v[i].z, v[i].z, ss);
      ss = fmaf(v[i].w, v[i].w, ss);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  const float tot = (red[0] + red[1]) + (red[2] + red[3]);
  const float rs = 1.0f / sqrtf(tot / static_cast<float>(d) + eps);
  const float4* g4 = reinterpret_cast<const float4*>(g);
  uint2* xr = reinterpret_cast<uint2*>(x + static_cast<size_t>(t) * d);
#pragma unroll
  for (int i = 0; i < kNormVec; ++i) {
    const int j = threadIdx.x + i * kNormThreads;
    if (j < nv) {
      const float4 gg = g4[j];
      const __nv_bfloat162 lo = __floats2bfloat162_rn(v[i].x * rs * gg.x, v[i].y * rs * gg.y);
      const __nv_bfloat162 hi = __floats2bfloat162_rn(v[i].z * rs * gg.z, v[i].w * rs * gg.w);
      xr[j] = make_uint2(*reinterpret_cast<const uint32_t*>(&lo), *reinterpret_cast<const uint32_t*>(&hi));
    }
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
};

constexpr int kGemvMaxNormTok = 64;

// TOK: tokens accumulated per pass (1 for single-token decode: fewer live
// registers, more loads in flight; 8 otherwise).  RPW: weight rows per warp --
// 4 for wide layers, 1 for narrow ones (N < ~9.5k: the draft's o / down /
// qkv / gate_up), which gives 4x the warps so the per-SM load queue stays
// full; the 4 rows an epilogue needs (SwiGLU / RoPE pairs) are then gathered
// from 4 warps through shared memory.  Per-row arithmetic (chunk order, FMA
// order, xor tree) is identical for every TOK and RPW (batch invariance).
// The block-level body: block `bid` of a GEMV grid (also run by the draft's
// persistent forward, draft_fwd_kernel, one virtual block at a time -- same
// arithmetic, same bits).  Needs 8 warps; s_rs / s_out are the block's smem.
template <int TOK, int RPW>
__device__ __forceinline__ void gemv_block(const bf16* __restrict__ W, const bf16* __restrict__ X, int M, int N, int K,
                                           const EpiArgs& e, const GemvNorm& nrm, int bid, float* s_rs, float* s_out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
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
    __syncthreads();
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
              bf16x8_to_f32(__ldg(reinterpret_cast<const uint4*>(X + static_cast<size_t>(t0 + t) * K + k)), xv);
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
      __syncthreads();
      const int grp = threadIdx.x / TOK, t = threadIdx.x % TOK;  // (row quad, token)
      const int nq = bid * kGemvWarps + 4 * grp;
      if (grp < kGemvWarps / 4 && t < mt && nq < N) {
        float v[4] = {s_out[(4 * grp) * TOK + t], s_out[(4 * grp + 1) * TOK + t], s_out[(4 * grp + 2) * TOK + t],
                      s_out[(4 * grp + 3) * TOK + t]};
        epilogue4(e, t0 + t, nq, v, N);
      }
      __syncthreads();
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

// ---------------------------------------------------------------------------
// K4: causal attention of the window's M queries over the KV cache.
// One block per (query head h, window token); its 4 warps take 32-position chunks of the
// context round-robin (chunk c -> warp c % 4).  Within a warp lane j owns
// position c*32+j: it computes the full fixed-order q.k dot product for every
// window token, the warp reduces max / sum-of-exp with shuffles, and the
// exp-weighted V sum is accumulated with lanes over head dims.  Each warp
// keeps a running (max, sum, o) per token over its chunks (online softmax in
// chunk order); the block then merges the 4 warps' states in warp order.
// Every step depends only on the token's own position and the cache, never
// on how many tokens share the launch (batch invariance), and there is no
// inter-block communication.
// ---------------------------------------------------------------------------
constexpr int kAttnWarps = 4;  // == the persistent kernel's epilogue warps (identical arithmetic)
constexpr int kAttnLanesPos = 32;  // positions per warp chunk
constexpr int kAttnMaxTokens = 16; // window tokens per block: AttnArgs::tpb <= this

struct AttnArgs {
  const bf16* q;      // [M, H, hd]
  const bf16* kc;     // layer cache [max_seq, KV, hd]
  const bf16* vc;
  bf16* o;            // [M, H, hd]
  const int32_t* pos;
  int pos_add, M, H, KV, hd;
  int tpb;            // window tokens per block (shares each K/V chunk load; no effect on the arithmetic)
  float scale;
  const int32_t* tok_pos;   // slot mode (tpb == 1): per-token position and KV slot
  const int32_t* tok_slot;
  long long slot_stride;
};

// Block-level body for head h, token group tg; run by warps 0..3 of the
// block (named barrier 2 over those 128 threads), also from the draft's
// persistent forward.
__device__ __forceinline__ void attn_bar() { asm volatile("bar.sync 2, 128;" ::: "memory"); }

template <int HD>
__device__ __forceinline__ void attention_block(AttnArgs a, int h, int tg, unsigned char* attn_smem) {
  constexpr int PER = HD / 32;  // dims per lane (2 or 4)
  const int t0 = tg * a.tpb;                          // first window token of this block
  const int MT = min(a.tpb, a.M - t0);                // tokens handled here
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int p0 = a.tok_pos ? a.tok_pos[t0] : *a.pos + a.pos_add + t0;  // position of the block's first token
  const int ctx_max = p0 + MT;
  const int n_chunks = (ctx_max + kAttnLanesPos - 1) / kAttnLanesPos;
  const int kvh = h / (a.H / a.KV);
  const size_t kstride = static_cast<size_t>(a.KV) * HD;
  if (a.tok_slot) {  // slot mode: this token's own sequence cache
    const size_t so = static_cast<size_t>(a.tok_slot[t0]) * static_cast<size_t>(a.slot_stride);
    a.kc += so;
    a.vc += so;
  }
  // per-warp state [M][HD + 2] in smem: o (HD), m, l
  float* st_all = reinterpret_cast<float*>(attn_smem);
  float* st = st_all + static_cast<size_t>(warp) * MT * (HD + 2);
  bf16* Qs = reinterpret_cast<bf16*>(st_all + static_cast<size_t>(kAttnWarps) * a.tpb * (HD + 2));  // [MT][HD]
  bf16* Vw = Qs + a.tpb * HD + static_cast<size_t>(warp) * kAttnLanesPos * HD;  // this warp's V chunk
  for (int i = threadIdx.x; i < MT * HD / 8; i += kAttnWarps * 32) {
    const int t = i / (HD / 8), v = i % (HD / 8);
    reinterpret_cast<uint4*>(Qs + t * HD)[v] =
        *reinterpret_cast<const uint4*>(a.q + (static_cast<size_t>(t0 + t) * a.H + h) * HD + v * 8);
  }
  for (int i = lane; i < MT * (HD + 2); i += 32) st[i] = (i % (HD + 2) == HD) ? -INFINITY : 0.f;
  attn_bar();
  for (int c = warp; c < n_chunks; c += kAttnWarps) {
    const int j = c * kAttnLanesPos + lane;  // this lane's position
    const bool have = j < ctx_max;
    // K row of position j and the chunk's V rows (flat 16-byte pieces
    // lane + 32 k) into registers, all loads in flight; V then to smem
    uint4 kr[HD / 8], vr[HD / 8];
#pragma unroll
    for (int v = 0; v < HD / 8; ++v)
      kr[v] = have ? *reinterpret_cast<const uint4*>(a.kc + j * kstride + kvh * HD + v * 8) : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int k = 0; k < HD / 8; ++k) {
      const int i = lane + 32 * k;
      const int jp = c * kAttnLanesPos + i / (HD / 8);
      vr[k] = jp < ctx_max ? *reinterpret_cast<const uint4*>(a.vc + jp * kstride + kvh * HD + (i % (HD / 8)) * 8)
                           : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int k = 0; k < HD / 8; ++k) {
      const int i = lane + 32 * k;
      reinterpret_cast<uint4*>(Vw + (i / (HD / 8)) * HD)[i % (HD / 8)] = vr[k];
    }
    __syncwarp();
    for (int t = 0; t < MT; ++t) {
      const int pt = p0 + t;
      if (c * kAttnLanesPos > pt) continue;  // chunk lies beyond this token's causal range
      const bf16* qr = Qs + t * HD;
      float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int v = 0; v < HD / 8; ++v) {
        const uint4 qv = *reinterpret_cast<const uint4*>(qr + v * 8);
        const uint32_t qw[4] = {qv.x, qv.y, qv.z, qv.w}, kw[4] = {kr[v].x, kr[v].y, kr[v].z, kr[v].w};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          acc[u] = fmaf(__uint_as_float(qw[u] << 16), __uint_as_float(kw[u] << 16), acc[u]);
          acc[u] = fmaf(__uint_as_float(qw[u] & 0xffff0000u), __uint_as_float(kw[u] & 0xffff0000u), acc[u]);
        }
      }
      const bool valid = have && j <= pt;
      const float s = valid ? ((acc[0] + acc[1]) + (acc[2] + acc[3])) * a.scale : -INFINITY;
      // chunk max (fixed xor tree)
      float cm = s;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) cm = fmaxf(cm, __shfl_xor_sync(0xffffffffu, cm, o));
      float* sr = st + t * (HD + 2);
      const float m_old = sr[HD];
      const float m_new = fmaxf(m_old, cm);
      const float p = valid ? expf(s - m_new) : 0.f;
      float ps = p;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) ps += __shfl_xor_sync(0xffffffffu, ps, o);
      const float corr = (m_old == -INFINITY) ? 0.f : expf(m_old - m_new);
      // o[d] = corr * o[d] + sum_j p_j v_j[d], lanes over dims, positions in order
      float ov[PER];
#pragma unroll
      for (int e = 0; e < PER; ++e) ov[e] = 0.f;
      const int jn = min(kAttnLanesPos, pt + 1 - c * kAttnLanesPos);
#pragma unroll 8
      for (int jj = 0; jj < jn; ++jj) {
        const float pj = __shfl_sync(0xffffffffu, p, jj);
        const bf16* vr = Vw + jj * HD + lane * PER;
        if (PER == 4) {
          const uint2 vv = *reinterpret_cast<const uint2*>(vr);
          ov[0] = fmaf(pj, __uint_as_float(vv.x << 16), ov[0]);
          ov[1] = fmaf(pj, __uint_as_float(vv.x & 0xffff0000u), ov[1]);
          ov[2 % PER] = fmaf(pj, __uint_as_float(vv.y << 16), ov[2 % PER]);
          ov[3 % PER] = fmaf(pj, __uint_as_float(vv.y & 0xffff0000u), ov[3 % PER]);
        } else {
          const uint32_t vv = *reinterpret_cast<const uint32_t*>(vr);
          ov[0] = fmaf(pj, __uint_as_float(vv << 16), ov[0]);
          ov[1 % PER] = fmaf(pj, __uint_as_float(vv & 0xffff0000u), ov[1 % PER]);
        }
      }
#pragma unroll
      for (int e = 0; e < PER; ++e) sr[lane * PER + e] = fmaf(corr, sr[lane * PER + e], ov[e]);
      __syncwarp();
      if (lane == 0) {
        sr[HD] = m_new;
        sr[HD + 1] = fmaf(corr, sr[HD + 1], ps);
      }
      __syncwarp();
    }
    __syncwarp();  // Vw is overwritten by the warp's next chunk
  }
  attn_bar();
  // merge the warps' states in warp order
  for (int i = threadIdx.x; i < MT * HD; i += kAttnWarps * 32) {
    const int t = i / HD, d = i % HD;
    float mx = -INFINITY;
#pragma unroll
    for (int w = 0; w < kAttnWarps; ++w) mx = fmaxf(mx, st_all[(static_cast<size_t>(w) * MT + t) * (HD + 2) + HD]);
    float L = 0.f, O = 0.f;
#pragma unroll
    for (int w = 0; w < kAttnWarps; ++w) {
      const float* sr = st_all + (static_cast<size_t>(w) * MT + t) * (HD + 2);
      if (sr[HD] != -INFINITY) {
        const float wt = expf(sr[HD] - mx);
        L = fmaf(wt, sr[HD + 1], L);
        O = fmaf(wt, sr[d], O);
      }
    }
    a.o[(static_cast<size_t>(t0 + t) * a.H + h) * HD + d] = __float2bfloat16(O / L);
  }
}

template <int HD>
__global__ void __launch_bounds__(kAttnWarps * 32, 2) attention_kernel(AttnArgs a) {
  extern __shared__ __align__(16) unsigned char attn_smem[];
  pdl_wait();
  pdl_trigger();
  attention_block<HD>(a, blockIdx.x, blockIdx.y, attn_smem);
}

size_t attention_smem_bytes(int tpb, int hd) {
  return static_cast<size_t>(kAttnWarps) * tpb * (hd + 2) * 4 + static_cast<size_t>(tpb) * hd * 2 +
         static_cast<size_t>(kAttnWarps) * kAttnLanesPos * hd * 2 + 64;
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
namespace {

int attention_tpb(int M, int H) {
  static const int forced = [] {
    const char* v = std::getenv("PEARL_ATTN_TPB");
    return v ? std::atoi(v) : 0;
  }();
  int t = forced > 0 ? forced : (M * H + 295) / 296;  // ~2 blocks per SM (measured best, llama2-7b)
  return std::max(1, std::min({t, kAttnMaxTokens, M}));
}

int launch_gemv(const bf16* W, const bf16* X, int M, int N, int K, const EpiArgs& e, cudaStream_t st,
                GemvNorm nrm = GemvNorm{nullptr, nullptr, 0.f}) {
  // narrow layers: one row per warp (4x the warps; same per-row arithmetic)
  const bool narrow = (N + kGemvWarps * kGemvRows - 1) / (kGemvWarps * kGemvRows) < 296;
  const dim3 block(kGemvWarps * 32);
  if (narrow) {
    const dim3 grid((N + kGemvWarps - 1) / kGemvWarps);
    if (M == 1) return launch_pdl(gemv_kernel<1, 1>, grid, block, 0, st, W, X, M, N, K, e, nrm);
    return launch_pdl(gemv_kernel<8, 1>, grid, block, 0, st, W, X, M, N, K, e, nrm);
  }
  const dim3 grid((N + kGemvWarps * kGemvRows - 1) / (kGemvWarps * kGemvRows));
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

// Diagnostics only (PEARL_ABLATE=attn|norm|gemm): skip a kernel class to
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

// The persistent forward serves a call when PEARL_FWD_PERSISTENT is set, or
// for every eligible call with PEARL_MEGA=1.  Off by default: on B200 its
// software phase barriers cost more than the per-op kernels' launch gaps
// with programmatic dependent launch ("persistent forward").
static bool mega_default() {
  static const bool on = [] {
    const char* v = std::getenv("PEARL_MEGA");
    return v != nullptr && std::string(v) == "1";
  }();
  return on;
}

// Experiment bits of the persistent kernel (PEARL_MEGA_OPTS).
static int mega_opts() {
  static const int o = [] {
    const char* v = std::getenv("PEARL_MEGA_OPTS");
    return v ? std::atoi(v) : 0;
  }();
  return o;
}

// Diagnostics only (PEARL_STOP=k): run only the first k ops / phases of a
// forward (embed, then per layer norm, qkv, attn, o, norm, gate_up, down,
// then final norm, lm_head), so both paths' intermediate buffers can be
// compared (pearl_llama_debug_buffer).
static int stop_after() {
  const char* v = std::getenv("PEARL_STOP");
  return v ? std::atoi(v) : -1;
}

int forward_chunk(Llama& m, const int32_t* tokens, int M, int32_t* pos, int pos_add, bool logits_all,
                  bool want_logits, float* logits, cudaStream_t st, bool use_mega, int adv_n = 0,
                  bool* advanced = nullptr, const int32_t* tok_slot = nullptr, const int32_t* tok_pos = nullptr) {
  if (tok_pos) use_mega = false;
  const int abl = ablate_mask();
  const int stop = stop_after();
  int n_ops = 0;
  auto halt = [&]() { return stop >= 0 && ++n_ops >= stop; };
  if (m.mega_ok && use_mega && !abl && !g_prof.on && M <= kMegaMaxTokens) {
    const int mode = !want_logits ? 0 : (logits_all ? 2 : 1);
    MegaArgs A{};
    A.phases = m.mg_phases + m.mg_off[M][mode];
    A.n_phases = stop >= 0 ? std::min(stop, m.mg_len[M][mode]) : m.mg_len[M][mode];
    A.maps = m.mg_maps;
    A.partials = m.tc.partials;
    A.tile_flags = m.tc.tile_flags;
    A.counter = m.mg_counter;
    A.tokens = tokens;
    A.pos = pos;
    A.pos_add = pos_add;
    A.logits = logits;
    A.trace = m.mg_trace;
    A.opts = mega_opts();
    return mega_launch(A, m.mega_grid, st);
  }
  const auto& c = m.cfg;
  const int d = c.d_model, hd = c.head_dim, H = c.n_heads, KV = c.n_kv_heads;
  const int nq = H * hd, nkv = KV * hd;
  int rc = launch_pdl(embed_kernel, dim3(M), dim3(256), 0, st, tokens, m.embed, m.h, d, c.vocab);
  if (rc) return rc;
  g_prof.mark(OP_EMBED, st);
  if (halt()) return PEARL_OK;
  const size_t slot_kv = static_cast<size_t>(c.max_seq) * nkv;
  const size_t layer_kv = static_cast<size_t>(std::max(1, c.n_slots)) * slot_kv;
  const float scale = 1.0f / sqrtf(static_cast<float>(hd));
  // tokens per attention block: ~2 blocks per SM, each
  // K/V chunk load shared by the block's tokens (PEARL_ATTN_TPB overrides)
  const int tpb = tok_pos ? 1 : attention_tpb(M, H);
  const size_t attn_smem = attention_smem_bytes(tpb, hd);
  // CUDA-core (draft) models fuse every RMSNorm into the consuming GEMV
  const bool fuse_norm = c.gemm_kind == PEARL_GEMM_CUDACORE;
  for (int l = 0; l < c.n_layers; ++l) {
    const LayerW& L = m.layers[l];
    if (!(abl & 2) && !fuse_norm) {
      rc = launch_pdl(rmsnorm_kernel, dim3(M), dim3(kNormThreads), 0, st, m.h, L.attn_norm, m.x, d, c.norm_eps, 0);
      if (rc) return rc;
      g_prof.mark(OP_NORM, st);
  if (halt()) return PEARL_OK;
    }
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
    rc = launch_gemm(m, L.wqkv, m.x, M, nq + 2 * nkv, d, e, st,
                     fuse_norm ? GemvNorm{m.h, L.attn_norm, c.norm_eps} : GemvNorm{nullptr, nullptr, 0.f});
    if (rc) return rc;
    g_prof.mark(OP_QKV, st);
  if (halt()) return PEARL_OK;
    AttnArgs aa{m.q, e.kc, e.vc, m.o, pos, pos_add, M, H, KV, hd, tpb, scale, tok_pos, tok_slot,
                static_cast<long long>(slot_kv)};
    if (abl & 1)
      rc = PEARL_OK;
    else if (hd == 128)
      rc = launch_pdl(attention_kernel<128>, dim3(H, (M + tpb - 1) / tpb), dim3(kAttnWarps * 32),
                      attn_smem, st, aa);
    else
      rc = launch_pdl(attention_kernel<64>, dim3(H, (M + tpb - 1) / tpb), dim3(kAttnWarps * 32),
                      attn_smem, st, aa);
    if (rc) return rc;
    g_prof.mark(OP_ATTN, st);
  if (halt()) return PEARL_OK;
    EpiArgs r{};
    r.kind = EPI_RESID;
    r.out_f32 = m.h;
    r.ld = d;
    rc = launch_gemm(m, L.wo, m.o, M, d, nq, r, st);
    if (rc) return rc;
    g_prof.mark(OP_O, st);
  if (halt()) return PEARL_OK;
    if (!(abl & 2) && !fuse_norm) {
      rc = launch_pdl(rmsnorm_kernel, dim3(M), dim3(kNormThreads), 0, st, m.h, L.mlp_norm, m.x, d, c.norm_eps, 0);
      if (rc) return rc;
      g_prof.mark(OP_NORM, st);
  if (halt()) return PEARL_OK;
    }
    EpiArgs g{};
    g.kind = EPI_SWIGLU;
    g.out_bf16 = m.act;
    g.ld = c.ffn;
    rc = launch_gemm(m, L.wgu, m.x, M, 2 * c.ffn, d, g, st,
                     fuse_norm ? GemvNorm{m.h, L.mlp_norm, c.norm_eps} : GemvNorm{nullptr, nullptr, 0.f});
    if (rc) return rc;
    g_prof.mark(OP_GU, st);
  if (halt()) return PEARL_OK;
    rc = launch_gemm(m, L.wdown, m.act, M, d, c.ffn, r, st);
    if (rc) return rc;
    g_prof.mark(OP_DOWN, st);
  if (halt()) return PEARL_OK;
  }
  if (!want_logits) return PEARL_OK;
  const int first = logits_all ? 0 : M - 1;
  const int rows = M - first;
  if (!fuse_norm) {
    rc = launch_pdl(rmsnorm_kernel, dim3(rows), dim3(kNormThreads), 0, st, m.h, m.final_norm, m.x, d, c.norm_eps,
                    first);
    if (rc) return rc;
    g_prof.mark(OP_NORM, st);
  if (halt()) return PEARL_OK;
  }
  EpiArgs s{};
  s.kind = EPI_STORE_F32;
  s.out_f32 = logits;
  s.ld = c.vocab;
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

std::once_flag g_attn_once;
cudaError_t g_attn_err = cudaSuccess;

// Phase lists of the persistent forward for every window size M <= 16 and
// logits mode (0 none, 1 last row, 2 all rows), mirroring forward_chunk op
// for op: same weights, same epilogues, same stream-K grid (num_sms), so the
// two paths produce identical bits.
int build_mega_plans(Llama& m) {
  const auto& c = m.cfg;
  if (c.gemm_kind != PEARL_GEMM_TCGEN05) return PEARL_OK;
  int per_sm = 0;
  PEARL_CUDA_TRY(mega_prepare());
  PEARL_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, mega_kernel_ptr(), mega_threads(),
                                                               mega_smem_bytes()));
  if (per_sm < 1) return PEARL_OK;
  const int G = m.tc.num_sms;
  const int d = c.d_model, hd = c.head_dim, H = c.n_heads, KV = c.n_kv_heads, L = c.n_layers;
  const int nq = H * hd, nkv = KV * hd;
  const size_t layer_kv = static_cast<size_t>(std::max(1, c.n_slots)) * c.max_seq * nkv;  // slot 0
  const int n_w = 4 * L + 1;
  const int Mmax = std::min(kMegaMaxTokens, c.max_tokens);
  std::vector<MegaMap> maps(static_cast<size_t>(n_w) + 4 * 16);
  const int wq[5][2] = {{nq + 2 * nkv, d}, {d, nq}, {2 * c.ffn, d}, {d, c.ffn}, {c.vocab, d}};
  for (int l = 0; l < L; ++l) {
    const LayerW& Lw = m.layers[l];
    const bf16* ws[4] = {Lw.wqkv, Lw.wo, Lw.wgu, Lw.wdown};
    for (int k = 0; k < 4; ++k) {
      int rc = tc_encode_2d(&maps[4 * l + k].map, ws[k], wq[k][1], wq[k][0], kMegaTileN);
      if (rc) return rc;
    }
  }
  int rc = tc_encode_2d(&maps[4 * L].map, m.lm_head, d, c.vocab, kMegaTileN);
  if (rc) return rc;
  auto xmap = [&](int M, int k) { return n_w + 4 * (M - 1) + k; };  // k: 0 x, 1 o, 2 act, 3 x last row
  for (int M = 1; M <= Mmax; ++M) {
    if ((rc = tc_encode_2d(&maps[xmap(M, 0)].map, m.x, d, M, kMegaMaxTokens))) return rc;
    if ((rc = tc_encode_2d(&maps[xmap(M, 1)].map, m.o, nq, M, kMegaMaxTokens))) return rc;
    if ((rc = tc_encode_2d(&maps[xmap(M, 2)].map, m.act, c.ffn, M, kMegaMaxTokens))) return rc;
    if ((rc = tc_encode_2d(&maps[xmap(M, 3)].map, m.x + static_cast<size_t>(M - 1) * d, d, 1, kMegaMaxTokens)))
      return rc;
  }
  std::vector<MegaPhase> all;
  auto gemm = [&](int M, int wmap, int xm, int N, int K, const EpiArgs& e) {
    MegaPhase p{};
    p.kind = MG_GEMM;
    p.M = M;
    p.N = N;
    p.K = K;
    p.KB = (K + kMegaTileK - 1) / kMegaTileK;
    const int tiles = (N + kMegaTileN - 1) / kMegaTileN;
    p.T = static_cast<long long>(tiles) * p.KB;
    p.seg_max = tc_seg_max(tiles, p.KB, static_cast<int>(std::min<long long>(G, p.T)));
    p.map_w = wmap;
    p.map_x = xm;
    p.e = e;
    all.push_back(p);
  };
  auto norm = [&](int M, const float* gain, int row0) {
    MegaPhase p{};
    p.kind = MG_NORM;
    p.M = M;
    p.h = m.h;
    p.gain = gain;
    p.xout = m.x;
    p.d = d;
    p.row0 = row0;
    p.eps = c.norm_eps;
    all.push_back(p);
  };
  const float scale = 1.0f / sqrtf(static_cast<float>(hd));
  for (int M = 1; M <= Mmax; ++M) {
    for (int mode = 0; mode < 3; ++mode) {
      m.mg_off[M][mode] = static_cast<int>(all.size());
      MegaPhase pe{};
      pe.kind = MG_EMBED;
      pe.M = M;
      pe.h = m.h;
      pe.d = d;
      pe.embed = m.embed;
      pe.V = c.vocab;
      all.push_back(pe);
      for (int l = 0; l < L; ++l) {
        const LayerW& Lw = m.layers[l];
        norm(M, Lw.attn_norm, 0);
        EpiArgs e{};
        e.kind = EPI_QKV;
        e.out_bf16 = m.q;
        e.kc = m.kcache + l * layer_kv;
        e.vc = m.vcache + l * layer_kv;
        e.cos_t = m.rope_cos;
        e.sin_t = m.rope_sin;
        e.n_q = nq;
        e.n_kv = nkv;
        e.hd = hd;
        gemm(M, 4 * l + 0, xmap(M, 0), nq + 2 * nkv, d, e);
        all.back().e_uses_pos = 1;
        MegaPhase pa{};
        pa.kind = MG_ATTN;
        pa.M = M;
        pa.q = m.q;
        pa.kc = e.kc;
        pa.vc = e.vc;
        pa.o = m.o;
        pa.H = H;
        pa.KV = KV;
        pa.hd = hd;
        pa.scale = scale;
        all.push_back(pa);
        EpiArgs r{};
        r.kind = EPI_RESID;
        r.out_f32 = m.h;
        r.ld = d;
        gemm(M, 4 * l + 1, xmap(M, 1), d, nq, r);
        norm(M, Lw.mlp_norm, 0);
        EpiArgs g{};
        g.kind = EPI_SWIGLU;
        g.out_bf16 = m.act;
        g.ld = c.ffn;
        gemm(M, 4 * l + 2, xmap(M, 0), 2 * c.ffn, d, g);
        gemm(M, 4 * l + 3, xmap(M, 2), d, c.ffn, r);
      }
      if (mode > 0) {
        const int first = mode == 2 ? 0 : M - 1;
        norm(M, m.final_norm, first);
        EpiArgs s{};
        s.kind = EPI_STORE_F32;
        s.ld = c.vocab;
        gemm(M - first, 4 * L, mode == 2 ? xmap(M, 0) : xmap(M, 3), c.vocab, d, s);
        all.back().e_is_logits = 1;
      }
      m.mg_len[M][mode] = static_cast<int>(all.size()) - m.mg_off[M][mode];
    }
  }
  for (const MegaPhase& p : all)
    if (p.kind == MG_GEMM) {
      const int tiles = static_cast<int>(p.T / p.KB);
      if (static_cast<size_t>(tiles) * p.seg_max * kMegaTileN * kMegaPartialTok > m.tc.partial_floats ||
          tiles > m.tc.n_flags) {
        set_error("persistent forward: shape exceeds the planned split-K workspace");
        return PEARL_ERR_ARG;
      }
    }
  PEARL_CUDA_TRY(cudaMalloc(&m.mg_maps, maps.size() * sizeof(MegaMap)));
  PEARL_CUDA_TRY(cudaMemcpy(m.mg_maps, maps.data(), maps.size() * sizeof(MegaMap), cudaMemcpyHostToDevice));
  PEARL_CUDA_TRY(cudaMalloc(&m.mg_phases, all.size() * sizeof(MegaPhase)));
  PEARL_CUDA_TRY(cudaMemcpy(m.mg_phases, all.data(), all.size() * sizeof(MegaPhase), cudaMemcpyHostToDevice));
  int max_len = 0;
  for (int M = 1; M <= Mmax; ++M)
    for (int mode = 0; mode < 3; ++mode) max_len = std::max(max_len, m.mg_len[M][mode]);
  const size_t ctr_bytes = static_cast<size_t>(max_len) * kMegaCtrStride * sizeof(unsigned);
  PEARL_CUDA_TRY(cudaMalloc(&m.mg_counter, ctr_bytes));
  PEARL_CUDA_TRY(cudaMemset(m.mg_counter, 0, ctr_bytes));
  m.mega_grid = G;
  m.mega_ok = true;
  return PEARL_OK;
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
  PEARL_ARG_CHECK(c.d_model <= 4 * kNormThreads * kNormVec, "d_model too large for the norm kernel");
  PEARL_ARG_CHECK(c.gemm_kind != PEARL_GEMM_CUDACORE || (c.max_tokens <= kGemvMaxNormTok && c.d_model % 256 == 0),
                  "CUDA-core models need max_tokens <= 64 and d_model % 256 == 0 (fused norm)");
  PEARL_ARG_CHECK(c.max_tokens >= 1 && c.max_tokens <= (c.gemm_kind == PEARL_GEMM_TCGEN05 ? 128 : 64),
                  "max_tokens in [1, 128] (tcgen05) / [1, 64] (CUDA-core)");
  PEARL_ARG_CHECK(c.max_seq >= 1 && c.max_seq <= 4096, "max_seq in [1, 4096]");
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
  std::call_once(g_attn_once, [] {
    g_attn_err = cudaFuncSetAttribute(attention_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(attention_smem_bytes(kAttnMaxTokens, 128)));
    if (g_attn_err == cudaSuccess)
      g_attn_err = cudaFuncSetAttribute(attention_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(attention_smem_bytes(kAttnMaxTokens, 64)));
  });
  if (g_attn_err) return fail(g_attn_err);
  if (c.gemm_kind == PEARL_GEMM_TCGEN05) {
    int rc = tc_init(m->tc, c);
    if (!rc) rc = build_mega_plans(*m);
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
  if (m->mg_maps) cudaFree(m->mg_maps);
  if (m->mg_phases) cudaFree(m->mg_phases);
  if (m->mg_counter) cudaFree(m->mg_counter);
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
  if (kind == PEARL_GEMM_CUDACORE)
    return launch_gemv(static_cast<const bf16*>(W), static_cast<const bf16*>(X), M, N, K, e, st);
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
  struct WindowScope {
    explicit WindowScope(const L2Window& w) { g_l2win = w; }
    ~WindowScope() { g_l2win = L2Window{}; }
  } window_scope(m->l2win);
  bool advanced = false;
  for (int c0 = 0; c0 < n_tokens; c0 += T) {
    const int mt = std::min(T, n_tokens - c0);
    const bool last_chunk = c0 + mt == n_tokens;
    int rc = forward_chunk(*m, tokens + c0, mt, pos, c0, !last_only, last_chunk && logits != nullptr, logits, st,
                           (flags & PEARL_FWD_PERSISTENT) != 0 || mega_default(),
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
                           logits ? logits + static_cast<size_t>(c0) * m->cfg.vocab : nullptr, st, false, 0, nullptr,
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
  const void* src[7] = {m->h, m->x, m->q, m->o, m->act, m->tc.tile_flags, m->mg_counter};
  PEARL_CUDA_TRY(cudaMemcpyAsync(dst, src[which], bytes, cudaMemcpyDeviceToDevice, static_cast<cudaStream_t>(stream)));
  return PEARL_OK;
}

// Diagnostic: one persistent-kernel forward with per-CTA phase timestamps.
// out[3p + 0] = phase kind, out[3p + 1] = us until the last CTA finished
// phase p, out[3p + 2] = us until the first CTA finished it (both from the
// earliest CTA start).  Returns the phase count (or a negative error).
extern "C" int pearl_llama_mega_trace(void* handle, const int32_t* tokens, int n_tokens, int32_t* pos, int flags,
                                      float* logits, float* out, int max_phases, void* stream) {
  Llama* m = static_cast<Llama*>(handle);
  PEARL_ARG_CHECK(m && tokens && pos && out && n_tokens >= 1, "bad trace arguments");
  PEARL_ARG_CHECK(m->mega_ok && n_tokens <= std::min(kMegaMaxTokens, m->cfg.max_tokens), "persistent forward not used");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int mode = logits == nullptr ? 0 : ((flags & PEARL_FWD_LAST_LOGITS) ? 1 : 2);
  const int np = m->mg_len[n_tokens][mode];
  const int G = m->mega_grid;
  PEARL_ARG_CHECK(np <= max_phases, "max_phases too small");
  const size_t n = static_cast<size_t>(np + 1) * G;
  PEARL_CUDA_TRY(cudaStreamSynchronize(st));
  PEARL_CUDA_TRY(cudaMalloc(&m->mg_trace, n * sizeof(unsigned long long)));
  int rc = forward_chunk(*m, tokens, n_tokens, pos, 0, mode == 2, mode != 0, logits, st, true);
  std::vector<unsigned long long> h(n);
  cudaError_t e = cudaStreamSynchronize(st);
  if (e == cudaSuccess) e = cudaMemcpy(h.data(), m->mg_trace, n * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  cudaFree(m->mg_trace);
  m->mg_trace = nullptr;
  if (rc) return rc;
  PEARL_CUDA_TRY(e);
  std::vector<MegaPhase> ph(np);
  PEARL_CUDA_TRY(cudaMemcpy(ph.data(), m->mg_phases + m->mg_off[n_tokens][mode], np * sizeof(MegaPhase),
                            cudaMemcpyDeviceToHost));
  unsigned long long t0 = ~0ull;
  for (int b = 0; b < G; ++b) t0 = std::min(t0, h[static_cast<size_t>(np) * G + b]);
  for (int p = 0; p < np; ++p) {
    unsigned long long lo = ~0ull, hi = 0;
    for (int b = 0; b < G; ++b) {
      lo = std::min(lo, h[static_cast<size_t>(p) * G + b]);
      hi = std::max(hi, h[static_cast<size_t>(p) * G + b]);
    }
    out[3 * p] = static_cast<float>(ph[p].kind);
    out[3 * p + 1] = static_cast<float>(hi - t0) * 1e-3f;
    out[3 * p + 2] = static_cast<float>(lo - t0) * 1e-3f;
  }
  return np;
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
