// K4: split-KV, GQA-grouped causal attention (see attention.cuh).
#include "attention.cuh"

#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "common.h"

namespace pearl {

namespace cg = cooperative_groups;
using bf16 = __nv_bfloat16;

namespace {

constexpr int kWarps = kAttnThreads / 32;



__device__ __forceinline__ int tok_position(const AttnArgs& a, int p0, int t) {
  return a.tok_pos ? a.tok_pos[t] : p0 + t;
}

template <int HD>
struct AttnSmem {
  static constexpr size_t kBytes =
      (static_cast<size_t>(kWarps + 1) * kAttnMaxRb * (HD + 2) + kAttnMaxRb * kWarps +
       kAttnMaxRb * kAttnCluster + kAttnMaxRb) * 4 + 64;
};

__device__ __forceinline__ uint32_t word(const uint4& u, int w) {
  return w == 0 ? u.x : (w == 1 ? u.y : (w == 2 ? u.z : u.w));
}

__device__ __forceinline__ void mma_bf16(float* c, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t trans8x8(uint32_t x) {
  uint32_t y;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&v);
}

// Register layout of a warp's 32-position segment (lane = 4 n + q):
//   kb[nt][j] = K[P0 + 8 nt + n][32 j + 8 q .. +7]  (16 bytes)
//   vb[i][j]  = V[P0 + 8 i  + n][32 j + 8 q .. +7]
// The q.k contraction runs over a PERMUTED head-dim order -- for k-step
// 2j + h the fragment's logical k = 2q + {0,1} / 2q + 8 + {0,1} is the
// physical dim 32 j + 8 q + 4 h + {0,1} / {2,3} -- applied identically to Q
// and K, so every fragment is one 16-byte load.  p.v's output dims are
// permuted the same way (logical tile c = 4 j + w, pair 2q + e <-> physical
// 32 j + 8 q + 2 w + e), and V's 8x8 blocks are transposed in registers
// (movmatrix) into the B-fragment layout.
template <int HD>
__device__ __forceinline__ void load_kv(const bf16* kc, const bf16* vc, size_t kvs, int P0, int lane, int lo, int hi,
                                        uint4 (*kb)[HD / 32], uint4 (*vb)[HD / 32]) {
  constexpr int J = HD / 32;
  const int n = lane >> 2, q = lane & 3;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int P = P0 + 8 * i + n;
    if (P >= lo && P <= hi) {
#pragma unroll
      for (int j = 0; j < J; ++j) {
        kb[i][j] = *reinterpret_cast<const uint4*>(kc + static_cast<size_t>(P) * kvs + 32 * j + 8 * q);
        vb[i][j] = *reinterpret_cast<const uint4*>(vc + static_cast<size_t>(P) * kvs + 32 * j + 8 * q);
      }
    }
  }
}

template <int HD, int MINB>
__global__ void __launch_bounds__(kAttnThreads, MINB) attn_kernel(AttnArgs a) {
  constexpr int J = HD / 32;    // 32-dim blocks
  constexpr int KS = HD / 16;   // q.k k-steps
  constexpr int NO = HD / 8;    // p.v output tiles
  constexpr int RS = HD + 2;    // state row: o[HD], m, l
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float* st = reinterpret_cast<float*>(smem_raw);          // [kWarps][kAttnMaxRb][RS] warp states
  float* cs = st + kWarps * kAttnMaxRb * RS;               // [kAttnMaxRb][RS] this CTA's folded state
  float* wgt = cs + kAttnMaxRb * RS;                       // fold weights / sums
  cg::cluster_group cluster = cg::this_cluster();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n = lane >> 2, q = lane & 3;
  const int crank = static_cast<int>(cluster.block_rank());
  const int CS = static_cast<int>(cluster.num_blocks());  // CTAs per (row block, KV head)
  const int g = a.H / a.KV;
  const int tpb = a.tpb;  // tokens per row block (tpb * g <= 16 rows)
  const bool seq_mode = a.tok_pos == nullptr;
  // Row blocks: runs of consecutive tokens sharing a KV slot (sequence mode:
  // one run), cut into chunks of tpb tokens.  Every CTA derives the same
  // table; tok_slot / tok_pos / *pos were written before this forward began
  // (its embedding kernel waited for them), so this runs before the wait.
  __shared__ int s_bstart[kAttnMaxTok + 1];
  __shared__ int s_nblk;
  if (seq_mode) {
    if (threadIdx.x == 0) s_nblk = (a.M + tpb - 1) / tpb;
  } else if (warp == 0) {
    int nb = 0, rs = 0, prev = -1;
    for (int c0 = 0; c0 < a.M; c0 += 32) {
      const int t = c0 + lane;
      const int sl = t < a.M ? a.tok_slot[t] : -2;
      int up = __shfl_up_sync(0xffffffffu, sl, 1);
      if (lane == 0) up = prev;
      const bool run0 = t < a.M && (t == 0 || sl != up);
      const unsigned rm = __ballot_sync(0xffffffffu, run0) & (0xffffffffu >> (31 - lane));
      const int my_rs = rm ? c0 + 31 - __clz(rm) : rs;  // this token's run start
      const bool bs = t < a.M && (t - my_rs) % tpb == 0;
      const unsigned bm = __ballot_sync(0xffffffffu, bs);
      if (bs) s_bstart[nb + __popc(bm & ((1u << lane) - 1))] = t;
      nb += __popc(bm);
      rs = __shfl_sync(0xffffffffu, my_rs, 31);
      prev = __shfl_sync(0xffffffffu, sl, 31);
    }
    if (lane == 0) {
      s_nblk = nb;
      s_bstart[nb] = a.M;
    }
  }
  __syncthreads();
  const int nblk = s_nblk;
  const int p0 = seq_mode ? *a.pos + a.pos_add : 0;
  const size_t kvs = static_cast<size_t>(a.KV) * HD;  // elements per cache position
  const int nclus = gridDim.x / CS;
  bool first = true;
  for (int item = blockIdx.x / CS; item < nblk * a.KV; item += nclus) {
  const int b = item / a.KV, kvh = item % a.KV;
  const int t0 = seq_mode ? b * tpb : s_bstart[b];
  const int t1 = seq_mode ? min(t0 + tpb, a.M) : s_bstart[b + 1];
  const int r0 = t0 * g, r1 = t1 * g, R = r1 - r0;
  const int pmax = tok_position(a, p0, t1 - 1);
  const size_t so = a.tok_slot ? static_cast<size_t>(a.tok_slot[t0]) * static_cast<size_t>(a.slot_stride) : 0;
  const bf16* kc = a.kc + so + static_cast<size_t>(kvh) * HD;
  const bf16* vc = a.vc + so + static_cast<size_t>(kvh) * HD;
  // segment js of this warp: 32 positions at 32 ((js CS + crank) 4 + warp)
  auto seg_p0 = [&](int js) { return 32 * ((js * CS + crank) * kWarps + warp); };

  uint4 kb[4][J], vb[4][J];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < J; ++j) kb[i][j] = vb[i][j] = make_uint4(0, 0, 0, 0);
  const int old_hi = (seq_mode && first) ? min(p0, pmax + 1) - 1 : -1;  // last position loadable before the wait
  if (first) {
    if (seg_p0(0) <= pmax) load_kv<HD>(kc, vc, kvs, seg_p0(0), lane, 0, old_hi, kb, vb);
    // later segments' old positions: warm L2 while the QKV GEMM drains
    for (int js = 1; js < a.spw; ++js) {
      const int P = seg_p0(js) + lane;
      if (P <= old_hi) {
        const bf16* kr = kc + static_cast<size_t>(P) * kvs;
        const bf16* vr = vc + static_cast<size_t>(P) * kvs;
#pragma unroll
        for (int o = 0; o < HD * 2; o += 128) {
          asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const char*>(kr) + o));
          asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const char*>(vr) + o));
        }
      }
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  }

  // query rows lo = n, hi = n + 8 of the 16-row tile (rows >= R are zero)
  uint4 qa[2][J];
  int prow[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int rr = n + 8 * h, r = r0 + rr;
    prow[h] = rr < R ? tok_position(a, p0, r / g) : -1;
#pragma unroll
    for (int j = 0; j < J; ++j) qa[h][j] = make_uint4(0, 0, 0, 0);
    if (rr < R && seg_p0(0) <= pmax) {
      const bf16* qr = a.q + (static_cast<size_t>(r / g) * a.H + kvh * g + r % g) * HD;
#pragma unroll
      for (int j = 0; j < J; ++j) qa[h][j] = *reinterpret_cast<const uint4*>(qr + 32 * j + 8 * q);
    }
  }
  // this warp's running state for rows lo / hi: max, sum, o (NO tiles x 4)
  float mrun[2] = {-INFINITY, -INFINITY}, lrun[2] = {0.f, 0.f};
  float o[NO][4];
#pragma unroll
  for (int c = 0; c < NO; ++c) o[c][0] = o[c][1] = o[c][2] = o[c][3] = 0.f;
  // the warp's segments in js order: a row's own positions decide what
  // contributes, and segments past a row's position are exact no-ops for it
  // (corr = exp(0) = 1, p = 0), so the fold never depends on the other rows
  for (int js = 0; js < a.spw; ++js) {
    const int P0 = seg_p0(js);
    if (P0 > pmax) break;
    if (js > 0) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < J; ++j) kb[i][j] = vb[i][j] = make_uint4(0, 0, 0, 0);
    }
    load_kv<HD>(kc, vc, kvs, P0, lane, js == 0 ? old_hi + 1 : 0, pmax, kb, vb);
    // ---- s = q . k (16 rows x 32 positions), fp32 accumulate
    float sc[4][4];
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      sc[nt][0] = sc[nt][1] = sc[nt][2] = sc[nt][3] = 0.f;
#pragma unroll
      for (int kk = 0; kk < KS; ++kk) {
        const int j = kk >> 1, h = kk & 1;
        mma_bf16(sc[nt], word(qa[0][j], 2 * h), word(qa[1][j], 2 * h), word(qa[0][j], 2 * h + 1),
                 word(qa[1][j], 2 * h + 1), word(kb[nt][j], 2 * h), word(kb[nt][j], 2 * h + 1));
      }
    }
    // ---- online softmax per row (lo: sc[.][0..1], hi: sc[.][2..3]) over
    // positions P0 + 8 nt + 2 q + e; p rounded to bf16 (the p.v operand), l
    // summed from the rounded values in a fixed (nt, e) order, then the quad
    uint32_t pp[4][2];
    float corr[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      float m = -INFINITY;
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int P = P0 + 8 * nt + 2 * q + e;
          sc[nt][2 * h + e] = P <= prow[h] ? sc[nt][2 * h + e] * a.scale : -INFINITY;
          m = fmaxf(m, sc[nt][2 * h + e]);
        }
      m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 1));
      m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 2));
      const float mn = fmaxf(mrun[h], m);
      corr[h] = mrun[h] == -INFINITY ? 0.f : expf(mrun[h] - mn);
      float l = 0.f;
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        const float x0 = sc[nt][2 * h] == -INFINITY ? 0.f : expf(sc[nt][2 * h] - mn);
        const float x1 = sc[nt][2 * h + 1] == -INFINITY ? 0.f : expf(sc[nt][2 * h + 1] - mn);
        pp[nt][h] = pack_bf16(x0, x1);
        const __nv_bfloat162 pb = *reinterpret_cast<const __nv_bfloat162*>(&pp[nt][h]);
        l += __low2float(pb);
        l += __high2float(pb);
      }
      l += __shfl_xor_sync(0xffffffffu, l, 1);
      l += __shfl_xor_sync(0xffffffffu, l, 2);
      lrun[h] = fmaf(lrun[h], corr[h], l);
      mrun[h] = mn;
    }
    // ---- o = corr * o + p . v: k = 32 positions (2 steps), n = HD dims
#pragma unroll
    for (int c = 0; c < NO; ++c) {
      const int j = c >> 2, w = c & 3;
      float oc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int s2 = 0; s2 < 2; ++s2)
        mma_bf16(oc, pp[2 * s2][0], pp[2 * s2][1], pp[2 * s2 + 1][0], pp[2 * s2 + 1][1],
                 trans8x8(word(vb[2 * s2][j], w)), trans8x8(word(vb[2 * s2 + 1][j], w)));
      o[c][0] = fmaf(o[c][0], corr[0], oc[0]);
      o[c][1] = fmaf(o[c][1], corr[0], oc[1]);
      o[c][2] = fmaf(o[c][2], corr[1], oc[2]);
      o[c][3] = fmaf(o[c][3], corr[1], oc[3]);
    }
  }
  // warp state -> smem: logical dims 2q + {0,1} of tile c = physical 32 j + 8 q + 2 w + {0,1}
  float* sw = st + warp * kAttnMaxRb * RS;
#pragma unroll
  for (int c = 0; c < NO; ++c) {
    const int d = 32 * (c >> 2) + 8 * q + 2 * (c & 3);
    *reinterpret_cast<float2*>(sw + n * RS + d) = make_float2(o[c][0], o[c][1]);
    *reinterpret_cast<float2*>(sw + (n + 8) * RS + d) = make_float2(o[c][2], o[c][3]);
  }
  if (q == 0) {
    sw[n * RS + HD] = mrun[0];
    sw[n * RS + HD + 1] = lrun[0];
    sw[(n + 8) * RS + HD] = mrun[1];
    sw[(n + 8) * RS + HD + 1] = lrun[1];
  }
  __syncthreads();
  // CTA fold over its warps in warp order (weights exp(m_w - max), 0 = empty)
  if (threadIdx.x < R * kWarps) {
    const int rr = threadIdx.x / kWarps, w = threadIdx.x % kWarps;
    float mx = -INFINITY;
#pragma unroll
    for (int x = 0; x < kWarps; ++x) mx = fmaxf(mx, st[(x * kAttnMaxRb + rr) * RS + HD]);
    const float mw = st[(w * kAttnMaxRb + rr) * RS + HD];
    wgt[rr * kWarps + w] = mw == -INFINITY ? 0.f : expf(mw - mx);
    if (w == 0) cs[rr * RS + HD] = mx;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < R * (HD + 1); i += kAttnThreads) {
    const int rr = i / (HD + 1), d = i % (HD + 1);  // d == HD: the row's l
    const int col = d < HD ? d : HD + 1;
    float acc = 0.f;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      const float wt = wgt[rr * kWarps + w];
      if (wt != 0.f) acc = fmaf(wt, st[(w * kAttnMaxRb + rr) * RS + col], acc);
    }
    cs[rr * RS + col] = acc;
  }
  // cluster fold over the CTAs in rank order (DSMEM); CTA `crank` produces
  // head dims [crank * HD / CS, (crank + 1) * HD / CS) of every row.  A
  // single-CTA "cluster" (CS = 1) folds its own state the same way.
  if (CS > 1) cluster.sync(); else __syncthreads();
  const int DC = HD / CS;  // dims per CTA
  float* cw = wgt + kAttnMaxRb * kWarps;  // [R][kAttnCluster] weights, then [R] sums
  if (threadIdx.x < R * CS) {
    const int rr = threadIdx.x / CS, c = threadIdx.x % CS;
    float mx = -INFINITY;
    for (int x = 0; x < CS; ++x) mx = fmaxf(mx, cluster.map_shared_rank(cs, x)[rr * RS + HD]);
    const float mc = cluster.map_shared_rank(cs, c)[rr * RS + HD];
    cw[rr * kAttnCluster + c] = mc == -INFINITY ? 0.f : expf(mc - mx);
  }
  __syncthreads();
  if (threadIdx.x < R) {
    const int rr = threadIdx.x;
    float L = 0.f;
    for (int c = 0; c < CS; ++c) {
      const float wt = cw[rr * kAttnCluster + c];
      if (wt != 0.f) L = fmaf(wt, cluster.map_shared_rank(cs, c)[rr * RS + HD + 1], L);
    }
    cw[kAttnMaxRb * kAttnCluster + rr] = L;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < R * DC; i += kAttnThreads) {
    const int rr = i / DC, d = crank * DC + i % DC;
    float O = 0.f;
    for (int c = 0; c < CS; ++c) {
      const float wt = cw[rr * kAttnCluster + c];
      if (wt != 0.f) O = fmaf(wt, cluster.map_shared_rank(cs, c)[rr * RS + d], O);
    }
    const int r = r0 + rr, t = r / g, h = kvh * g + r % g;
    a.o[(static_cast<size_t>(t) * a.H + h) * HD + d] = __float2bfloat16(O / cw[kAttnMaxRb * kAttnCluster + rr]);
  }
  if (CS > 1) cluster.sync();  // the peers' states stay alive until every CTA has read them
  else __syncthreads();         // smem reuse by the next item
  first = false;
  }
  if (first) {  // no work for this cluster: still order after the producer
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  }
}

std::once_flag g_once;
cudaError_t g_err = cudaSuccess;

}  // namespace

int attn_init() {
  std::call_once(g_once, [] {
    g_err = cudaFuncSetAttribute(attn_kernel<128, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(AttnSmem<128>::kBytes));
    if (g_err == cudaSuccess)
      g_err = cudaFuncSetAttribute(attn_kernel<128, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(AttnSmem<128>::kBytes));
    if (g_err == cudaSuccess)
      g_err = cudaFuncSetAttribute(attn_kernel<64, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(AttnSmem<64>::kBytes));
    if (g_err == cudaSuccess)
      g_err = cudaFuncSetAttribute(attn_kernel<64, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(AttnSmem<64>::kBytes));
  });
  PEARL_CUDA_TRY(g_err);
  return PEARL_OK;
}

int attn_cluster_size(bool slot_mode) {
  // slot mode (batched sequences): many short token runs, one item each --
  // single-CTA clusters keep every item's latency chain short
  if (slot_mode) return 1;
  static const int cs = [] {
    const char* v = std::getenv("PEARL_ATTN_CLUSTER");
    const int x = v ? std::atoi(v) : kAttnClusterDefault;
    return (x == 1 || x == 2 || x == 4 || x == 8) ? x : kAttnClusterDefault;
  }();
  return cs;
}

static int attn_minb() {
  static const int m = [] {
    const char* v = std::getenv("PEARL_ATTN_MINB");
    return v && std::atoi(v) == 3 ? 3 : 2;
  }();
  return m;
}

void attn_plan(const AttnShape& s, int* tpb, int* spw, int* grid) {
  const int g = s.H / s.KV;
  // tokens per row block: one 16-row MMA tile of (token, query head) rows
  *tpb = std::max(1, kAttnMaxRb / g);
  // segments per warp: the cluster's CS CTAs x 4 warps cover the whole
  // cache in spw rounds of 128 CS positions (a function of max_seq only)
  const int CS = attn_cluster_size(s.slot_mode);
  *spw = (s.max_seq + 128 * CS - 1) / (128 * CS);
  // row blocks: sequence mode ceil(M / tpb); slot mode at most one per token
  // run chunk, bounded by M.  One cluster per (block, KV head) item: items
  // past the device-side block count exit at once
  const int nblk_max = s.slot_mode ? s.M : (s.M + *tpb - 1) / *tpb;
  *grid = nblk_max * s.KV * CS;
}

int attn_launch(const AttnArgs& a, int hd, int grid, cudaStream_t st) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kAttnThreads);
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = attn_cluster_size(a.tok_pos != nullptr);
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  const bool m3 = attn_minb() == 3;
  if (hd == 128) {
    cfg.dynamicSmemBytes = AttnSmem<128>::kBytes;
    if (m3) PEARL_CUDA_TRY(cudaLaunchKernelEx(&cfg, attn_kernel<128, 3>, a));
    else PEARL_CUDA_TRY(cudaLaunchKernelEx(&cfg, attn_kernel<128, 2>, a));
  } else {
    cfg.dynamicSmemBytes = AttnSmem<64>::kBytes;
    if (m3) PEARL_CUDA_TRY(cudaLaunchKernelEx(&cfg, attn_kernel<64, 3>, a));
    else PEARL_CUDA_TRY(cudaLaunchKernelEx(&cfg, attn_kernel<64, 2>, a));
  }
  count_launch();
  return PEARL_OK;
}

}  // namespace pearl
