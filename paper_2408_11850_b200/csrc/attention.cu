// K4: split-KV, GQA-grouped causal attention (see attention.cuh).
#include "attention.cuh"

#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "attention_core.cuh"
#include "tc_common.cuh"
#include "common.h"

namespace pearl {

namespace cg = cooperative_groups;
using bf16 = __nv_bfloat16;

namespace {

using namespace attn_core;

template <int HD>
struct AttnSmem {
  // warp states + weights, kAttnLCS logical folded states (at most), fold area
  static constexpr size_t kBytes =
      static_cast<size_t>(Smem<HD>::kWarpFloats + kAttnLCS * Smem<HD>::kStateFloats + Smem<HD>::kFoldFloats) * 4 + 64;
};

template <int HD, int MINB>
__global__ void __launch_bounds__(kAttnThreads, MINB) attn_kernel(AttnArgs a) {
  constexpr int J = HD / 32;    // 32-dim blocks
  constexpr int RS = HD + 2;    // state row: o[HD], m, l
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float* st = reinterpret_cast<float*>(smem_raw);          // [kWarps][kAttnMaxRb][RS] warp states
  float* wgt = st + kWarps * kAttnMaxRb * RS;              // [kAttnMaxRb][kWarps] warp weights
  float* cs = wgt + kAttnMaxRb * kWarps;                   // [per][kAttnMaxRb][RS] logical CTA states
  cg::cluster_group cluster = cg::this_cluster();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) PEARL_TL(a.tl, 0);
  const int crank = static_cast<int>(cluster.block_rank());
  const int CS = static_cast<int>(cluster.num_blocks());  // physical CTAs per (row block, KV head)
  const int per = kAttnLCS / CS;                          // logical CTAs per physical CTA
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
  // segment js of this warp in logical CTA lc: 32 positions at 32 ((js kAttnLCS + lc) 4 + warp)
  auto seg_p0 = [&](int js, int lc) { return 32 * ((js * kAttnLCS + lc) * kWarps + warp); };
  const int lc0 = crank * per;  // this CTA's first logical CTA

  uint4 kb[4][J], vb[4][J];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < J; ++j) kb[i][j] = vb[i][j] = make_uint4(0, 0, 0, 0);
  const int old_hi = (seq_mode && first) ? min(p0, pmax + 1) - 1 : -1;  // last position loadable before the wait
  if (first) {
    if (seg_p0(0, lc0) <= pmax) load_kv<HD>(kc, vc, kvs, seg_p0(0, lc0), lane, 0, old_hi, kb, vb);
    // the other segments' old positions: warm L2 while the QKV GEMM drains
    for (int x = 1; x < a.spw * per; ++x) {
      const int P = seg_p0(x / per, lc0 + x % per) + lane;
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
    if (threadIdx.x == 0) PEARL_TL(a.tl, 1);
  }

  // this CTA's logical CTAs one after another: warp passes, then the fold of
  // the 4 warp states into the logical CTA's state
  for (int l = 0; l < per; ++l) {
    if (l > 0) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < J; ++j) kb[i][j] = vb[i][j] = make_uint4(0, 0, 0, 0);
    }
    warp_pass<HD>(a, kc, vc, kvs, p0, r0, R, g, kvh, pmax, kAttnLCS, lc0 + l, warp, lane, a.spw,
                  l == 0 ? old_hi : -1, kb, vb, st + warp * kAttnMaxRb * RS);
    __syncthreads();
    if (threadIdx.x == 0 && first && l == 0) PEARL_TL(a.tl, 2);
    cta_fold<HD>(st, cs + l * kAttnMaxRb * RS, wgt, R, threadIdx.x, kAttnThreads, [] { __syncthreads(); });
    __syncthreads();
  }
  if (threadIdx.x == 0 && first) PEARL_TL(a.tl, 3);
  // fold of the kAttnLCS logical states in order (DSMEM across the cluster);
  // logical CTA lc produces head dims [lc HD / kAttnLCS, (lc + 1) HD / kAttnLCS)
  if (CS > 1) cluster.sync();
  if (threadIdx.x == 0 && first) PEARL_TL(a.tl, 5);
  auto peer = [&](int c) -> const float* {
    return cluster.map_shared_rank(cs + (c % per) * kAttnMaxRb * RS, c / per);
  };
  for (int l = 0; l < per; ++l)
    cluster_fold_out<HD>(a, peer, kAttnLCS, lc0 + l, R, r0, g, kvh, threadIdx.x, kAttnThreads);
  if (threadIdx.x == 0 && first) PEARL_TL(a.tl, 6);
  if (CS > 1) cluster.sync();  // the peers' states stay alive until every CTA has read them
  else __syncthreads();         // smem reuse by the next item
  first = false;
  }
  if (first) {  // no work for this cluster: still order after the producer
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  }
  if (threadIdx.x == 0) PEARL_TL(a.tl, 4);
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
  // slot mode (batched sequences): many short token runs, one item each.
  // The fold is the same for any physical cluster (kAttnLCS logical CTAs),
  // so this is purely a speed choice (PEARL_ATTN_CLUSTER_SLOT: 1, 2, 4).
  if (slot_mode) {
    static const int css = [] {
      const char* v = std::getenv("PEARL_ATTN_CLUSTER_SLOT");
      const int x = v ? std::atoi(v) : 1;
      return (x == 1 || x == 2 || x == 4) ? x : 1;
    }();
    return css;
  }
  static const int cs = [] {
    const char* v = std::getenv("PEARL_ATTN_CLUSTER");
    const int x = v ? std::atoi(v) : kAttnClusterDefault;
    return (x == 1 || x == 2 || x == 4) ? x : kAttnClusterDefault;
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
  // segments per warp: the kAttnLCS logical CTAs x 4 warps cover the whole
  // cache in spw rounds of 512 positions (a function of max_seq only)
  const int CS = attn_cluster_size(s.slot_mode);
  *spw = (s.max_seq + 128 * kAttnLCS - 1) / (128 * kAttnLCS);
  // row blocks: sequence mode ceil(M / tpb); slot mode at most one per token
  // run chunk, bounded by M.  One cluster per (block, KV head) item: items
  // past the device-side block count exit at once
  const int nblk_max = s.slot_mode ? s.M : (s.M + *tpb - 1) / *tpb;
  *grid = nblk_max * s.KV * CS;
}

int attn_launch(const AttnArgs& a_in, int hd, int grid, cudaStream_t st) {
  AttnArgs a = a_in;
#ifdef PEARL_TIMELINE
  a.tl = timeline_next(1);
#endif
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
