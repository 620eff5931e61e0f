// Persistent whole-forward kernel for tcgen05 (target) models, windows of
// M <= 16 tokens.
//
// Why: a batch-1 decode forward of a 7B target is 129 weight-streaming GEMMs
// of 33-262 MB.  Launched one by one, every GEMM pays ~5 us of launch, ramp
// and tail on top of streaming at ~6.3 TB/s (tools/gemm_sweep.py), plus the
// attention and norm kernels in between -- ~40% of the forward.  Here one
// cooperative grid (one CTA per SM) runs the whole forward as an ordered list
// of phases:
//
//   embed, per layer [norm1, QKV GEMM, attention, O GEMM, norm2, gate/up
//   GEMM, down GEMM], final norm, lm_head GEMM
//
// CTA roles (7 warps):
//   warp 0 / lane 0 : W producer.  Streams the weight tiles of every GEMM
//                     phase (stream-K ranges, as gemm_tc.cu) into the smem
//                     ring without ever waiting on activations, so HBM stays
//                     busy across phase boundaries.
//   warp 6 / lane 0 : X producer.  Before the first stage of GEMM phase p it
//                     waits until every CTA has finished phase p - 1 (a
//                     release/acquire counter per phase), then TMA-loads the activation
//                     tiles of that phase into the same stages.
//   warp 1          : TMEM allocator; lane 0 issues tcgen05.mma into four
//                     rotating accumulators.
//   warps 2..5      : epilogues (stream-K fixup, fused RoPE/KV, residual,
//                     SwiGLU, logits), and the non-GEMM phases -- attention
//                     items (head, token), RMSNorm rows, embedding rows --
//                     distributed round-robin over CTAs.  After each phase a
//                     CTA adds 1 to that phase's counter (release).  One
//                     counter per phase: a CTA with no work in a phase runs
//                     ahead, so a single running total could reach p * G
//                     before every CTA has finished phase p - 1.  ctr[p-1] ==
//                     G means every CTA is past phase p - 1, hence past all
//                     earlier phases too (each CTA walks the list in order).
//
// Every per-token computation keeps the fixed order of the per-op kernels'
// design (same stream-K split points, fixed-order fixup, attention chunk
// order), so results are independent of M (batch invariance) and identical
// between a graph replay and the next.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <string>
#include <vector>

#include "common.h"
#include "epilogue.cuh"
#include "fwd_mega.cuh"
#include "tc_common.cuh"

namespace pearl {

constexpr int kMgThreads = 224;  // 7 warps
constexpr int kMgEpiWarp0 = 2;
constexpr int kMgXWarp = 6;
constexpr int kMgStages = 8;
constexpr int kMgStageBytes = kWBytes + kXBytes;        // NT = 1
constexpr int kMgRing = kMgStages * kMgStageBytes;      // 144 KB
constexpr int kMgEBytes = kTileN * 16 * 4;               // [128][16] fp32
constexpr int kMgAttnWarps = 4;
constexpr int kMgChunk = 32;
constexpr int kMgTmemCols = 64;                          // 4 accumulators x 16

__host__ __device__ constexpr int mg_attn_bytes(int hd) {
  return kMgAttnWarps * (hd + 2) * 4 + hd * 2 + kMgAttnWarps * kMgChunk * hd * 2;
}
constexpr size_t kMgSmem = 1024 + kMgRing + kMgEBytes + mg_attn_bytes(128) + 512;

__device__ __forceinline__ void mg_epi_bar() { asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads) : "memory"); }

__device__ __forceinline__ unsigned ld_relaxed(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Phase counters sit on their own 128-byte lines (kMgCtrStride words apart).
constexpr int kMgCtrStride = kMegaCtrStride;

// Spin until ctr reaches target (every CTA finished that phase).  Polls with
// relaxed loads (an acquire load would invalidate the SM's L1 on every poll)
// and acquires once.  Bounded: a stuck grid traps instead of hanging the GPU.
__device__ __forceinline__ void wait_phase(const unsigned* ctr, unsigned target) {
  long long spins = 0;
  while (ld_relaxed(ctr) < target) {
    __nanosleep(64);
    if (++spins > (1ll << 26)) asm volatile("trap;");
  }
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
}

__device__ __forceinline__ void signal_phase(unsigned* ctr) {
  asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
}

// Stream-K range of this CTA in a GEMM phase of T (tile, k-block) units: the
// first min(G, T) CTAs split the units as the per-GEMM kernel's grid of
// min(num_sms, T) CTAs does (identical segments => identical sums).
__device__ __forceinline__ int mg_range(long long T, int G, long long* r0, long long* r1) {
  const int Gp = static_cast<int>(T < G ? T : G);
  const long long b = blockIdx.x;
  *r0 = b < Gp ? b * T / Gp : T;
  *r1 = b < Gp ? (b + 1) * T / Gp : T;
  return Gp;
}

__device__ __forceinline__ unsigned long long mg_clock() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// ---------------------------------------------------------------------------
// non-GEMM phase bodies (128 epilogue threads, et = 0..127)
// ---------------------------------------------------------------------------
__device__ void mg_embed_row(const MegaPhase& ph, const int32_t* tokens, int t, int et) {
  int tok = tokens[t];
  tok = tok < 0 ? 0 : (tok >= ph.V ? ph.V - 1 : tok);
  const uint4* row = reinterpret_cast<const uint4*>(ph.embed + static_cast<size_t>(tok) * ph.d);
  float4* h = reinterpret_cast<float4*>(ph.h + static_cast<size_t>(t) * ph.d);
#pragma unroll 4
  for (int i = et; i < ph.d / 8; i += kEpiThreads) {
    const uint4 u = row[i];
    h[2 * i] = make_float4(__uint_as_float(u.x << 16), __uint_as_float(u.x & 0xffff0000u), __uint_as_float(u.y << 16),
                           __uint_as_float(u.y & 0xffff0000u));
    h[2 * i + 1] = make_float4(__uint_as_float(u.z << 16), __uint_as_float(u.z & 0xffff0000u),
                               __uint_as_float(u.w << 16), __uint_as_float(u.w & 0xffff0000u));
  }
}

// rmsnorm of row t: fixed order (thread-strided float4 sums in k order, warp
// xor tree, warps summed in order) -- rmsnorm_kernel's arithmetic.  The row
// stays in registers: all loads in flight at once.
constexpr int kMgNormVec = 16;  // d <= 4 * 128 * 16
__device__ void mg_norm_row(const MegaPhase& ph, int t, int et, float* red) {
  const int d = ph.d, nv = d / 4;
  const float4* hr = reinterpret_cast<const float4*>(ph.h + static_cast<size_t>(t) * d);
  float4 v[kMgNormVec];
#pragma unroll
  for (int i = 0; i < kMgNormVec; ++i) {
    const int j = et + i * kEpiThreads;
    v[i] = j < nv ? __ldcg(hr + j) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < kMgNormVec; ++i) {
    if (et + i * kEpiThreads < nv) {
      ss = fmaf(v[i].x, v[i].x, ss);
      ss = fmaf(v[i].y, v[i].y, ss);
      ss = fmaf(v[i].z, v[i].z, ss);
      ss = fmaf(v[i].w, v[i].w, ss);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if ((et & 31) == 0) red[et >> 5] = ss;
  mg_epi_bar();
  const float tot = (red[0] + red[1]) + (red[2] + red[3]);
  const float rs = 1.0f / sqrtf(tot / static_cast<float>(d) + ph.eps);
  const float4* g4 = reinterpret_cast<const float4*>(ph.gain);
  uint2* xr = reinterpret_cast<uint2*>(ph.xout + static_cast<size_t>(t) * d);
#pragma unroll
  for (int i = 0; i < kMgNormVec; ++i) {
    const int j = et + i * kEpiThreads;
    if (j < nv) {
      const float4 gg = g4[j];
      const __nv_bfloat162 lo = __floats2bfloat162_rn(v[i].x * rs * gg.x, v[i].y * rs * gg.y);
      const __nv_bfloat162 hi = __floats2bfloat162_rn(v[i].z * rs * gg.z, v[i].w * rs * gg.w);
      xr[j] = make_uint2(*reinterpret_cast<const uint32_t*>(&lo), *reinterpret_cast<const uint32_t*>(&hi));
    }
  }
  mg_epi_bar();  // red[] reused by the next row
}

// Attention of window token t, query head h: 4 warps over 32-position chunks
// (chunk c -> warp c % 4), online softmax per warp in chunk order, warps
// merged in order.  Same arithmetic as attention_kernel in llama.cu.
template <int HD>
__device__ void mg_attn_item(const MegaPhase& ph, const MegaArgs& A, int h, int t, int et, unsigned char* sm) {
  constexpr int PER = HD / 32;
  const int warp = et >> 5, lane = et & 31;
  float* st_all = reinterpret_cast<float*>(sm);                     // [4][HD + 2]
  bf16* Qs = reinterpret_cast<bf16*>(st_all + kMgAttnWarps * (HD + 2));
  bf16* Vw = Qs + HD + static_cast<size_t>(warp) * kMgChunk * HD;  // this warp's chunk
  const int pt = *A.pos + A.pos_add + t;                            // token position
  const int ctx = pt + 1;
  const int n_chunks = (ctx + kMgChunk - 1) / kMgChunk;
  const int kvh = h / (ph.H / ph.KV);
  const size_t kstride = static_cast<size_t>(ph.KV) * HD;
  float* st = st_all + warp * (HD + 2);
  for (int i = et; i < HD / 8; i += kEpiThreads)
    reinterpret_cast<uint4*>(Qs)[i] = *reinterpret_cast<const uint4*>(ph.q + (static_cast<size_t>(t) * ph.H + h) * HD + i * 8);
  for (int i = lane; i < HD + 2; i += 32) st[i] = (i == HD) ? -INFINITY : 0.f;
  mg_epi_bar();
  for (int c = warp; c < n_chunks; c += kMgAttnWarps) {
    const int j = c * kMgChunk + lane;
    const bool have = j < ctx;
    // the chunk's K row (this lane's position) and V rows (flat 16-byte
    // pieces lane + 32 k): all loads in flight together, then V to smem
    uint4 kr[HD / 8], vr[HD / 8];
#pragma unroll
    for (int v = 0; v < HD / 8; ++v)
      kr[v] = have ? *reinterpret_cast<const uint4*>(ph.kc + j * kstride + kvh * HD + v * 8) : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int k = 0; k < HD / 8; ++k) {
      const int i = lane + 32 * k;
      const int jp = c * kMgChunk + i / (HD / 8);
      vr[k] = jp < ctx ? *reinterpret_cast<const uint4*>(ph.vc + jp * kstride + kvh * HD + (i % (HD / 8)) * 8)
                       : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int k = 0; k < HD / 8; ++k) {
      const int i = lane + 32 * k;
      reinterpret_cast<uint4*>(Vw + (i / (HD / 8)) * HD)[i % (HD / 8)] = vr[k];
    }
    __syncwarp();
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int v = 0; v < HD / 8; ++v) {
      const uint4 qv = reinterpret_cast<const uint4*>(Qs)[v];
      const uint32_t qw[4] = {qv.x, qv.y, qv.z, qv.w}, kw[4] = {kr[v].x, kr[v].y, kr[v].z, kr[v].w};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        acc[u] = fmaf(__uint_as_float(qw[u] << 16), __uint_as_float(kw[u] << 16), acc[u]);
        acc[u] = fmaf(__uint_as_float(qw[u] & 0xffff0000u), __uint_as_float(kw[u] & 0xffff0000u), acc[u]);
      }
    }
    const float s = have ? ((acc[0] + acc[1]) + (acc[2] + acc[3])) * ph.scale : -INFINITY;
    float cm = s;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) cm = fmaxf(cm, __shfl_xor_sync(0xffffffffu, cm, o));
    const float m_old = st[HD];
    const float m_new = fmaxf(m_old, cm);
    const float p = have ? expf(s - m_new) : 0.f;
    float ps = p;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ps += __shfl_xor_sync(0xffffffffu, ps, o);
    const float corr = (m_old == -INFINITY) ? 0.f : expf(m_old - m_new);
    float ov[PER];
#pragma unroll
    for (int e = 0; e < PER; ++e) ov[e] = 0.f;
    const int jn = min(kMgChunk, ctx - c * kMgChunk);
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
    for (int e = 0; e < PER; ++e) st[lane * PER + e] = fmaf(corr, st[lane * PER + e], ov[e]);
    __syncwarp();
    if (lane == 0) {
      st[HD] = m_new;
      st[HD + 1] = fmaf(corr, st[HD + 1], ps);
    }
    __syncwarp();
  }
  mg_epi_bar();
  for (int d = et; d < HD; d += kEpiThreads) {
    float mx = -INFINITY;
#pragma unroll
    for (int w = 0; w < kMgAttnWarps; ++w) mx = fmaxf(mx, st_all[w * (HD + 2) + HD]);
    float L = 0.f, O = 0.f;
#pragma unroll
    for (int w = 0; w < kMgAttnWarps; ++w) {
      const float* sr = st_all + w * (HD + 2);
      if (sr[HD] != -INFINITY) {
        const float wt = expf(sr[HD] - mx);
        L = fmaf(wt, sr[HD + 1], L);
        O = fmaf(wt, sr[d], O);
      }
    }
    ph.o[(static_cast<size_t>(t) * ph.H + h) * HD + d] = __float2bfloat16(O / L);
  }
  mg_epi_bar();  // smem reused by the next item
}

// ---------------------------------------------------------------------------
// the kernel
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kMgThreads, 1) fwd_mega_kernel(MegaArgs A) {
  extern __shared__ __align__(1024) unsigned char mg_smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(mg_smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  float* E = reinterpret_cast<float*>(smem + kMgRing);
  unsigned char* attn_sm = smem + kMgRing + kMgEBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(attn_sm + mg_attn_bytes(128));
  uint64_t* empty = full + kMgStages;
  uint64_t* acc_full = empty + kMgStages;
  uint64_t* acc_empty = acc_full + kAccs;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + kAccs);
  int* s_last = reinterpret_cast<int*>(tmem_slot + 1);
  float* red = reinterpret_cast<float*>(s_last + 4);  // [4]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = gridDim.x;
  const MegaPhase* phases = A.phases;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kMgStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);  // released by the MMA commit; W and X producers both wait on it
    }
    for (int b = 0; b < kAccs; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], kEpiThreads);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(kMgTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  if (A.trace && threadIdx.x == 0) A.trace[static_cast<size_t>(A.n_phases) * G + blockIdx.x] = mg_clock();

  if (warp == 0) {
    if (lane == 0) {
      // ---- W producer: every GEMM phase's stream-K range, never blocked by activations
      int it = 0;
      for (int p = 0; p < A.n_phases; ++p) {
        const MegaPhase& ph = phases[p];
        if (ph.kind != MG_GEMM) continue;
        long long r0, r1;
        mg_range(ph.T, G, &r0, &r1);
        for (long long x = r0; x < r1; ++x, ++it) {
          const int s = it % kMgStages;
          if (it >= kMgStages) mbar_wait(&empty[s], ((it / kMgStages) - 1) & 1);
          mbar_expect_tx(&full[s], kMgStageBytes);
          tma_load_2d(smem + s * kMgStageBytes, &A.maps[ph.map_w].map, &full[s], static_cast<int>(x % ph.KB) * kTileK,
                      static_cast<int>(x / ph.KB) * kTileN);
        }
      }
    }
  } else if (warp == kMgXWarp) {
    if (lane == 0) {
      // ---- X producer: waits for the phases before each GEMM phase
      int it = 0;
      for (int p = 0; p < A.n_phases; ++p) {
        const MegaPhase& ph = phases[p];
        if (ph.kind != MG_GEMM) continue;
        long long r0, r1;
        const int Gp = mg_range(ph.T, G, &r0, &r1);
        if (r1 > r0) {
          if (p > 0) wait_phase(A.counter + (p - 1) * kMgCtrStride, G);
          // generic-proxy writes of the previous phases -> async-proxy (TMA) reads
          asm volatile("fence.proxy.async.global;" ::: "memory");
        }
        for (long long x = r0; x < r1; ++x, ++it) {
          const int s = it % kMgStages;
          if (it >= kMgStages) mbar_wait(&empty[s], ((it / kMgStages) - 1) & 1);
          tma_load_2d(smem + s * kMgStageBytes + kWBytes, &A.maps[ph.map_x].map, &full[s],
                      static_cast<int>(x % ph.KB) * kTileK, 0);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---- MMA issuer
      int it = 0, ui = 0;
      for (int p = 0; p < A.n_phases; ++p) {
        const MegaPhase& ph = phases[p];
        if (ph.kind != MG_GEMM) continue;
        long long r0, r1;
        const int Gp = mg_range(ph.T, G, &r0, &r1);
        SkShape sk{ph.T, Gp, ph.KB};
        for (long long x = r0; x < r1; ++ui) {
          const Unit u = unit_at(sk, x, r1);
          x += u.kb1 - u.kb0;
          const int b = ui % kAccs;
          if (ui >= kAccs) mbar_wait(&acc_empty[b], ((ui / kAccs) - 1) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t acc = tmem + b * kTokTile;
          for (int kb = u.kb0; kb < u.kb1; ++kb, ++it) {
            const int s = it % kMgStages;
            mbar_wait(&full[s], (it / kMgStages) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            unsigned char* st = smem + s * kMgStageBytes;
            const uint64_t adesc = umma_desc_sw128(st);
            const uint64_t bdesc = umma_desc_sw128(st + kWBytes);
#pragma unroll
            for (int kk = 0; kk < kTileK / 16; ++kk)
              umma_bf16(acc, adesc + 2 * kk, bdesc + 2 * kk, (kb > u.kb0 || kk > 0) ? 1u : 0u);
            umma_commit(&empty[s]);
          }
          umma_commit(&acc_full[b]);
        }
      }
    }
  } else {
    // ---- epilogue / phase warps 2..5
    const int lanegrp = warp & 3;
    const int row = lanegrp * 32 + lane;
    const int et = threadIdx.x - kMgEpiWarp0 * 32;
    int ui = 0;
    for (int p = 0; p < A.n_phases; ++p) {
      const MegaPhase& ph = phases[p];
      if (ph.kind == MG_GEMM) {
        long long r0, r1;
        const int Gp = mg_range(ph.T, G, &r0, &r1);
        SkShape sk{ph.T, Gp, ph.KB};
        const int Mp = (ph.M + 3) & ~3;
        for (long long x = r0; x < r1; ++ui) {
          const Unit u = unit_at(sk, x, r1);
          x += u.kb1 - u.kb0;
          const int tile = u.tile;
          const int b = ui % kAccs;
          mbar_wait(&acc_full[b], (ui / kAccs) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          float v[16];
          tmem_ld16(tmem + (static_cast<uint32_t>(lanegrp * 32) << 16) + b * kTokTile, v);
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          mbar_arrive(&acc_empty[b]);
          if (u.nseg == 1) {
#pragma unroll
            for (int q = 0; q < 4; ++q)
              *reinterpret_cast<float4*>(E + row * 16 + 4 * q) = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
          } else {
            float* dst = A.partials + ((static_cast<size_t>(tile) * ph.seg_max + u.seg) * kTileN + row) * Mp;
#pragma unroll
            for (int q = 0; q < 4; ++q)
              if (4 * q < Mp)
                *reinterpret_cast<float4*>(dst + 4 * q) = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
            mg_epi_bar();
            if (et == 0) {
              int old;
              asm volatile("atom.add.release.gpu.global.s32 %0, [%1], 1;" : "=r"(old) : "l"(A.tile_flags + tile) : "memory");
              *s_last = (old == u.nseg - 1);
            }
            mg_epi_bar();
            if (!*s_last) continue;
            asm volatile("fence.acq_rel.gpu;" ::: "memory");
            // fixup: gemm_tc.cu's batched split-order sum (NT = 1)
            const float* src = A.partials + (static_cast<size_t>(tile) * ph.seg_max * kTileN + row) * Mp;
            const size_t sstride = static_cast<size_t>(kTileN) * Mp;
            const int nq = Mp / 4;
            float4 acc[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int s0 = 0; s0 < u.nseg; s0 += 4) {
              float4 pp[4][4];
#pragma unroll
              for (int sb = 0; sb < 4; ++sb)
#pragma unroll
                for (int q = 0; q < 4; ++q)
                  if (s0 + sb < u.nseg && q < nq)
                    pp[sb][q] = __ldcg(reinterpret_cast<const float4*>(src + (s0 + sb) * sstride + 4 * q));
#pragma unroll
              for (int sb = 0; sb < 4; ++sb)
#pragma unroll
                for (int q = 0; q < 4; ++q)
                  if (s0 + sb < u.nseg && q < nq) {
                    acc[q].x += pp[sb][q].x;
                    acc[q].y += pp[sb][q].y;
                    acc[q].z += pp[sb][q].z;
                    acc[q].w += pp[sb][q].w;
                  }
            }
#pragma unroll
            for (int q = 0; q < 4; ++q)
              if (q < nq) *reinterpret_cast<float4*>(E + row * 16 + 4 * q) = acc[q];
            if (et == 0) A.tile_flags[tile] = 0;
          }
          mg_epi_bar();
          EpiArgs e = ph.e;
          if (ph.e_uses_pos) {
            e.pos = A.pos;
            e.pos_add = A.pos_add;
          }
          if (ph.e_is_logits) e.out_f32 = A.logits;
          epilogue_tile<4>(e, tile, E, 16, ph.M, ph.N, et);
          mg_epi_bar();
        }
      } else {
        // non-GEMM phase: all previous phases must be complete
        if (et == 0 && p > 0) wait_phase(A.counter + (p - 1) * kMgCtrStride, G);
        mg_epi_bar();
        if (!(A.opts & 1)) asm volatile("fence.acq_rel.gpu;" ::: "memory");
        if (ph.kind == MG_EMBED) {
          for (int t = blockIdx.x; t < ph.M; t += G) mg_embed_row(ph, A.tokens, t, et);
        } else if (ph.kind == MG_NORM) {
          for (int t = ph.row0 + blockIdx.x; t < ph.M; t += G) mg_norm_row(ph, t, et, red);
        } else if (ph.kind == MG_ATTN) {
          const int items = ph.H * ph.M;
          for (int i = blockIdx.x; i < items; i += G) {
            if (ph.hd == 128)
              mg_attn_item<128>(ph, A, i % ph.H, i / ph.H, et, attn_sm);
            else
              mg_attn_item<64>(ph, A, i % ph.H, i / ph.H, et, attn_sm);
          }
        }
      }
      // this CTA is done with phase p: its generic writes must be visible to
      // later TMA (async-proxy) reads and to other CTAs before the release
      if (!(A.opts & 6)) asm volatile("fence.proxy.async.global;" ::: "memory");
      mg_epi_bar();
      if (et == 0) {
        if ((A.opts & 6) == 2) asm volatile("fence.proxy.async.global;" ::: "memory");
        signal_phase(A.counter + p * kMgCtrStride);
        if (A.trace) A.trace[static_cast<size_t>(p) * G + blockIdx.x] = mg_clock();
      }
    }
  }
  __syncwarp();
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kMgTmemCols));
  // Once every CTA has finished the last phase nobody reads the counters any
  // more: CTA 0 zeroes them for the next launch (no memset node per forward).
  if (blockIdx.x == 0) {
    if (threadIdx.x == 0) wait_phase(A.counter + (A.n_phases - 1) * kMgCtrStride, G);
    __syncthreads();
    for (int i = threadIdx.x; i < A.n_phases; i += blockDim.x) A.counter[i * kMgCtrStride] = 0;
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
namespace {
std::once_flag g_mg_once;
cudaError_t g_mg_err = cudaSuccess;
}  // namespace

int mega_supported(int M) { return M >= 1 && M <= kTokTile; }

size_t mega_smem_bytes() { return kMgSmem; }

static_assert(kMegaTileN == kTileN && kMegaTileK == kTileK && kMegaPartialTok == kMaxTokTiles * kTokTile &&
                  kMegaMaxTokens == kTokTile,
              "fwd_mega.cuh constants out of sync with tc_common.cuh");

int mega_threads() { return kMgThreads; }
const void* mega_kernel_ptr() { return reinterpret_cast<const void*>(fwd_mega_kernel); }
cudaError_t mega_prepare() {
  std::call_once(g_mg_once, [] {
    g_mg_err = cudaFuncSetAttribute(fwd_mega_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(kMgSmem));
  });
  return g_mg_err;
}

int mega_launch(const MegaArgs& a, int grid, cudaStream_t st) {
  PEARL_CUDA_TRY(mega_prepare());
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kMgThreads);
  cfg.dynamicSmemBytes = kMgSmem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  PEARL_CUDA_TRY(cudaLaunchKernelEx(&cfg, fwd_mega_kernel, a));
  count_launch();
  return PEARL_OK;
}

}  // namespace pearl
