// Shared device building blocks of the tcgen05 contraction kernels (K3):
// tile constants, PTX wrappers for mbarrier / TMA / tcgen05, the K-major
// SWIZZLE_128B UMMA descriptor, and the stream-K unit walker.  Used by the
// tcgen05 GEMM kernel (gemm_tc.cu).
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace pearl {

constexpr int kTileN = 128;    // weight rows per tile (MMA-M)
constexpr int kTileK = 64;     // K per stage (one 128-byte swizzle row)
constexpr int kTokTile = 16;   // tokens per MMA (MMA-N)
constexpr int kMaxTokTiles = 8;  // windows / batched passes up to 128 tokens
constexpr int kWBytes = kTileN * kTileK * 2;   // 16 KB
constexpr int kXBytes = kTokTile * kTileK * 2; // 2 KB per token tile
#ifndef PEARL_MAX_STAGES
#define PEARL_MAX_STAGES 8
#endif
constexpr int kMaxStages = PEARL_MAX_STAGES;
constexpr int kTcThreads = 192;
constexpr int kEpiThreads = 128;
constexpr int kAccs = 4;  // TMEM accumulators (x NT*16 fp32 columns) in flight

// Per token-tile-count (NT) configuration.  One CTA per SM with a deep ring
// (8 stages of 16 KB weight tiles in flight per SM) beats two co-resident
// CTAs with a 90 KB ring (which let the next kernel's CTAs start streaming
// under programmatic dependent launch): 7B forward M=4 3.43 -> 3.31 ms,
// M=16 4.0 -> 3.77 ms, M=24 5.15 -> 4.35 ms (B200, graph replay).  A
// 200 KB / 12-stage ring measured no better.
// Diagnostic builds may override the ring size / co-residency (A/B probes).
#ifndef PEARL_RING_KB
#define PEARL_RING_KB 144
#endif
#ifndef PEARL_GEMM_MINB
#define PEARL_GEMM_MINB 1
#endif
template <int NT>
struct TcCfg {
  // NT <= 2 (decode windows): W and X of a k-block share one stage of a
  // 144 KB ring.  NT >= 3 (wide windows, prefill): X tiles would take up to
  // half of every stage, halving the weight bytes in flight (latency-bound
  // streaming: 4 stages = 64 KB of W per SM at NT = 8), so X gets its own
  // 3-stage ring (L2-resident activations need little lead) and W keeps
  // up to 8 x 16 KB stages.
  static constexpr bool kSplitX = NT >= 3;
  static constexpr int kXStages = 3;
  static constexpr int kXStageBytes = NT * kXBytes;
  static constexpr int kRing = PEARL_RING_KB * 1024;
  // staged tile, token-major: E[t * kEStride + row] (+4 pad keeps rows 16-byte aligned)
  static constexpr int kEStride = kTileN + 4;
  static constexpr int kEBytes = NT * 16 * kEStride * 4;
  static constexpr int kStageBytes = kSplitX ? kWBytes : kWBytes + NT * kXBytes;
  static constexpr int kXRingBytes = kSplitX ? kXStages * kXStageBytes : 0;
  static constexpr int kBudget = 227 * 1024 - 1024 - 512 - kEBytes - kXRingBytes;
  static constexpr int kStagesFit = kSplitX ? kBudget / kStageBytes : kRing / kStageBytes;
  static constexpr int kStages = kStagesFit < kMaxStages ? kStagesFit : kMaxStages;
  static constexpr int kCols = kAccs * NT * 16;
  static constexpr int kTmemCols = kCols <= 32 ? 32 : kCols <= 64 ? 64 : kCols <= 128 ? 128 : kCols <= 256 ? 256 : 512;
  static constexpr size_t kSmem = 1024 + static_cast<size_t>(kStages) * kStageBytes + kXRingBytes + kEBytes + 512;
  // NT = 1: registers capped for two CTAs per SM (<= 170), so the attention
  // kernel (or the next GEMM after it) can be resident beside a GEMM CTA
  static constexpr int kMinBlocks = NT == 1 ? 2 : PEARL_GEMM_MINB;
  // wide windows: 8 epilogue warps (each TMEM lane quarter read by two warps,
  // one per half of the token chunks) for the 128-token tiles' epilogues
  static constexpr int kEpiWarps = NT >= 2 ? 8 : 4;
  static constexpr int kEpi = 32 * kEpiWarps;
  static constexpr int kThreads = 64 + kEpi;
};


// ---- PTX helpers -----------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
  } while (!done);
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ uint64_t umma_desc_sw128(const void* smem_tile) {
  // K-major SWIZZLE_128B canonical layout: rows of 128 B, 8-row groups 1024 B
  // apart (SBO = 1024 B), LBO = 16 B (unused for swizzled K-major), version 1.
  const uint64_t addr = smem_u32(smem_tile);
  return ((addr & 0x3FFFFull) >> 4) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}

// instruction descriptor: D=f32, A=B=bf16, K-major both, N=16, M=128
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | ((kTokTile >> 3) << 17) | ((kTileN >> 4) << 24);

__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(kIdesc), "r"(accumulate));
}

// Same MMA with N = n columns (n % 16 == 0, <= 256): the NT token tiles of a
// stage are one contiguous K-major SW128 operand of n rows.
__host__ __device__ constexpr uint32_t umma_idesc(int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((static_cast<uint32_t>(n) >> 3) << 17) | ((kTileN >> 4) << 24);
}

__device__ __forceinline__ void umma_bf16_n(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t accumulate,
                                            uint32_t idesc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads) : "memory"); }
template <int N>
__device__ __forceinline__ void epi_bar_n() { asm volatile("bar.sync 1, %0;" ::"n"(N) : "memory"); }

// Stream-K: CTA c owns iterations [c*T/G, (c+1)*T/G) of the flattened
// (tile, k-block) space.  cta_of(x) is the CTA whose range contains x.
template <class A>
__device__ __forceinline__ int cta_of(const A& a, long long x) {
  return static_cast<int>(((x + 1) * a.G + a.T - 1) / a.T) - 1;
}

struct Unit {
  int tile, kb0, kb1, seg, nseg;
};

// The unit (maximal run inside one tile) starting at iteration x, capped at r1.
template <class A>
__device__ __forceinline__ Unit unit_at(const A& a, long long x, long long r1) {
  Unit u;
  u.tile = static_cast<int>(x / a.KB);
  u.kb0 = static_cast<int>(x % a.KB);
  u.kb1 = static_cast<int>(min(static_cast<long long>(a.KB), u.kb0 + (r1 - x)));
  const long long t0 = static_cast<long long>(u.tile) * a.KB;
  const int c0 = cta_of(a, t0);
  u.seg = cta_of(a, x) - c0;
  u.nseg = cta_of(a, t0 + a.KB - 1) - c0 + 1;
  return u;
}


__device__ __forceinline__ unsigned long long tl_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#ifdef PEARL_TIMELINE
#define PEARL_TL(buf, slot)                                                                        \
  do {                                                                                             \
    if ((buf) != nullptr && blockIdx.x < 160) (buf)[blockIdx.x * 16 + (slot)] = ::pearl::tl_now(); \
  } while (0)
#else
#define PEARL_TL(buf, slot) \
  do {                      \
  } while (0)
#endif

}  // namespace pearl
