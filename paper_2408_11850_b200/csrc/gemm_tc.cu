// K3: tcgen05 + TMA small-M contraction (see gemm_tc.cuh).
//
// Persistent, warp-specialised CTA (one per SM), 6 warps:
//   warp 0 / lane 0 : TMA producer.  Streams the 128x64 W tile and the NT
//                     16x64 X tiles of every k-block of every work unit the
//                     CTA owns into a multi-stage smem ring (SWIZZLE_128B),
//                     running ahead across unit boundaries.  W tiles of the
//                     first stages are requested before griddepcontrol.wait
//                     (PDL), i.e. while the previous kernel is still running.
//   warp 1          : TMEM allocator; lane 0 issues tcgen05.mma
//                     (M=128 weight rows, N=16 tokens, K=16, bf16 -> fp32)
//                     into one of two TMEM accumulators and tcgen05.commit
//                     releases smem stages / publishes finished units.
//   warps 2..5      : epilogue.  tcgen05.ld 32x32b (warp w owns TMEM lanes
//                     32(w%4)..+31 = weight rows), frees the accumulator for
//                     the unit after next, then either applies the fused
//                     epilogue (no split) or stores an fp32 partial; the last
//                     CTA to finish a row tile sums its partials in split
//                     order and applies the epilogue.
// Work unit = (row tile, K split); the split count is a function of (N, K)
// only and units are assigned round-robin, so every output element is the
// same fp32 computation whatever the number of tokens M (batch invariance).
#include "gemm_tc.cuh"

#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <string>

#include "epilogue.cuh"
#include "tc_common.cuh"

namespace pearl {

struct TcArgs {
  int M, N, K, KB;
  long long T;   // total (tile, k-block) iterations
  int G;         // CTAs sharing them (stream-K); a function of (N, K) only
  int seg_max;   // partial slots per tile
  int w_tiled;   // W stored tile-major: [tiles][KB][128 rows][64 cols], one 16 KB box contiguous
  EpiArgs e;
  float* partials;
  int* flags;
  unsigned long long* tl;  // PEARL_TIMELINE builds: this launch's stamps
};

// W tile (tile, kb): row-major [N, K] -> box at (k = 64 kb, row = 128 tile);
// tile-major -> the 128 consecutive 128-byte rows at row (tile KB + kb) 128
// (a contiguous 16 KB: a CTA's run of k-blocks streams one contiguous range)
__device__ __forceinline__ void tma_load_w(void* dst, const CUtensorMap* map, uint64_t* bar, const TcArgs& a, int tile,
                                           int kb) {
  if (a.w_tiled) tma_load_2d(dst, map, bar, 0, (tile * a.KB + kb) * kTileN);
  else tma_load_2d(dst, map, bar, kb * kTileK, tile * kTileN);
}

// ---- kernel ------------------------------------------------------------------
template <int NT>
__global__ void __launch_bounds__(TcCfg<NT>::kThreads, TcCfg<NT>::kMinBlocks)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX, TcArgs a) {
  using C = TcCfg<NT>;
  constexpr int stage_bytes = C::kStageBytes;
  constexpr int stages = C::kStages;
  constexpr int ES = C::kEStride;
  extern __shared__ __align__(1024) unsigned char tc_smem_raw[];
  __shared__ float s_rs[kMaxTokTiles * kTokTile];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(tc_smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  unsigned char* xring = smem + stages * stage_bytes;  // kSplitX: [kXStages][NT x 2 KB]
  float* E = reinterpret_cast<float*>(xring + C::kXRingBytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(xring + C::kXRingBytes + C::kEBytes);
  uint64_t* empty = full + kMaxStages;
  uint64_t* acc_full = empty + kMaxStages;   // [kAccs]
  uint64_t* acc_empty = acc_full + kAccs;    // [kAccs]
  uint64_t* xfull = acc_empty + kAccs;       // [kXStages] (kSplitX)
  uint64_t* xempty = xfull + C::kXStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(xempty + C::kXStages);
  int* s_last = reinterpret_cast<int*>(tmem_slot + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) PEARL_TL(a.tl, 0);
  const long long r0 = static_cast<long long>(blockIdx.x) * a.T / a.G;
  const long long r1 = static_cast<long long>(blockIdx.x + 1) * a.T / a.G;
  const int total = static_cast<int>(r1 - r0);

  if (threadIdx.x == 0) {
    for (int s = 0; s < kMaxStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < kAccs; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], C::kEpi);
    }
    for (int b = 0; b < C::kXStages; ++b) {
      mbar_init(&xfull[b], 1);
      mbar_init(&xempty[b], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmW)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmX)) : "memory");
  }
  if (warp == 1) {
    // kAccs accumulators x NT*16 fp32 columns
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(C::kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // every CTA of this persistent grid is resident: dependents may launch now
  // (they block in griddepcontrol.wait until this grid has completed)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---- TMA producer: iterations r0..r1 in order (tile = x / KB, kb = x % KB),
      // walked with incremental (tile, kb) counters: no 64-bit divisions in the
      // issue loop (this single thread's loop is on the streaming critical path)
      const uint32_t bytes = stage_bytes;
      const int npre = min(stages, total);
      const int kb_start = static_cast<int>(r0 % a.KB), tile_start = static_cast<int>(r0 / a.KB);
      int kb = kb_start, tile = tile_start;
      if constexpr (C::kSplitX) {
        // W ring `stages` deep, X ring kXStages deep: X of iteration c is issued
        // together with W of iteration c + D (D = stages - kXStages), both
        // waiting on MMA(c + D - stages), so neither ring can wait on the other
        constexpr int XS = C::kXStages;
        constexpr int D = stages - XS;
        static_assert(D >= 0, "W ring shallower than the X ring");
        int xi = 0, kx = kb_start;
        auto issue_x = [&]() {
          const int sx = xi % XS;
          if (xi >= XS) mbar_wait(&xempty[sx], ((xi / XS) - 1) & 1);
          unsigned char* xs = xring + sx * C::kXStageBytes;
          mbar_expect_tx(&xfull[sx], C::kXStageBytes);
          tma_load_2d(xs, &tmX, &xfull[sx], kx * kTileK, 0);  // one box of 16 NT token rows
          if (++kx == a.KB) kx = 0;
          ++xi;
        };
        for (int it = 0; it < npre; ++it) {
          mbar_expect_tx(&full[it], kWBytes);
          tma_load_w(smem + it * stage_bytes, &tmW, &full[it], a, tile, kb);
          if (++kb == a.KB) { kb = 0; ++tile; }
        }
        asm volatile("griddepcontrol.wait;" ::: "memory");
        PEARL_TL(a.tl, 1);
        if (blockIdx.x == 0 && a.e.adv_pos != nullptr) *a.e.adv_pos += a.e.adv_n;
        while (xi < total && xi < XS) issue_x();
        for (int it = npre; it < total; ++it) {
          const int s = it % stages;
          mbar_wait(&empty[s], ((it / stages) - 1) & 1);
          mbar_expect_tx(&full[s], kWBytes);
          tma_load_w(smem + s * stage_bytes, &tmW, &full[s], a, tile, kb);
          if (++kb == a.KB) { kb = 0; ++tile; }
          if (xi < total && xi <= it - D) issue_x();
        }
        while (xi < total) issue_x();
      } else {
      // W does not depend on the previous kernel: request it before the PDL wait
      for (int it = 0; it < npre; ++it) {
        unsigned char* st = smem + it * stage_bytes;
        mbar_expect_tx(&full[it], bytes);
        tma_load_w(st, &tmW, &full[it], a, tile, kb);
        if (++kb == a.KB) { kb = 0; ++tile; }
      }
      asm volatile("griddepcontrol.wait;" ::: "memory");
      PEARL_TL(a.tl, 1);
      if (blockIdx.x == 0 && a.e.adv_pos != nullptr) *a.e.adv_pos += a.e.adv_n;
      int kx = kb_start;
      for (int it = 0; it < npre; ++it) {
        unsigned char* st = smem + it * stage_bytes;
        tma_load_2d(st + kWBytes, &tmX, &full[it], kx * kTileK, 0);  // one box of 16 NT token rows
        if (++kx == a.KB) kx = 0;
      }
      for (int it = npre; it < total; ++it) {
        const int s = it % stages;
        mbar_wait(&empty[s], ((it / stages) - 1) & 1);
        unsigned char* st = smem + s * stage_bytes;
        const int kc = kb * kTileK;
        mbar_expect_tx(&full[s], bytes);
        tma_load_w(st, &tmW, &full[s], a, tile, kb);
        tma_load_2d(st + kWBytes, &tmX, &full[s], kc, 0);
        if (++kb == a.KB) { kb = 0; ++tile; }
      }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---- MMA issuer: one accumulator per unit (run of k-blocks inside a tile)
      int it = 0, ui = 0;
      for (long long x = r0; x < r1; ++ui) {
        const Unit u = unit_at(a, x, r1);
        x += u.kb1 - u.kb0;
        const int b = ui % kAccs;
        if (ui >= kAccs) mbar_wait(&acc_empty[b], ((ui / kAccs) - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t acc = tmem + b * NT * kTokTile;
        for (int kb = u.kb0; kb < u.kb1; ++kb, ++it) {
          const int s = it % stages;
          mbar_wait(&full[s], (it / stages) & 1);
          const int sx = it % C::kXStages;
          if constexpr (C::kSplitX) mbar_wait(&xfull[sx], (it / C::kXStages) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          unsigned char* st = smem + s * stage_bytes;
#ifdef PEARL_TIMELINE
          if (it == 0) PEARL_TL(a.tl, 2);
#endif
          const uint64_t adesc = umma_desc_sw128(st);
          // all NT token tiles in ONE MMA of N = 16 NT columns (the tiles are
          // contiguous rows of one SW128 operand); per-column arithmetic is the
          // same for any N (tests/test_gemm_gpu.py::test_batch_invariance)
          const uint64_t bdesc =
              umma_desc_sw128(C::kSplitX ? xring + sx * C::kXStageBytes : st + kWBytes);
#pragma unroll
          for (int kk = 0; kk < kTileK / 16; ++kk)
            umma_bf16_n(acc, adesc + 2 * kk, bdesc + 2 * kk, (kb > u.kb0 || kk > 0) ? 1u : 0u,
                        umma_idesc(NT * kTokTile));
          umma_commit(&empty[s]);
          if constexpr (C::kSplitX) umma_commit(&xempty[sx]);
        }
        umma_commit(&acc_full[b]);
      }
      PEARL_TL(a.tl, 3);
    }
  } else {
    // ---- epilogue warps 2..(2 + kEpiWarps); with 8 of them, warps w and
    // w + 4 read the same TMEM lane quarter and take alternate token chunks
    constexpr int EPI = C::kEpi;
    constexpr int HALVES = C::kEpiWarps / 4;
    const int lanegrp = warp & 3;  // TMEM lane quarter this warp may access
    const int row = lanegrp * 32 + lane;
    const int et = threadIdx.x - 64;  // 0..EPI-1
    const int half = et / 128;
    const int Mp = (a.M + 3) & ~3;  // partial row stride (float4 aligned)
    // folded RMSNorm: the per-token scales, once per CTA, while the first
    // accumulator is still being filled
    const float* rsp = nullptr;
    if (a.e.ss_in != nullptr) {
      asm volatile("griddepcontrol.wait;" ::: "memory");
      for (int t = et; t < a.M; t += EPI) s_rs[t] = norm_rs(a.e, t);
      epi_bar_n<EPI>();
      rsp = s_rs;
    }
    // QKV (sequence mode): the window's first position, read once (the
    // epilogue's RoPE-table loads then need no dependent position load)
    int pos0 = INT_MIN;
    if (a.e.kind == EPI_QKV && a.e.tok_pos == nullptr) {
      asm volatile("griddepcontrol.wait;" ::: "memory");
      pos0 = *a.e.pos + a.e.pos_add;
    }
    int ui = 0;
    for (long long x = r0; x < r1; ++ui) {
      const Unit u = unit_at(a, x, r1);
      x += u.kb1 - u.kb0;
      const int tile = u.tile;
      const int b = ui % kAccs;
      mbar_wait(&acc_full[b], (ui / kAccs) & 1);
      if (et == 0) PEARL_TL(a.tl, 5);  // (timeline builds) the last unit's accumulator is ready
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      // the accumulator in 16-column chunks (16 registers live, not 16 NT):
      // token-major staging of the tile (a warp's 32 rows of one token are
      // 128 contiguous bytes) or this split's fp32 partial [t][row] (coalesced)
      float* dst = a.partials + (static_cast<size_t>(tile) * a.seg_max + u.seg) * Mp * kTileN + row;
#pragma unroll 1
      for (int j = half; j < NT; j += HALVES) {
        float v[16];
        tmem_ld16(tmem + (static_cast<uint32_t>(lanegrp * 32) << 16) + b * NT * kTokTile + j * kTokTile, v);
        if (u.nseg == 1) {
#pragma unroll
          for (int c = 0; c < 16; ++c) E[(16 * j + c) * ES + row] = v[c];
        } else {
#pragma unroll
          for (int c = 0; c < 16; ++c)
            if (16 * j + c < a.M) dst[static_cast<size_t>(16 * j + c) * kTileN] = v[c];
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      mbar_arrive(&acc_empty[b]);  // the MMA warp may reuse this accumulator
      if (u.nseg != 1) {
        epi_bar_n<EPI>();  // all partial stores of the CTA precede the releasing atomic
        if (et == 0) {
          int old;
          // release this CTA's partial stores (ordered before by the barrier)
          // and, on the last arrival, acquire everyone else's: the CTA barrier
          // below then orders every thread's partial loads after it
          asm volatile("atom.add.acq_rel.gpu.global.s32 %0, [%1], 1;" : "=r"(old) : "l"(a.flags + tile) : "memory");
          *s_last = (old == u.nseg - 1);
        }
        epi_bar_n<EPI>();
        if (!*s_last) continue;
        if (et == 0) PEARL_TL(a.tl, 6);  // (timeline builds) last arriver starts the reduction
        if (et == 0) PEARL_TL(a.tl, 9);
        // Fixed split order => independent of arrival order and of M: each
        // element is ((0 + p_0) + p_1) + ... over the splits in order.  One
        // 16-token tile at a time, its 16 loads per split in flight together.
        const float* src = a.partials + static_cast<size_t>(tile) * a.seg_max * Mp * kTileN + row;
        const size_t sstride = static_cast<size_t>(Mp) * kTileN;
        if (a.M <= 4) {
          // short windows: up to 8 splits' (<= 4) values in flight at once,
          // then summed in split order -- the same additions as below, one
          // L2 round trip instead of one per split (the tail of the GEMM)
          float acc[4] = {0.f, 0.f, 0.f, 0.f};
          for (int sg0 = 0; sg0 < u.nseg; sg0 += 8) {
            float p[8][4];
#pragma unroll
            for (int q = 0; q < 8; ++q)
#pragma unroll
              for (int c = 0; c < 4; ++c)
                p[q][c] = (sg0 + q < u.nseg && c < a.M)
                              ? __ldcg(src + (sg0 + q) * sstride + static_cast<size_t>(c) * kTileN) : 0.f;
#pragma unroll
            for (int q = 0; q < 8; ++q)
              if (sg0 + q < u.nseg)
#pragma unroll
                for (int c = 0; c < 4; ++c) acc[c] += p[q][c];
          }
#pragma unroll
          for (int c = 0; c < 4; ++c) E[c * ES + row] = acc[c];
        } else if (a.M > 32) {
          // wide windows / prefill: every (token, 4-row group) item of the
          // tile as a float4 (item idx = et + 128 i: the epilogue's mapping),
          // 8 items' loads in flight per round, splits added in order
          const float* base = a.partials + static_cast<size_t>(tile) * a.seg_max * Mp * kTileN;
          const int nit = (32 * a.M - et + EPI - 1) / EPI;
          for (int i0 = 0; i0 < nit; i0 += 8) {
            float4 acc[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int sg = 0; sg < u.nseg; ++sg) {
              float4 pv[8];
#pragma unroll
              for (int q = 0; q < 8; ++q) {
                const int idx = et + EPI * (i0 + q);
                pv[q] = i0 + q < nit ? __ldcg(reinterpret_cast<const float4*>(
                                           base + sg * sstride + static_cast<size_t>(idx / 32) * kTileN + 4 * (idx % 32)))
                                     : make_float4(0.f, 0.f, 0.f, 0.f);
              }
#pragma unroll
              for (int q = 0; q < 8; ++q) {
                acc[q].x += pv[q].x;
                acc[q].y += pv[q].y;
                acc[q].z += pv[q].z;
                acc[q].w += pv[q].w;
              }
            }
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const int idx = et + EPI * (i0 + q);
              if (i0 + q < nit) *reinterpret_cast<float4*>(E + (idx / 32) * ES + 4 * (idx % 32)) = acc[q];
            }
          }
        } else {
#pragma unroll 1
          for (int j = half; j < NT; j += HALVES) {  // 8 warps: the two warps of a row take alternate chunks
            if (16 * j >= a.M) break;
            float acc[16];
#pragma unroll
            for (int c = 0; c < 16; ++c) acc[c] = 0.f;
            // SGB splits' 16 values in flight per round, summed in split order
            constexpr int SGB = NT == 1 ? 4 : 2;
            for (int sg = 0; sg < u.nseg; sg += SGB) {
              float p[SGB][16];
#pragma unroll
              for (int q = 0; q < SGB; ++q)
#pragma unroll
                for (int c = 0; c < 16; ++c)
                  p[q][c] = (sg + q < u.nseg && 16 * j + c < a.M)
                                ? __ldcg(src + (sg + q) * sstride + static_cast<size_t>(16 * j + c) * kTileN) : 0.f;
#pragma unroll
              for (int q = 0; q < SGB; ++q)
                if (sg + q < u.nseg)
#pragma unroll
                  for (int c = 0; c < 16; ++c) acc[c] += p[q][c];
            }
#pragma unroll
            for (int c = 0; c < 16; ++c) E[(16 * j + c) * ES + row] = acc[c];
          }
        }
        if (et == 0) a.flags[tile] = 0;
      }
      epi_bar_n<EPI>();
      if (et == 0) PEARL_TL(a.tl, 7);  // (timeline builds) tile staged in E
      if (NT <= 2) {
        // MAXI * EPI / 32 = 16 NT tokens: exactly the window's tiles
        epilogue_tile<NT * 512 / EPI, true, EPI>(a.e, tile, E, ES, a.M, a.N, et, rsp, 0, pos0);
      } else {  // 64-token slices: 8 items per thread at a time over the 8 warps
        for (int t0 = 0; t0 < a.M; t0 += 64) epilogue_tile<8, true, EPI>(a.e, tile, E, ES, a.M, a.N, et, rsp, t0, pos0);
      }
      epi_bar_n<EPI>();
      if (et == 0) PEARL_TL(a.tl, 8);  // (timeline builds) epilogue done
    }
  }
  __syncwarp();
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 64) PEARL_TL(a.tl, 4);
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(C::kTmemCols));
}

// ---- host side ---------------------------------------------------------------

namespace {

PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::once_flag g_enc_once;

int get_encoder() {
  std::call_once(g_enc_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  if (!g_encode) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return PEARL_ERR_CUDA;
  }
  return PEARL_OK;
}

int encode_2d(CUtensorMap* map, const void* base, int inner, int rows, int box_rows) {
  int rc = get_encoder();
  if (rc) return rc;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(inner) * 2};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(kTileK), static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed: " + std::to_string(static_cast<int>(r)));
    return PEARL_ERR_CUDA;
  }
  return PEARL_OK;
}

std::once_flag g_attr_once;
cudaError_t g_attr_err = cudaSuccess;

template <int NT>
cudaError_t set_attr() {
  return cudaFuncSetAttribute(tc_gemm_kernel<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              static_cast<int>(TcCfg<NT>::kSmem));
}

}  // namespace

int tc_encode_2d(CUtensorMap* map, const void* base, int inner, int rows, int box_rows) {
  return encode_2d(map, base, inner, rows, box_rows);
}

// Split-K factor for an (N, K) weight: enough (tile, split) units to keep
// every SM's pipeline busy while per-SM work stays balanced.  Depends on the
// shape only (batch invariance).
int tc_splits(int N, int K, int num_sms) {
  const int tiles = (N + kTileN - 1) / kTileN;
  const int KB = (K + kTileK - 1) / kTileK;
  int best = 1;
  double best_cost = -1;
  for (int S = 1; S <= std::min(KB, 16); ++S) {
    if (KB / S < 4 && S > 1) break;  // keep >= 4 k-blocks of streaming per unit
    const long long units = static_cast<long long>(tiles) * S;
    const long long waves = (units + num_sms - 1) / num_sms;
    // busiest SM: its streamed k-blocks + a per-unit overhead (~1.5 k-block
    // times) + the split-K reduction tail; measured on B200 (tools/gemm_sweep.py)
    const double cost = static_cast<double>(waves * ((KB + S - 1) / S)) + 1.5 * waves + 0.5 * (S - 1);
    if (best_cost < 0 || cost < best_cost - 1e-9) {
      best_cost = cost;
      best = S;
    }
  }
  return best;
}

// Stream-K grid of an (N, K) GEMM on num_sms SMs -- a function of the shape
// only (batch invariance).  Narrow GEMMs (fewer tiles than SMs / 2) whose
// k-blocks divide evenly get tiles x S CTAs, every tile cut into exactly S
// equal splits and every CTA owning one unit: no CTA straddles two tiles, so
// the split-K last arrivers start together and the tail is one reduction
// (7B O / down: 32 tiles x 4 splits on 128 CTAs).  Otherwise all SMs.
int tc_grid(int N, int K, int num_sms) {
  const int tiles = (N + kTileN - 1) / kTileN;
  const int KB = (K + kTileK - 1) / kTileK;
  const long long T = static_cast<long long>(tiles) * KB;
  static const bool even = [] {
    const char* env = std::getenv("PEARL_EVEN_SPLITS");  // 0: plain stream-K (A/B)
    return !(env && env[0] == '0');
  }();
  if (even) {
    for (int S = num_sms / tiles; S >= 2; --S) {
      if (KB % S == 0 && KB / S >= 4 && tiles * S * 5 >= num_sms * 4) return tiles * S;
    }
  }
  return static_cast<int>(std::min<long long>(num_sms, T));
}

// Largest number of stream-K segments any tile is cut into.
int tc_seg_max(int tiles, int KB, int G) {
  const long long T = static_cast<long long>(tiles) * KB;
  auto cta_of = [&](long long x) { return static_cast<int>(((x + 1) * G + T - 1) / T) - 1; };
  int mx = 1;
  for (int t = 0; t < tiles; ++t) {
    const long long t0 = static_cast<long long>(t) * KB;
    mx = std::max(mx, cta_of(t0 + KB - 1) - cta_of(t0) + 1);
  }
  return mx;
}

int tc_init(TcGemmCtx& ctx, const pearl_llama_config& c) {
  if (c.max_tokens > kMaxTokTiles * kTokTile) {
    set_error("tcgen05 path supports max_tokens <= 128");
    return PEARL_ERR_ARG;
  }
  int dev = 0;
  PEARL_CUDA_TRY(cudaGetDevice(&dev));
  PEARL_CUDA_TRY(cudaDeviceGetAttribute(&ctx.num_sms, cudaDevAttrMultiProcessorCount, dev));
  if (c.sm_count > 0) ctx.num_sms = std::min(ctx.num_sms, c.sm_count);
  std::call_once(g_attr_once, [] {
    cudaError_t e = set_attr<1>();
    if (e == cudaSuccess) e = set_attr<2>();
    if (e == cudaSuccess) e = set_attr<3>();
    if (e == cudaSuccess) e = set_attr<4>();
    if (e == cudaSuccess) e = set_attr<5>();
    if (e == cudaSuccess) e = set_attr<6>();
    if (e == cudaSuccess) e = set_attr<7>();
    if (e == cudaSuccess) e = set_attr<8>();
    g_attr_err = e;
  });
  PEARL_CUDA_TRY(g_attr_err);
  ctx.max_tokens = c.max_tokens;
  const int hd = c.head_dim;
  const int shapes[5][2] = {{(c.n_heads + 2 * c.n_kv_heads) * hd, c.d_model},
                            {c.d_model, c.n_heads * hd},
                            {2 * c.ffn, c.d_model},
                            {c.d_model, c.ffn},
                            {c.vocab, c.d_model}};
  size_t pf = 0;
  int flags = 0;
  for (auto& s : shapes) {
    const int tiles = (s[0] + kTileN - 1) / kTileN;
    const int KB = (s[1] + kTileK - 1) / kTileK;
    int Sa = tc_seg_max(tiles, KB, tc_grid(s[0], s[1], ctx.num_sms));
    Sa = std::max(Sa, ctx.min_plan_splits);
    pf = std::max(pf, static_cast<size_t>(tiles) * Sa * kTileN * kMaxTokTiles * kTokTile);
    flags = std::max(flags, tiles);
  }
  ctx.partial_floats = pf;
  ctx.n_flags = flags;
  PEARL_CUDA_TRY(cudaMalloc(&ctx.partials, pf * sizeof(float)));
  PEARL_CUDA_TRY(cudaMalloc(&ctx.tile_flags, static_cast<size_t>(flags) * sizeof(int)));
  PEARL_CUDA_TRY(cudaMemset(ctx.tile_flags, 0, static_cast<size_t>(flags) * sizeof(int)));
  return get_encoder();
}

void tc_free(TcGemmCtx& ctx) {
  if (ctx.partials) cudaFree(ctx.partials);
  if (ctx.tile_flags) cudaFree(ctx.tile_flags);
  ctx.partials = nullptr;
  ctx.tile_flags = nullptr;
}

int tc_gemm(TcGemmCtx& ctx, const __nv_bfloat16* W, const __nv_bfloat16* X, int M, int N, int K, const EpiArgs& e,
            cudaStream_t st, int force_splits, bool w_tiled) {
  if (M < 1 || M > kMaxTokTiles * kTokTile) {
    set_error("tc_gemm: M must be in [1, 128]");
    return PEARL_ERR_ARG;
  }
  if (K % 8 != 0) {
    set_error("tc_gemm: K must be a multiple of 8");
    return PEARL_ERR_ARG;
  }
  if (w_tiled && (N % kTileN != 0 || K % kTileK != 0)) {
    set_error("tc_gemm: tile-major weights need N % 128 == 0 and K % 64 == 0");
    return PEARL_ERR_ARG;
  }
  const auto key = std::make_tuple(static_cast<const void*>(W), w_tiled ? -N : N, K);
  auto it = ctx.wmaps.find(key);
  if (it == ctx.wmaps.end()) {
    TcWeightMap wm;
    // tile-major: a [N K / 64, 64] matrix of 128-byte rows, box 64 x 128
    int rc = w_tiled ? encode_2d(&wm.map, W, kTileK, static_cast<int>(static_cast<long long>(N) * K / kTileK), kTileN)
                     : encode_2d(&wm.map, W, K, N, kTileN);
    if (rc) return rc;
    it = ctx.wmaps.emplace(key, wm).first;
  }
  // the window's NT token tiles as ONE box (16 NT rows of 128 B; the SW128
  // layout of stacked 16-row boxes and of one tall box is the same), so the
  // producer issues one X copy per stage instead of NT
  alignas(64) CUtensorMap xmap;
  int rc = encode_2d(&xmap, X, K, M, kTokTile * ((M + kTokTile - 1) / kTokTile));
  if (rc) return rc;
  TcArgs a;
  a.M = M;
  a.N = N;
  a.K = K;
  a.KB = (K + kTileK - 1) / kTileK;
  const int tiles = (N + kTileN - 1) / kTileN;
  a.T = static_cast<long long>(tiles) * a.KB;
  a.G = force_splits > 0 ? static_cast<int>(std::min<long long>(force_splits, a.T)) : tc_grid(N, K, ctx.num_sms);
  a.seg_max = tc_seg_max(tiles, a.KB, a.G);
  a.w_tiled = w_tiled ? 1 : 0;
  a.e = e;
  a.partials = ctx.partials;
  a.flags = ctx.tile_flags;
#ifdef PEARL_TIMELINE
  a.tl = timeline_next(0);
#else
  a.tl = nullptr;
#endif
  if (static_cast<size_t>(tiles) * a.seg_max * kTileN * kMaxTokTiles * kTokTile > ctx.partial_floats ||
      tiles > ctx.n_flags) {
    set_error("tc_gemm: shape exceeds the planned split-K workspace");
    return PEARL_ERR_ARG;
  }
  const int NT = (M + kTokTile - 1) / kTokTile;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(a.G);
  cfg.blockDim = dim3(kTcThreads);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  switch (NT) {
    case 1:
      cfg.dynamicSmemBytes = TcCfg<1>::kSmem;
      cfg.blockDim = dim3(TcCfg<1>::kThreads);
      PEARL_CUDA_TRY(cudaLaunchKernelEx(&cfg, tc_gemm_kernel<1>, it->second.map, xmap, a));
      break;
    case 2:
      cfg.dynamicSmemBytes = TcCfg<2>::kSmem;
      cfg.blockDim = dim3(TcCfg<2>::kThreads);
      PEARL_CUDA_TRY(cudaLaunchKernelEx(&cfg, tc_gemm_kernel<2>, it->second.map, xmap, a));
      break;
    case 3:
      cfg.dynamicSmemBytes = TcCfg<3>::kSmem;
      cfg.blockDim = dim3(TcCfg<3>::kThreads);
      PEARL_CUDA_TRY(cudaLaunchKernelEx(&cfg, tc_gemm_kernel<3>, it->second.map, xmap, a));
      break;
    case 4:
      cfg.dynamicSmemBytes = TcCfg<4>::kSmem;
      cfg.blockDim = dim3(TcCfg<4>::kThreads);
      PEARL_CUDA_TRY(cudaLaunchKernelEx(&cfg, tc_gemm_kernel<4>, it->second.map, xmap, a));
      break;
    case 5:
      cfg.dynamicSmemBytes = TcCfg<5>::kSmem;
      cfg.blockDim = dim3(TcCfg<5>::kThreads);
      PEARL_CUDA_TRY(cudaLaunchKernelEx(&cfg, tc_gemm_kernel<5>, it->second.map, xmap, a));
      break;
    case 6:
      cfg.dynamicSmemBytes = TcCfg<6>::kSmem;
      cfg.blockDim = dim3(TcCfg<6>::kThreads);
      PEARL_CUDA_TRY(cudaLaunchKernelEx(&cfg, tc_gemm_kernel<6>, it->second.map, xmap, a));
      break;
    case 7:
      cfg.dynamicSmemBytes = TcCfg<7>::kSmem;
      cfg.blockDim = dim3(TcCfg<7>::kThreads);
      PEARL_CUDA_TRY(cudaLaunchKernelEx(&cfg, tc_gemm_kernel<7>, it->second.map, xmap, a));
      break;
    default:
      cfg.dynamicSmemBytes = TcCfg<8>::kSmem;
      cfg.blockDim = dim3(TcCfg<8>::kThreads);
      PEARL_CUDA_TRY(cudaLaunchKernelEx(&cfg, tc_gemm_kernel<8>, it->second.map, xmap, a));
      break;
  }
  count_launch();
  return PEARL_OK;
}

}  // namespace pearl
