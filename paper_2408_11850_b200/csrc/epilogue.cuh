// Fused GEMM epilogues shared by the CUDA-core GEMV (K2) and the tcgen05
// GEMM (K3): fp32 store (logits), residual add, RoPE + Q store + K/V cache
// append, SwiGLU.  Both GEMMs call epilogue4 on identical fp32 values, so the
// epilogue never introduces a difference between the two engines.
#pragma once

#include <cuda_bf16.h>
#include <stdint.h>

#include <climits>

namespace pearl {

using bf16 = __nv_bfloat16;

// ---------------------------------------------------------------------------
// Epilogues shared by the CUDA-core and tcgen05 GEMMs
// ---------------------------------------------------------------------------
enum EpiKind { EPI_STORE_F32 = 0, EPI_RESID = 1, EPI_QKV = 2, EPI_SWIGLU = 3 };

struct EpiArgs {
  int kind;
  float* out_f32;   // STORE_F32: [M, N]; RESID: h [M, N]
  bf16* out_bf16;   // QKV: q [M, H hd]; SWIGLU: act [M, N/2]
  bf16* kc;         // QKV: layer k cache [max_seq, KV, hd]
  bf16* vc;
  const float* cos_t;
  const float* sin_t;
  const int32_t* pos;
  int pos_add;
  int n_q;          // H * hd
  int n_kv;         // KV * hd
  int hd;
  int ld;           // leading dimension of out
  // slot mode (batched sequences, pearl_llama_forward_slots): token t sits at
  // position tok_pos[t] of KV slot tok_slot[t] (cache base + slot * slot_stride)
  const int32_t* tok_pos;
  const int32_t* tok_slot;
  long long slot_stride;
  int32_t* adv_pos; // optional: one thread adds adv_n to *adv_pos once the kernel's
  int adv_n;        //   inputs are ready (folds the forward's position advance into
                    //   its last GEMM: every earlier reader of pos has completed)
  // RMSNorm folded into the tcgen05 GEMMs (no norm kernel; see llama.cu):
  //  * producer side (RESID): also write the next GEMM's operand
  //    x_out[t] = bf16(h[t] * gain) and, per 128-row tile, the tile's sum of
  //    h^2 into ss_out[tile * ss_ld + t];
  //  * consumer side (QKV / SWIGLU / STORE_F32): scale every output by
  //    rs[t] = 1 / sqrt(sum_tiles ss_in[tile * ss_ld + t] / d + eps), computed
  //    once per CTA (norm_rs) and passed to epilogue_tile.
  bf16* x_out;
  const float* gain;
  float* ss_out;
  const float* ss_in;
  int ss_ld;        // tokens per ss row (the model's max_tokens)
  int ss_tiles;     // tiles summed by the consumer (ceil(d / 128))
  int norm_d;
  float norm_eps;
};

// Sum of squares of four consecutive h values, reduced over a warp's 32
// lanes (= the 32 four-row groups of one 128-row tile) in a fixed xor tree.
// The embedding kernel and the residual epilogue use exactly this order.
__device__ __forceinline__ float tile_sumsq(float4 h) {
  float s = h.x * h.x;
  s = fmaf(h.y, h.y, s);
  s = fmaf(h.z, h.z, s);
  s = fmaf(h.w, h.w, s);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  return s;
}

// rs[t] of token t from the producer's per-tile partial sums (fixed order).
// The tile sums are loaded 16 at a time (independent loads in flight, one L2
// round trip per 16 tiles instead of one per tile) and added in tile order.
__device__ __forceinline__ float norm_rs(const EpiArgs& e, int t) {
  float tot = 0.f;
  for (int k0 = 0; k0 < e.ss_tiles; k0 += 16) {
    float v[16];
#pragma unroll
    for (int q = 0; q < 16; ++q)
      v[q] = k0 + q < e.ss_tiles ? __ldcg(e.ss_in + static_cast<size_t>(k0 + q) * e.ss_ld + t) : 0.f;
#pragma unroll
    for (int q = 0; q < 16; ++q)
      if (k0 + q < e.ss_tiles) tot += v[q];
  }
  return 1.0f / sqrtf(tot / static_cast<float>(e.norm_d) + e.norm_eps);
}

// The per-element arithmetic, with explicit rounding (no FMA contraction), so
// every call site -- GEMV, per-GEMM tcgen05 kernel, persistent forward --
// produces the same bits whatever the compiler does around it.
__device__ __forceinline__ float swiglu1(float gt, float up) {
  return __fmul_rn(__fdiv_rn(gt, __fadd_rn(1.0f, expf(-gt))), up);
}

__device__ __forceinline__ void rope2(float x0, float x1, float c, float s, float* y0, float* y1) {
  *y0 = __fsub_rn(__fmul_rn(x0, c), __fmul_rn(x1, s));
  *y1 = __fadd_rn(__fmul_rn(x0, s), __fmul_rn(x1, c));
}

// Position and KV-slot offset (elements) of window token t.
__device__ __forceinline__ int epi_pos(const EpiArgs& e, int t) {
  return e.tok_pos ? e.tok_pos[t] : *e.pos + e.pos_add + t;
}
__device__ __forceinline__ size_t epi_slot_off(const EpiArgs& e, int t) {
  return e.tok_slot ? static_cast<size_t>(e.tok_slot[t]) * static_cast<size_t>(e.slot_stride) : 0;
}

// Handle four consecutive output rows n0..n0+3 (n0 % 4 == 0) for token t.
__device__ __forceinline__ void epilogue4(const EpiArgs& e, int t, int n0, const float* v, int N) {
  switch (e.kind) {
    case EPI_STORE_F32:
      for (int r = 0; r < 4; ++r)
        if (n0 + r < N) e.out_f32[static_cast<size_t>(t) * e.ld + n0 + r] = v[r];
      break;
    case EPI_RESID:
      for (int r = 0; r < 4; ++r)
        if (n0 + r < N) e.out_f32[static_cast<size_t>(t) * e.ld + n0 + r] += v[r];
      break;
    case EPI_SWIGLU: {
      // rows (2j, 2j+1) = (gate_j, up_j)
      for (int r = 0; r < 4; r += 2) {
        e.out_bf16[static_cast<size_t>(t) * e.ld + (n0 + r) / 2] = __float2bfloat16(swiglu1(v[r], v[r + 1]));
      }
      break;
    }
    case EPI_QKV: {
      const int p = epi_pos(e, t);
      const size_t so = epi_slot_off(e, t);
      const int half = e.hd >> 1;
      if (n0 < e.n_q + e.n_kv) {
        float w[4];
        for (int r = 0; r < 4; r += 2) {
          const int n = n0 + r;
          const int i = (n % e.hd) >> 1;  // rotation pair index within the head
          const float c = e.cos_t[static_cast<size_t>(p) * half + i];
          const float s = e.sin_t[static_cast<size_t>(p) * half + i];
          rope2(v[r], v[r + 1], c, s, &w[r], &w[r + 1]);
        }
        if (n0 < e.n_q) {
          for (int r = 0; r < 4; ++r) e.out_bf16[static_cast<size_t>(t) * e.n_q + n0 + r] = __float2bfloat16(w[r]);
        } else {
          const int nk = n0 - e.n_q;
          for (int r = 0; r < 4; ++r)
            e.kc[so + static_cast<size_t>(p) * e.n_kv + nk + r] = __float2bfloat16(w[r]);
        }
      } else {
        const int nv = n0 - e.n_q - e.n_kv;
        for (int r = 0; r < 4; ++r) e.vc[so + static_cast<size_t>(p) * e.n_kv + nv + r] = __float2bfloat16(v[r]);
      }
      break;
    }
  }
}

// Epilogue of one 128-row output tile for tokens 0..M-1 on the tcgen05 paths
// (per-GEMM kernel and persistent forward): E is the tile's fp32 result in
// smem -- row-major E[row * ES + t] (TR = false, persistent forward) or
// token-major E[t * ES + row] (TR = true, per-GEMM kernel: conflict-free
// staging stores and one 16-byte read per item); 128 threads (et) take items
// (4-row group g, token t) = (idx % 32, idx / 32), idx = et + 128 i.  Same
// arithmetic as epilogue4, but every global load of all of a thread's items
// (residual rows, RoPE tables, the position) is issued before any store, so a
// tile's epilogue costs one memory round trip instead of one per item.
template <bool TR>
__device__ __forceinline__ float4 epi_rows4(const float* E, int ES, int g, int t) {
  if (TR) return *reinterpret_cast<const float4*>(E + t * ES + g * 4);
  return make_float4(E[(g * 4) * ES + t], E[(g * 4 + 1) * ES + t], E[(g * 4 + 2) * ES + t], E[(g * 4 + 3) * ES + t]);
}

__device__ __forceinline__ float4 scale4(float4 v, float r) {
  return make_float4(__fmul_rn(v.x, r), __fmul_rn(v.y, r), __fmul_rn(v.z, r), __fmul_rn(v.w, r));
}

// rs: per-token norm scales in smem (nullptr: no folded norm).
// t_base: this call covers tokens t_base .. min(M, t_base + MAXI * 4) - 1
// (wide windows run it in 64-token slices, bounding the registers per thread).
// NTHR: the epilogue threads sharing the items (idx = et + NTHR i); a call
// covers up to MAXI * NTHR / 32 tokens.
// pos0: the window's first position when the caller already read it (QKV,
// sequence mode; INT_MIN: read *e.pos here).
template <int MAXI, bool TR = false, int NTHR = 128>
__device__ __forceinline__ void epilogue_tile(const EpiArgs& e, int tile, const float* E, int ES, int M, int N,
                                              int et, const float* rs = nullptr, int t_base = 0,
                                              int pos0 = INT_MIN) {
  constexpr int kGroups = 32;  // 128 rows / 4
  constexpr int kTok = MAXI * NTHR / kGroups;
  E += static_cast<size_t>(t_base) * (TR ? ES : 1);
  if (rs) rs += t_base;
  const int nitems = kGroups * (M - t_base < kTok ? M - t_base : kTok);
  switch (e.kind) {
    case EPI_STORE_F32:
#pragma unroll
      for (int i = 0; i < MAXI; ++i) {
        const int idx = et + NTHR * i, g = idx % kGroups, t = idx / kGroups, n0 = tile * 128 + g * 4;
        if (idx >= nitems || n0 >= N) continue;
        float* o = e.out_f32 + static_cast<size_t>(t_base + t) * e.ld + n0;
        float4 v = epi_rows4<TR>(E, ES, g, t);
        if (rs) v = scale4(v, rs[t]);
        if (n0 + 3 < N && (e.ld & 3) == 0) {
          *reinterpret_cast<float4*>(o) = v;
        } else {
          const float w[4] = {v.x, v.y, v.z, v.w};
          for (int r = 0; r < 4; ++r)
            if (n0 + r < N) o[r] = w[r];
        }
      }
      break;
    case EPI_RESID: {
      // a thread's items share their 4-row group g (NTHR is a multiple of
      // 32), so the gain slice is one load, issued with the residual loads
      float4 gv = make_float4(0.f, 0.f, 0.f, 0.f);
      {
        const int n0 = tile * 128 + (et % kGroups) * 4;
        if (e.x_out && n0 + 3 < N) gv = __ldg(reinterpret_cast<const float4*>(e.gain + n0));
      }
      float4 hv[MAXI];
#pragma unroll
      for (int i = 0; i < MAXI; ++i) {
        const int idx = et + NTHR * i, g = idx % kGroups, t = idx / kGroups, n0 = tile * 128 + g * 4;
        if (idx < nitems && n0 + 3 < N)
          hv[i] = *reinterpret_cast<const float4*>(e.out_f32 + static_cast<size_t>(t_base + t) * e.ld + n0);
      }
#pragma unroll
      for (int i = 0; i < MAXI; ++i) {
        const int idx = et + NTHR * i, g = idx % kGroups, t = idx / kGroups, n0 = tile * 128 + g * 4;
        if (idx >= nitems) continue;  // uniform per warp: a warp's 32 lanes are one token's 32 groups
        float4 hn = make_float4(0.f, 0.f, 0.f, 0.f);
        if (n0 < N) {
          float* o = e.out_f32 + static_cast<size_t>(t_base + t) * e.ld + n0;
          const float4 v = epi_rows4<TR>(E, ES, g, t);
          if (n0 + 3 < N) {
            hn = make_float4(hv[i].x + v.x, hv[i].y + v.y, hv[i].z + v.z, hv[i].w + v.w);
            *reinterpret_cast<float4*>(o) = hn;
          } else {
            const float w[4] = {v.x, v.y, v.z, v.w};
            for (int r = 0; r < 4; ++r)
              if (n0 + r < N) o[r] += w[r];
          }
        }
        if (e.x_out) {
          if (n0 + 3 < N) {
            const __nv_bfloat162 lo = __floats2bfloat162_rn(hn.x * gv.x, hn.y * gv.y);
            const __nv_bfloat162 hi = __floats2bfloat162_rn(hn.z * gv.z, hn.w * gv.w);
            *reinterpret_cast<uint2*>(e.x_out + static_cast<size_t>(t_base + t) * e.ld + n0) =
                make_uint2(*reinterpret_cast<const uint32_t*>(&lo), *reinterpret_cast<const uint32_t*>(&hi));
          }
          const float ss = tile_sumsq(hn);
          if (g == 0) e.ss_out[static_cast<size_t>(tile) * e.ss_ld + t_base + t] = ss;
        }
      }
      break;
    }
    case EPI_SWIGLU:
#pragma unroll
      for (int i = 0; i < MAXI; ++i) {
        const int idx = et + NTHR * i, g = idx % kGroups, t = idx / kGroups, n0 = tile * 128 + g * 4;
        if (idx >= nitems || n0 >= N) continue;
        float4 v = epi_rows4<TR>(E, ES, g, t);
        if (rs) v = scale4(v, rs[t]);
        e.out_bf16[static_cast<size_t>(t_base + t) * e.ld + n0 / 2] = __float2bfloat16(swiglu1(v.x, v.y));
        e.out_bf16[static_cast<size_t>(t_base + t) * e.ld + (n0 + 2) / 2] = __float2bfloat16(swiglu1(v.z, v.w));
      }
      break;
    case EPI_QKV: {
      const int p0 = e.tok_pos ? 0 : (pos0 != INT_MIN ? pos0 : *e.pos + e.pos_add);  // slot mode: per-token positions
      const int half = e.hd >> 1;
      float2 cs[MAXI], sn[MAXI];
#pragma unroll
      for (int i = 0; i < MAXI; ++i) {
        const int idx = et + NTHR * i, g = idx % kGroups, t = idx / kGroups, n0 = tile * 128 + g * 4;
        if (idx < nitems && n0 < e.n_q + e.n_kv) {
          const size_t off = static_cast<size_t>(e.tok_pos ? e.tok_pos[t_base + t] : p0 + t_base + t) * half + ((n0 % e.hd) >> 1);
          cs[i] = *reinterpret_cast<const float2*>(e.cos_t + off);
          sn[i] = *reinterpret_cast<const float2*>(e.sin_t + off);
        }
      }
#pragma unroll
      for (int i = 0; i < MAXI; ++i) {
        const int idx = et + NTHR * i, g = idx % kGroups, t = idx / kGroups, n0 = tile * 128 + g * 4;
        if (idx >= nitems || n0 >= N) continue;
        const int p = e.tok_pos ? e.tok_pos[t_base + t] : p0 + t_base + t;
        const size_t so = epi_slot_off(e, t_base + t);
        float4 v4 = epi_rows4<TR>(E, ES, g, t);
        if (rs) v4 = scale4(v4, rs[t]);
        const float v[4] = {v4.x, v4.y, v4.z, v4.w};
        if (n0 < e.n_q + e.n_kv) {
          float w[4];
          rope2(v[0], v[1], cs[i].x, sn[i].x, &w[0], &w[1]);
          rope2(v[2], v[3], cs[i].y, sn[i].y, &w[2], &w[3]);
          bf16* dst = n0 < e.n_q ? e.out_bf16 + static_cast<size_t>(t_base + t) * e.n_q + n0
                                 : e.kc + so + static_cast<size_t>(p) * e.n_kv + (n0 - e.n_q);
          for (int r = 0; r < 4; ++r) dst[r] = __float2bfloat16(w[r]);
        } else {
          bf16* dst = e.vc + so + static_cast<size_t>(p) * e.n_kv + (n0 - e.n_q - e.n_kv);
          for (int r = 0; r < 4; ++r) dst[r] = __float2bfloat16(v[r]);
        }
      }
      break;
    }
  }
}

}  // namespace pearl
