// Fused GEMM epilogues shared by the CUDA-core GEMV (K2) and the tcgen05
// GEMM (K3): fp32 store (logits), residual add, RoPE + Q store + K/V cache
// append, SwiGLU.  Both GEMMs call epilogue4 on identical fp32 values, so the
// epilogue never introduces a difference between the two engines.
#pragma once

#include <cuda_bf16.h>
#include <stdint.h>

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
};

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
        const float gt = v[r], up = v[r + 1];
        const float s = gt / (1.0f + expf(-gt));
        e.out_bf16[static_cast<size_t>(t) * e.ld + (n0 + r) / 2] = __float2bfloat16(s * up);
      }
      break;
    }
    case EPI_QKV: {
      const int p = *e.pos + e.pos_add + t;
      const int half = e.hd >> 1;
      if (n0 < e.n_q + e.n_kv) {
        float w[4];
        for (int r = 0; r < 4; r += 2) {
          const int n = n0 + r;
          const int i = (n % e.hd) >> 1;  // rotation pair index within the head
          const float c = e.cos_t[static_cast<size_t>(p) * half + i];
          const float s = e.sin_t[static_cast<size_t>(p) * half + i];
          w[r] = v[r] * c - v[r + 1] * s;
          w[r + 1] = v[r] * s + v[r + 1] * c;
        }
        if (n0 < e.n_q) {
          for (int r = 0; r < 4; ++r) e.out_bf16[static_cast<size_t>(t) * e.n_q + n0 + r] = __float2bfloat16(w[r]);
        } else {
          const int nk = n0 - e.n_q;
          for (int r = 0; r < 4; ++r)
            e.kc[static_cast<size_t>(p) * e.n_kv + nk + r] = __float2bfloat16(w[r]);
        }
      } else {
        const int nv = n0 - e.n_q - e.n_kv;
        for (int r = 0; r < 4; ++r) e.vc[static_cast<size_t>(p) * e.n_kv + nv + r] = __float2bfloat16(v[r]);
      }
      break;
    }
  }
}


}  // namespace pearl
