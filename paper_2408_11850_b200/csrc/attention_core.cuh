// K4 device core of the clustered attention kernel (attention.cu): one warp's
// pass over its 32-position segments, the fold of a (logical) CTA's 4 warp
// states, and the fold of the kAttnLCS logical CTA states (see attention.cuh
// for the algorithm).  Kept apart so that every execution shape of the fold
// (4-CTA clusters, one CTA running the logical CTAs in turn) runs exactly the
// same instructions.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "attention.cuh"

namespace pearl {
namespace attn_core {

using bf16 = __nv_bfloat16;
constexpr int kWarps = kAttnThreads / 32;  // warps of one (virtual) CTA

template <int HD>
struct Smem {
  static constexpr int RS = HD + 2;  // state row: o[HD], m, l
  // warp states [kWarps][kAttnMaxRb][RS] (reused per logical CTA) + warp weights
  static constexpr int kWarpFloats = kWarps * kAttnMaxRb * RS + kAttnMaxRb * kWarps;
  // one logical CTA's folded state [kAttnMaxRb][RS]
  static constexpr int kStateFloats = kAttnMaxRb * RS;
  // cluster fold weights [kAttnMaxRb][kAttnCluster] + row sums [kAttnMaxRb]
  static constexpr int kFoldFloats = kAttnMaxRb * kAttnCluster + kAttnMaxRb;
};

__device__ __forceinline__ int tok_position(const AttnArgs& a, int p0, int t) {
  return a.tok_pos ? a.tok_pos[t] : p0 + t;
}

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

// One warp's pass: rows r0..r0+R-1 of the item (row r = token r / g, query
// head kvh g + r % g), segments P0(js) = 32 ((js CS + crank) 4 + warp),
// js = 0..spw-1, folded in js order with an online softmax; the state
// (o[HD], m, l per row, 16 rows) goes to sw[16][HD + 2].  kb / vb may hold
// segment 0's positions <= old_hi already (loaded before a PDL wait).
template <int HD>
__device__ __forceinline__ void warp_pass(const AttnArgs& a, const bf16* kc, const bf16* vc, size_t kvs, int p0,
                                          int r0, int R, int g, int kvh, int pmax, int CS, int crank, int warp,
                                          int lane, int spw, int old_hi, uint4 (*kb)[HD / 32], uint4 (*vb)[HD / 32],
                                          float* sw) {
  constexpr int J = HD / 32;    // 32-dim blocks
  constexpr int KS = HD / 16;   // q.k k-steps
  constexpr int NO = HD / 8;    // p.v output tiles
  constexpr int RS = HD + 2;
  const int n = lane >> 2, q = lane & 3;
  auto seg_p0 = [&](int js) { return 32 * ((js * CS + crank) * kWarps + warp); };
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
  for (int js = 0; js < spw; ++js) {
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
}

// CTA fold over its kWarps warp states st[w][16][RS] in warp order (weights
// exp(m_w - max), 0 = empty) into cs[16][RS]; threads tid = 0..nthr-1 of the
// (virtual) CTA; `sync` is the CTA's barrier.
template <int HD, typename Sync>
__device__ __forceinline__ void cta_fold(const float* st, float* cs, float* wgt, int R, int tid, int nthr, Sync sync) {
  constexpr int RS = HD + 2;
  if (tid < R * kWarps) {
    const int rr = tid / kWarps, w = tid % kWarps;
    float mx = -INFINITY;
#pragma unroll
    for (int x = 0; x < kWarps; ++x) mx = fmaxf(mx, st[(x * kAttnMaxRb + rr) * RS + HD]);
    const float mw = st[(w * kAttnMaxRb + rr) * RS + HD];
    wgt[rr * kWarps + w] = mw == -INFINITY ? 0.f : expf(mw - mx);
    if (w == 0) cs[rr * RS + HD] = mx;
  }
  sync();
  // items in groups of 2: every load of the group before any store (the
  // compiler cannot move a load above a store to the same shared array)
  constexpr int G = 2;
  const int n = R * (HD + 1);  // d == HD: the row's l
  for (int i0 = tid; i0 < n; i0 += G * nthr) {
    float wt[G][kWarps], sv[G][kWarps];
#pragma unroll
    for (int q = 0; q < G; ++q) {
      const int i = i0 + q * nthr;
      const int rr = (i < n ? i : 0) / (HD + 1), d = (i < n ? i : 0) % (HD + 1);
      const int col = d < HD ? d : HD + 1;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) {
        wt[q][w] = wgt[rr * kWarps + w];
        sv[q][w] = st[(w * kAttnMaxRb + rr) * RS + col];
      }
    }
#pragma unroll
    for (int q = 0; q < G; ++q) {
      const int i = i0 + q * nthr;
      if (i >= n) break;
      const int rr = i / (HD + 1), d = i % (HD + 1);
      const int col = d < HD ? d : HD + 1;
      float acc = 0.f;
#pragma unroll
      for (int w = 0; w < kWarps; ++w)
        if (wt[q][w] != 0.f) acc = fmaf(wt[q][w], sv[q][w], acc);
      cs[rr * RS + col] = acc;
    }
  }
}

// Cluster fold, step 1: weights of the CS CTA states of each row (into
// cw[rr * kAttnCluster + c]); peer(c) is CTA c's folded state.
template <int HD, typename Peer>
__device__ __forceinline__ void cluster_weights(Peer peer, int CS, int R, float* cw, int tid) {
  constexpr int RS = HD + 2;
  if (tid < R * CS) {
    const int rr = tid / CS, c = tid % CS;
    float mx = -INFINITY;
    for (int x = 0; x < CS; ++x) mx = fmaxf(mx, peer(x)[rr * RS + HD]);
    const float mc = peer(c)[rr * RS + HD];
    cw[rr * kAttnCluster + c] = mc == -INFINITY ? 0.f : expf(mc - mx);
  }
}

// step 2: each row's softmax denominator L (into cw[kAttnMaxRb * kAttnCluster + rr])
template <int HD, typename Peer>
__device__ __forceinline__ void cluster_sums(Peer peer, int CS, int R, float* cw, int tid) {
  constexpr int RS = HD + 2;
  if (tid < R) {
    const int rr = tid;
    float L = 0.f;
    for (int c = 0; c < CS; ++c) {
      const float wt = cw[rr * kAttnCluster + c];
      if (wt != 0.f) L = fmaf(wt, peer(c)[rr * RS + HD + 1], L);
    }
    cw[kAttnMaxRb * kAttnCluster + rr] = L;
  }
}

// step 3: output dims [crank HD / CS, (crank + 1) HD / CS) of every row
template <int HD, typename Peer>
__device__ __forceinline__ void cluster_out(const AttnArgs& a, Peer peer, int CS, int crank, int R, int r0, int g,
                                            int kvh, const float* cw, int tid, int nthr) {
  constexpr int RS = HD + 2;
  const int DC = HD / CS;  // dims per CTA
  for (int i = tid; i < R * DC; i += nthr) {
    const int rr = i / DC, d = crank * DC + i % DC;
    float O = 0.f;
    for (int c = 0; c < CS; ++c) {
      const float wt = cw[rr * kAttnCluster + c];
      if (wt != 0.f) O = fmaf(wt, peer(c)[rr * RS + d], O);
    }
    const int r = r0 + rr, t = r / g, h = kvh * g + r % g;
    a.o[(static_cast<size_t>(t) * a.H + h) * HD + d] = __float2bfloat16(O / cw[kAttnMaxRb * kAttnCluster + rr]);
  }
}

// The three fold steps above in ONE pass: each output thread (row rr, dim d)
// loads the CS states' m, l and o[d] together (one DSMEM / smem round trip,
// no barriers), recomputes the row's weights and denominator in the same
// order with the same operations, and writes o -- bitwise the same rows as
// cluster_weights + cluster_sums + cluster_out.
template <int HD, typename Peer>
__device__ __forceinline__ void cluster_fold_out(const AttnArgs& a, Peer peer, int CS, int crank, int R, int r0, int g,
                                                 int kvh, int tid, int nthr) {
  constexpr int RS = HD + 2;
  const int DC = HD / CS;
  // items in groups of 4: all peers' (m, l, o) of the group loaded before any
  // global store (a store through a generic pointer pins the loads after it)
  constexpr int G = 4;
  const int n = R * DC;
  for (int i0 = tid; i0 < n; i0 += G * nthr) {
    float m4[G][kAttnCluster], l4[G][kAttnCluster], o4[G][kAttnCluster];
#pragma unroll
    for (int q = 0; q < G; ++q) {
      const int i = i0 + q * nthr < n ? i0 + q * nthr : i0;
      const int rr = i / DC, d = crank * DC + i % DC;
#pragma unroll
      for (int c = 0; c < kAttnCluster; ++c) {
        if (c < CS) {
          const float* st = peer(c) + rr * RS;
          m4[q][c] = st[HD];
          l4[q][c] = st[HD + 1];
          o4[q][c] = st[d];
        }
      }
    }
#pragma unroll
    for (int q = 0; q < G; ++q) {
      const int i = i0 + q * nthr;
      if (i >= n) break;
      const int rr = i / DC, d = crank * DC + i % DC;
      const float* m = m4[q];
      const float* l = l4[q];
      const float* o = o4[q];
      float mx = -INFINITY;
#pragma unroll
      for (int c = 0; c < kAttnCluster; ++c)
        if (c < CS) mx = fmaxf(mx, m[c]);
      float L = 0.f, O = 0.f;
#pragma unroll
      for (int c = 0; c < kAttnCluster; ++c) {
        if (c < CS) {
          const float wt = m[c] == -INFINITY ? 0.f : expf(m[c] - mx);
          if (wt != 0.f) {
            L = fmaf(wt, l[c], L);
            O = fmaf(wt, o[c], O);
          }
        }
      }
      const int r = r0 + rr, t = r / g, h = kvh * g + r % g;
      a.o[(static_cast<size_t>(t) * a.H + h) * HD + d] = __float2bfloat16(O / L);
    }
  }
}

}  // namespace attn_core
}  // namespace pearl
