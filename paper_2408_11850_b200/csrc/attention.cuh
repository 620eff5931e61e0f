// K4: causal attention of a forward's window over the KV cache (replaces the
// attention inside SequenceModel.next_dist, pearl_lab/models.py:58-71, for
// the draft's token forward and the target's window forward,
// engines.py:277-282 / 492).
//
// Split-KV over a thread-block cluster, GQA-grouped, on the tensor cores
// (mma.sync m16n8k16, bf16 -> fp32):
//   * a cluster of 8 CTAs x 4 warps serves one (row block, KV head).  The
//     rows of a KV head are its (token t, group member j) pairs -- every
//     query head that reads that KV head -- so each K/V row is loaded once
//     for all of them (GQA 8:1 reads K/V once, not 8 times), up to 16 rows
//     per block (one MMA row tile);
//   * warp w of CTA c owns the 32-position segments 32 js + 4 c + w, js =
//     0..spw-1 (spw = max_seq / 1024 rounded up: one round covers 1024
//     positions), folded in js order with an online softmax.  s = q.k for 16
//     rows x 32 positions is 32 MMAs, o += p.v another 32; Q, K and V
//     fragments are 16-byte loads straight from global into registers (a
//     head-dim permutation makes them contiguous; V is transposed with
//     movmatrix), so K/V never touch shared memory and a CTA (~42 KB of
//     smem) can sit beside a GEMM CTA under programmatic dependent launch;
//   * K/V of positions before the window (written by earlier forwards) are
//     loaded -- or prefetched into L2 -- BEFORE griddepcontrol.wait, under
//     the QKV GEMM's tail;
//   * a CTA folds its 4 warps in warp order, then the cluster folds its 8
//     CTAs in rank order through distributed shared memory (each CTA writes
//     an eighth of the head dims).  No global partials, no atomics.
// Every fold is over FIXED position ranges in a fixed order and a masked
// (empty) state is skipped exactly, so a token's output depends only on its
// own position and the cache -- never on M, the row blocking or the grid
// (batch invariance: an M=1 AR step, an M=gamma PEARL window and an
// M=gamma+1 SD window give bitwise identical rows).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace pearl {

constexpr int kAttnThreads = 128;   // 4 warps
// The fold is defined over kAttnLCS LOGICAL CTAs x 4 warps per (row block,
// KV head) -- the arithmetic of every output row -- whatever the physical
// cluster: a cluster of CS CTAs (1, 2 or 4) runs kAttnLCS / CS logical CTAs
// per physical CTA one after another, and the fold reads logical state c
// from physical rank c / (kAttnLCS / CS).  Sequence mode (CS = 4) and slot
// mode (CS = 1) therefore give bitwise the same rows (batched == single).
constexpr int kAttnLCS = 4;
constexpr int kAttnCluster = kAttnLCS;  // fold width (logical CTAs)
constexpr int kAttnClusterDefault = 4;  // physical, sequence mode: measured best on B200 (7B M=4: 1 -> 3.09, 2 -> 2.98, 4 -> 2.97 ms)
constexpr int kAttnMaxRb = 16;      // rows per block (one m16n8k16 row tile)
constexpr int kAttnMaxTok = 128;    // tokens per launch (a model's max_tokens)

struct AttnArgs {
  const __nv_bfloat16* q;   // [M, H, hd] (post-RoPE)
  const __nv_bfloat16* kc;  // layer cache base [n_slots][max_seq][KV][hd]
  const __nv_bfloat16* vc;
  __nv_bfloat16* o;         // [M, H, hd]
  const int32_t* pos;       // sequence mode: token t sits at *pos + pos_add + t
  int pos_add;
  const int32_t* tok_pos;   // slot mode: per-token position and KV slot
  const int32_t* tok_slot;
  long long slot_stride;    // elements per slot
  int M, H, KV;
  float scale;
  int tpb;                  // tokens per row block (rows t * g + j, <= 16); slot mode
                            // blocks never straddle a run of same-slot tokens
  int spw;                  // segments per warp (rounds of 512 positions)
  unsigned long long* tl;   // PEARL_TIMELINE builds: this launch's stamps
};

// Host: plan (rb, nrb) for a window of M tokens, launch on stream st.
struct AttnShape {
  int M, H, KV, hd, max_seq, num_sms;
  bool slot_mode;
};
void attn_plan(const AttnShape& s, int* tpb, int* spw, int* grid);
int attn_cluster_size(bool slot_mode);  // physical CTAs per cluster (PEARL_ATTN_CLUSTER: 1, 2, 4)
int attn_launch(const AttnArgs& a, int hd, int grid, cudaStream_t st);
int attn_init();  // one-time kernel attributes

}  // namespace pearl
