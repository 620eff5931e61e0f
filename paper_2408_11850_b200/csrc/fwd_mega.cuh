// Persistent whole-forward kernel (fwd_mega.cu): phase descriptors and host API.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "epilogue.cuh"

namespace pearl {

constexpr int kMegaMaxTokens = 16;   // window sizes served by the persistent forward
constexpr int kMegaTileN = 128;      // == kTileN  (tc_common.cuh)
constexpr int kMegaTileK = 64;       // == kTileK
constexpr int kMegaCtrStride = 32;  // words between phase counters (one 128 B line each)
constexpr int kMegaPartialTok = 128;  // == kMaxTokTiles * kTokTile (partials row pitch bound)

enum MegaKind { MG_EMBED = 0, MG_NORM = 1, MG_GEMM = 2, MG_ATTN = 3 };

struct alignas(64) MegaMap {
  CUtensorMap map;
};

// One phase of the forward.  Per-call values (token ids, positions, logits)
// are not stored here: the kernel takes them from MegaArgs, so a phase list
// depends only on the window size M and the logits mode and is built once.
struct MegaPhase {
  int kind;
  int M;
  // GEMM
  int N, K, KB, seg_max, map_w, map_x;
  long long T;
  EpiArgs e;           // e.pos / e.out_f32 (logits) patched from MegaArgs when flagged
  int e_uses_pos;      // QKV epilogue: pos = A.pos, pos_add = A.pos_add
  int e_is_logits;     // lm_head: out_f32 = A.logits
  // norm / embed
  float* h;
  const float* gain;
  bf16* xout;
  int d;
  int row0;            // first row normalised (final norm, last-only logits)
  float eps;
  const bf16* embed;
  int V;
  // attention
  const bf16* q;
  const bf16* kc;
  const bf16* vc;
  bf16* o;
  int H, KV, hd;
  float scale;
};

struct MegaArgs {
  const MegaPhase* phases;
  int n_phases;
  const MegaMap* maps;
  float* partials;
  int* tile_flags;
  unsigned* counter;   // [n_phases * kMegaCtrStride] CTAs done with phase p; zero between launches
  // per call
  const int32_t* tokens;
  const int32_t* pos;
  int pos_add;
  float* logits;
  int opts;            // experiment bits (PEARL_MEGA_OPTS)
  // diagnostics: globaltimer at each CTA's end of phase p ([p * G + cta]) and
  // at its start ([n_phases * G + cta]); null in production
  unsigned long long* trace;
};

struct SkShape {
  long long T;
  int G;
  int KB;
};

int mega_supported(int M);
size_t mega_smem_bytes();
int mega_threads();
const void* mega_kernel_ptr();
cudaError_t mega_prepare();  // sets the kernel's dynamic smem limit (once)
int mega_launch(const MegaArgs& a, int grid, cudaStream_t st);

}  // namespace pearl
