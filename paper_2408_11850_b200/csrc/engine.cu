// Device-resident PEARL step bookkeeping: K5 KV rollback, state commit and
// next-step input assembly.
//
// The reference keeps DecodeState as an immutable host value
// (engines.py:80-99) and rebuilds it after every verification
// (pre-verify engines.py:431-446, post-verify engines.py:500-515, SD commit
// engines.py:376-381 + _commit engines.py:322-341).  Here the same
// transitions run in one tiny kernel right after K1, on the stream that
// produced the verdict, so a whole step (draft block || target window ->
// verify -> commit) is one CUDA graph and the host only reads a summary.
#include <cuda_runtime.h>

#include "common.h"

namespace pearl {

// summary layout written for the host (int32)
enum {
  SUM_STATUS = 0,
  SUM_ACCEPTED,
  SUM_CORRECTION,
  SUM_EXAMINED,
  SUM_DRAWS,
  SUM_BONUS,
  SUM_COMMITTED,
  SUM_MODE,
  SUM_NPENDING,
  SUM_TPOS,
  SUM_DPOS,
  SUM_VCUR,
  SUM_DCUR,
  SUM_FALLBACK,
  SUM_HDR = 16
};

__global__ void kv_rollback_kernel(int32_t* len, const int32_t* new_len, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) len[i] = new_len[i];
}

__global__ void commit_kernel(pearl_commit_args a) {
  const pearl_verify_result v = *a.verdict;
  const bool ok = v.status == PEARL_OK;
  const bool full_accept = ok && v.correction < 0;
  // carry the unverified fresh drafts' q rows over as the next pending block
  // (pending_rows == NULL: the draft rank of a split pair, which keeps no q rows)
  if (!a.sd_mode && full_accept && a.pending_rows && blockIdx.x < a.gamma - 1) {
    const float* srow = a.draft_rows + static_cast<size_t>(blockIdx.x + 1) * a.V;
    float* drow = a.pending_rows + static_cast<size_t>(blockIdx.x) * a.V;
    // rows start 16-byte aligned only when V % 4 == 0 (e.g. not V = 32001)
    const int nvec = (a.V % 4 == 0) ? a.V / 4 : 0;
    const float4* src = reinterpret_cast<const float4*>(srow);
    float4* dst = reinterpret_cast<float4*>(drow);
    for (int i = threadIdx.x; i < nvec; i += blockDim.x) dst[i] = src[i];
    for (int i = nvec * 4 + threadIdx.x; i < a.V; i += blockDim.x) drow[i] = srow[i];
  }
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  pearl_seq_state s = *a.state;
  int status = v.status;
  if (ok) {
    const int C = s.committed_len;
    int add = 0;
    if (!full_accept) {
      add = v.accepted + 1;  // chain[:n] + correction
    } else if (a.sd_mode) {
      add = a.gamma + 1;     // SD: all gamma drafts + bonus (k == 0)
    } else {
      add = a.k + 1;         // pending + first fresh draft
    }
    if (C + add > a.max_len) {
      status = PEARL_ERR_VALUE;
    } else {
      if (!full_accept) {
        for (int i = 0; i < v.accepted; ++i) a.seq_tokens[C + i] = a.chain[i];
        a.seq_tokens[C + v.accepted] = v.correction;
        s.n_pending = 0;
        s.mode = 0;
      } else if (a.sd_mode) {
        for (int i = 0; i < a.gamma; ++i) a.seq_tokens[C + i] = a.chain[i];
        a.seq_tokens[C + a.gamma] = v.bonus;
        s.n_pending = 0;
        s.mode = 0;
      } else {
        for (int i = 0; i <= a.k; ++i) a.seq_tokens[C + i] = a.chain[i];
        for (int i = 0; i < a.gamma - 1; ++i) a.pending_tok[i] = a.chain[a.k + 1 + i];
        s.n_pending = a.gamma - 1;
        s.mode = 1;
      }
      s.committed_len = C + add;
      // K5: in-place rollback -- both caches shrink to the accepted prefix
      s.target_pos = s.committed_len - 1;
      s.draft_pos = min(s.draft_pos, s.committed_len + s.n_pending - 1);
    }
  }
  s.last_status = status;
  *a.state = s;
  if (a.out_host_view) {
    int32_t* o = a.out_host_view;
    o[SUM_STATUS] = status;
    o[SUM_ACCEPTED] = v.accepted;
    o[SUM_CORRECTION] = v.correction;
    o[SUM_EXAMINED] = v.examined;
    o[SUM_DRAWS] = v.draws_used;
    o[SUM_BONUS] = v.bonus;
    o[SUM_COMMITTED] = s.committed_len;
    o[SUM_MODE] = s.mode;
    o[SUM_NPENDING] = s.n_pending;
    o[SUM_TPOS] = s.target_pos;
    o[SUM_DPOS] = s.draft_pos;
    o[SUM_VCUR] = s.verify_cursor;
    o[SUM_DCUR] = s.draft_cursor;
    o[SUM_FALLBACK] = v.fallback;
    for (int i = 0; i < a.gamma; ++i) o[SUM_HDR + i] = a.chain[a.k + i];
  }
}

__global__ void assemble_kernel(pearl_seq_state* state, const int32_t* seq, const int32_t* pending,
                                int32_t* target_in, int32_t* draft_in, int32_t* draft_in_count) {
  const pearl_seq_state s = *state;
  const int C = s.committed_len, k = s.n_pending;
  // a split pair's ranks assemble only their own model's input (the other pointer is NULL)
  if (target_in)
    for (int i = threadIdx.x; i <= k; i += blockDim.x) target_in[i] = (i == 0) ? seq[C - 1] : pending[i - 1];
  if (!draft_in) return;
  const int cnt = C + k - s.draft_pos;
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
    const int idx = s.draft_pos + i;
    draft_in[i] = idx < C ? seq[idx] : pending[idx - C];
  }
  if (threadIdx.x == 0 && draft_in_count) *draft_in_count = cnt;
}

}  // namespace pearl

using namespace pearl;

extern "C" int pearl_kv_rollback(int32_t* cache_len, const int32_t* new_len, int n, void* stream) {
  PEARL_ARG_CHECK(cache_len && new_len && n >= 1, "bad rollback arguments");
  kv_rollback_kernel<<<(n + 127) / 128, 128, 0, static_cast<cudaStream_t>(stream)>>>(cache_len, new_len, n);
  PEARL_CUDA_TRY(cudaGetLastError());
  count_launch();
  return PEARL_OK;
}

extern "C" int pearl_pearl_commit(const pearl_commit_args* args, void* stream) {
  PEARL_ARG_CHECK(args && args->state && args->seq_tokens && args->chain && args->verdict, "bad commit arguments");
  PEARL_ARG_CHECK(args->gamma >= 1, "gamma >= 1");
  PEARL_ARG_CHECK(args->sd_mode || args->gamma == 1 || (args->pending_tok && (!args->pending_rows || args->draft_rows)),
                  "pending buffers required");
  const int blocks = args->sd_mode ? 1 : (args->gamma > 1 ? args->gamma - 1 : 1);
  commit_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(*args);
  PEARL_CUDA_TRY(cudaGetLastError());
  count_launch();
  return PEARL_OK;
}

extern "C" int pearl_step_assemble(pearl_seq_state* state, const int32_t* seq_tokens, const int32_t* pending_tok,
                                   int32_t* target_in, int32_t* draft_in, int32_t* draft_in_count, void* stream) {
  PEARL_ARG_CHECK(state && seq_tokens && (target_in || draft_in), "bad assemble arguments");
  assemble_kernel<<<1, 64, 0, static_cast<cudaStream_t>(stream)>>>(state, seq_tokens, pending_tok, target_in, draft_in,
                                                                    draft_in_count);
  PEARL_CUDA_TRY(cudaGetLastError());
  count_launch();
  return PEARL_OK;
}
