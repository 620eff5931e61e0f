/*
 * pearl_b200.h -- C ABI of libpearl_b200.so, the B200 (sm_100a) hot path of
 * PEARL's parallel draft-and-verify decoding loop.
 *
 * Drop-in boundary.  The reference (pearl_lab, pure Python) has no FFI: its
 * hot path is the Python call graph decode_pearl -> pearl_{pre,post}verify_step
 * -> SequenceModel.next_dist / _draft_block / _verify -> verify_chain ->
 * accept_prob / residual_dist / sample.  Each entry point below replaces one
 * of those reference operations; the Python package paper_2408_11850_b200
 * binds them with ctypes and re-exposes the reference's
 * own Python API on top.
 *
 * Conventions
 *   - Every function returns int: 0 = OK, >0 = a domain error that the Python
 *     layer maps to the reference exception class (codes below), <0 = CUDA or
 *     argument error (pearl_last_error() has the message).
 *   - All array arguments are DEVICE pointers unless stated; sizes are plain
 *     ints.  `stream` is a cudaStream_t passed as void*.  No call allocates
 *     device memory or synchronises the stream, except the *_create / *_prepare
 *     setup calls, so every launch sequence is CUDA-graph capturable.
 *   - Row arrays (`p_rows`, `q_rows`) are device arrays of device pointers,
 *     one per row: fp64 ProbDist.probs rows (PEARL_ROWS_PROBS64) or fp32 logits
 *     rows (PEARL_ROWS_LOGITS32).
 */
#ifndef PEARL_B200_H_
#define PEARL_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (map to pearl_lab exceptions, core.py:27-36) ---------- */
#define PEARL_OK 0
#define PEARL_ERR_INVALID_DISTRIBUTION 1 /* core.InvalidDistribution */
#define PEARL_ERR_ALL_ZERO_RESIDUAL 2    /* core.AllZeroResidual     */
#define PEARL_ERR_ZERO_DRAFT_PROB 3      /* core.ZeroDraftProb       */
#define PEARL_ERR_VALUE 4                /* ValueError (bad lengths, exhausted uniforms) */
#define PEARL_ERR_TIMEOUT 5              /* split pair: the peer never delivered (DeviceError) */
#define PEARL_ERR_CUDA (-1)
#define PEARL_ERR_ARG (-2)

/* ---- row encodings ------------------------------------------------------ */
#define PEARL_ROWS_PROBS64 0  /* normalised ProbDist.probs, float64       */
#define PEARL_ROWS_LOGITS32 1 /* raw logits, float32; law = device softmax */

/* ---- verify / sample flags --------------------------------------------- */
#define PEARL_F_GREEDY 1   /* argmax rule: engines._verify_chain_greedy / _pick */
#define PEARL_F_BONUS 2    /* SD: one extra target row; bonus pick on full accept */
#define PEARL_F_ADVANCE 4  /* advance *cursor by the draws consumed */
#define PEARL_F_PROBE 8    /* only compute per-position accept probabilities */

/* Result of one chain verification (sampling.VerifyResult, sampling.py:44-58,
 * plus the RNG consumption the reference tracks in RandomStream.n_draws). */
typedef struct {
  int32_t status;     /* PEARL_OK or a PEARL_ERR_* domain code            */
  int32_t accepted;   /* VerifyResult.accepted_count                      */
  int32_t correction; /* VerifyResult.correction, -1 for None             */
  int32_t examined;   /* VerifyResult.examined                            */
  int32_t draws_used; /* uniforms consumed from the verify stream         */
  int32_t bonus;      /* SD bonus token (engines.py:377-378), -1 if none  */
  int32_t fallback;   /* 1 if an exact sequential CDF replay was needed   */
  int32_t reserved;
} pearl_verify_result;

/* Library identity / errors */
int pearl_version(void);
const char* pearl_last_error(void);
/* Number of kernel launches the library has issued (captured nodes count
 * once per capture); used to report gpu_launches per timed step. */
unsigned long long pearl_launch_count(void);

/* Size in bytes of the scratch `work` buffer pearl_spec_verify needs for a
 * chain of n positions.  The buffer must be zero-initialised once; the
 * kernel leaves it zeroed again on exit. */
size_t pearl_verify_work_bytes(int n);

/* Pre-plan the pairwise-summation tree for vocabulary size V (host work +
 * one upload).  Must be called once per V before any capture. */
int pearl_prepare_vocab(int V);

/*
 * K1 -- fused speculative verify.
 * Replaces engines._verify (engines.py:229-238) -> sampling.verify_chain
 * (sampling.py:61-93) -> accept_prob (sampling.py:24-41) -> residual_dist
 * (core.py:193-214) -> sample (core.py:182-190); greedy twin
 * engines._verify_chain_greedy (engines.py:220-226); SD bonus pick
 * engines.py:377-378 (PEARL_F_BONUS: p_rows has n+1 rows).
 * Position i uses uniforms[*cursor + i] for its accept test and
 * uniforms[*cursor + i + 1] for a correction drawn at i; the bonus uses
 * uniforms[*cursor + n].  Bit-exact with the reference for PROBS64 rows and
 * with ProbDist(device softmax) for LOGITS32 rows.
 * accept_probs (optional, may be NULL): float64[n] accept probabilities.
 */
int pearl_spec_verify(int row_mode, const void* const* p_rows, const void* const* q_rows,
                      const int32_t* drafted, int n, int V, const double* uniforms,
                      int n_uniforms, int32_t* cursor, float inv_temperature, int flags,
                      pearl_verify_result* out, double* accept_probs, void* work, void* stream);

/* One chain of a batched K1 launch (pearl_spec_verify_multi). All pointers
 * are device pointers. Position i of the chain verifies the id
 * drafted[i * stride], except that with `tail` non-NULL the last position
 * (n - 1) reads *tail (a draft pick that never went through the host). */
typedef struct pearl_verify_chain {
  const void* const* p_rows;   /* n rows (n + 1 with PEARL_F_BONUS)           */
  const void* const* q_rows;   /* n rows (ignored with PEARL_F_GREEDY)        */
  const int32_t* drafted;
  const int32_t* tail;         /* may be NULL                                 */
  const double* uniforms;      /* this chain's verify stream (NULL if greedy) */
  int32_t* cursor;             /* its device cursor (may be NULL)             */
  pearl_verify_result* out;
  void* work;                  /* pearl_verify_work_bytes(n), zeroed once     */
  int32_t n;
  int32_t cluster_base;        /* sum over the previous chains of n (+1 with PEARL_F_BONUS) */
  int32_t stride;
  int32_t reserved;
} pearl_verify_chain;

/*
 * K1 over many independent chains in ONE launch: the B sequences of a
 * lockstep batch, each with its own rows, drafted ids,
 * uniform stream, cursor, verdict and work buffer. Chain s is exactly
 * pearl_spec_verify on its own arguments (bit-identical verdicts), its
 * positions running as clusters cluster_base .. cluster_base + n (+1) - 1.
 * `chains`: device array of n_chains descriptors sorted by cluster_base;
 * n_clusters = the sum of all chains' cluster counts.
 */
int pearl_spec_verify_multi(int row_mode, const pearl_verify_chain* chains, int n_chains, int n_clusters,
                            int V, int n_uniforms, float inv_temperature, int flags, void* stream);

/*
 * Inverse-CDF / argmax pick from `rows` rows of one law each.
 * Replaces core.sample (core.py:182-190) and engines._pick (engines.py:214-217).
 * Row r uses uniforms[*cursor + r].  out_tokens: int32[rows].  If
 * append_dst is non-NULL the token of row 0 is also written there (the next
 * input slot of a decode loop).
 */
int pearl_sample_rows(int row_mode, const void* const* rows, int n_rows, int V,
                      const double* uniforms, int n_uniforms, int32_t* cursor,
                      float inv_temperature, int flags, int32_t* out_tokens,
                      int32_t* append_dst, int32_t* status, void* work, void* stream);

/* pearl_sample_rows with one uniform stream per row (B independent
 * sequences decoded in lockstep): row r draws tables[r][*cursors[r]] and
 * advances cursors[r] by one (PEARL_F_ADVANCE).  tables / cursors are device
 * arrays of device pointers; both may be NULL with PEARL_F_GREEDY. */
int pearl_sample_rows_multi(int row_mode, const void* const* rows, int n_rows, int V,
                            const double* const* tables, int n_uniforms, int32_t* const* cursors,
                            float inv_temperature, int flags, int32_t* out_tokens, int32_t* status,
                            void* stream);

/* Device law of fp32 logits rows as float64 p1 = softmax rows (the vector a
 * SequenceModel.next_dist adapter hands to ProbDist, models.py:64-71).
 * logits: float32[n_rows, V] contiguous; out: float64[n_rows, V]. */
int pearl_logits_to_probs(const float* logits, int n_rows, int V, float inv_temperature,
                          double* out, int32_t* status, void* stream);

/* residual_dist (core.py:193-214) numerator: out = max(p-q,0)/sum(max(p-q,0))
 * for one pair of PROBS64 rows; status gets PEARL_ERR_ALL_ZERO_RESIDUAL when
 * the mass is below 1e-15. */
int pearl_residual(const double* p, const double* q, int V, double* out, int32_t* status,
                   void* stream);


/* ======================================================================== *
 * Llama decoder runtime (replaces SequenceModel.next_dist, models.py:58-71,
 * for GPU models: the draft's per-token forward inside _draft_block,
 * engines.py:277-282, and the target's window forward,
 * engines.py:302 / 373 / 425 / 492).
 * ======================================================================== */

/* Linear-layer engine of a model. */
#define PEARL_GEMM_CUDACORE 0 /* batch-invariant 128-bit GEMV (draft, K2) */
#define PEARL_GEMM_TCGEN05 1  /* tcgen05 + TMA small-M contraction (target, K3) */
/* OR-ed into pearl_gemm's kind (tcgen05 only): W is stored tile-major,
 * [N/128][K/64][128][64] bf16, so every 128x64 TMA box is 16 contiguous KB */
#define PEARL_GEMM_W_TILED 0x100

typedef struct {
  int32_t n_layers, d_model, n_heads, n_kv_heads, head_dim, ffn, vocab;
  int32_t max_seq;    /* KV-cache capacity (positions)                  */
  int32_t max_tokens; /* largest window processed in one pass (chunking) */
  int32_t gemm_kind;  /* PEARL_GEMM_*                                    */
  float norm_eps;
  int32_t sm_count;  /* SMs the model's stream-K grids span (0: all);  \
                        must match the partition it runs on            */
  int32_t n_slots;   /* KV-cache slots (independent sequences, >= 1);   \
                        the cache is [L, n_slots, max_seq, KV, hd]      */
} pearl_llama_config;

/* Weight / cache pointer table, in this order (all device pointers):
 *   0 embed      bf16 [V, d]          1 final_norm fp32 [d]
 *   2 lm_head    bf16 [V, d]          3 rope_cos   fp32 [max_seq, hd/2]
 *   4 rope_sin   fp32 [max_seq, hd/2] 5 k_cache    bf16 [L, n_slots, max_seq, KV, hd]
 *   6 v_cache    bf16 [L, n_slots, max_seq, KV, hd]
 *   then per layer l (base 7 + 6 l):
 *     attn_norm fp32 [d], wqkv bf16 [(H+2KV) hd, d], wo bf16 [d, H hd],
 *     mlp_norm fp32 [d], w_gate_up bf16 [2 ffn, d] (rows 2j = gate_j,
 *     2j+1 = up_j), w_down bf16 [d, ffn]                                  */
#define PEARL_LLAMA_FIXED_PTRS 7
#define PEARL_LLAMA_PTRS_PER_LAYER 6

int pearl_llama_create(const pearl_llama_config* cfg, const void* const* ptrs, int n_ptrs,
                       void** handle);
int pearl_llama_destroy(void* handle);

/* Forward flags */
#define PEARL_FWD_ADVANCE 1     /* *pos += n_tokens when done              */
#define PEARL_FWD_LAST_LOGITS 2 /* logits only for the last token ([1, V]) */

/* Run n_tokens tokens (device int32[n_tokens]) at positions *pos .. *pos+n-1
 * (pos is a device int32 so graph replays see its current value), append
 * their K/V to the cache and write fp32 logits [n_tokens, V] (or [1, V]).
 * Per-token results are bitwise independent of n_tokens (batch invariance),
 * which is what makes GPU PEARL / SD greedy output token-identical to AR. */
int pearl_llama_forward(void* handle, const int32_t* tokens, int n_tokens, int32_t* pos,
                        int flags, float* logits, void* stream);

/* Batched (slot-mode) forward: token i belongs to KV slot tok_slot[i] and
 * sits at position tok_pos[i] of that slot (device int32[n_tokens] each);
 * K/V are appended there and fp32 logits [n_tokens, V] written for every
 * token.  Tokens of different slots may be mixed in any order; each token's
 * logits are bitwise the ones a single-sequence forward would produce
 * (batch invariance), which makes a batched decode token-identical to
 * independent per-prompt decodes.  Replaces the per-sequence next_dist
 * calls of B independent decodes (cli.py:204-208 runs prompts as separate
 * decodes). */
int pearl_llama_forward_slots(void* handle, const int32_t* tokens, int n_tokens, const int32_t* tok_slot,
                              const int32_t* tok_pos, float* logits, void* stream);

size_t pearl_llama_workspace_bytes(void* handle, int n_tokens);

/* Keep [base, base + bytes) -- a model's packed streamed weights -- in
 * persisting L2 lines: every kernel of the model's forwards carries an L2
 * access-policy window over it (hit ratio = granted / bytes).  For a draft
 * model this serves its per-token weight reads from L2 instead of HBM,
 * which the concurrently running target saturates.  *granted (optional) =
 * the device's persisting-L2 size after the call; bytes = 0 clears it. */
int pearl_llama_set_l2_window(void* handle, const void* base, size_t bytes, size_t* granted);

/* SM partition for two concurrently running models (green contexts):
 * *first_stream runs on first_sms SMs (rounded up to the partition
 * granularity, count in *first_count), *rest_stream on the remaining
 * *rest_count SMs.  Created once per process; later calls with the same
 * first_sms return the same streams. */
int pearl_green_streams(int first_sms, void** first_stream, void** rest_stream, int* first_count,
                        int* rest_count);

/* Diagnostic: copy an internal activation buffer of the last forward
 * (0 residual h fp32 [T, d]; 1 x, 2 q, 3 o, 4 act bf16; 5 stream-K tile
 * flags int32; 6 folded-norm per-tile sums of h^2 fp32 [ceil(d/128), T])
 * to device dst.  With
 * PEARL_STOP=k in the environment a forward runs only its first k ops. */
int pearl_llama_debug_buffer(void* handle, int which, void* dst, size_t bytes, void* stream);

/* Diagnostic: one eager forward with an event after every launch; out_ms
 * (float[10]) receives device ms per op {embed, (unused), qkv, attention, o,
 * gate_up, down, lm_head, other} and the total. */
int pearl_llama_profile(void* handle, const int32_t* tokens, int n_tokens, int32_t* pos, float* logits,
                        float* out_ms, void* stream);

/* Standalone contraction Y[M, N] (fp32) = X[M, K] (bf16) . W[N, K]^T (bf16)
 * on the given engine (PEARL_GEMM_*), for tests and microbenchmarks.
 * splits = 0 lets the planner pick the split-K factor (tcgen05 only). */
int pearl_gemm(int kind, const void* W, const void* X, float* Y, int M, int N, int K, int splits, void* stream);
/* Split-K factor the tcgen05 planner uses for an (N, K) weight. */
int pearl_gemm_splits(int N, int K);

/* ======================================================================== *
 * PEARL step bookkeeping on the device (engines.py:397-526 state updates)
 * ======================================================================== */

typedef struct {
  int32_t committed_len; /* len(DecodeState.committed), prefix included  */
  int32_t n_pending;     /* len(DecodeState.pending)                     */
  int32_t mode;          /* 0 PRE_VERIFY, 1 POST_VERIFY                  */
  int32_t target_pos;    /* target KV length (== committed_len - 1)      */
  int32_t draft_pos;     /* draft KV length                              */
  int32_t verify_cursor; /* uniforms used from the verify stream table   */
  int32_t draft_cursor;  /* uniforms used from the draft stream table    */
  int32_t last_status;
} pearl_seq_state;

/* K5 -- in-place KV rollback: cache length[i] = new_len[i] (no data moves;
 * positions past the new length are overwritten by the next window). */
int pearl_kv_rollback(int32_t* cache_len, const int32_t* new_len, int n, void* stream);

typedef struct {
  pearl_seq_state* state;
  int32_t* seq_tokens;        /* committed tokens, capacity max_len       */
  int32_t max_len;
  const int32_t* chain;       /* k pending + fresh drafts xs[0..gamma)    */
  int32_t k;                  /* pending count verified this step         */
  int32_t gamma;              /* fresh drafts this step                   */
  const pearl_verify_result* verdict;
  int32_t* pending_tok;       /* [gamma_max] next pending ids             */
  float* pending_rows;        /* [gamma_max, V] next pending q logits     */
  const float* draft_rows;    /* [gamma, V] this step's draft logits      */
  int32_t V;
  int32_t sd_mode;            /* 1: draft-then-verify commit (bonus), no pending */
  int32_t* out_host_view;     /* optional: [16 + gamma] summary for the host */
} pearl_commit_args;

/* Apply one verified step to the device-resident DecodeState: append the
 * accepted chain plus correction (or SD bonus), roll both KV caches back to
 * the accepted prefix, carry the unverified drafts (and their q rows) over
 * as the next pending block, switch PRE/POST mode (engines.py:431-446,
 * 500-515, 376-381). */
int pearl_pearl_commit(const pearl_commit_args* args, void* stream);

/* Build the next step's inputs from the device state: target window
 * [committed[-1]] + pending, and the draft catch-up tokens
 * committed+pending [draft_pos ..]. */
int pearl_step_assemble(pearl_seq_state* state, const int32_t* seq_tokens, const int32_t* pending_tok,
                        int32_t* target_in, int32_t* draft_in, int32_t* draft_in_count, void* stream);

/* ======================================================================== *
 * K6 -- split pair: draft and target on different GPUs (one process each).
 * Replaces the _PhaseRunner rendezvous (engines.py:241-262) when the two
 * closures run on different devices: the draft rank pushes its gamma ids and
 * q-logit rows into a mailbox in the TARGET GPU's memory, the target rank
 * verifies (K1) and pushes the verdict into a mailbox in the DRAFT GPU's
 * memory.  Mailboxes are plain device allocations shared through CUDA IPC
 * (peer-mapped over NVLink / NVSwitch); push and wait are kernels, so a
 * split step stays one CUDA graph per rank.
 *
 * Mailbox layout: [0, 8) uint64 sequence flag; ids int32 at
 * PEARL_MAILBOX_IDS_OFFSET (<= PEARL_MAILBOX_MAX_IDS); fp32 rows at
 * PEARL_MAILBOX_ROWS_OFFSET (16-byte aligned).
 * ======================================================================== */
#define PEARL_MAILBOX_IDS_OFFSET 256
#define PEARL_MAILBOX_MAX_IDS 1024
#define PEARL_MAILBOX_ROWS_OFFSET (256 + 4 * 1024)
#define PEARL_IPC_HANDLE_BYTES 64

/* Bytes of a mailbox holding n_rows fp32 rows of V (plus header and ids). */
size_t pearl_mailbox_bytes(int n_rows, int V);
/* Setup calls (allocate / synchronise): a zeroed mailbox in the current
 * device's memory, and its release. */
int pearl_mailbox_alloc(size_t bytes, void** dptr);
int pearl_mailbox_free(void* dptr);
/* CUDA-IPC export of a mailbox (64 opaque bytes into host handle_out) and
 * import of a peer's handle (maps the peer allocation, enabling NVLink peer
 * access); the importing process must be a different process. */
int pearl_ipc_export(void* dptr, void* handle_out);
int pearl_ipc_import(const void* handle, void** dptr);
int pearl_ipc_close(void* dptr);

typedef struct {
  void* peer_box;                /* receiver's mailbox (peer-mapped)          */
  const int32_t* ids;            /* n_ids int32 -> box ids                    */
  int32_t n_ids;
  const float* rows;             /* n_rows x V fp32, contiguous -> box rows   */
  int32_t n_rows;
  int32_t V;
  unsigned long long* send_seq;  /* sender's device counter (starts at 0)     */
  unsigned int* arrive;          /* sender's zeroed device int (CTA election) */
} pearl_xfer_send_args;

/* One push: copy ids and rows into the peer mailbox, then release
 * ++(*send_seq) into its flag (system-scope fence before the flag store). */
int pearl_xfer_send(const pearl_xfer_send_args* args, void* stream);

/* Copy-engine push for GPU pairs that cannot map each other's memory
 * (cudaDeviceCanAccessPeer == 0; also PEARL_K6_COPY=1 for tests): the same
 * message as pearl_xfer_send, moved by stream-ordered cudaMemcpyAsync --
 * payload first, then the new sequence number (computed on the device into
 * the sender's 8-byte `staging` word) into the peer's flag, so the flag can
 * only land after the payload.  Graph-capturable (memcpy nodes). */
int pearl_xfer_send_copy(const pearl_xfer_send_args* args, unsigned long long* staging, void* stream);

/* 1 if a kernel on the current device can store into memory of the device
 * whose PCI bus id is `peer_pci_bus_id` (same device or peer access
 * supported), 0 if not, negative on error. */
int pearl_peer_storable(const char* peer_pci_bus_id);
/* PCI bus id of the current device into out (>= 16 bytes). */
int pearl_pci_bus_id(char* out, int len);

/* One receive: spin (acquire, system scope) until the local mailbox's flag
 * reaches ++(*recv_seq), then copy n_ids ids out of it into dst_ids.  If
 * timeout_ns > 0 and the flag does not arrive in time, *status (optional)
 * becomes PEARL_ERR_TIMEOUT and the kernel returns (no GPU hang). */
int pearl_xfer_wait(const void* box, unsigned long long* recv_seq, int32_t* dst_ids, int n_ids,
                    int32_t* status, long long timeout_ns, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* PEARL_B200_H_ */
