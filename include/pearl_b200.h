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

#ifdef __cplusplus
}
#endif

#endif /* PEARL_B200_H_ */
