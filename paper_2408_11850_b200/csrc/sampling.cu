// K1 fused speculative verify + inverse-CDF pick + device softmax/residual.
//
// One thread-block cluster (C CTAs, C from the vocabulary plan) owns one
// chain position; CTA r of the cluster owns the r-th subtree slice of the
// vocabulary and keeps that slice of p and q in shared memory as fp64.
//
//   pearl_spec_verify  <- engines._verify / sampling.verify_chain /
//                         accept_prob / residual_dist / sample
//                         (engines.py:229-238, sampling.py:24-93,
//                          core.py:182-214) and the greedy twin
//                         (engines.py:220-226) and SD bonus (engines.py:377-378)
//   pearl_sample_rows  <- core.sample / engines._pick (core.py:182-190,
//                         engines.py:214-217)
//   pearl_logits_to_probs, pearl_residual <- the law a next_dist adapter hands
//                         to ProbDist, and residual_dist's numerator.
//
// Every position is evaluated speculatively and in parallel (its accept
// test, and -- only if it rejects -- its residual correction); the last
// cluster to finish reduces the per-position verdicts with a warp ballot to
// find the first rejection, exactly as the sequential reference walk would,
// and reports the draws the reference would have consumed.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <string>
#include <type_traits>

#include "common.h"
#include "probdist.cuh"

namespace pearl {

constexpr int kThreads = 256;

struct Rec {
  int status;
  int accept;
  int corr;
  int fb;
  double a;
  double pad;
};

struct WorkHdr {
  int arrived;
  int pad[7];
};

struct RowJob {
  int mode;
  float inv_temp;
  int V;
  const int* plan;
  int cap;
};

extern __shared__ __align__(16) unsigned char g_smem[];

// Loads the (static) plan, then waits for the producing kernel (PDL) and lets
// dependents launch: every kernel here calls it before touching any input.
__device__ __forceinline__ void load_plan(int* splan, const int* gplan, int rank) {
  for (int i = threadIdx.x; i < kPlanStride; i += blockDim.x) splan[i] = gplan[rank * kPlanStride + i];
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  __syncthreads();
}

// block-wide max of floats and OR of ints; result valid in every thread
__device__ __forceinline__ void block_max_or(Scratch& s, float& m, int& flag) {
  m = warp_max_f(m);
  flag = warp_or_i(flag);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) { s.warp_f[w] = m; s.warp_j[w] = flag; }
  __syncthreads();
  if (threadIdx.x < 32) {
    const int nw = blockDim.x >> 5;
    float x = threadIdx.x < nw ? s.warp_f[threadIdx.x] : -INFINITY;
    int f = threadIdx.x < nw ? s.warp_j[threadIdx.x] : 0;
    x = warp_max_f(x);
    f = warp_or_i(f);
    if (threadIdx.x == 0) { s.res_d[3] = x; s.res_i[3] = f; }
  }
  __syncthreads();
  m = static_cast<float>(s.res_d[3]);
  flag = s.res_i[3];
  __syncthreads();
}

// Per-row normalisation constants (identical in every thread of the cluster).
struct RowNorm {
  float m;      // max logit (logits mode)
  double S;     // pairwise sum of e
  double Pn;    // pairwise sum of e/S (ProbDist renormaliser)
};

// Fill the smem slices of NR rows with their law and return the constants.
//   logits mode: slice = e (if !normalize) or ((e/S)/Pn) (ProbDist probs)
//   probs  mode: slice = the given fp64 row
// Returns PEARL_ERR_INVALID_DISTRIBUTION if any row has NaN/+inf or is all -inf.
template <int NR>
__device__ int prepare_rows(ClusterCtx& cc, Scratch& s, const int* plan, const RowJob& job,
                            const void* const* rows, double* const* slices, bool normalize,
                            RowNorm* norm) {
  const int lo = plan[3], hi = plan[4];
  if (job.mode == PEARL_ROWS_PROBS64) {
    for (int r = 0; r < NR; ++r) {
      const double* g = static_cast<const double*>(rows[r]);
      double* sl = slices[r];
      for (int i = lo + threadIdx.x; i < hi; i += blockDim.x) sl[i - lo] = g[i];
      norm[r] = RowNorm{0.f, 1.0, 1.0};
    }
    __syncthreads();
    return PEARL_OK;
  }
  // logits: max + validity.  One pass over global memory: a thread's
  // elements (stride kThreads) are all requested before any is used, kept in
  // registers, and the exp pass below reuses them (NR == 1; slices of up to
  // 16 * kThreads elements -- V <= 32768 per CTA slice of 8 -- or 36 * kThreads).
  constexpr int kMaxPer = 36;
  float xr[NR == 1 ? kMaxPer : 1];
  const int len = hi - lo;
  const int per_mode = NR != 1 ? 0 : (len <= 16 * kThreads ? 16 : (len <= kMaxPer * kThreads ? kMaxPer : 0));
  double mv[4];
  int bad_any = 0;
  auto load_regs = [&](const float* g, float& m, int& bad, auto per_c) {
    constexpr int PER = decltype(per_c)::value;
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int i = lo + threadIdx.x + u * kThreads;
      xr[u] = i < hi ? g[i] : -INFINITY;
    }
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      if (isnan(xr[u]) || xr[u] == INFINITY) bad = 1;
      m = fmaxf(m, xr[u]);
    }
  };
  for (int r = 0; r < NR; ++r) {
    const float* g = static_cast<const float*>(rows[r]);
    float m = -INFINITY;
    int bad = 0;
    if (per_mode == 16) {
      load_regs(g, m, bad, std::integral_constant<int, 16>{});
    } else if (per_mode == kMaxPer) {
      load_regs(g, m, bad, std::integral_constant<int, (NR == 1 ? kMaxPer : 1)>{});
    } else {
      for (int i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        float x = g[i];
        if (isnan(x) || x == INFINITY) bad = 1;
        m = fmaxf(m, x);
      }
    }
    block_max_or(s, m, bad);
    mv[r] = m;
    bad_any |= bad;
  }
  mv[NR] = bad_any;
  PEARL_TR(2);
  const double* all = cluster_gather_d(cc, s, mv, NR + 1);
  PEARL_TR(3);
  int invalid = 0;
  for (int r = 0; r < NR; ++r) {
    float m = -INFINITY;
    for (int k = 0; k < cc.size; ++k) {
      m = fmaxf(m, static_cast<float>(all[4 * k + r]));
      invalid |= (all[4 * k + NR] != 0.0);
    }
    norm[r].m = m;
    if (m == -INFINITY) invalid = 1;
  }
  if (invalid) return PEARL_ERR_INVALID_DISTRIBUTION;
  auto exp_regs = [&](double* sl, float m, auto per_c) {
    constexpr int PER = decltype(per_c)::value;
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int i = lo + threadIdx.x + u * kThreads;
      if (i < hi) sl[i - lo] = static_cast<double>(dev_expf(__fmul_rn(__fsub_rn(xr[u], m), job.inv_temp)));
    }
  };
  for (int r = 0; r < NR; ++r) {
    const float* g = static_cast<const float*>(rows[r]);
    double* sl = slices[r];
    const float m = norm[r].m;
    if (per_mode == 16) {
      exp_regs(sl, m, std::integral_constant<int, 16>{});
    } else if (per_mode == kMaxPer) {
      exp_regs(sl, m, std::integral_constant<int, (NR == 1 ? kMaxPer : 1)>{});
    } else {
      for (int i = lo + threadIdx.x; i < hi; i += blockDim.x)
        sl[i - lo] = static_cast<double>(dev_expf(__fmul_rn(__fsub_rn(g[i], m), job.inv_temp)));
    }
  }
  __syncthreads();
  if (!normalize) {
    for (int r = 0; r < NR; ++r) { norm[r].S = 1.0; norm[r].Pn = 1.0; }
    return PEARL_OK;
  }
  PEARL_TR(4);
  double S[NR];
  cluster_pairwise<NR>(cc, s, plan, [&](int c, int i) { return slices[c][i - lo]; }, S);
  PEARL_TR(5);
  PEARL_TR(6);
  // arr = e / S is formed inside the second pairwise sum's leaf pass (each
  // element is evaluated exactly once there and written back)
  double Pn[NR];
  cluster_pairwise<NR>(cc, s, plan, [&](int c, int i) {
    const double a = __ddiv_rn(slices[c][i - lo], S[c]);
    slices[c][i - lo] = a;
    return a;
  }, Pn);
  PEARL_TR(7);
  for (int r = 0; r < NR; ++r) {
    double* sl = slices[r];
    for (int i = lo + threadIdx.x; i < hi; i += blockDim.x) sl[i - lo] = __ddiv_rn(sl[i - lo], Pn[r]);
    norm[r].S = S[r];
    norm[r].Pn = Pn[r];
  }
  __syncthreads();
  return PEARL_OK;
}

// Element x of a row's ProbDist probs, recomputed from global memory with the
// exact op sequence prepare_rows used (so any CTA can read any element).
__device__ __forceinline__ double row_prob(const RowJob& job, const void* row, const RowNorm& nm, int x) {
  if (job.mode == PEARL_ROWS_PROBS64) return static_cast<const double*>(row)[x];
  const float l = static_cast<const float*>(row)[x];
  double e = static_cast<double>(dev_expf(__fmul_rn(__fsub_rn(l, nm.m), job.inv_temp)));
  return __ddiv_rn(__ddiv_rn(e, nm.S), nm.Pn);
}

// argmax over the smem slice (first index on ties)
__device__ int slice_argmax(ClusterCtx& cc, Scratch& s, const int* plan, const double* sl) {
  const int lo = plan[3], hi = plan[4];
  double bv = -1.0;
  int bi = 0x7fffffff;
  for (int i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    double v = sl[i - lo];
    if (v > bv) { bv = v; bi = i; }  // increasing i per thread: first max kept
  }
  return cluster_argmax(cc, s, bv, bi);
}

// records written by other CTAs are read through the L2 (never a stale L1 line)
__device__ __forceinline__ Rec load_rec(const Rec* p) {
  Rec r;
  r.status = __ldcg(&p->status);
  r.accept = __ldcg(&p->accept);
  r.corr = __ldcg(&p->corr);
  r.fb = __ldcg(&p->fb);
  r.a = __ldcg(&p->a);
  r.pad = 0.0;
  return r;
}

// ---------------------------------------------------------------------------
// K1
// ---------------------------------------------------------------------------
struct VerifyArgs {
  RowJob job;
  int flags;
  int n;
  const void* const* p_rows;
  const void* const* q_rows;
  const int32_t* drafted;
  const double* uniforms;
  int n_uniforms;
  int32_t* cursor;
  WorkHdr* work;
  pearl_verify_result* out;
  double* accept_out;
};

// one chain as the verify body sees it (a pearl_spec_verify call, or one
// descriptor of a pearl_spec_verify_multi launch)
struct ChainView {
  RowJob job;
  int flags;
  int n;
  const void* const* p_rows;
  const void* const* q_rows;
  const int32_t* drafted;
  const int32_t* tail;
  int stride;
  const double* uniforms;
  int n_uniforms;
  int32_t* cursor;
  WorkHdr* work;
  pearl_verify_result* out;
  double* accept_out;
  __device__ __forceinline__ int id(int pos) const {
    return (tail != nullptr && pos == n - 1) ? *tail : drafted[pos * stride];
  }
};

// position `pos` of chain A on this cluster; the chain's last-arriving
// cluster reduces the verdict (first reject by ballot) and advances its cursor
__device__ __forceinline__ void verify_position(ClusterCtx& cc, const int* plan, Scratch& s, double* P,
                                                double* Q, const ChainView& A, int pos) {
  const int lo = plan[3];
  const bool greedy = (A.flags & PEARL_F_GREEDY) != 0;
  const bool probe = (A.flags & PEARL_F_PROBE) != 0;
  const bool bonus_row = pos == A.n;  // only launched with PEARL_F_BONUS
  const int cur = A.cursor ? *A.cursor : 0;
  Rec rec{PEARL_OK, 0, -1, 0, 0.0, 0.0};

  if (bonus_row) {
    const void* rows[1] = {A.p_rows[pos]};
    double* sl[1] = {P};
    RowNorm nm[1];
    int st = prepare_rows<1>(cc, s, plan, A.job, rows, sl, !greedy, nm);
    if (st != PEARL_OK) {
      rec.status = st;
    } else if (greedy) {
      rec.corr = slice_argmax(cc, s, plan, P);
    } else {
      const int ui = cur + A.n;
      if (ui >= A.n_uniforms) {
        rec.status = PEARL_ERR_VALUE;
      } else {
        int fb = 0;
        rec.corr = cluster_search(cc, s, plan, A.job.V, [&](int i) { return P[i - lo]; },
                                  A.uniforms[ui], &fb);
        rec.fb = fb;
      }
    }
  } else {
    const int x = A.id(pos);
    const void* rows[2] = {A.p_rows[pos], A.q_rows[pos]};
    double* sl[2] = {P, Q};
    RowNorm nm[2];
    int st;
    if (greedy) {
      // greedy never reads q (engines.py:220-226); argmax of e == argmax of p
      st = prepare_rows<1>(cc, s, plan, A.job, rows, sl, false, nm);
      if (st == PEARL_OK) {
        const int best = slice_argmax(cc, s, plan, P);
        rec.accept = (x == best);
        rec.corr = best;
        rec.a = rec.accept ? 1.0 : 0.0;
      }
    } else {
      st = prepare_rows<2>(cc, s, plan, A.job, rows, sl, true, nm);
      if (st == PEARL_OK) {
        if (x < 0 || x >= A.job.V) {
          st = PEARL_ERR_VALUE;
        } else {
          const double qx = row_prob(A.job, rows[1], nm[1], x);
          const double px = row_prob(A.job, rows[0], nm[0], x);
          if (qx <= 0.0) {
            st = PEARL_ERR_ZERO_DRAFT_PROB;
          } else {
            const double a = (px >= qx) ? 1.0 : __ddiv_rn(px, qx);  // sampling.py:37-41
            rec.a = a;
            if (probe) {
              rec.accept = 1;
            } else if (cur + pos >= A.n_uniforms) {
              st = PEARL_ERR_VALUE;
            } else {
              const double u = A.uniforms[cur + pos];
              rec.accept = (u <= a);  // sampling.py:89
              if (!rec.accept) {
                // residual_dist (core.py:209-214) + sample (core.py:182-190)
                double mass;
                cluster_pairwise<1>(cc, s, plan, [&](int, int i) {
                  return fmax(__dsub_rn(P[i - lo], Q[i - lo]), 0.0);
                }, &mass);
                if (mass < 1e-15) {
                  st = PEARL_ERR_ALL_ZERO_RESIDUAL;
                } else if (cur + pos + 1 >= A.n_uniforms) {
                  st = PEARL_ERR_VALUE;
                } else {
                  double total;
                  cluster_pairwise<1>(cc, s, plan, [&](int, int i) {
                    return __ddiv_rn(fmax(__dsub_rn(P[i - lo], Q[i - lo]), 0.0), mass);
                  }, &total);
                  int fb = 0;
                  rec.corr = cluster_search(cc, s, plan, A.job.V, [&](int i) {
                    return __ddiv_rn(__ddiv_rn(fmax(__dsub_rn(P[i - lo], Q[i - lo]), 0.0), mass), total);
                  }, A.uniforms[cur + pos + 1], &fb);
                  rec.fb = fb;
                }
              }
            }
          }
        }
      }
    }
    rec.status = st;
  }

  // no CTA may exit while a peer could still read its shared memory
  if (cc.size > 1) cluster_sync_all();
  // publish this position's verdict; the last cluster reduces
  __shared__ int s_last;
  Rec* recs = reinterpret_cast<Rec*>(A.work + 1);
  if (cc.rank == 0 && threadIdx.x == 0) {
    recs[pos] = rec;
    __threadfence();
    const int total = A.n + ((A.flags & PEARL_F_BONUS) ? 1 : 0);
    const int old = atomicAdd(&A.work->arrived, 1);
    s_last = (old == total - 1);
  }
  __syncthreads();
  if (cc.rank != 0 || !s_last) return;
  __threadfence();
  if (threadIdx.x >= 32) return;
  // warp 0 of the last cluster: first non-accepted position via ballot
  const int lane = threadIdx.x;
  int stop = A.n;
  for (int base = 0; base < A.n; base += 32) {
    const int i = base + lane;
    int bad = 0;
    if (i < A.n) {
      const Rec r = load_rec(recs + i);
      bad = (r.status != PEARL_OK) || !r.accept;
    }
    const unsigned bal = __ballot_sync(0xffffffffu, bad);
    if (bal) { stop = base + __ffs(bal) - 1; break; }
  }
  if (lane != 0) return;
  pearl_verify_result res{};
  res.correction = -1;
  res.bonus = -1;
  int fb = 0;
  if (A.accept_out)
    for (int i = 0; i < A.n; ++i) A.accept_out[i] = load_rec(recs + i).a;
  if (stop < A.n) {
    const Rec r = load_rec(recs + stop);
    fb = r.fb;
    if (r.status == PEARL_ERR_ZERO_DRAFT_PROB) {
      res.status = r.status;
      res.draws_used = stop;  // accept draws of the positions before
    } else if (r.status == PEARL_ERR_ALL_ZERO_RESIDUAL) {
      res.status = r.status;
      res.draws_used = stop + 1;
    } else if (r.status != PEARL_OK) {
      res.status = r.status;
    } else {
      res.accepted = stop;
      res.correction = r.corr;
      res.examined = stop + 1;
      res.draws_used = greedy ? 0 : stop + 2;
    }
  } else {
    res.accepted = A.n;
    res.examined = A.n;
    res.draws_used = greedy || probe ? 0 : A.n;
    if (A.flags & PEARL_F_BONUS) {
      const Rec r = load_rec(recs + A.n);
      if (r.status != PEARL_OK) {
        res.status = r.status;
      } else {
        res.bonus = r.corr;
        fb = r.fb;
        res.draws_used += greedy ? 0 : 1;
      }
    }
  }
  res.fallback = fb;
  *A.out = res;
  if (A.cursor && (A.flags & PEARL_F_ADVANCE) && res.status == PEARL_OK) *A.cursor = cur + res.draws_used;
  A.work->arrived = 0;
}

__device__ __forceinline__ void verify_smem(const RowJob& job, int*& plan, Scratch*& s, double*& P, double*& Q) {
  plan = reinterpret_cast<int*>(g_smem);
  s = reinterpret_cast<Scratch*>(g_smem + kPlanStride * sizeof(int));
  P = reinterpret_cast<double*>(g_smem + kPlanStride * sizeof(int) + sizeof(Scratch));
  Q = P + job.cap;
}

__global__ void __launch_bounds__(kThreads) spec_verify_kernel(VerifyArgs A) {
  cg::cluster_group cl = cg::this_cluster();
  ClusterCtx cc{static_cast<int>(cl.block_rank()), static_cast<int>(cl.num_blocks()), 0};
  int* plan;
  Scratch* s;
  double *P, *Q;
  verify_smem(A.job, plan, s, P, Q);
  load_plan(plan, A.job.plan, cc.rank);
  const ChainView v{A.job, A.flags, A.n, A.p_rows, A.q_rows, A.drafted, nullptr, 1, A.uniforms, A.n_uniforms,
                    A.cursor, A.work, A.out, A.accept_out};
  verify_position(cc, plan, *s, P, Q, v, blockIdx.x / cc.size);
}

static_assert(sizeof(pearl_verify_chain) == 80, "pearl_verify_chain layout (batched.py packs it)");

struct VerifyMultiArgs {
  RowJob job;
  int flags;
  int n_chains;
  int n_uniforms;
  const pearl_verify_chain* chains;
};

__global__ void __launch_bounds__(kThreads) spec_verify_multi_kernel(VerifyMultiArgs A) {
  cg::cluster_group cl = cg::this_cluster();
  ClusterCtx cc{static_cast<int>(cl.block_rank()), static_cast<int>(cl.num_blocks()), 0};
  int* plan;
  Scratch* s;
  double *P, *Q;
  verify_smem(A.job, plan, s, P, Q);
  load_plan(plan, A.job.plan, cc.rank);
  const int c = blockIdx.x / cc.size;
  __shared__ int s_chain;
  // chain of cluster c = (number of chains with cluster_base <= c) - 1 (sorted bases)
  if (threadIdx.x < 32) {
    int cnt = 0;
    for (int b = 0; b < A.n_chains; b += 32) {
      const int i = b + threadIdx.x;
      cnt += __popc(__ballot_sync(0xffffffffu, i < A.n_chains && A.chains[i].cluster_base <= c));
    }
    if (threadIdx.x == 0) s_chain = cnt - 1;
  }
  __syncthreads();
  const pearl_verify_chain& d = A.chains[s_chain];
  const ChainView v{A.job, A.flags, d.n, d.p_rows, d.q_rows, d.drafted, d.tail, d.stride, d.uniforms,
                    d.uniforms ? A.n_uniforms : 0, d.cursor, static_cast<WorkHdr*>(d.work), d.out, nullptr};
  verify_position(cc, plan, *s, P, Q, v, c - d.cluster_base);
}

// ---------------------------------------------------------------------------
// pick kernel: one row per cluster
// ---------------------------------------------------------------------------
struct SampleArgs {
  RowJob job;
  int flags;
  int n_rows;
  const void* const* rows;
  const double* uniforms;
  int n_uniforms;
  int32_t* cursor;
  int32_t* out;
  int32_t* append_dst;
  int32_t* status;
  WorkHdr* work;
  // per-row streams (pearl_sample_rows_multi): row r draws tables[r][*cursors[r]]
  // and advances its own cursor; NULL for the shared-stream form
  const double* const* tables;
  int32_t* const* cursors;
  int multi;  // pearl_sample_rows_multi launch: no shared cursor / arrival counter
};

__global__ void __launch_bounds__(kThreads) sample_rows_kernel(SampleArgs A) {
  cg::cluster_group cl = cg::this_cluster();
  ClusterCtx cc{static_cast<int>(cl.block_rank()), static_cast<int>(cl.num_blocks()), 0};
  const int row = blockIdx.x / cc.size;
  int* plan = reinterpret_cast<int*>(g_smem);
  Scratch& s = *reinterpret_cast<Scratch*>(g_smem + kPlanStride * sizeof(int));
  double* P = reinterpret_cast<double*>(g_smem + kPlanStride * sizeof(int) + sizeof(Scratch));
  PEARL_TR(0);
  load_plan(plan, A.job.plan, cc.rank);
  PEARL_TR(1);
  const int lo = plan[3];
  const bool greedy = (A.flags & PEARL_F_GREEDY) != 0;
  const bool per_row = A.tables != nullptr;
  const int cur = per_row ? *A.cursors[row] - row : (A.cursor ? *A.cursor : 0);  // (row r reads cur + r)
  const double* table = per_row ? A.tables[row] : A.uniforms;
  const void* rows[1] = {A.rows[row]};
  double* sl[1] = {P};
  RowNorm nm[1];
  int st = prepare_rows<1>(cc, s, plan, A.job, rows, sl, !greedy, nm);
  int tok = -1;
  if (st == PEARL_OK) {
    if (greedy) {
      tok = slice_argmax(cc, s, plan, P);
    } else if (cur + row >= A.n_uniforms) {
      st = PEARL_ERR_VALUE;
    } else {
      tok = cluster_search(cc, s, plan, A.job.V, [&](int i) { return P[i - lo]; },
                           table[cur + row], nullptr);
    }
  }
  PEARL_TR(20);
  if (cc.size > 1) cluster_sync_all();
  PEARL_TR(21);
  if (cc.rank != 0 || threadIdx.x != 0) return;
  A.out[row] = tok;
  if (row == 0 && A.append_dst) *A.append_dst = tok;
  if (st != PEARL_OK && A.status) atomicMax(A.status, st);
  if (A.multi) {
    if (per_row && (A.flags & PEARL_F_ADVANCE) && !greedy && st == PEARL_OK) *A.cursors[row] = cur + row + 1;
    return;
  }
  __threadfence();
  const int old = atomicAdd(&A.work->arrived, 1);
  if (old == A.n_rows - 1) {
    __threadfence();
    if (A.cursor && (A.flags & PEARL_F_ADVANCE) && !greedy) *A.cursor = cur + A.n_rows;
    A.work->arrived = 0;
  }
}

// ---------------------------------------------------------------------------
// device law (p1 = e / S) and residual numerator
// ---------------------------------------------------------------------------
struct ProbsArgs {
  RowJob job;
  const float* logits;
  double* out;
  int32_t* status;
};

__global__ void __launch_bounds__(kThreads) logits_to_probs_kernel(ProbsArgs A) {
  cg::cluster_group cl = cg::this_cluster();
  ClusterCtx cc{static_cast<int>(cl.block_rank()), static_cast<int>(cl.num_blocks()), 0};
  const int row = blockIdx.x / cc.size;
  int* plan = reinterpret_cast<int*>(g_smem);
  Scratch& s = *reinterpret_cast<Scratch*>(g_smem + kPlanStride * sizeof(int));
  double* P = reinterpret_cast<double*>(g_smem + kPlanStride * sizeof(int) + sizeof(Scratch));
  load_plan(plan, A.job.plan, cc.rank);
  const int lo = plan[3], hi = plan[4];
  const void* rows[1] = {A.logits + static_cast<size_t>(row) * A.job.V};
  double* sl[1] = {P};
  RowNorm nm[1];
  int st = prepare_rows<1>(cc, s, plan, A.job, rows, sl, false, nm);
  double S = 1.0;
  if (st == PEARL_OK) cluster_pairwise<1>(cc, s, plan, [&](int, int i) { return P[i - lo]; }, &S);
  if (cc.size > 1) cluster_sync_all();
  if (st != PEARL_OK) {
    if (cc.rank == 0 && threadIdx.x == 0 && A.status) atomicMax(A.status, st);
    return;
  }
  double* o = A.out + static_cast<size_t>(row) * A.job.V;
  for (int i = lo + threadIdx.x; i < hi; i += blockDim.x) o[i] = __ddiv_rn(P[i - lo], S);
}

struct ResidArgs {
  RowJob job;
  const double* p;
  const double* q;
  double* out;
  int32_t* status;
};

__global__ void __launch_bounds__(kThreads) residual_kernel(ResidArgs A) {
  cg::cluster_group cl = cg::this_cluster();
  ClusterCtx cc{static_cast<int>(cl.block_rank()), static_cast<int>(cl.num_blocks()), 0};
  int* plan = reinterpret_cast<int*>(g_smem);
  Scratch& s = *reinterpret_cast<Scratch*>(g_smem + kPlanStride * sizeof(int));
  double* P = reinterpret_cast<double*>(g_smem + kPlanStride * sizeof(int) + sizeof(Scratch));
  double* Q = P + A.job.cap;
  load_plan(plan, A.job.plan, cc.rank);
  const int lo = plan[3], hi = plan[4];
  for (int i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    P[i - lo] = A.p[i];
    Q[i - lo] = A.q[i];
  }
  __syncthreads();
  double mass;
  cluster_pairwise<1>(cc, s, plan, [&](int, int i) { return fmax(__dsub_rn(P[i - lo], Q[i - lo]), 0.0); },
                      &mass);
  if (cc.size > 1) cluster_sync_all();
  if (mass < 1e-15) {
    if (cc.rank == 0 && threadIdx.x == 0 && A.status) atomicMax(A.status, PEARL_ERR_ALL_ZERO_RESIDUAL);
    return;
  }
  for (int i = lo + threadIdx.x; i < hi; i += blockDim.x)
    A.out[i] = __ddiv_rn(fmax(__dsub_rn(P[i - lo], Q[i - lo]), 0.0), mass);
}

// ---------------------------------------------------------------------------
// host launch helpers
// ---------------------------------------------------------------------------
namespace {

size_t smem_bytes(const VocabPlan& p, int nslices) {
  return kPlanStride * sizeof(int) + sizeof(Scratch) + static_cast<size_t>(nslices) * p.cap * sizeof(double);
}

template <class K>
int configure(K kernel, size_t smem) {
  PEARL_CUDA_TRY(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem)));
  PEARL_CUDA_TRY(cudaFuncSetAttribute(kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  return PEARL_OK;
}

template <class K, class Args>
int launch_clustered(K kernel, int n_clusters, int C, size_t smem, void* stream, const Args& args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(n_clusters * C);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = static_cast<cudaStream_t>(stream);
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  // programmatic dependent launch: the kernels load their vocabulary plan
  // (static) before griddepcontrol.wait, overlapping the producer's tail
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  PEARL_CUDA_TRY(cudaLaunchKernelEx(&cfg, kernel, args));
  count_launch();
  return PEARL_OK;
}

std::once_flag g_cfg_once;
int g_cfg_status = PEARL_OK;

int configure_all() {
  std::call_once(g_cfg_once, [] {
    // worst case slice: V=131072 over 16 CTAs -> 8192 (+ rounding) elements, 2 slices
    const size_t smem = kPlanStride * sizeof(int) + sizeof(Scratch) + 2 * 8320 * sizeof(double);
    int st = configure(spec_verify_kernel, smem);
    if (st == PEARL_OK) st = configure(spec_verify_multi_kernel, smem);
    if (st == PEARL_OK) st = configure(sample_rows_kernel, smem);
    if (st == PEARL_OK) st = configure(logits_to_probs_kernel, smem);
    if (st == PEARL_OK) st = configure(residual_kernel, smem);
    g_cfg_status = st;
  });
  return g_cfg_status;
}

}  // namespace
}  // namespace pearl

using namespace pearl;

#ifdef PEARL_TRACE_PICK
extern "C" int pearl_debug_trace(long long* out) {
  return cudaMemcpyFromSymbol(out, g_trace, sizeof(long long) * 32) == cudaSuccess ? 0 : -1;
}
#endif

extern "C" size_t pearl_verify_work_bytes(int n) {
  return sizeof(WorkHdr) + static_cast<size_t>(std::max(n, 1) + 1) * sizeof(Rec);
}

extern "C" int pearl_prepare_vocab(int V) {
  int st = configure_all();
  if (st != PEARL_OK) return st;
  return prepare_plan(V);
}

extern "C" int pearl_spec_verify(int row_mode, const void* const* p_rows, const void* const* q_rows,
                                 const int32_t* drafted, int n, int V, const double* uniforms,
                                 int n_uniforms, int32_t* cursor, float inv_temperature, int flags,
                                 pearl_verify_result* out, double* accept_probs, void* work,
                                 void* stream) {
  PEARL_ARG_CHECK(n >= 1 && n <= 1024, "chain length must be in [1, 1024]");
  PEARL_ARG_CHECK(row_mode == PEARL_ROWS_PROBS64 || row_mode == PEARL_ROWS_LOGITS32, "bad row mode");
  PEARL_ARG_CHECK(p_rows && drafted && out && work, "null argument");
  PEARL_ARG_CHECK((flags & PEARL_F_GREEDY) || q_rows, "q_rows required unless greedy");
  PEARL_ARG_CHECK(inv_temperature > 0.0f, "inverse temperature must be positive");
  int st = configure_all();
  if (st != PEARL_OK) return st;
  const VocabPlan* plan = get_plan(V);
  if (!plan) return PEARL_ERR_ARG;
  VerifyArgs a{};
  a.job = RowJob{row_mode, inv_temperature, V, plan->d_plan, plan->cap};
  a.flags = flags;
  a.n = n;
  a.p_rows = p_rows;
  a.q_rows = q_rows ? q_rows : p_rows;
  a.drafted = drafted;
  a.uniforms = uniforms;
  a.n_uniforms = uniforms ? n_uniforms : 0;
  a.cursor = cursor;
  a.work = static_cast<WorkHdr*>(work);
  a.out = out;
  a.accept_out = accept_probs;
  const int clusters = n + ((flags & PEARL_F_BONUS) ? 1 : 0);
  return launch_clustered(spec_verify_kernel, clusters, plan->C, smem_bytes(*plan, 2), stream, a);
}

extern "C" int pearl_spec_verify_multi(int row_mode, const pearl_verify_chain* chains, int n_chains,
                                       int n_clusters, int V, int n_uniforms, float inv_temperature, int flags,
                                       void* stream) {
  PEARL_ARG_CHECK(n_chains >= 1 && n_clusters >= n_chains, "need at least one chain of one position");
  PEARL_ARG_CHECK(row_mode == PEARL_ROWS_PROBS64 || row_mode == PEARL_ROWS_LOGITS32, "bad row mode");
  PEARL_ARG_CHECK(chains != nullptr, "null argument");
  PEARL_ARG_CHECK(inv_temperature > 0.0f, "inverse temperature must be positive");
  int st = configure_all();
  if (st != PEARL_OK) return st;
  const VocabPlan* plan = get_plan(V);
  if (!plan) return PEARL_ERR_ARG;
  VerifyMultiArgs a{};
  a.job = RowJob{row_mode, inv_temperature, V, plan->d_plan, plan->cap};
  a.flags = flags;
  a.n_chains = n_chains;
  a.n_uniforms = n_uniforms;
  a.chains = chains;
  return launch_clustered(spec_verify_multi_kernel, n_clusters, plan->C, smem_bytes(*plan, 2), stream, a);
}

extern "C" int pearl_sample_rows(int row_mode, const void* const* rows, int n_rows, int V,
                                 const double* uniforms, int n_uniforms, int32_t* cursor,
                                 float inv_temperature, int flags, int32_t* out_tokens,
                                 int32_t* append_dst, int32_t* status, void* work, void* stream) {
  PEARL_ARG_CHECK(n_rows >= 1, "need at least one row");
  PEARL_ARG_CHECK(rows && out_tokens && work, "null argument");
  PEARL_ARG_CHECK(inv_temperature > 0.0f, "inverse temperature must be positive");
  int st = configure_all();
  if (st != PEARL_OK) return st;
  const VocabPlan* plan = get_plan(V);
  if (!plan) return PEARL_ERR_ARG;
  SampleArgs a{};
  a.job = RowJob{row_mode, inv_temperature, V, plan->d_plan, plan->cap};
  a.flags = flags;
  a.n_rows = n_rows;
  a.rows = rows;
  a.uniforms = uniforms;
  a.n_uniforms = uniforms ? n_uniforms : 0;
  a.cursor = cursor;
  a.out = out_tokens;
  a.append_dst = append_dst;
  a.status = status;
  a.work = static_cast<WorkHdr*>(work);
  return launch_clustered(sample_rows_kernel, n_rows, plan->C, smem_bytes(*plan, 1), stream, a);
}

extern "C" int pearl_sample_rows_multi(int row_mode, const void* const* rows, int n_rows, int V,
                                       const double* const* tables, int n_uniforms, int32_t* const* cursors,
                                       float inv_temperature, int flags, int32_t* out_tokens, int32_t* status,
                                       void* stream) {
  PEARL_ARG_CHECK(n_rows >= 1, "need at least one row");
  PEARL_ARG_CHECK(rows && out_tokens && ((flags & PEARL_F_GREEDY) || (tables && cursors)), "null argument");
  PEARL_ARG_CHECK(inv_temperature > 0.0f, "inverse temperature must be positive");
  int st = configure_all();
  if (st != PEARL_OK) return st;
  const VocabPlan* plan = get_plan(V);
  if (!plan) return PEARL_ERR_ARG;
  SampleArgs a{};
  a.job = RowJob{row_mode, inv_temperature, V, plan->d_plan, plan->cap};
  a.flags = flags;
  a.n_rows = n_rows;
  a.rows = rows;
  a.n_uniforms = n_uniforms;
  a.out = out_tokens;
  a.status = status;
  a.tables = (flags & PEARL_F_GREEDY) ? nullptr : tables;
  a.cursors = (flags & PEARL_F_GREEDY) ? nullptr : cursors;
  a.multi = 1;
  return launch_clustered(sample_rows_kernel, n_rows, plan->C, smem_bytes(*plan, 1), stream, a);
}

extern "C" int pearl_logits_to_probs(const float* logits, int n_rows, int V, float inv_temperature,
                                     double* out, int32_t* status, void* stream) {
  PEARL_ARG_CHECK(n_rows >= 1 && logits && out, "bad arguments");
  PEARL_ARG_CHECK(inv_temperature > 0.0f, "inverse temperature must be positive");
  int st = configure_all();
  if (st != PEARL_OK) return st;
  const VocabPlan* plan = get_plan(V);
  if (!plan) return PEARL_ERR_ARG;
  ProbsArgs a{};
  a.job = RowJob{PEARL_ROWS_LOGITS32, inv_temperature, V, plan->d_plan, plan->cap};
  a.logits = logits;
  a.out = out;
  a.status = status;
  return launch_clustered(logits_to_probs_kernel, n_rows, plan->C, smem_bytes(*plan, 1), stream, a);
}

extern "C" int pearl_residual(const double* p, const double* q, int V, double* out, int32_t* status,
                              void* stream) {
  PEARL_ARG_CHECK(p && q && out, "bad arguments");
  int st = configure_all();
  if (st != PEARL_OK) return st;
  const VocabPlan* plan = get_plan(V);
  if (!plan) return PEARL_ERR_ARG;
  ResidArgs a{};
  a.job = RowJob{PEARL_ROWS_PROBS64, 1.0f, V, plan->d_plan, plan->cap};
  a.p = p;
  a.q = q;
  a.out = out;
  a.status = status;
  return launch_clustered(residual_kernel, 1, plan->C, smem_bytes(*plan, 2), stream, a);
}
