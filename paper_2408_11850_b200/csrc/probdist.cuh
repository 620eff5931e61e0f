// Device-side ProbDist arithmetic, bit-exact with the reference's numpy code.
//
// The reference keeps every next-token law as a numpy float64 vector
// (pearl_lab/core.py:67-120).  Three numpy behaviours decide its sampled
// tokens and must be reproduced exactly on the GPU:
//   * ndarray.sum()   -- numpy pairwise summation (ProbDist core.py:91,
//                        residual_dist core.py:210).  Emulated here with the
//                        same tree: leaves of <=128 elements summed with 8
//                        strided accumulators, split rule n2 = n/2 - (n/2)%8.
//                        The tree is pre-planned on the host (plan.cpp) and
//                        partitioned across the CTAs of a thread-block
//                        cluster at depth log2(C), so each CTA owns one
//                        subtree and the cluster combines C subtree sums in
//                        the balanced top-level order.
//   * np.cumsum       -- a strictly sequential fp64 scan (core.py:98).  We
//                        run a parallel scan with a rigorous error bound and
//                        resolve searchsorted exactly whenever u is farther
//                        than the bound from every CDF value; otherwise we
//                        replay the sequential scan (probability ~1e-11).
//   * searchsorted(..., 'right') with cdf[-1] = 1.0 (core.py:99, 189-190).
// All fp64 arithmetic uses explicit __d*_rn intrinsics so nvcc can never
// contract an add with a multiply into an FMA (that would change rounding).
//
// It also defines the device's next-token law from fp32 logits
// (pearl_dev_expf / logits -> p1), mirrored bit-for-bit by
// oracle/probdist.py:dev_expf / logits_to_p1.
#pragma once

#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace cg = cooperative_groups;

namespace pearl {

// Phase timestamps of one CTA (diagnostics: built only with -DPEARL_TRACE_PICK,
// read with pearl_debug_trace).
#ifdef PEARL_TRACE_PICK
__device__ long long g_trace[32];
#define PEARL_TR(k) \
  do { if (blockIdx.x == 0 && threadIdx.x == 0) g_trace[k] = clock64(); } while (0)
#else
#define PEARL_TR(k) do { } while (0)
#endif

// ---------------------------------------------------------------------------
// plan layout (int32), one block of kPlanStride ints per CTA of the cluster
//   [0] n_leaves [1] n_nodes [2] n_levels [3] lo [4] hi
//   [kPlanHdr ..)            leaves: (start, len) absolute element indices
//   then nodes: (left, right) value-slot indices (leaves occupy slots
//               [0, n_leaves), node j occupies slot n_leaves + j)
//   then level_end[n_levels]: exclusive end (node index) of each height level
// ---------------------------------------------------------------------------
constexpr int kPlanStride = 1024;
constexpr int kPlanHdr = 8;
constexpr int kMaxLeaves = 160;
constexpr int kMaxNodes = 160;
constexpr int kMaxCluster = 16;

// ---------------------------------------------------------------------------
// device exp (fp32, IEEE RN ops only) -- twin of oracle/probdist.py:dev_expf
// ---------------------------------------------------------------------------
__device__ __forceinline__ float dev_expf(float x) {
  if (!(x >= -80.0f)) return 0.0f;  // flush (also -inf)
  const float kLog2e = __int_as_float(0x3fb8aa3b);
  const float kLn2Hi = __int_as_float(0x3f318000);
  const float kLn2Lo = __int_as_float(0xb95e8083);
  float t = __fmul_rn(x, kLog2e);
  float k = rintf(t);
  float r = __fsub_rn(x, __fmul_rn(k, kLn2Hi));
  r = __fsub_rn(r, __fmul_rn(k, kLn2Lo));
  float p = __int_as_float(0x39500d01);
  p = __fadd_rn(__fmul_rn(p, r), __int_as_float(0x3ab60b61));
  p = __fadd_rn(__fmul_rn(p, r), __int_as_float(0x3c088889));
  p = __fadd_rn(__fmul_rn(p, r), __int_as_float(0x3d2aaaab));
  p = __fadd_rn(__fmul_rn(p, r), __int_as_float(0x3e2aaaab));
  p = __fadd_rn(__fmul_rn(p, r), __int_as_float(0x3f000000));
  p = __fadd_rn(__fmul_rn(p, r), __int_as_float(0x3f800000));
  p = __fadd_rn(__fmul_rn(p, r), __int_as_float(0x3f800000));
  int ki = static_cast<int>(k);
  return __fmul_rn(p, __int_as_float((ki + 127) << 23));
}

// ---------------------------------------------------------------------------
// small block / warp helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ float warp_max_f(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// (value, index) argmax with first-index tie break
__device__ __forceinline__ void warp_argmax(double& v, int& i) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double ov = __shfl_xor_sync(0xffffffffu, v, o);
    int oi = __shfl_xor_sync(0xffffffffu, i, o);
    if (ov > v || (ov == v && oi < i)) { v = ov; i = oi; }
  }
}

__device__ __forceinline__ int warp_min_i(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__device__ __forceinline__ int warp_or_i(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v |= __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Shared scratch for the block/cluster collectives below.
struct Scratch {
  double xchg[2][4];       // cluster exchange, double-buffered (see ClusterCtx)
  int xchg_i[2][4];
  double gath_d[kMaxCluster * 4];  // gathered values, row r = CTA r
  int gath_i[kMaxCluster * 4];
  double warp_d[32];
  int warp_i[32];
  int warp_j[32];
  float warp_f[32];
  double vals[kMaxLeaves + kMaxNodes];  // pairwise leaf / node values
  double res_d[4];
  int res_i[4];
};

// Cluster context: rank, size and the exchange-buffer parity.  Every
// collective writes its local contribution into xchg[parity], syncs the
// cluster, reads every rank's slot, and flips parity.  Alternating two
// buffers is race-free: a rank can only overwrite buffer b again after the
// *next* cluster barrier, which every reader of b has passed only after
// finishing its reads of b.
struct ClusterCtx {
  int rank;
  int size;
  int parity;
};

// Non-.aligned cluster barrier: callers may arrive from divergent code
// (e.g. after a thread-0-only block), which the .aligned form used by
// cg::cluster_group::sync() does not allow (compute-sanitizer synccheck).
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release;\n\tbarrier.cluster.wait.acquire;" ::: "memory");
}

// Gather up to 4 values from every CTA of the cluster.  After the cluster
// barrier, threads (r, k) < (size, 4) each read ONE remote value into the
// local gather table (row r = CTA r, 4 slots per row), then a block barrier
// publishes it: one DSMEM round trip per collective instead of every thread
// walking every rank.  The returned table stays valid until the next gather
// of the same type (a CTA can only pass the next cluster barrier once all
// its threads are done with it).
__device__ __forceinline__ const double* cluster_gather_d(ClusterCtx& cc, Scratch& s, const double* v, int nv) {
  if (threadIdx.x == 0)
    for (int k = 0; k < nv; ++k) s.xchg[cc.parity][k] = v[k];
  __syncwarp();  // reconverge warp 0 before the (cluster) barrier
  if (cc.size == 1) {
    __syncthreads();
    if (threadIdx.x < nv) s.gath_d[threadIdx.x] = s.xchg[cc.parity][threadIdx.x];
  } else {
    cluster_sync_all();
    if (threadIdx.x < cc.size * 4 && (threadIdx.x & 3) < nv)
      s.gath_d[threadIdx.x] = cg::this_cluster().map_shared_rank(&s.xchg[cc.parity][0], threadIdx.x >> 2)[threadIdx.x & 3];
  }
  __syncwarp();
  __syncthreads();
  cc.parity ^= 1;
  return s.gath_d;
}

__device__ __forceinline__ const int* cluster_gather_i(ClusterCtx& cc, Scratch& s, const int* v, int nv) {
  if (threadIdx.x == 0)
    for (int k = 0; k < nv; ++k) s.xchg_i[cc.parity][k] = v[k];
  __syncwarp();  // reconverge warp 0 before the (cluster) barrier
  if (cc.size == 1) {
    __syncthreads();
    if (threadIdx.x < nv) s.gath_i[threadIdx.x] = s.xchg_i[cc.parity][threadIdx.x];
  } else {
    cluster_sync_all();
    if (threadIdx.x < cc.size * 4 && (threadIdx.x & 3) < nv)
      s.gath_i[threadIdx.x] = cg::this_cluster().map_shared_rank(&s.xchg_i[cc.parity][0], threadIdx.x >> 2)[threadIdx.x & 3];
  }
  __syncwarp();
  __syncthreads();
  cc.parity ^= 1;
  return s.gath_i;
}

// balanced top-level combine of n (power of two <= 16) subtree sums g[i*stride],
// bottom-up, the association of numpy's recursive halving at the top levels
// (fully unrolled: register-resident)
__device__ __forceinline__ double tree_combine(const double* g, int stride, int n) {
  double b[kMaxCluster];
#pragma unroll
  for (int i = 0; i < kMaxCluster; ++i) b[i] = i < n ? g[i * stride] : 0.0;
#pragma unroll
  for (int w = kMaxCluster; w > 1; w >>= 1) {
    if (n >= w) {
#pragma unroll
      for (int i = 0; i < w / 2; ++i) b[i] = __dadd_rn(b[2 * i], b[2 * i + 1]);
    }
  }
  return b[0];
}

// ---------------------------------------------------------------------------
// CTA-subtree pairwise sum.  f(i) returns element i (absolute index) as an
// fp64 value; it is evaluated exactly once per element.
// Returns the cluster-wide numpy pairwise sum, identical in every thread.
// ---------------------------------------------------------------------------
template <int kNv, class F>
__device__ void cluster_pairwise(ClusterCtx& cc, Scratch& s, const int* plan, F f, double* result) {
  const int nl = plan[0], nn = plan[1], nlev = plan[2];
  const int* leaves = plan + kPlanHdr;
  const int* nodes = leaves + 2 * nl;
  const int* lev_end = nodes + 2 * nn;
  const int lane = threadIdx.x & 31;
  const int l8 = threadIdx.x & 7;
  const int grp = threadIdx.x >> 3;
  const int ngrp = blockDim.x >> 3;
  double sums[kNv];
  for (int c = 0; c < kNv; ++c) {
    for (int base = 0; base < nl; base += ngrp) {
      const int L = base + grp;
      const bool act = L < nl;
      const int st = act ? leaves[2 * L] : 0;
      const int n = act ? leaves[2 * L + 1] : 8;
      double r = 0.0;
      double res = 0.0;
      if (n < 8) {
        if (act && l8 == 0) {
          for (int i = 0; i < n; ++i) res = __dadd_rn(res, f(c, st + i));
        }
      } else {
        const int stop = n - (n & 7);
        if (act) {
          r = f(c, st + l8);
          for (int i = 8; i < stop; i += 8) r = __dadd_rn(r, f(c, st + i + l8));
        }
      }
      // combine ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)); all lanes shuffle
      double o = __shfl_xor_sync(0xffffffffu, r, 1);
      double g = __dadd_rn(r, o);
      o = __shfl_xor_sync(0xffffffffu, g, 2);
      double h = __dadd_rn(g, o);
      o = __shfl_xor_sync(0xffffffffu, h, 4);
      double full = __dadd_rn(h, o);
      (void)lane;
      if (act && l8 == 0) {
        if (n >= 8) {
          res = full;
          const int stop = n - (n & 7);
          for (int i = stop; i < n; ++i) res = __dadd_rn(res, f(c, st + i));
        }
        s.vals[L] = res;
      }
    }
    __syncthreads();
    int j0 = 0;
    for (int lev = 0; lev < nlev; ++lev) {
      const int j1 = lev_end[lev];
      for (int j = j0 + threadIdx.x; j < j1; j += blockDim.x)
        s.vals[nl + j] = __dadd_rn(s.vals[nodes[2 * j]], s.vals[nodes[2 * j + 1]]);
      j0 = j1;
      __syncthreads();
    }
    sums[c] = nn > 0 ? s.vals[nl + nn - 1] : s.vals[0];
    __syncthreads();
  }
  if (cc.size == 1) {
    for (int c = 0; c < kNv; ++c) result[c] = sums[c];
    return;
  }
  const double* all = cluster_gather_d(cc, s, sums, kNv);
  for (int c = 0; c < kNv; ++c) result[c] = tree_combine(all + c, 4, cc.size);
}

// ---------------------------------------------------------------------------
// block / cluster max of floats, argmax of doubles
// ---------------------------------------------------------------------------
__device__ float cluster_max_f(ClusterCtx& cc, Scratch& s, float v) {
  v = warp_max_f(v);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) s.warp_f[w] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    float x = threadIdx.x < (blockDim.x >> 5) ? s.warp_f[threadIdx.x] : -INFINITY;
    x = warp_max_f(x);
    if (threadIdx.x == 0) s.res_d[0] = x;
  }
  __syncthreads();
  double m = s.res_d[0];
  __syncthreads();
  const double* all = cluster_gather_d(cc, s, &m, 1);
  float out = -INFINITY;
  for (int r = 0; r < cc.size; ++r) out = fmaxf(out, static_cast<float>(all[4 * r]));
  return out;
}

__device__ int cluster_argmax(ClusterCtx& cc, Scratch& s, double v, int i) {
  warp_argmax(v, i);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) { s.warp_d[w] = v; s.warp_i[w] = i; }
  __syncthreads();
  if (threadIdx.x < 32) {
    double x = -1.0;
    int xi = 0x7fffffff;
    if (threadIdx.x < (blockDim.x >> 5)) { x = s.warp_d[threadIdx.x]; xi = s.warp_i[threadIdx.x]; }
    warp_argmax(x, xi);
    if (threadIdx.x == 0) { s.res_d[0] = x; s.res_i[0] = xi; }
  }
  __syncthreads();
  double bv = s.res_d[0];
  int bi = s.res_i[0];
  __syncthreads();
  const double* allv = cluster_gather_d(cc, s, &bv, 1);
  const int* alli = cluster_gather_i(cc, s, &bi, 1);
  double best = -1.0;
  int besti = 0x7fffffff;
  for (int r = 0; r < cc.size; ++r) {
    double x = allv[4 * r];
    int xi = alli[4 * r];
    if (x > best || (x == best && xi < besti)) { best = x; besti = xi; }
  }
  return besti;
}

// ---------------------------------------------------------------------------
// Exact searchsorted(cumsum(a), u, 'right') with cdf[-1] := 1.0 over the
// cluster's slices [lo, hi).  a(i) returns the fp64 element i.
// ---------------------------------------------------------------------------
template <class F>
__device__ int cluster_search(ClusterCtx& cc, Scratch& s, const int* plan, int V, F a, double u,
                              int* used_fallback) {
  const int lo = plan[3], hi = plan[4];
  const int len = hi - lo;
  const int nt = blockDim.x;
  // odd chunk length: thread chunks start 8*per bytes apart, so an odd per
  // spreads a warp's fp64 reads over all banks (an even 16 put all 32 lanes
  // on one bank pair).  The answer does not depend on the chunking: the scan
  // is exact up to the rigorous bound delta, and ambiguous draws replay the
  // sequential scan.
  const int per = ((len + nt - 1) / nt) | 1;
  const int st = lo + threadIdx.x * per;
  const int en = min(st + per, hi);
  // rigorous bound on |parallel prefix - sequential prefix| for values
  // summing to ~1: (#adds on either chain) * 2^-53, doubled for margin
  const double delta = static_cast<double>(V + 2048) * 2.220446049250313e-16;
  PEARL_TR(10);
  // 1) chunk totals
  double t = 0.0;
  for (int i = st; i < en; ++i) t = __dadd_rn(t, a(i));
  // 2) block exclusive scan of chunk totals (ordered)
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double incl = t;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    double y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl = __dadd_rn(y, incl);
  }
  if (lane == 31) s.warp_d[w] = incl;
  __syncthreads();
  if (threadIdx.x == 0) {
    double run = 0.0;
    const int nw = nt >> 5;
    for (int k = 0; k < nw; ++k) {
      double x = s.warp_d[k];
      s.warp_d[k] = run;
      run = __dadd_rn(run, x);
    }
    s.res_d[1] = run;  // CTA total
  }
  __syncthreads();
  const double thread_off = __dadd_rn(s.warp_d[w], __dsub_rn(incl, t));
  const double cta_total = s.res_d[1];
  __syncthreads();
  PEARL_TR(11);
  const double* allT = cluster_gather_d(cc, s, &cta_total, 1);
  PEARL_TR(12);
  double cta_off = 0.0;
  for (int r = 0; r < cc.rank; ++r) cta_off = __dadd_rn(cta_off, allT[4 * r]);
  // 3) walk the chunk
  const double ulo = u - delta, uhi = u + delta;
  int cand = 0x7fffffff;
  int amb = 0;
  double c = __dadd_rn(cta_off, thread_off);
  for (int i = st; i < en; ++i) {
    c = __dadd_rn(c, a(i));
    if (i == V - 1) { cand = i; break; }  // cdf[-1] = 1.0 > u always
    if (c > uhi) { cand = i; break; }
    if (c >= ulo) amb = 1;
  }
  PEARL_TR(13);
  // 4) reduce: j = min cand; ambiguity only counts before j.  Per CTA:
  // (first local candidate jl, ambiguity in the chunks up to jl); chunks are
  // in thread order, so the global answer is j = min over CTAs of jl and the
  // draw is ambiguous iff some CTA starting at or before j flagged it --
  // one cluster exchange of both values.
  int wc = warp_min_i(cand);
  if (lane == 0) s.warp_i[w] = wc;
  __syncthreads();
  if (threadIdx.x < 32) {
    int x = threadIdx.x < (nt >> 5) ? s.warp_i[threadIdx.x] : 0x7fffffff;
    x = warp_min_i(x);
    if (threadIdx.x == 0) s.res_i[1] = x;
  }
  __syncthreads();
  const int jl = s.res_i[1];
  int mine = (amb && st <= jl) ? 1 : 0;
  int wa = warp_or_i(mine);
  if (lane == 0) s.warp_j[w] = wa;
  __syncthreads();
  if (threadIdx.x < 32) {
    int x = threadIdx.x < (nt >> 5) ? s.warp_j[threadIdx.x] : 0;
    x = warp_or_i(x);
    if (threadIdx.x == 0) s.res_i[2] = x;
  }
  __syncthreads();
  int both[2] = {jl, s.res_i[2]};
  __syncthreads();
  PEARL_TR(14);
  const int* jj = cluster_gather_i(cc, s, both, 2);
  PEARL_TR(15);
  int j = 0x7fffffff;
  for (int r = 0; r < cc.size; ++r) j = min(j, jj[4 * r]);
  int ambiguous = 0;
  bool starts_before = true;  // CTA r's slice starts at or before j iff no earlier CTA found a candidate
  for (int r = 0; r < cc.size; ++r) {
    // (slices are ordered; r's flag already stops at its own first candidate)
    if (starts_before) ambiguous |= jj[4 * r + 1];
    starts_before &= (jj[4 * r] == 0x7fffffff);
  }
  if (!ambiguous) {
    if (used_fallback) *used_fallback = 0;
    return j;
  }
  // 5) exact sequential replay, CTA by CTA (probability ~ 1e-11 per draw)
  if (used_fallback) *used_fallback = 1;
  double carry = 0.0;
  int ans = -1;
  for (int r = 0; r < cc.size; ++r) {
    double v2[2] = {0.0, 0.0};
    // the whole of warp 0 runs the replay in lockstep (every lane the same
    // values; lane 0's are published), so no warp reaches the following
    // barriers partially diverged
    if (cc.rank == r && threadIdx.x < 32) {
      double cc_ = carry;
      int an = ans;
      for (int i = lo; i < hi && an < 0; ++i) {
        cc_ = __dadd_rn(cc_, a(i));
        if (i == V - 1 || cc_ > u) an = i;
      }
      v2[0] = cc_;
      v2[1] = static_cast<double>(an);
    }
    __syncwarp();
    const double* got = cluster_gather_d(cc, s, v2, 2);
    carry = got[4 * r];
    if (ans < 0) ans = static_cast<int>(got[4 * r + 1]);
    __syncthreads();
  }
  return ans;
}

}  // namespace pearl
