// Host planner for the numpy pairwise-summation tree (see probdist.cuh).
//
// numpy sums a contiguous float64 vector of n elements as
//   n <= 128 : one leaf (8 strided accumulators, or sequential for n < 8)
//   n  > 128 : pairwise(first n2) + pairwise(rest), n2 = n/2 - (n/2) % 8
// The planner cuts that tree at depth log2(C) into C subtrees, one per CTA of
// a thread-block cluster, and for each subtree lists its leaves (left to
// right) and its internal nodes grouped by height so a CTA can combine a
// whole level in parallel.  Only the shape depends on V, so one plan per V
// serves every row of that vocabulary.
#include <cuda_runtime.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "common.h"

namespace pearl {

constexpr int kPlanStride = 1024;
constexpr int kPlanHdr = 8;

namespace {

struct Node {
  int left, right;  // child slots (leaf slot or -1-nodeIndex before relabel)
  int height;
};

struct Builder {
  std::vector<std::pair<int, int>> leaves;  // (start, len)
  std::vector<Node> nodes;                  // unsorted internal nodes
  // returns encoded child: >=0 leaf index, <0 => -(node index + 1)
  int build(int lo, int n) {
    if (n <= 128) {
      leaves.push_back({lo, n});
      return static_cast<int>(leaves.size()) - 1;
    }
    int n2 = n / 2;
    n2 -= n2 % 8;
    int l = build(lo, n2);
    int r = build(lo + n2, n - n2);
    int hl = l >= 0 ? 0 : nodes[-l - 1].height;
    int hr = r >= 0 ? 0 : nodes[-r - 1].height;
    nodes.push_back({l, r, 1 + std::max(hl, hr)});
    return -static_cast<int>(nodes.size());
  }
};

void split_ranges(int lo, int n, int depth, std::vector<std::pair<int, int>>& out) {
  if (depth == 0) {
    out.push_back({lo, n});
    return;
  }
  int n2 = n / 2;
  n2 -= n2 % 8;
  split_ranges(lo, n2, depth - 1, out);
  split_ranges(lo + n2, n - n2, depth - 1, out);
}

bool fill_block(int lo, int n, int* blk) {
  Builder b;
  b.build(lo, n);
  const int nl = static_cast<int>(b.leaves.size());
  const int nn = static_cast<int>(b.nodes.size());
  // order internal nodes by height (stable); remember new positions
  std::vector<int> order(nn);
  for (int i = 0; i < nn; ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(),
                   [&](int a, int c) { return b.nodes[a].height < b.nodes[c].height; });
  std::vector<int> pos(nn);
  for (int i = 0; i < nn; ++i) pos[order[i]] = i;
  int nlev = 0;
  for (auto& nd : b.nodes) nlev = std::max(nlev, nd.height);
  const int need = kPlanHdr + 2 * nl + 2 * nn + nlev;
  if (need > kPlanStride || nl > 160 || nn > 160) return false;
  blk[0] = nl;
  blk[1] = nn;
  blk[2] = nlev;
  blk[3] = lo;
  blk[4] = lo + n;
  int* lv = blk + kPlanHdr;
  for (int i = 0; i < nl; ++i) {
    lv[2 * i] = b.leaves[i].first;
    lv[2 * i + 1] = b.leaves[i].second;
  }
  int* nd = lv + 2 * nl;
  auto slot = [&](int enc) { return enc >= 0 ? enc : nl + pos[-enc - 1]; };
  for (int i = 0; i < nn; ++i) {
    const Node& x = b.nodes[order[i]];
    nd[2 * i] = slot(x.left);
    nd[2 * i + 1] = slot(x.right);
  }
  int* le = nd + 2 * nn;
  for (int h = 1; h <= nlev; ++h) {
    int cnt = 0;
    for (auto& x : b.nodes) cnt += (x.height <= h);
    le[h - 1] = cnt;
  }
  return true;
}

std::mutex g_mu;
std::map<int, VocabPlan> g_plans;

}  // namespace

// Cluster size per vocabulary: one CTA below 4096 ids, then 8 (<= 65536),
// then 16 (<= 131072, Llama-3).  Depth log2(C) of the tree must still be
// made of internal nodes (n > 128), which these thresholds guarantee.
static int choose_cluster(int V) {
  if (V < 4096) return 1;
  if (V <= 65536) return 8;
  return 16;
}

int prepare_plan(int V) {
  if (V < 2 || V > 131072) {
    set_error("vocabulary size must be in [2, 131072], got " + std::to_string(V));
    return PEARL_ERR_ARG;
  }
  std::lock_guard<std::mutex> lk(g_mu);
  if (g_plans.count(V)) return PEARL_OK;
  VocabPlan p;
  p.V = V;
  p.C = choose_cluster(V);
  int depth = 0;
  while ((1 << depth) < p.C) ++depth;
  std::vector<std::pair<int, int>> ranges;
  split_ranges(0, V, depth, ranges);
  std::vector<int> host(static_cast<size_t>(p.C) * kPlanStride, 0);
  for (int r = 0; r < p.C; ++r) {
    if (!fill_block(ranges[r].first, ranges[r].second, host.data() + r * kPlanStride)) {
      set_error("pairwise plan does not fit for V=" + std::to_string(V));
      return PEARL_ERR_ARG;
    }
    p.cap = std::max(p.cap, ranges[r].second);
  }
  PEARL_CUDA_TRY(cudaMalloc(&p.d_plan, host.size() * sizeof(int)));
  PEARL_CUDA_TRY(cudaMemcpy(p.d_plan, host.data(), host.size() * sizeof(int), cudaMemcpyHostToDevice));
  g_plans[V] = p;
  return PEARL_OK;
}

const VocabPlan* get_plan(int V) {
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_plans.find(V);
  if (it == g_plans.end()) {
    set_error("vocabulary size " + std::to_string(V) + " not prepared (call pearl_prepare_vocab)");
    return nullptr;
  }
  return &it->second;
}

}  // namespace pearl
