// Clique sharding across ranks (the paper's "in parallel",
// P:253, mapped onto one process per GPU).
//
//  * cliques are assigned to ranks by LPT on the cost k^3 + 16 (Jacobi / tridiagonal work grows as
//    k^3; the constant keeps tiny cliques from being free): the most expensive clique first, each to
//    the least-loaded rank (ties: lowest rank) -- max-cut's giant cliques spread over the ranks
//    instead of landing in one contiguous range; every rank keeps its cliques in canonical order;
//  * every pattern coordinate t is owned by the rank of the first clique that
//    contains it (its first stacked position); a rank touches t when one of its
//    cliques contains t; t is shared when two or more ranks touch it;
//  * per iteration only the partial sums of shared coordinates (scatter), the
//    m-vector u = A D^-1 r1 (column-sharded by owner) and a few residual
//    scalars cross ranks.
#include <algorithm>

#include "internal.h"

namespace sdp {

ShardPlan make_shard_plan(const std::vector<int32_t>& ksz, const std::vector<int64_t>& off,
                          const std::vector<int32_t>& seg_ptr, const std::vector<int32_t>& seg_idx, int world,
                          int rank) {
  ShardPlan sp;
  sp.world = world;
  sp.rank = rank;
  const int64_t p = (int64_t)ksz.size();
  const int64_t N = (int64_t)seg_ptr.size() - 1;
  // LPT on the clique cost (deterministic: stable order of equal costs, lowest rank on ties)
  std::vector<int32_t> order(p);
  for (int64_t k = 0; k < p; ++k) order[k] = (int32_t)k;
  auto cost = [&](int64_t k) { return (double)ksz[k] * ksz[k] * ksz[k] + 16.0; };
  std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return cost(a) > cost(b); });
  std::vector<double> load(world, 0.0);
  sp.clique_rank.assign(p, 0);
  for (int32_t k : order) {
    int best = 0;
    for (int r = 1; r < world; ++r)
      if (load[r] < load[best]) best = r;
    sp.clique_rank[k] = best;
    load[best] += cost(k);
  }
  // every rank gets at least one clique (world <= p): move the cheapest clique of the most
  // loaded rank with >= 2 cliques to an empty rank
  for (int r = 0; r < world; ++r) {
    bool has = false;
    for (int64_t k = 0; k < p && !has; ++k) has = sp.clique_rank[k] == r;
    if (has) continue;
    std::vector<int> cnt(world, 0);
    for (int64_t k = 0; k < p; ++k) cnt[sp.clique_rank[k]]++;
    for (auto it = order.rbegin(); it != order.rend(); ++it)
      if (cnt[sp.clique_rank[*it]] >= 2) {
        sp.clique_rank[*it] = r;
        break;
      }
  }
  for (int64_t k = 0; k < p; ++k)
    if (sp.clique_rank[k] == rank) sp.my_cliques.push_back((int32_t)k);
  std::vector<int32_t> clique_of(off.back());
  for (int64_t k = 0; k < p; ++k)
    for (int64_t s = off[k]; s < off[k + 1]; ++s) clique_of[s] = (int32_t)k;
  const std::vector<int32_t>& crank = sp.clique_rank;
  for (int64_t t = 0; t < N; ++t) {
    const int b = seg_ptr[t], e = seg_ptr[t + 1];
    const int first = crank[clique_of[seg_idx[b]]];  // seg_idx ascends: the first clique's rank owns t
    bool touch = false, multi = false;
    for (int i = b; i < e; ++i) {
      const int ri = crank[clique_of[seg_idx[i]]];
      touch |= ri == rank;
      multi |= ri != first;
    }
    if (multi) {
      sp.shared_coords.push_back((int32_t)t);
      sp.shared_local.push_back(touch ? (int32_t)sp.local_coords.size() : -1);
    }
    if (touch) {
      sp.local_coords.push_back((int32_t)t);
      sp.owned.push_back(first == rank ? 1 : 0);
    }
  }
  return sp;
}

}  // namespace sdp
