// Clique sharding across ranks (the paper's "in parallel",
// P:253, mapped onto one process per GPU).
//
//  * cliques (canonical order) are split into contiguous ranges balanced by
//    cost k^3 + 16 (Jacobi work grows as k^3; the constant keeps tiny cliques
//    from being free);
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
  // contiguous clique ranges balanced by cost
  std::vector<double> prefix(p + 1, 0.0);
  for (int64_t k = 0; k < p; ++k) prefix[k + 1] = prefix[k] + (double)ksz[k] * ksz[k] * ksz[k] + 16.0;
  sp.clique_begin.assign(world + 1, 0);
  for (int r = 1; r < world; ++r) {
    const double target = prefix[p] * r / world;
    int64_t b = std::lower_bound(prefix.begin(), prefix.end(), target) - prefix.begin();
    // every rank gets at least one clique (a giant clique can outweigh a share)
    b = std::min<int64_t>(std::max<int64_t>(b, sp.clique_begin[r - 1] + 1), p - (world - r));
    sp.clique_begin[r] = b;
  }
  sp.clique_begin[world] = p;
  // rank of every stacked position
  auto rank_of_clique = [&](int64_t k) {
    return (int)(std::upper_bound(sp.clique_begin.begin(), sp.clique_begin.end(), k) - sp.clique_begin.begin()) - 1;
  };
  std::vector<int32_t> clique_of(off.back());
  for (int64_t k = 0; k < p; ++k)
    for (int64_t s = off[k]; s < off[k + 1]; ++s) clique_of[s] = (int32_t)k;
  std::vector<int32_t> crank(p);
  for (int64_t k = 0; k < p; ++k) crank[k] = rank_of_clique(k);
  for (int64_t t = 0; t < N; ++t) {
    const int b = seg_ptr[t], e = seg_ptr[t + 1];
    const int first = crank[clique_of[seg_idx[b]]], last = crank[clique_of[seg_idx[e - 1]]];
    bool touch = false;
    for (int i = b; i < e && !touch; ++i) touch = crank[clique_of[seg_idx[i]]] == rank;
    if (first != last) {
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
