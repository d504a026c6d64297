// Sparse Cholesky of the KKT Schur complement S = A D^-1 A^T (the factorisation
// is computed once and cached).  For problems whose constraints touch few common pattern
// entries (SDPA-type inputs, e.g. distance constraints on a geometric graph) S is sparse and so is
// its Cholesky factor under a fill-reducing order: the dense O(m^3) factorisation and the dense
// triangular inverse are replaced by
//   1. ordering + symbolic factorisation: the chordal analysis of S's graph (exact minimum degree,
//      setup_host.cpp) -- the later neighbours of v are the rows of column v of the factor;
//   2. left-looking numeric factorisation S = L L^T in that order (L(i, v) stored per column);
//   3. G = L^-1 column by column: L g = e_j has its nonzeros on the elimination-tree path from j
//      to the root, so each column costs the sum of the column lengths along that path;
// after which S^-1 = G^T G is one (DMMA) SYRK on the GPU and the iteration's y = S^-1 u stays the
// dense mat-vec.  Host code, O(sum |col|^2) + O(m * path * |col|), OpenMP over the columns of G.
#include <omp.h>

#include <algorithm>
#include <cmath>
#include <string>

#include "internal.h"

namespace sdp {

bool sparse_inverse_factor(int m, const std::vector<int64_t>& sp, const std::vector<int32_t>& si,
                           const std::vector<double>& sv, int64_t ldg, std::vector<double>& GT, int64_t* nnz_l,
                           double max_fill_frac, bool force, std::string* why) {
  // 1. ordering + symbolic (S's graph: the off-diagonal pattern, upper pairs)
  std::vector<std::pair<int32_t, int32_t>> edges;
  for (int a = 0; a < m; ++a)
    for (int64_t e = sp[a]; e < sp[a + 1]; ++e)
      if (si[e] > a) edges.push_back({a, si[e]});
  ChordalResult cr = chordal_analysis(m, edges);
  std::vector<int32_t> pos(m);
  for (int q = 0; q < m; ++q) pos[cr.order[q]] = q;
  // column v: [v, later(v) sorted by elimination position]
  std::vector<int64_t> cp(m + 1, 0);
  for (int v = 0; v < m; ++v) cp[v + 1] = cp[v] + 1 + (cr.later_ptr[v + 1] - cr.later_ptr[v]);
  const int64_t nnz = cp[m];
  *nnz_l = nnz;
  if (!force && (double)nnz > max_fill_frac * (double)m * (double)m) {
    if (why) *why = "factor too dense";
    return false;
  }
  std::vector<int32_t> ci(nnz);
  std::vector<double> cv(nnz, 0.0);
  for (int v = 0; v < m; ++v) {
    int64_t e = cp[v];
    ci[e++] = v;
    for (int64_t l = cr.later_ptr[v]; l < cr.later_ptr[v + 1]; ++l) ci[e++] = cr.later_idx[l];
    std::sort(ci.begin() + cp[v] + 1, ci.begin() + cp[v + 1], [&](int32_t x, int32_t y) { return pos[x] < pos[y]; });
  }
  // row structure: for every column u and every row v > u of it, (u, the entry index of v in col(u))
  std::vector<int64_t> rp(m + 1, 0);
  for (int u = 0; u < m; ++u)
    for (int64_t e = cp[u] + 1; e < cp[u + 1]; ++e) rp[ci[e] + 1]++;
  for (int v = 0; v < m; ++v) rp[v + 1] += rp[v];
  std::vector<int64_t> rent(rp[m]);
  std::vector<int32_t> rcol(rp[m]);
  {
    std::vector<int64_t> fillp(rp.begin(), rp.end() - 1);
    for (int q = 0; q < m; ++q) {  // columns in elimination order: rows see their columns in order
      const int u = cr.order[q];
      for (int64_t e = cp[u] + 1; e < cp[u + 1]; ++e) {
        rcol[fillp[ci[e]]] = u;
        rent[fillp[ci[e]]++] = e;
      }
    }
  }
  // 2. left-looking numeric factorisation in elimination order
  std::vector<double> w(m, 0.0), diag(m, 0.0);
  for (int a = 0; a < m; ++a)
    for (int64_t e = sp[a]; e < sp[a + 1]; ++e)
      if (si[e] == a) diag[a] = sv[e];
  for (int q = 0; q < m; ++q) {
    const int v = cr.order[q];
    // S(:, v) on col(v)
    for (int64_t e = sp[v]; e < sp[v + 1]; ++e) w[si[e]] = sv[e];
    for (int64_t r = rp[v]; r < rp[v + 1]; ++r) {
      const int64_t ev = rent[r];  // entry of v in col(u)
      const int u = rcol[r];
      const double lvu = cv[ev];
      for (int64_t e = ev; e < cp[u + 1]; ++e) w[ci[e]] -= cv[e] * lvu;  // rows at or after v
    }
    const double d = w[v];
    if (!(d > 1e-12 * diag[v]) || !std::isfinite(d)) {
      if (why) *why = "S = A D^-1 A^T is not positive definite";
      return false;
    }
    const double lvv = std::sqrt(d);
    cv[cp[v]] = lvv;
    for (int64_t e = cp[v] + 1; e < cp[v + 1]; ++e) cv[e] = w[ci[e]] / lvv;
    for (int64_t e = cp[v]; e < cp[v + 1]; ++e) w[ci[e]] = 0.0;
    for (int64_t e = sp[v]; e < sp[v + 1]; ++e) w[si[e]] = 0.0;
  }
  // 3. G = L^-1, column j of G = row j of GT: L g = e_j along the elimination-tree path
  std::vector<int32_t> parent(m, -1);
  for (int v = 0; v < m; ++v)
    if (cp[v + 1] - cp[v] > 1) parent[v] = ci[cp[v] + 1];  // first later row in elimination order
  GT.assign((size_t)m * ldg, 0.0);
#pragma omp parallel
  {
    std::vector<double> g(m, 0.0);
#pragma omp for schedule(dynamic, 16)
    for (int j = 0; j < m; ++j) {
      g[j] = 1.0;
      double* out = GT.data() + (size_t)j * ldg;
      for (int k = j; k >= 0; k = parent[k]) {
        const double gk = g[k] / cv[cp[k]];
        g[k] = 0.0;
        out[k] = gk;
        for (int64_t e = cp[k] + 1; e < cp[k + 1]; ++e) g[ci[e]] -= cv[e] * gk;
      }
    }
  }
  return true;
}

}  // namespace sdp
