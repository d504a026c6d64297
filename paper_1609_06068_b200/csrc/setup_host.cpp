// Host-side chordal analysis, run once in sdp_setup ("Setup: Chordal
// decomposition").  Independent of oracle/ (which is Python); the two are
// checked against each other by tests/test_library_host.py.
//
//  * aggregate pattern arrives as off-diagonal upper edges;
//  * chordal extension: exact minimum-degree symbolic elimination with
//    lowest-index ties (reading G13) -- the fill edges are E' \ E;
//  * maximal cliques from the elimination tree: the
//    candidate K_v = {v} U adj+(v) is maximal iff no child w of v in the
//    elimination tree has |K_w| = |K_v| + 1;
//  * cliques sorted ascending inside and lexicographically as a list
//    (reading G14); coordinates of E' in column-major upper order.
//
// Adjacency is a dense bitset (n^2/8 bytes) for n <= 46340, sorted adjacency lists beyond.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <set>
#include <stdexcept>

#include "internal.h"

namespace sdp {

namespace {
inline int popc(uint64_t x) { return __builtin_popcountll(x); }

// Minimum-degree queue, smallest degree then smallest index (reading G13), as a binary heap with
// lazy deletion: an update pushes the new key, stale entries are skipped when they surface (no
// per-update allocation, unlike an ordered set).
struct MinDegQueue {
  std::vector<std::pair<int32_t, int32_t>> heap;  // (degree, vertex), min-heap
  const std::vector<int32_t>* deg = nullptr;
  const std::vector<char>* dead = nullptr;
  static bool later_first(const std::pair<int32_t, int32_t>& a, const std::pair<int32_t, int32_t>& b) {
    return a > b;  // std heap is a max-heap: invert for the smallest (degree, index)
  }
  void push(int32_t d, int32_t v) {
    heap.push_back({d, v});
    std::push_heap(heap.begin(), heap.end(), later_first);
  }
  int32_t pop() {
    for (;;) {
      std::pop_heap(heap.begin(), heap.end(), later_first);
      const auto e = heap.back();
      heap.pop_back();
      if (!(*dead)[e.second] && (*deg)[e.second] == e.first) return e.second;
    }
  }
};
}  // namespace

// Exact minimum degree on a dense bitset (fast for n up to ~5e4: one word op per 64 vertices).
// Fills later[v] (v's not-yet-eliminated neighbours when it is eliminated) and pos[v].
int64_t eliminate_bitset(int32_t n, const std::vector<std::pair<int32_t, int32_t>>& edges,
                         std::vector<std::vector<int32_t>>& later, std::vector<int32_t>& pos) {
  const int64_t W = (n + 63) / 64;
  std::vector<uint64_t> adj((size_t)n * W, 0ull);
  auto row = [&](int v) { return adj.data() + (size_t)v * W; };
  int64_t e0 = 0;
  for (auto& e : edges) {
    int i = e.first, j = e.second;
    if (i == j) continue;
    uint64_t* ri = row(i);
    if (!(ri[j >> 6] >> (j & 63) & 1ull)) {
      ri[j >> 6] |= 1ull << (j & 63);
      row(j)[i >> 6] |= 1ull << (i & 63);
      ++e0;
    }
  }
  std::vector<uint64_t> alive(W, ~0ull);
  if (n % 64) alive[W - 1] = (1ull << (n % 64)) - 1ull;
  std::vector<int32_t> deg(n);
  std::vector<char> dead(n, 0);
  MinDegQueue queue;
  queue.deg = &deg;
  queue.dead = &dead;
  queue.heap.reserve((size_t)4 * n);
  for (int v = 0; v < n; ++v) {
    int d = 0;
    const uint64_t* r = row(v);
    for (int64_t w = 0; w < W; ++w) d += popc(r[w]);
    deg[v] = d;
    queue.push(d, v);
  }
  std::vector<uint64_t> nbmask(W, 0ull);
  std::vector<int32_t> nzw;  // words of nbmask with bits set
  for (int step = 0; step < n; ++step) {
    const int v = queue.pop();
    dead[v] = 1;
    pos[v] = step;
    alive[v >> 6] &= ~(1ull << (v & 63));
    const uint64_t* rv = row(v);
    std::vector<int32_t>& nb = later[v];
    nzw.clear();
    for (int64_t w = 0; w < W; ++w) {
      uint64_t m = rv[w] & alive[w];
      if (!m) continue;
      nbmask[w] = m;
      nzw.push_back((int32_t)w);
      while (m) {
        int b = __builtin_ctzll(m);
        nb.push_back((int32_t)(w * 64 + b));
        m &= m - 1;
      }
    }
    // eliminate v: its remaining neighbourhood becomes a clique (fill edges).  Only the words of
    // N(v) change in a neighbour's row, so its alive degree is updated from them: -1 for v, + the
    // members of N(v) \ {u} it was not adjacent to
    for (int u : nb) {
      uint64_t* ru = row(u);
      int added = 0;
      for (int32_t w : nzw) {
        uint64_t fresh = nbmask[w] & ~ru[w];
        if (w == (u >> 6)) fresh &= ~(1ull << (u & 63));
        added += popc(fresh);
        ru[w] |= fresh;
      }
      const int d = deg[u] - 1 + added;
      if (d != deg[u]) {
        deg[u] = d;
        queue.push(d, u);
      }
    }
    for (int32_t w : nzw) nbmask[w] = 0ull;
  }
  return e0;
}

// The same elimination on sorted adjacency lists of the alive vertices (O(n + fill) memory; no
// order limit): eliminating v replaces adj(u) by (adj(u) U N(v)) \ {u, v} for every u in N(v).
int64_t eliminate_sparse(int32_t n, const std::vector<std::pair<int32_t, int32_t>>& edges,
                         std::vector<std::vector<int32_t>>& later, std::vector<int32_t>& pos) {
  std::vector<std::vector<int32_t>> adj(n);
  for (auto& e : edges) {
    if (e.first == e.second) continue;
    adj[e.first].push_back(e.second);
    adj[e.second].push_back(e.first);
  }
  int64_t e0 = 0;
  for (int v = 0; v < n; ++v) {
    std::sort(adj[v].begin(), adj[v].end());
    adj[v].erase(std::unique(adj[v].begin(), adj[v].end()), adj[v].end());
    e0 += (int64_t)adj[v].size();
  }
  e0 /= 2;
  std::vector<int32_t> deg(n);
  std::vector<char> dead(n, 0);
  MinDegQueue queue;
  queue.deg = &deg;
  queue.dead = &dead;
  queue.heap.reserve((size_t)4 * n);
  for (int v = 0; v < n; ++v) {
    deg[v] = (int32_t)adj[v].size();
    queue.push(deg[v], v);
  }
  std::vector<int32_t> merged;
  for (int step = 0; step < n; ++step) {
    const int v = queue.pop();
    dead[v] = 1;
    pos[v] = step;
    std::vector<int32_t>& nb = later[v];
    nb = std::move(adj[v]);  // alive neighbours only (eliminated vertices are removed below)
    adj[v].clear();
    for (int u : nb) {
      const std::vector<int32_t>& au = adj[u];
      merged.clear();
      size_t a = 0, b = 0;
      while (a < au.size() || b < nb.size()) {
        int32_t x;
        if (b == nb.size() || (a < au.size() && au[a] < nb[b]))
          x = au[a++];
        else if (a == au.size() || nb[b] < au[a])
          x = nb[b++];
        else {
          x = au[a++];
          ++b;
        }
        if (x != u && x != v) merged.push_back(x);
      }
      adj[u].swap(merged);
      if ((int32_t)adj[u].size() != deg[u]) {
        deg[u] = (int32_t)adj[u].size();
        queue.push(deg[u], u);
      }
    }
  }
  return e0;
}

ChordalResult chordal_analysis(int32_t n, const std::vector<std::pair<int32_t, int32_t>>& edges) {
  // bitset for n <= 46340 (n^2 / 8 bytes), sorted lists beyond (or SDP_CHORDAL_SPARSE=1);
  // both give the same elimination (exact minimum degree, lowest index on ties)
  const char* sp = getenv("SDP_CHORDAL_SPARSE");
  const bool sparse = n > 46340 || (sp && *sp == '1');
  std::vector<std::vector<int32_t>> later(n);
  std::vector<int32_t> pos(n);
  const auto tq0 = std::chrono::steady_clock::now();
  const int64_t e0 = sparse ? eliminate_sparse(n, edges, later, pos) : eliminate_bitset(n, edges, later, pos);
  if (getenv("SDP_SETUP_TRACE"))
    fprintf(stderr, "[setup]   minimum-degree elimination %9.2f ms\n",
            std::chrono::duration<double>(std::chrono::steady_clock::now() - tq0).count() * 1e3);
  ChordalResult cr;
  cr.order.resize(n);
  for (int v = 0; v < n; ++v) cr.order[pos[v]] = v;
  cr.later_ptr.assign(n + 1, 0);
  for (int v = 0; v < n; ++v) cr.later_ptr[v + 1] = cr.later_ptr[v] + (int64_t)later[v].size();
  cr.later_idx.reserve(cr.later_ptr[n]);
  for (int v = 0; v < n; ++v) cr.later_idx.insert(cr.later_idx.end(), later[v].begin(), later[v].end());
  // elimination tree: parent(v) = first-eliminated later neighbour
  std::vector<int32_t> parent(n, -1);
  for (int v = 0; v < n; ++v) {
    int best = -1;
    for (int u : later[v])
      if (best < 0 || pos[u] < pos[best]) best = u;
    parent[v] = best;
  }
  std::vector<char> maximal(n, 1);
  for (int w = 0; w < n; ++w) {
    int v = parent[w];
    if (v >= 0 && later[w].size() == later[v].size() + 1) maximal[v] = 0;
  }
  for (int v = 0; v < n; ++v) {
    if (!maximal[v]) continue;
    std::vector<int32_t> K = later[v];
    K.push_back(v);
    std::sort(K.begin(), K.end());
    cr.cliques.push_back(std::move(K));
  }
  std::sort(cr.cliques.begin(), cr.cliques.end());
  // extended pattern E' (+ diagonal) in canonical order: every edge of the filled graph joins a
  // vertex to one of its later neighbours
  std::vector<int64_t> cnt(n + 1, 0);
  for (int v = 0; v < n; ++v)
    for (int u : later[v]) cnt[std::max(u, v) + 1]++;
  for (int j = 0; j < n; ++j) cnt[j + 1] += cnt[j] + 1;  // + the diagonal entry of each column
  const int64_t tot = cnt[n];
  cr.coord_row.assign(tot, 0);
  cr.coord_col.assign(tot, 0);
  std::vector<int64_t> fillp(cnt.begin(), cnt.end() - 1);
  for (int v = 0; v < n; ++v)
    for (int u : later[v]) {
      const int j = std::max(u, v);
      cr.coord_row[fillp[j]++] = std::min(u, v);
    }
  cr.col_ptr.assign(n + 1, 0);
  for (int j = 0; j < n; ++j) {
    std::sort(cr.coord_row.begin() + cnt[j], cr.coord_row.begin() + fillp[j]);
    cr.coord_row[fillp[j]] = j;  // diagonal last (rows < j first)
    for (int64_t e = cnt[j]; e <= fillp[j]; ++e) cr.coord_col[e] = j;
    cr.col_ptr[j + 1] = cnt[j + 1];
  }
  cr.fill_edges = (tot - n) - e0;
  return cr;
}

int64_t coord_index(const ChordalResult& cr, int32_t i, int32_t j) {
  if (i > j) std::swap(i, j);
  const int32_t* b = cr.coord_row.data() + cr.col_ptr[j];
  const int32_t* e = cr.coord_row.data() + cr.col_ptr[j + 1];
  const int32_t* p = std::lower_bound(b, e, i);
  if (p == e || *p != i) return -1;
  return (int64_t)(p - cr.coord_row.data());
}

}  // namespace sdp
