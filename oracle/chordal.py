"""ORACLE (test infrastructure only): chordal analysis of the aggregate pattern.

PAPER.md passages followed:
  P:71-72   cliques, maximal cliques
  P:75-79   Definition 1 (chordal graph) and chordal extension by heuristics
  P:83      every node has a self-loop
  P:99      E_k with the clique's vertices "sorted in the natural ordering"
  P:153     aggregate sparsity pattern of C, A_1..A_m

Readings:
  G13  the paper names no extension heuristic; we take exact minimum degree
       (ties -> lowest vertex index) and symbolic elimination: the fill edges
       are the chordal extension.
  G14  cliques are sorted ascending inside, and the list is sorted
       lexicographically (hence by smallest vertex first).
  Structural support: an entry listed in the input is present even if its
       value is 0.
"""
from __future__ import annotations

import numpy as np


def aggregate_adjacency(prob) -> np.ndarray:
    """Boolean n x n adjacency of the aggregate sparsity pattern.

    (i, j) is an edge iff entry ij is listed in C, in some A_i or in the
    optional user pattern E (the pattern "described by the graph
    G(V,E)"; attributes e_row / e_col, may be absent or None); diagonal
    self-loops are implicit and not stored here."""
    n = prob.n
    adj = np.zeros((n, n), dtype=bool)
    pairs = [(prob.c_row, prob.c_col), (prob.a_row, prob.a_col)]
    if getattr(prob, "e_row", None) is not None:
        pairs.append((prob.e_row, prob.e_col))
    for r, c in pairs:
        r = np.asarray(r, dtype=np.int64)
        c = np.asarray(c, dtype=np.int64)
        adj[r, c] = True
        adj[c, r] = True
    np.fill_diagonal(adj, False)
    return adj


def minimum_degree_elimination(adj: np.ndarray):
    """Symbolic elimination under the exact minimum-degree rule (reading G13).

    Step t: among the vertices not yet eliminated pick v with the smallest
    number of not-yet-eliminated neighbours (ties: smallest index), record its
    neighbourhood ("later neighbours"), turn that neighbourhood into a clique
    (these added edges are the fill) and delete v.

    Returns (order, later, filled) where later[v] is the sorted array of
    neighbours of v at the moment it was eliminated and filled is the
    adjacency of the chordal extension G'(V, E')."""
    n = adj.shape[0]
    g = adj.copy()
    np.fill_diagonal(g, False)
    alive = np.ones(n, dtype=bool)
    deg = g.sum(axis=1).astype(np.int64)
    big = np.iinfo(np.int64).max
    order = []
    later = [None] * n
    for _ in range(n):
        v = int(np.argmin(np.where(alive, deg, big)))  # argmin: first (lowest) index on ties
        nb = np.flatnonzero(g[v] & alive)
        later[v] = nb
        g[np.ix_(nb, nb)] = True
        g[nb, nb] = False
        alive[v] = False
        deg[nb] = (g[nb] & alive).sum(axis=1)
        order.append(v)
    return order, later, g


def maximal_cliques_from_elimination(order, later):
    """Maximal cliques of the filled (chordal) graph (Theorems 1-2).

    Candidates are K_v = {v} U later[v] (each is a clique after elimination).
    Every maximal clique of a chordal graph is one of them.  K_v is dropped
    iff K_v is a subset of some other K_u; since v is the first-eliminated
    vertex of K_v, such a u must contain v as a later neighbour, so only
    those u are checked.  Output: each clique sorted ascending, list
    sorted lexicographically (reading G14)."""
    n = len(order)
    K = [None] * n
    containing = [[] for _ in range(n)]
    for v in range(n):
        K[v] = frozenset([v, *later[v].tolist()])
        for w in later[v].tolist():
            containing[w].append(v)
    out = []
    for v in range(n):
        if not any(K[v] <= K[u] for u in containing[v]):
            out.append(tuple(sorted(K[v])))
    out.sort()
    return [np.array(c, dtype=np.int64) for c in out]


def chordal_decomposition(prob, dense: bool = False):
    """Aggregate pattern -> chordal extension -> maximal cliques.

    With dense=True the whole index set is one clique (p = 1; the
    undecomposed cone) and the pattern is complete.
    Returns (cliques, filled_adjacency)."""
    n = prob.n
    if dense:
        filled = np.ones((n, n), dtype=bool)
        np.fill_diagonal(filled, False)
        return [np.arange(n, dtype=np.int64)], filled
    adj = aggregate_adjacency(prob)
    order, later, filled = minimum_degree_elimination(adj)
    return maximal_cliques_from_elimination(order, later), filled
