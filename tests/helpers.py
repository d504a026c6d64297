"""Test-side brute-force utilities (independent of oracle/ and of the CUDA path)."""
from __future__ import annotations

import itertools
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def adj_from_edges(n, edges):
    A = np.zeros((n, n), dtype=bool)
    for i, j in edges:
        A[i, j] = A[j, i] = True
    return A


def is_chordal_bruteforce(adj: np.ndarray) -> bool:
    """Definition 1 checked literally: every simple cycle of length
    >= 4 has a chord.  Enumerates cycles by DFS; only for n <= 8."""
    n = adj.shape[0]

    def has_chord(cyc):
        L = len(cyc)
        for a in range(L):
            for b in range(a + 2, L):
                if a == 0 and b == L - 1:
                    continue
                if adj[cyc[a], cyc[b]]:
                    return True
        return False

    for start in range(n):
        # cycles whose smallest vertex is `start`
        stack = [(start, [start])]
        while stack:
            v, path = stack.pop()
            for w in range(start + 1, n):
                if not adj[v, w] or w in path:
                    continue
                stack.append((w, path + [w]))
            if len(path) >= 4 and adj[path[-1], start] and path[1] < path[-1]:
                if not has_chord(path):
                    return False
    return True


def maximal_cliques_bruteforce(adj: np.ndarray):
    """All maximal cliques by exhaustive subset enumeration (n <= 10)."""
    n = adj.shape[0]
    cliques = []
    for r in range(1, n + 1):
        for S in itertools.combinations(range(n), r):
            if all(adj[a, b] for a, b in itertools.combinations(S, 2)):
                cliques.append(frozenset(S))
    maximal = [c for c in cliques if not any(c < d for d in cliques)]
    return sorted(tuple(sorted(c)) for c in maximal)


def random_graph(n, p, rng):
    A = np.triu(rng.random((n, n)) < p, 1)
    return A | A.T


def grone_completion(X: np.ndarray, known: np.ndarray, order, later):
    """PSD completion of a partial matrix on a chordal pattern (Theorem 1).

    Vertices are added in reverse perfect-elimination order; when v is added
    its known later-neighbours alpha form a clique, and each unknown X[v,u]
    (u already placed) is set to X[v,alpha] X[alpha,alpha]^+ X[alpha,u]."""
    X = X.copy()
    done = [order[-1]]
    for v in reversed(order[:-1]):
        alpha = list(later[v])
        P = np.linalg.pinv(X[np.ix_(alpha, alpha)]) if alpha else None
        for u in done:
            if known[v, u] or u == v:
                continue
            val = X[v, alpha] @ P @ X[alpha, u] if alpha else 0.0
            X[v, u] = X[u, v] = val
        done.append(v)
    return X
