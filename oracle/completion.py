"""ORACLE (test infrastructure only): PSD completion of a partial matrix on a chordal pattern.

PAPER.md passages followed:
  P:90-97   PSD-completable partial matrices S(E,?)_+
  P:104-108 Theorem 1 (Grone et al.): X in S(E,?) is PSD-completable iff every maximal-clique block is PSD
The paper proves existence only; the completion written out here is the classical clique-tree /
perfect-elimination construction (the maximum-determinant completion when the blocks are definite):
vertices are placed in reverse perfect-elimination order, and when v is placed its later neighbours
alpha (a clique of the chordal pattern) give every still unknown entry
    X[v, u] = X[v, alpha] X[alpha, alpha]^+ X[alpha, u]      (u already placed).
The pseudo-inverse is numpy's (eigenvalues with |lambda| <= rtol max|lambda| dropped).
Pinned in tests/test_oracle_completion.py by properties that hold whatever the implementation:
agreement on the pattern, PSD-ness, and the maximum-determinant characterisation (the inverse of the
completion of a definite partial matrix vanishes off the pattern).
"""
from __future__ import annotations

import numpy as np


def complete_psd(X: np.ndarray, known: np.ndarray, order, later, rtol: float = 1e-12) -> np.ndarray:
    """Completion of the partial symmetric matrix X (entries where `known`) on a chordal pattern with
    perfect elimination `order` and later-neighbour sets `later` (oracle.chordal)."""
    Y = np.array(X, dtype=np.float64, copy=True)
    Y[~known] = 0.0
    done = [order[-1]]
    for v in reversed(order[:-1]):
        alpha = list(later[v])
        if alpha:
            P = np.linalg.pinv(Y[np.ix_(alpha, alpha)], rcond=rtol, hermitian=True)
            r = Y[v, alpha] @ P
        for u in done:
            if known[v, u] or u == v:
                continue
            val = float(r @ Y[alpha, u]) if alpha else 0.0
            Y[v, u] = Y[u, v] = val
        done.append(v)
    return Y
