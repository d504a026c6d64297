"""Pins of oracle.completion (Theorem 1) by implementation-independent
properties: agreement on the pattern, PSD-ness, and the maximum-determinant characterisation."""
import numpy as np

from oracle import chordal
from oracle import completion


def _chordal_instance(n, p, seed):
    rng = np.random.default_rng(seed)
    A = np.triu(rng.random((n, n)) < p, 1)
    adj = A | A.T
    order, later, filled = chordal.minimum_degree_elimination(adj)
    known = filled | np.eye(n, dtype=bool)
    return rng, order, later, known


def test_completion_of_a_definite_partial_matrix_is_the_max_det_one():
    """A partial matrix cut from a random positive definite matrix: the completion agrees on the
    pattern, is positive definite, and its inverse is zero off the pattern (the first-order
    condition of max log det over the completions), which pins every filled entry."""
    for seed in range(4):
        rng, order, later, known = _chordal_instance(14, 0.25, seed)
        G = rng.standard_normal((14, 14))
        S = G @ G.T + 14 * np.eye(14)
        Y = completion.complete_psd(S, known, order, later)
        assert np.allclose(Y[known], S[known], rtol=0, atol=1e-12)
        assert np.linalg.eigvalsh(Y).min() > 0
        Yi = np.linalg.inv(Y)
        assert np.abs(Yi[~known]).max() <= 1e-9 * np.abs(Yi).max()


def test_completion_of_a_low_rank_partial_matrix():
    """Blocks of a rank-2 PSD matrix on a chain (singular 2x2 clique blocks when the chain is cut
    from a rank-1 part): the completion is PSD and exact on the pattern."""
    rng = np.random.default_rng(7)
    n = 9
    adj = np.zeros((n, n), dtype=bool)
    for i in range(n - 1):
        adj[i, i + 1] = adj[i + 1, i] = True
    order, later, filled = chordal.minimum_degree_elimination(adj)
    known = filled | np.eye(n, dtype=bool)
    B = rng.standard_normal((n, 2))
    S = B @ B.T
    Y = completion.complete_psd(S, known, order, later)
    assert np.allclose(Y[known], S[known], atol=1e-12)
    assert np.linalg.eigvalsh(Y).min() >= -1e-10 * np.linalg.norm(S)
    # rank-1: every 2x2 block singular (pseudo-inverse path); the completion is then the matrix itself
    b = rng.standard_normal(n)
    S1 = np.outer(b, b)
    Y1 = completion.complete_psd(S1, known, order, later)
    assert np.allclose(Y1, S1, atol=1e-9 * np.abs(S1).max())


def test_two_block_closed_form():
    """Two cliques {0,1}, {1,2} sharing vertex 1: the only unknown entry is
    X02 = X01 X11^{-1} X12 (the Schur-complement / max-det value)."""
    X = np.array([[2.0, 0.6, 0.0], [0.6, 1.5, -0.4], [0.0, -0.4, 3.0]])
    adj = np.array([[0, 1, 0], [1, 0, 1], [0, 1, 0]], dtype=bool)
    order, later, filled = chordal.minimum_degree_elimination(adj)
    known = filled | np.eye(3, dtype=bool)
    Y = completion.complete_psd(X, known, order, later)
    assert abs(Y[0, 2] - 0.6 * (-0.4) / 1.5) <= 1e-15
