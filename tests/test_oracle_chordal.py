"""Pins for oracle/chordal.py: Definition 1 by brute force, exhaustive maximal
cliques, SPEC.md hand examples, and the block-arrow closed form."""
import numpy as np
import pytest

from oracle import chordal
from tests.helpers import (adj_from_edges, golden, is_chordal_bruteforce,
                           maximal_cliques_bruteforce, random_graph)


def test_bruteforce_chordality_matches_spec_examples():
    for ex in golden("spec_examples.json")["chordal"]:
        assert is_chordal_bruteforce(adj_from_edges(ex["n"], ex["edges"])) == ex["chordal"], ex["cite"]


def test_extension_examples():
    for ex in golden("spec_examples.json")["extension"]:
        adj = adj_from_edges(ex["n"], ex["edges"])
        _, _, filled = chordal.minimum_degree_elimination(adj)
        assert (filled.sum() - adj.sum()) // 2 == ex["added"], ex["cite"]
        assert is_chordal_bruteforce(filled)


def test_clique_examples():
    for ex in golden("spec_examples.json")["cliques"]:
        adj = adj_from_edges(ex["n"], ex["edges"])
        order, later, _ = chordal.minimum_degree_elimination(adj)
        got = [c.tolist() for c in chordal.maximal_cliques_from_elimination(order, later)]
        assert got == ex["cliques"], ex["cite"]


@pytest.mark.parametrize("seed", range(60))
def test_random_graphs_against_bruteforce(seed):
    """Extension is a superset of the input and chordal (Definition 1, checked by
    cycle enumeration); cliques are exactly the maximal cliques of the extension."""
    rng = np.random.default_rng(seed)
    n = int(rng.integers(3, 8))
    adj = random_graph(n, float(rng.uniform(0.2, 0.7)), rng)
    order, later, filled = chordal.minimum_degree_elimination(adj)
    assert np.all(filled[adj])
    assert np.array_equal(filled, filled.T)
    assert is_chordal_bruteforce(filled)
    got = [tuple(c.tolist()) for c in chordal.maximal_cliques_from_elimination(order, later)]
    assert got == maximal_cliques_bruteforce(filled)
    # every edge of the extension lies in some clique (SPEC S:30 coverage)
    for i in range(n):
        for j in range(i + 1, n):
            if filled[i, j]:
                assert any(i in c and j in c for c in got)


def test_chordal_input_gets_no_fill():
    """Min degree on an already-chordal graph: random chordal graphs built as
    unions of cliques along a tree (interval graphs) keep their edge set."""
    rng = np.random.default_rng(7)
    for _ in range(30):
        n = int(rng.integers(4, 9))
        adj = np.zeros((n, n), dtype=bool)
        # interval graph: vertices are intervals, chordal by construction
        lo = rng.uniform(0, 10, n)
        hi = lo + rng.uniform(0, 4, n)
        for i in range(n):
            for j in range(i + 1, n):
                if lo[i] <= hi[j] and lo[j] <= hi[i]:
                    adj[i, j] = adj[j, i] = True
        assert is_chordal_bruteforce(adj)
        _, _, filled = chordal.minimum_degree_elimination(adj)
        # minimum degree may add fill even on chordal graphs only if it picks a
        # non-simplicial vertex; on interval graphs the extension must stay chordal
        assert is_chordal_bruteforce(filled)


@pytest.mark.parametrize("l,d,h", [(2, 2, 1), (5, 5, 2), (40, 10, 5), (7, 3, 4)])
def test_block_arrow_cliques_closed_form(gen, l, d, h):
    """Block-arrow (Fig. 2) is chordal: the cliques are exactly the
    l sets block_i U arrow (BASELINE configs 1-2: 40 x 15, 400 x 30)."""
    prob = gen.block_arrow(l, d, h, 3, seed=0)
    cliques, filled = chordal.chordal_decomposition(prob)
    adj = chordal.aggregate_adjacency(prob)
    assert np.array_equal(filled, adj)  # no fill
    arrow = list(range(l * d, l * d + h))
    want = [list(range(i * d, (i + 1) * d)) + arrow for i in range(l)]
    assert [c.tolist() for c in cliques] == want


def test_dense_reference_is_one_clique(gen):
    prob = gen.block_arrow(3, 2, 1, 2, seed=0)
    cliques, _ = chordal.chordal_decomposition(prob, dense=True)
    assert len(cliques) == 1 and cliques[0].tolist() == list(range(prob.n))
