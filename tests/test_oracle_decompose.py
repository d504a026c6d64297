"""Pins for oracle/decompose.py: selectors, D, block
elimination of the KKT system against a full dense LU solve."""
import numpy as np
import pytest
import scipy.sparse

from oracle import decompose as dc
from tests.helpers import golden


def path_problem():
    """Path 0-1-2 pattern, one constraint picking X_11."""
    import sdp_inputs as gen
    return gen.Problem(name="path", n=3, m=1,
                       c_row=np.array([0, 0, 1, 1, 2], np.int32), c_col=np.array([0, 1, 1, 2, 2], np.int32),
                       c_val=np.array([1.0, 0.1, 1.0, 0.1, 1.0]), b=np.array([1.0]), a_fmt="coo",
                       a_con=np.array([0], np.int32), a_row=np.array([1], np.int32),
                       a_col=np.array([1], np.int32), a_val=np.array([1.0]))


def test_path_D_and_S():
    dec = dc.decompose(path_problem())
    ex = golden("spec_examples.json")
    assert [c.tolist() for c in dec.cliques] == [[0, 1], [1, 2]]
    assert dec.D.tolist() == ex["D"][0]["D"]
    S = dec.factor()
    assert np.allclose(S, ex["kkt"][0]["S"])


@pytest.mark.parametrize("seed", range(4))
def test_selectors(gen, seed):
    prob = gen.block_arrow(3, 3, 2, 4, seed)
    dec = dc.decompose(prob)
    rng = np.random.default_rng(seed)
    N, St = dec.N, int(dec.offsets[-1])
    # dense H_k from the definition x_k = vec(E_k X E_k^T) = H_k x
    Hd = np.zeros((St, N))
    for k, C in enumerate(dec.cliques):
        lr, lc = dc.packed_upper_local(len(C))
        for a, (i, j) in enumerate(zip(C[lr], C[lc])):
            t = np.flatnonzero((dec.coord_row == min(i, j)) & (dec.coord_col == max(i, j)))
            Hd[dec.offsets[k] + a, t] = 1.0
    x = rng.standard_normal(N)
    w = rng.standard_normal(St)
    assert np.allclose(dec.gather(x), Hd @ x)
    assert np.allclose(dec.scatter(w), Hd.T @ w)
    # orthonormal rows within each clique: H_k H_k^T = I
    for k in range(dec.p):
        Hk = Hd[dec.offsets[k]:dec.offsets[k + 1]]
        assert np.array_equal(Hk @ Hk.T, np.eye(Hk.shape[0]))
    # D = sum_k H_k^T H_k is diagonal with integer multiplicities
    Dm = Hd.T @ Hd
    assert np.array_equal(Dm, np.diag(dec.D))
    # svec isometry: <C, X> = c . x for X on the pattern
    X = dec.dense_from_pattern(x)
    Cm = np.zeros((prob.n, prob.n))
    Cm[prob.c_row, prob.c_col] = prob.c_val
    Cm[prob.c_col, prob.c_row] = prob.c_val
    assert abs(np.sum(Cm * X) - dec.c @ x) < 1e-10
    # <A_i, X> = (A x)_i
    for i in range(dec.m):
        Ai = np.zeros((prob.n, prob.n))
        Ai[prob.a_row, prob.a_col] = prob.a_val[i]
        Ai[prob.a_col, prob.a_row] = prob.a_val[i]
        assert abs(np.sum(Ai * X) - (dec.A @ x)[i]) < 1e-10


@pytest.mark.parametrize("seed", range(5))
def test_block_elimination_matches_dense_lu(gen, seed):
    """E:OptCondMinYPrimal solved by block elimination equals an LU solve of the
    whole (N+m) KKT matrix; both block rows hold to 1e-12."""
    rng = np.random.default_rng(seed)
    prob = gen.block_arrow(3, 3, 2, 5, seed) if seed % 2 == 0 else gen.maxcut_er(9, seed, p=0.4)
    dec = dc.decompose(prob)
    r1 = rng.standard_normal(dec.N)
    r2 = rng.standard_normal(dec.m)
    x, y = dec.solve_kkt(r1, r2)
    K = dec.kkt_matrix_dense()
    sol = np.linalg.solve(K, np.concatenate([r1, r2]))
    assert np.allclose(x, sol[:dec.N], atol=1e-11)
    assert np.allclose(y, sol[dec.N:], atol=1e-11)
    A = dec.A.toarray() if scipy.sparse.issparse(dec.A) else dec.A
    assert np.linalg.norm(dec.D * x + A.T @ y - r1) <= 1e-12 * np.linalg.norm(r1)
    assert np.linalg.norm(A @ x - r2) <= 1e-12 * max(np.linalg.norm(r2), 1)


def test_rank_deficient_raises(gen):
    prob = gen.trace_one_tridiagonal(5)
    # duplicate the constraint: A has two equal rows -> S singular
    prob.a_con = np.concatenate([prob.a_con, np.ones_like(prob.a_con)])
    prob.a_row = np.concatenate([prob.a_row, prob.a_row])
    prob.a_col = np.concatenate([prob.a_col, prob.a_col])
    prob.a_val = np.concatenate([prob.a_val, prob.a_val])
    prob.m = 2
    prob.b = np.ones(2)
    with pytest.raises(dc.RankDeficient):
        dc.decompose(prob)


def test_invalid_inputs(gen):
    prob = gen.scalar_primal()
    prob.c_row = np.array([0, 0], np.int32)
    prob.c_col = np.array([0, 0], np.int32)
    prob.c_val = np.array([1.0, 2.0])
    with pytest.raises(dc.InvalidProblem):
        dc.decompose(prob)
