"""CPU checks of the sparse Cholesky of S = A D^-1 A^T (the factorisation is
computed once and cached): the library's host-only entry point sdp_schur_inverse_host
(minimum-degree order from the chordal analysis, left-looking factorisation, G = L^-1 along
elimination-tree paths, S^-1 = G^T G) against numpy's inverse, on sparse SPD matrices with
the structure of distance-constraint SDPs, a dense one, and a singular one."""
import numpy as np
import pytest
import scipy.sparse as sp

L = pytest.importorskip("paper_1609_06068_b200._lib", reason="libchordal_sdp.so not built")


def geometric_spd(n, r, seed, shift=0.1):
    from scipy.spatial import cKDTree
    rng = np.random.default_rng(seed)
    P = rng.random((n, 2))
    E = np.array(sorted(cKDTree(P).query_pairs(r)))
    W = sp.coo_matrix((rng.random(len(E)), (E[:, 0], E[:, 1])), shape=(n, n))
    W = W + W.T
    return (sp.diags(np.asarray(W.sum(1)).ravel()) - W + shift * sp.eye(n)).tocsr()


@pytest.mark.parametrize("n,r,seed", [(50, 0.3, 0), (300, 0.1, 1), (700, 0.06, 2)])
def test_sparse_inverse_matches_numpy(n, r, seed):
    S = geometric_spd(n, r, seed)
    Sinv, nnz = L.schur_inverse_host(S)
    want = np.linalg.inv(S.toarray())
    assert np.abs(Sinv - want).max() <= 1e-11 * np.abs(want).max()
    assert np.allclose(Sinv, Sinv.T, rtol=0, atol=1e-14 * np.abs(want).max())
    assert n <= nnz <= n * (n + 1) // 2


def test_schur_of_distance_constraints_is_sparse(gen):
    """S of the sensor-network SDP (constraints share a vertex => S_ab != 0): the factor stays
    sparse under minimum degree and the inverse is exact."""
    from oracle import decompose as dc
    prob = gen.sensor_network(300, 0.09, seed=3)
    dec = dc.decompose(prob, factor=False)
    A = sp.csr_matrix(dec.A)
    S = (A @ sp.diags(1.0 / dec.D) @ A.T).tocsr()
    Sinv, nnz = L.schur_inverse_host(S, force_sparse=False)
    m = S.shape[0]
    assert nnz < m * m / 8
    want = np.linalg.inv(S.toarray())
    assert np.abs(Sinv - want).max() <= 1e-10 * np.abs(want).max()


def test_dense_and_singular():
    rng = np.random.default_rng(4)
    G = rng.standard_normal((120, 120))
    D = G @ G.T / 120 + np.eye(120)
    with pytest.raises(L.SdpError, match="STATE"):
        L.schur_inverse_host(D, force_sparse=False)   # factor dense: the library keeps the dense path
    Sinv, nnz = L.schur_inverse_host(D, force_sparse=True)
    assert nnz == 120 * 121 // 2
    assert np.abs(Sinv @ D - np.eye(120)).max() <= 1e-12
    S = geometric_spd(100, 0.2, 5, shift=0.0)          # a graph Laplacian: singular
    with pytest.raises(L.SdpError, match="RANK_DEFICIENT"):
        L.schur_inverse_host(S)
