"""Pins for oracle/psd.py: SPEC hand values, the 2x2 closed form,
the variational characterisation of a Euclidean projection onto a convex cone,
the Moreau decomposition, idempotence, equivariance and zero padding."""
import math

import numpy as np
import pytest

from oracle import psd
from oracle.decompose import smat_dense, svec_dense
from tests.helpers import golden


def rand_sym(k, rng, scale=1.0):
    G = rng.standard_normal((k, k)) * scale
    return 0.5 * (G + G.T)


def test_spec_hand_values():
    for ex in golden("spec_examples.json")["project_psd"]:
        got = psd.project_psd(np.array(ex["in"], dtype=float))
        assert np.allclose(got, np.array(ex["out"], dtype=float), atol=1e-15), ex["cite"]


def test_two_by_two_closed_form():
    """P_+ of [[a,b],[b,c]] from the explicit 2x2 spectral formulas."""
    rng = np.random.default_rng(0)
    for _ in range(200):
        a, b, c = rng.standard_normal(3)
        t = math.hypot((a - c) / 2, b)
        m = (a + c) / 2
        l1, l2 = m + t, m - t
        if t == 0:
            want = np.eye(2) * max(m, 0.0)
        else:
            # spectral projector onto the l1 eigenvector
            P1 = (np.array([[a, b], [b, c]]) - l2 * np.eye(2)) / (l1 - l2)
            P2 = np.eye(2) - P1
            want = max(l1, 0.0) * P1 + max(l2, 0.0) * P2
        got = psd.project_psd(np.array([[a, b], [b, c]]))
        assert np.allclose(got, want, atol=1e-13)


@pytest.mark.parametrize("k", [1, 2, 3, 7, 16, 33])
def test_projection_characterisation(k):
    """For a closed convex cone K, P = P_K(X) iff P in K, X - P in -K* = -K
    (self-dual) and <X - P, P> = 0.  Also <X - P, Y - P> <= 0 for every Y in K."""
    rng = np.random.default_rng(k)
    for _ in range(20):
        X = rand_sym(k, rng)
        P = psd.project_psd(X)
        R = X - P
        nrm = np.linalg.norm(X)
        assert np.linalg.eigvalsh(P).min() >= -1e-13 * nrm
        assert np.linalg.eigvalsh(R).max() <= 1e-13 * nrm
        assert abs(np.sum(R * P)) <= 1e-12 * nrm ** 2
        for _ in range(5):
            G = rng.standard_normal((k, k))
            Y = G @ G.T
            assert np.sum(R * (Y - P)) <= 1e-11 * nrm * (nrm + np.linalg.norm(Y))


@pytest.mark.parametrize("k", [1, 4, 12, 30])
def test_moreau_idempotence_equivariance(k):
    rng = np.random.default_rng(100 + k)
    for _ in range(10):
        X = rand_sym(k, rng, 3.0)
        P = psd.project_psd(X)
        Pm = psd.project_psd(-X)
        nrm = np.linalg.norm(X)
        # Moreau: X = P_+(X) - P_+(-X), <P_+(X), P_+(-X)> = 0
        assert np.allclose(X, P - Pm, atol=1e-13 * nrm)
        assert abs(np.sum(P * Pm)) <= 1e-12 * nrm ** 2
        # idempotence
        assert np.allclose(psd.project_psd(P), P, atol=1e-13 * nrm)
        # orthogonal equivariance P(Q X Q^T) = Q P(X) Q^T
        Q, _ = np.linalg.qr(rng.standard_normal((k, k)))
        assert np.allclose(psd.project_psd(Q @ X @ Q.T), Q @ P @ Q.T, atol=1e-12 * nrm)
        # zero padding P(diag(X, 0)) = diag(P(X), 0)
        Z = np.zeros((k + 3, k + 3))
        Z[:k, :k] = X
        assert np.allclose(psd.project_psd(Z)[:k, :k], P, atol=1e-13 * nrm)
        assert np.allclose(psd.project_psd(Z)[k:, :], 0.0, atol=1e-13 * nrm)
        # non-expansive
        Y = rand_sym(k, rng, 3.0)
        assert np.linalg.norm(psd.project_psd(Y) - P) <= np.linalg.norm(Y - X) * (1 + 1e-12)


def test_psd_and_nsd_inputs():
    rng = np.random.default_rng(5)
    G = rng.standard_normal((9, 9))
    S = G @ G.T
    assert np.allclose(psd.project_psd(S), S, atol=1e-12 * np.linalg.norm(S))
    assert np.allclose(psd.project_psd(-S), 0.0, atol=1e-12 * np.linalg.norm(S))


def test_svec_hand_values_and_isometry():
    ex = golden("spec_examples.json")["svec"]
    assert np.allclose(svec_dense(np.array(ex[0]["matrix"], float)), ex[0]["svec"], atol=1e-15)
    assert np.allclose(svec_dense(np.array(ex[1]["matrix"], float)), ex[1]["svec"])
    A = np.array(ex[2]["A"], float)
    B = np.array(ex[2]["B"], float)
    assert abs(svec_dense(A) @ svec_dense(B) - ex[2]["inner"]) < 1e-14
    rng = np.random.default_rng(1)
    for k in (1, 2, 5, 9):
        X = rand_sym(k, rng)
        Y = rand_sym(k, rng)
        assert abs(svec_dense(X) @ svec_dense(Y) - np.sum(X * Y)) < 1e-12
        assert np.array_equal(smat_dense(svec_dense(X), k), X) or np.allclose(smat_dense(svec_dense(X), k), X, atol=1e-15)


def test_packed_batch_layout():
    rng = np.random.default_rng(3)
    ks = [3, 1, 5]
    mats = [rand_sym(k, rng) for k in ks]
    vals = np.concatenate([psd.pack_upper(M) for M in mats])
    out = psd.project_psd_packed_batch(ks, vals)
    off = 0
    for k, M in zip(ks, mats):
        s = k * (k + 1) // 2
        assert np.allclose(psd.unpack_upper(out[off:off + s], k), psd.project_psd(M))
        off += s
