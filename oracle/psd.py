"""ORACLE (test infrastructure only): projection onto the PSD cone.

P:244-253 (E:XkUpdate) and P:403-410 (E:zkUpdate): P_k is the projection onto
S_+^{|C_k|}, i.e. the Frobenius-nearest PSD matrix, computed from an eigenvalue
decomposition X = V diag(w) V^T as V diag(max(w, 0)) V^T.

The eigendecomposition is the library routine numpy.linalg.eigh (LAPACK
syevd); it is one step of the plain definition, not a re-implementation.
Reading G15: eigenvalues are clipped at exactly 0.
"""
from __future__ import annotations

import numpy as np

from .decompose import smat_dense, svec_dense, packed_upper_local


def project_psd(X: np.ndarray) -> np.ndarray:
    """argmin_{P >= 0} ||P - X||_F for symmetric X."""
    X = 0.5 * (X + X.T)
    w, V = np.linalg.eigh(X)
    P = (V * np.maximum(w, 0.0)) @ V.T
    return 0.5 * (P + P.T)


def project_psd_svec(v: np.ndarray, k: int) -> np.ndarray:
    """E:XkUpdate in vector form: vec{ P_k [ vec^-1(v) ] } with svec coordinates."""
    return svec_dense(project_psd(smat_dense(v, k)))


def unpack_upper(vals: np.ndarray, k: int) -> np.ndarray:
    """Unscaled packed-upper column-major values -> dense symmetric matrix."""
    r, c = packed_upper_local(k)
    M = np.zeros((k, k))
    M[r, c] = vals
    M[c, r] = vals
    return M


def pack_upper(M: np.ndarray) -> np.ndarray:
    r, c = packed_upper_local(M.shape[0])
    return M[r, c]


def project_psd_packed_batch(ks, vals: np.ndarray) -> np.ndarray:
    """Batch P_+ over matrices given as unscaled packed-upper column-major
    values, concatenated in order (the boundary layout of sdp_project_psd_batch)."""
    out = np.empty_like(vals)
    off = 0
    for k in np.asarray(ks).tolist():
        s = k * (k + 1) // 2
        out[off:off + s] = pack_upper(project_psd(unpack_upper(vals[off:off + s], k)))
        off += s
    return out
