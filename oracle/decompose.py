"""ORACLE (test infrastructure only): vectorisation, entry selectors, KKT system.

PAPER.md passages followed:
  P:165-176  vectorised data c, A, variables x, x_k and H_k = E_k (x) E_k,
             "entry-selector matrices ... whose rows are orthonormal"
  P:222-233  D = sum_k H_k^T H_k (diagonal); KKT system E:OptCondMinYPrimal,
             solved "by block elimination" with a factorisation cached once
  P:355-360, P:401  the dual KKT system E:OptCondMinYDual has the same matrix

Readings:
  G1   vectors live on the extended-pattern support in svec form (off-diagonal
       entries times sqrt(2)); this is an isometry of the paper's vec for
       symmetric matrices, keeps H_k a 0/1 selector with orthonormal rows and
       makes D positive definite.
  G2   "A_0 ... A_m" means A_1 ... A_m.
  Coordinate order: upper-triangle entries (i <= j) sorted by column, then
       row ("column-major upper").  Inside a clique the local svec order is the
       same rule applied to local indices.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import scipy.linalg
import scipy.sparse

from .chordal import chordal_decomposition

SQRT2 = math.sqrt(2.0)


class RankDeficient(Exception):
    """S = A D^-1 A^T is not positive definite."""


class InvalidProblem(Exception):
    pass


def packed_upper_local(k: int):
    """Local (row, col) of the packed upper column-major order of a k x k block."""
    rows, cols = [], []
    for j in range(k):
        for i in range(j + 1):
            rows.append(i)
            cols.append(j)
    return np.array(rows, dtype=np.int64), np.array(cols, dtype=np.int64)


def svec_dense(M: np.ndarray) -> np.ndarray:
    """svec of a dense symmetric matrix in packed upper column-major order."""
    r, c = packed_upper_local(M.shape[0])
    return np.where(r == c, 1.0, SQRT2) * M[r, c]


def smat_dense(v: np.ndarray, k: int) -> np.ndarray:
    """Inverse of svec_dense (vec^-1)."""
    r, c = packed_upper_local(k)
    vals = np.where(r == c, 1.0, 1.0 / SQRT2) * v
    M = np.zeros((k, k))
    M[r, c] = vals
    M[c, r] = vals
    return M


@dataclass
class Decomposition:
    n: int
    m: int
    cliques: list           # list of sorted int arrays
    coord_row: np.ndarray   # row i of coordinate t (i <= j)
    coord_col: np.ndarray   # col j of coordinate t
    H: list                 # H[k][a] = global coordinate of local svec entry a
    offsets: np.ndarray     # clique k occupies [offsets[k], offsets[k+1]) of stacked vectors
    D: np.ndarray           # D = sum_k H_k^T H_k (diagonal entries)
    c: np.ndarray           # svec(C) on the pattern
    A: object               # m x N, dense ndarray or scipy CSR (rows = svec(A_i))
    b: np.ndarray
    L: np.ndarray = None    # Cholesky factor of S = A D^-1 A^T (cached)

    @property
    def N(self):
        return self.coord_row.shape[0]

    @property
    def p(self):
        return len(self.cliques)

    @property
    def sizes(self):
        return np.array([len(c) for c in self.cliques], dtype=np.int64)

    # --- entry selectors ------------------------------------
    def gather(self, x: np.ndarray) -> np.ndarray:
        """Stacked H_k x for k = 1..p."""
        return np.concatenate([x[h] for h in self.H]) if self.H else np.zeros(0)

    def scatter(self, w: np.ndarray) -> np.ndarray:
        """sum_k H_k^T w_k for a stacked clique vector w."""
        out = np.zeros(self.N)
        for k, h in enumerate(self.H):
            np.add.at(out, h, w[self.offsets[k]:self.offsets[k + 1]])
        return out

    def block(self, w: np.ndarray, k: int) -> np.ndarray:
        return w[self.offsets[k]:self.offsets[k + 1]]

    # --- KKT --------------------------------------------------
    def A_mul(self, v):
        return self.A @ v

    def AT_mul(self, y):
        return self.A.T @ y

    def factor(self):
        """S = A D^-1 A^T and its Cholesky factor, computed once."""
        if scipy.sparse.issparse(self.A):
            S = (self.A @ scipy.sparse.diags(1.0 / self.D) @ self.A.T).toarray()
        else:
            S = (self.A / self.D) @ self.A.T
        S = 0.5 * (S + S.T)
        try:
            self.L = np.linalg.cholesky(S)
        except np.linalg.LinAlgError as e:
            raise RankDeficient(str(e))
        if not np.all(np.isfinite(self.L)):
            raise RankDeficient("non-finite Cholesky factor")
        return S

    def solve_kkt(self, r1: np.ndarray, r2: np.ndarray):
        """Solve [D A^T; A 0][x; y] = [r1; r2] by block elimination:
        y = S^-1 (A D^-1 r1 - r2), x = D^-1 (r1 - A^T y)."""
        u = self.A_mul(r1 / self.D) - r2
        t = scipy.linalg.solve_triangular(self.L, u, lower=True)
        y = scipy.linalg.solve_triangular(self.L.T, t, lower=False)
        x = (r1 - self.AT_mul(y)) / self.D
        return x, y

    def kkt_matrix_dense(self):
        """The full (N+m) x (N+m) KKT coefficient matrix (tiny problems only)."""
        A = self.A.toarray() if scipy.sparse.issparse(self.A) else self.A
        N, m = self.N, self.m
        K = np.zeros((N + m, N + m))
        K[:N, :N] = np.diag(self.D)
        K[:N, N:] = A.T
        K[N:, :N] = A
        return K

    # --- canonical outputs --------------------------------------------------
    def unsvec_pattern(self, x: np.ndarray) -> np.ndarray:
        """Unscaled matrix entries X_ij on the pattern coordinates."""
        return np.where(self.coord_row == self.coord_col, 1.0, 1.0 / SQRT2) * x

    def dense_from_pattern(self, x: np.ndarray) -> np.ndarray:
        """Dense symmetric matrix with the pattern entries of x (0 elsewhere)."""
        X = np.zeros((self.n, self.n))
        v = self.unsvec_pattern(x)
        X[self.coord_row, self.coord_col] = v
        X[self.coord_col, self.coord_row] = v
        return X


def decompose(prob, dense: bool = False, factor: bool = True) -> Decomposition:
    """Build the decomposed problem E:PrimalVectorForm from data."""
    n, m = prob.n, prob.m
    cliques, filled = chordal_decomposition(prob, dense=dense)
    # extended pattern E' (plus diagonal), column-major upper order
    up = np.triu(filled) | np.eye(n, dtype=bool)
    cols, rows = np.nonzero(up.T)          # row-major scan of up.T = column-major of up
    coord_row = rows.astype(np.int64)
    coord_col = cols.astype(np.int64)
    N = coord_row.shape[0]
    key = coord_col * n + coord_row
    assert np.all(np.diff(key) > 0)

    def index_of(i, j):
        i = np.asarray(i, dtype=np.int64)
        j = np.asarray(j, dtype=np.int64)
        lo, hi = np.minimum(i, j), np.maximum(i, j)
        k = hi * n + lo
        t = np.searchsorted(key, k)
        if np.any(t >= N) or np.any(key[np.minimum(t, N - 1)] != k):
            raise InvalidProblem("entry outside the extended pattern")
        return t

    H = []
    offsets = [0]
    for C in cliques:
        lr, lc = packed_upper_local(len(C))
        H.append(index_of(C[lr], C[lc]))
        offsets.append(offsets[-1] + len(lr))
    offsets = np.array(offsets, dtype=np.int64)
    D = np.zeros(N)
    for h in H:
        np.add.at(D, h, 1.0)
    if np.any(D <= 0):
        raise InvalidProblem("a pattern coordinate is covered by no clique")

    def scale(i, j):
        return np.where(np.asarray(i) == np.asarray(j), 1.0, SQRT2)

    for arr in (prob.c_row, prob.c_col):
        if np.any(np.asarray(arr) < 0) or np.any(np.asarray(arr) >= n):
            raise InvalidProblem("C index out of range")
    if np.any(np.asarray(prob.c_row) > np.asarray(prob.c_col)):
        raise InvalidProblem("C entry below the diagonal")
    ct = index_of(prob.c_row, prob.c_col)
    if np.unique(ct).shape[0] != ct.shape[0]:
        raise InvalidProblem("duplicate C entry")
    c = np.zeros(N)
    c[ct] = scale(prob.c_row, prob.c_col) * np.asarray(prob.c_val, dtype=np.float64)

    if prob.a_fmt == "dense":
        at = index_of(prob.a_row, prob.a_col)
        if np.unique(at).shape[0] != at.shape[0]:
            raise InvalidProblem("duplicate A pattern entry")
        A = np.zeros((m, N))
        A[:, at] = np.asarray(prob.a_val) * scale(prob.a_row, prob.a_col)[None, :]
    else:
        if np.any(np.asarray(prob.a_row) > np.asarray(prob.a_col)):
            raise InvalidProblem("A entry below the diagonal")
        at = index_of(prob.a_row, prob.a_col)
        con = np.asarray(prob.a_con, dtype=np.int64)
        if np.any(con < 0) or np.any(con >= m):
            raise InvalidProblem("constraint index out of range")
        pair = con * N + at
        if np.unique(pair).shape[0] != pair.shape[0]:
            raise InvalidProblem("duplicate A entry")
        vals = np.asarray(prob.a_val, dtype=np.float64) * scale(prob.a_row, prob.a_col)
        A = scipy.sparse.csr_matrix((vals, (con, at)), shape=(m, N))
    dec = Decomposition(n=n, m=m, cliques=cliques, coord_row=coord_row, coord_col=coord_col,
                        H=H, offsets=offsets, D=D, c=c, A=A,
                        b=np.asarray(prob.b, dtype=np.float64).copy())
    if factor:
        dec.factor()
    return dec
