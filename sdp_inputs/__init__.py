"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the method (no chordal analysis, no svec
scaling, no projections, no KKT algebra).  It only draws random numbers in a
fixed order and writes down SDP data in plain matrix-entry form:

  * ``C``       upper-triangle COO entries (i <= j) of the cost matrix C,
  * ``A``       either COO entries (con, i, j, value), i <= j, of A_1..A_m, or
                "dense on pattern": one (i, j) list shared by every A_con plus an
                m x |pattern| value matrix,
  * ``b``       right-hand side of A(X) = b  (E:PrimalSDP).

Entries are *unscaled* matrix values; whoever consumes them applies its own
vectorisation.  Recipes follow SURVEY.md section 8(d) "Generator specification"
and DESIGN.md "Input recipe"; the workloads stand in for the paper's block-arrow
family (Fig. 2) and SDPLIB max-cut problems (PAPER.md:509-513,
files not available here).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import numpy as np


@dataclass
class Problem:
    """SDP data in matrix-entry form.  All index arrays are 0-based int32."""

    name: str
    n: int
    m: int
    c_row: np.ndarray
    c_col: np.ndarray
    c_val: np.ndarray
    b: np.ndarray
    # A, format "coo" or "dense"
    a_fmt: str
    a_con: Optional[np.ndarray] = None
    a_row: Optional[np.ndarray] = None
    a_col: Optional[np.ndarray] = None
    a_val: Optional[np.ndarray] = None  # coo: (nnz,), dense: (m, npat)
    meta: dict = field(default_factory=dict)
    # optional user sparsity pattern E ("described by the graph G(V,E)"): upper entries
    # that belong to the pattern even though C and every A_i are zero there
    e_row: Optional[np.ndarray] = None
    e_col: Optional[np.ndarray] = None

    def a_support(self):
        """(row, col) arrays of every structurally present A entry (may repeat across cons)."""
        return self.a_row, self.a_col


# ----------------------------------------------------------------------------
# Block-arrow (Fig. 2): l diagonal blocks of size d plus an
# arrow head of width h, n = l*d + h.
# ----------------------------------------------------------------------------

def block_arrow_pattern(l: int, d: int, h: int):
    """Upper-triangle (i <= j) entries of the block-arrow pattern, ordered by
    column then row (column-major upper).  Returns (row, col) int32 arrays."""
    n = l * d + h
    rows, cols = [], []
    for j in range(n):
        if j < l * d:
            start = (j // d) * d
        else:
            start = 0
        r = np.arange(start, j + 1, dtype=np.int32)
        rows.append(r)
        cols.append(np.full(r.shape, j, dtype=np.int32))
    return np.concatenate(rows), np.concatenate(cols)


def block_arrow(l: int, d: int, h: int, m: int, seed: int, name: str = "") -> Problem:
    """Strictly feasible block-arrow SDP (SURVEY.md 8(d) generator, reading G21).

    Draw order: A ~ U(-1,1)^(m x N); G ~ N(0,1)^(n x n); y0 ~ N(0,1)^m;
    Zoff ~ U(-1,1)^N.  X0 = G G^T / n (PSD, only pattern entries needed);
    b_i = <A_i, X0>; Z0 = pattern-sparse, diagonally dominant (Z0_ii = sum_{j!=i}|Z0_ij| + 1);
    C = sum_i y0_i A_i + Z0.  So X0 > 0 and Z0 > 0: strong duality, optimum attained.
    """
    rng = np.random.default_rng(seed)
    n = l * d + h
    row, col = block_arrow_pattern(l, d, h)
    npat = row.shape[0]
    A = rng.uniform(-1.0, 1.0, (m, npat))
    G = rng.standard_normal((n, n))
    # X0_ij = G_i . G_j / n on pattern entries only (chunked to bound memory)
    x0 = np.empty(npat)
    step = 1 << 16
    for s in range(0, npat, step):
        e = min(npat, s + step)
        x0[s:e] = np.einsum("ij,ij->i", G[row[s:e]], G[col[s:e]]) / n
    offdiag = row != col
    # <A_i, X0> = sum over upper entries with weight 1 (diag) or 2 (off-diag)
    w = np.where(offdiag, 2.0, 1.0)
    b = A @ (w * x0)
    y0 = rng.standard_normal(m)
    zoff = rng.uniform(-1.0, 1.0, npat)
    z0 = np.where(offdiag, zoff, 0.0)
    rowsum = np.zeros(n)
    np.add.at(rowsum, row[offdiag], np.abs(z0[offdiag]))
    np.add.at(rowsum, col[offdiag], np.abs(z0[offdiag]))
    z0[~offdiag] = rowsum[row[~offdiag]] + 1.0
    cval = A.T @ y0 + z0
    return Problem(
        name=name or f"block_arrow_l{l}_d{d}_h{h}_m{m}_s{seed}",
        n=n, m=m,
        c_row=row.copy(), c_col=col.copy(), c_val=cval,
        b=b, a_fmt="dense", a_row=row, a_col=col, a_val=A,
        meta={"kind": "block_arrow", "l": l, "d": d, "h": h, "seed": seed},
    )


# ----------------------------------------------------------------------------
# Max-cut relaxation on an Erdos-Renyi graph (stands in for SDPLIB maxG*,
# PAPER.md:509-513): min <-L/4, X> s.t. X_ii = 1.
# ----------------------------------------------------------------------------

def graph_maxcut(n: int, edges_i: np.ndarray, edges_j: np.ndarray, name: str, meta=None) -> Problem:
    """Max-cut SDP data for a simple graph given by edges (i < j)."""
    ei = np.asarray(edges_i, dtype=np.int32)
    ej = np.asarray(edges_j, dtype=np.int32)
    deg = np.zeros(n)
    np.add.at(deg, ei, 1.0)
    np.add.at(deg, ej, 1.0)
    diag = np.arange(n, dtype=np.int32)
    c_row = np.concatenate([diag, np.minimum(ei, ej)])
    c_col = np.concatenate([diag, np.maximum(ei, ej)])
    c_val = np.concatenate([-deg / 4.0, np.full(ei.shape[0], 0.25)])
    return Problem(
        name=name, n=n, m=n,
        c_row=c_row, c_col=c_col, c_val=c_val,
        b=np.ones(n), a_fmt="coo",
        a_con=diag.copy(), a_row=diag.copy(), a_col=diag.copy(), a_val=np.ones(n),
        meta=dict(meta or {}, kind="maxcut", n_edges=int(ei.shape[0])),
    )


def maxcut_er(n: int, seed: int, p: Optional[float] = None, name: str = "") -> Problem:
    """ER(n, 4/n) max-cut: mask = rng.random(n(n-1)/2) < p over np.triu_indices(n, 1)."""
    rng = np.random.default_rng(seed)
    prob = 4.0 / n if p is None else p
    iu, ju = np.triu_indices(n, 1)
    mask = rng.random(iu.shape[0]) < prob
    return graph_maxcut(n, iu[mask], ju[mask], name or f"maxcut_er_n{n}_s{seed}",
                        meta={"seed": seed, "p": prob})


def cycle_maxcut(n: int) -> Problem:
    i = np.arange(n)
    j = (i + 1) % n
    return graph_maxcut(n, np.minimum(i, j), np.maximum(i, j), f"maxcut_C{n}")


# ----------------------------------------------------------------------------
# Closed-form instances (no randomness)
# ----------------------------------------------------------------------------

def trace_one_tridiagonal(n: int = 12, a: float = 1.0, b: float = -0.7) -> Problem:
    """min <C,X> s.t. tr X = 1, C = tridiag(b, a, b)."""
    diag = np.arange(n, dtype=np.int32)
    off = np.arange(n - 1, dtype=np.int32)
    return Problem(
        name=f"trace1_tridiag_n{n}", n=n, m=1,
        c_row=np.concatenate([diag, off]), c_col=np.concatenate([diag, off + 1]),
        c_val=np.concatenate([np.full(n, a), np.full(n - 1, b)]),
        b=np.ones(1), a_fmt="coo",
        a_con=np.zeros(n, dtype=np.int32), a_row=diag.copy(), a_col=diag.copy(), a_val=np.ones(n),
        meta={"kind": "trace1", "a": a, "b": b},
    )


def lovasz_theta_cycle(n: int = 5) -> Problem:
    """Lovasz theta of C_n as min <-J, X> s.t. tr X = 1, X_ij = 0 on edges (i, i+1)."""
    iu, ju = np.triu_indices(n)
    c_row, c_col = iu.astype(np.int32), ju.astype(np.int32)
    c_val = -np.ones(c_row.shape[0])
    con, ar, ac, av = [], [], [], []
    for i in range(n):
        con.append(0); ar.append(i); ac.append(i); av.append(1.0)
    bvec = [1.0]
    for e in range(n):
        i, j = e, (e + 1) % n
        con.append(e + 1); ar.append(min(i, j)); ac.append(max(i, j)); av.append(1.0)
        bvec.append(0.0)
    return Problem(
        name=f"theta_C{n}", n=n, m=n + 1,
        c_row=c_row, c_col=c_col, c_val=c_val, b=np.array(bvec), a_fmt="coo",
        a_con=np.array(con, dtype=np.int32), a_row=np.array(ar, dtype=np.int32),
        a_col=np.array(ac, dtype=np.int32), a_val=np.array(av),
        meta={"kind": "theta"},
    )


def sensor_network(n: int, radius: float, seed: int, name: str = "") -> Problem:
    """Distance-constraint SDP on a random geometric graph (the sparse SDP class of sensor network
    localisation, SDPA-type input with a sparse Schur complement; SURVEY 8(f) #3 stand-in for the
    SDPLIB theta / qp instances of P:509-532, whose files are not available).

    Draw order: P ~ U[0,1]^(n x 2) (vertex positions; edges = pairs closer than `radius`),
    G ~ N(0,1)^(n x n), Coff ~ U(-1,1)^(#edges).  X0 = G G^T / n (strictly positive definite).
    Constraint per edge (i, j): X_ii + X_jj - 2 X_ij = b_ij := the same of X0.
    C = diagonally dominant on the graph: C_ij = Coff_ij / 2 on edges,
    C_ii = 1 + sum_j |C_ij| (C > 0, so y = 0 is strictly dual feasible)."""
    from scipy.spatial import cKDTree
    rng = np.random.default_rng(seed)
    P = rng.random((n, 2))
    G = rng.standard_normal((n, n))
    E = np.array(sorted(cKDTree(P).query_pairs(radius)), dtype=np.int64).reshape(-1, 2)
    m = E.shape[0]
    coff = 0.5 * rng.uniform(-1.0, 1.0, m)
    i, j = E[:, 0], E[:, 1]
    gi = np.einsum("ij,ij->i", G, G) / n                      # X0_ii
    xij = np.einsum("ij,ij->i", G[i], G[j]) / n               # X0_ij on the edges
    b = gi[i] + gi[j] - 2.0 * xij
    cdiag = np.ones(n)
    np.add.at(cdiag, i, np.abs(coff))
    np.add.at(cdiag, j, np.abs(coff))
    c_row = np.concatenate([np.arange(n), i]).astype(np.int32)
    c_col = np.concatenate([np.arange(n), j]).astype(np.int32)
    c_val = np.concatenate([cdiag, coff])
    k = np.arange(m)
    a_con = np.concatenate([k, k, k]).astype(np.int32)
    a_row = np.concatenate([i, j, i]).astype(np.int32)
    a_col = np.concatenate([i, j, j]).astype(np.int32)
    a_val = np.concatenate([np.ones(m), np.ones(m), -np.ones(m)])
    return Problem(name=name or f"sensor_n{n}_r{radius}_s{seed}", n=n, m=m, c_row=c_row, c_col=c_col,
                   c_val=c_val, b=b, a_fmt="coo", a_con=a_con, a_row=a_row, a_col=a_col, a_val=a_val,
                   meta={"kind": "sensor", "seed": seed, "edges": m})


def scalar_primal() -> Problem:
    """n=1, min x s.t. x = 2, x >= 0 (objective 2)."""
    z = np.zeros(1, dtype=np.int32)
    return Problem(name="scalar", n=1, m=1, c_row=z, c_col=z.copy(), c_val=np.ones(1),
                   b=np.array([2.0]), a_fmt="coo", a_con=z.copy(), a_row=z.copy(),
                   a_col=z.copy(), a_val=np.ones(1), meta={"kind": "scalar"})


# ----------------------------------------------------------------------------
# Batched PSD projection input (BASELINE configs[4])
# ----------------------------------------------------------------------------

def packed_upper_index(k: int):
    """(row, col) of the packed-upper column-major order: col-major over i <= j."""
    tr, tc = np.tril_indices(k)
    return tc.astype(np.int32), tr.astype(np.int32)


def psd_batch(count: int, seed: int, sizes=(8, 16, 32, 64)):
    """k ~ U(sizes); X = (G + G^T)/2, G ~ N(0,1)^(k x k), packed upper column-major.

    Returns (k array int32, packed values float64 concatenated)."""
    rng = np.random.default_rng(seed)
    ks = rng.choice(np.asarray(sizes), count).astype(np.int32)
    tot = int(np.sum(ks.astype(np.int64) * (ks + 1) // 2))
    out = np.empty(tot)
    idx_cache = {}
    off = 0
    for k in ks:
        k = int(k)
        if k not in idx_cache:
            idx_cache[k] = packed_upper_index(k)
        r, c = idx_cache[k]
        G = rng.standard_normal((k, k))
        X = 0.5 * (G + G.T)
        s = k * (k + 1) // 2
        out[off:off + s] = X[r, c]
        off += s
    return ks, out


# ----------------------------------------------------------------------------
# Named BASELINE configurations
# ----------------------------------------------------------------------------

CONFIG_SEEDS = {0: 1000, 1: 1001, 2: 1002, 3: 1003, 4: 1004}


def config(idx: int, batch_count: int = 200_000):
    if idx == 0:
        return block_arrow(5, 5, 2, 10, CONFIG_SEEDS[0], name="cfg0_block_arrow_l5_d5_h2_m10")
    if idx == 1:
        return block_arrow(40, 10, 5, 200, CONFIG_SEEDS[1], name="cfg1_block_arrow_l40_d10_h5_m200")
    if idx == 2:
        return block_arrow(400, 20, 10, 2000, CONFIG_SEEDS[2], name="cfg2_block_arrow_l400_d20_h10_m2000")
    if idx == 3:
        return maxcut_er(3000, CONFIG_SEEDS[3], name="cfg3_maxcut_er_n3000")
    if idx == 4:
        return psd_batch(batch_count, CONFIG_SEEDS[4])
    raise ValueError(idx)
