"""SDPA sparse format (".dat-s") reader / writer for the solver's problem data.

The SDPA pair (SDPA manual; the format of the SDPLIB problems the paper uses,
P:509-513) is
    primal  min  sum_i c_i x_i   s.t.  sum_i F_i x_i - F_0 = X >= 0
    dual    max  <F_0, Y>        s.t.  <F_i, Y> = c_i,  Y >= 0.
The dual is this library's standard primal form with X := Y,
C = -F_0, A_i = F_i and b = c, so `objective` of a solve equals -(SDPA dual
objective).  Block-diagonal SDPA structure (several SDP blocks, negative sizes
for diagonal / LP blocks) becomes one n x n matrix whose aggregate sparsity
pattern is block diagonal; the chordal decomposition then keeps the
blocks apart.  Entries are read as given on or above the diagonal (i <= j),
duplicates are summed.

This module is argument marshalling only (host-side parsing); every step of
the solve runs in libchordal_sdp.so.
"""
from __future__ import annotations

import re
from dataclasses import dataclass, field
from typing import Optional

import numpy as np


@dataclass
class SdpData:
    """Problem data in the form `Solver` takes (0-based int32 indices, upper entries)."""
    name: str
    n: int
    m: int
    c_row: np.ndarray
    c_col: np.ndarray
    c_val: np.ndarray
    b: np.ndarray
    a_fmt: str = "coo"
    a_con: Optional[np.ndarray] = None
    a_row: Optional[np.ndarray] = None
    a_col: Optional[np.ndarray] = None
    a_val: Optional[np.ndarray] = None
    meta: dict = field(default_factory=dict)


def _numbers(line: str):
    return [t for t in re.split(r"[\s,{}()]+", line.strip()) if t]


def read_sdpa(path_or_text: str, name: str | None = None) -> SdpData:
    """Parse an SDPA sparse file (path, or the text itself if it contains a newline)."""
    if "\n" in path_or_text:
        text = path_or_text
        name = name or "sdpa"
    else:
        with open(path_or_text) as f:
            text = f.read()
        name = name or path_or_text
    lines = []
    for raw in text.splitlines():
        s = raw.strip()
        if not s or s[0] in "\"*":
            continue
        lines.append(s)
    it = iter(lines)
    m = int(float(_numbers(next(it))[0]))
    nblocks = int(float(_numbers(next(it))[0]))
    sizes = []
    while len(sizes) < nblocks:
        sizes += [int(float(t)) for t in _numbers(next(it))]
    sizes = sizes[:nblocks]
    c = []
    while len(c) < m:
        c += [float(t) for t in _numbers(next(it))]
    c = np.array(c[:m], dtype=np.float64)
    offs = np.concatenate([[0], np.cumsum(np.abs(sizes))]).astype(np.int64)
    n = int(offs[-1])
    ent = {}
    for s in it:
        tok = _numbers(s)
        if len(tok) < 5:
            continue
        mat, blk, i, j = (int(float(t)) for t in tok[:4])
        v = float(tok[4])
        if not (0 <= mat <= m and 1 <= blk <= nblocks):
            raise ValueError(f"SDPA entry out of range: {s!r}")
        bs = sizes[blk - 1]
        i, j = min(i, j), max(i, j)
        if not (1 <= i <= abs(bs) and 1 <= j <= abs(bs)) or (bs < 0 and i != j):
            raise ValueError(f"SDPA entry outside its block: {s!r}")
        key = (mat, int(offs[blk - 1]) + i - 1, int(offs[blk - 1]) + j - 1)
        ent[key] = ent.get(key, 0.0) + v
    cr, cc, cv, ac, ar, acl, av = [], [], [], [], [], [], []
    for (mat, r, col), v in sorted(ent.items(), key=lambda kv: (kv[0][0], kv[0][2], kv[0][1])):
        if mat == 0:                      # C = -F_0
            cr.append(r), cc.append(col), cv.append(-v)
        else:                             # A_i = F_i
            ac.append(mat - 1), ar.append(r), acl.append(col), av.append(v)
    # every diagonal / LP block coordinate must be in the pattern even if no
    # matrix mentions it: the diagonal is always part of the pattern
    i32 = lambda a: np.asarray(a, dtype=np.int32)  # noqa: E731
    return SdpData(name=name, n=n, m=m, c_row=i32(cr), c_col=i32(cc), c_val=np.asarray(cv, np.float64), b=c,
                   a_con=i32(ac), a_row=i32(ar), a_col=i32(acl), a_val=np.asarray(av, np.float64),
                   meta={"kind": "sdpa", "blocks": sizes, "sign": "objective = -(SDPA dual objective)"})


def write_sdpa(prob, path: str, blocks=None, comment: str = "written by paper_1609_06068_b200.sdpa"):
    """Write problem data (this library's form) as SDPA sparse; one SDP block
    of order n unless `blocks` (SDPA block sizes, summing to n in absolute
    value) is given."""
    blocks = list(blocks) if blocks is not None else [prob.n]
    offs = np.concatenate([[0], np.cumsum(np.abs(blocks))])
    if offs[-1] != prob.n:
        raise ValueError("block sizes do not add up to n")

    def loc(r, c):
        b = int(np.searchsorted(offs, r, side="right") - 1)
        return b + 1, int(r - offs[b] + 1), int(c - offs[b] + 1)

    out = [f'"{comment}"', str(prob.m), str(len(blocks)), " ".join(str(b) for b in blocks),
           " ".join(repr(float(v)) for v in prob.b)]
    for r, c, v in zip(prob.c_row, prob.c_col, prob.c_val):
        b, i, j = loc(min(r, c), max(r, c))
        out.append(f"0 {b} {i} {j} {-float(v)!r}")
    if prob.a_fmt != "coo":
        raise ValueError("write_sdpa needs COO constraint data")
    for k, r, c, v in zip(prob.a_con, prob.a_row, prob.a_col, prob.a_val):
        b, i, j = loc(min(r, c), max(r, c))
        out.append(f"{int(k) + 1} {b} {i} {j} {float(v)!r}")
    with open(path, "w") as f:
        f.write("\n".join(out) + "\n")
