"""SDPA sparse reader (paper_1609_06068_b200.sdpa): parse hand-written golden
files whose optima have closed forms and solve them with the oracle (CPU)."""
import math
import os

import numpy as np
import pytest

from oracle import admm
from oracle import decompose as dc

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

CASES = [("theta_c5.dat-s", -math.sqrt(5.0)),                  # Lovasz 1979
         ("maxcut_c5.dat-s", -(25 + 5 * math.sqrt(5.0)) / 8),   # Goemans-Williamson on C5
         ("mixed_blocks.dat-s", -1.5)]                           # lambda_max over the blocks


@pytest.fixture(scope="module")
def sdpa():
    from paper_1609_06068_b200 import sdpa as m
    return m


def test_parse_structure(sdpa):
    p = sdpa.read_sdpa(os.path.join(GOLD, "mixed_blocks.dat-s"))
    assert (p.n, p.m) == (4, 1) and p.meta["blocks"] == [2, -2]
    assert np.allclose(p.b, [1.0])
    # C = -F0, upper entries, column-major sorted
    assert sorted(zip(p.c_row.tolist(), p.c_col.tolist(), p.c_val.tolist())) == [
        (0, 0, -1.0), (0, 1, -0.5), (1, 1, -1.0), (2, 2, -0.7), (3, 3, -0.2)]
    assert p.a_con.tolist() == [0, 0, 0, 0] and np.allclose(p.a_val, 1.0)


def test_parse_rejects_entries_outside_blocks(sdpa):
    bad = '"x"\n1\n1\n-2\n1.0\n0 1 1 2 1.0\n1 1 1 1 1.0\n'  # off-diagonal entry in a diagonal block
    with pytest.raises(ValueError):
        sdpa.read_sdpa(bad)


def test_duplicates_are_summed(sdpa):
    txt = '"x"\n1\n1\n2\n1.0\n0 1 1 2 0.25\n0 1 2 1 0.25\n1 1 1 1 1.0\n1 1 2 2 1.0\n'
    p = sdpa.read_sdpa(txt)
    assert p.c_row.tolist() == [0] and p.c_col.tolist() == [1] and np.allclose(p.c_val, [-0.5])


def test_roundtrip(sdpa, tmp_path):
    p = sdpa.read_sdpa(os.path.join(GOLD, "theta_c5.dat-s"))
    out = tmp_path / "t.dat-s"
    sdpa.write_sdpa(p, str(out))
    q = sdpa.read_sdpa(str(out))
    for f in ("c_row", "c_col", "c_val", "b", "a_con", "a_row", "a_col", "a_val"):
        assert np.array_equal(getattr(p, f), getattr(q, f)), f


@pytest.mark.parametrize("fname,want", CASES)
def test_golden_optima_with_oracle(sdpa, fname, want):
    p = sdpa.read_sdpa(os.path.join(GOLD, fname))
    dec = dc.decompose(p)
    for form in ("primal", "dual"):
        st, status = admm.solve(dec, 1.0, form, 1e-10, 20000)
        assert status == "solved"
        assert abs(st.objective - want) <= 1e-7 * abs(want), (form, st.objective, want)
