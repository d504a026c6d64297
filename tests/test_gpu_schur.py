"""S^-1 on the device (kernels_schur.cu: blocked Gauss-Jordan sweep of the SPD Schur complement
S = A D^-1 A^T) against the host Cholesky + L^-1 route (SDP_SCHUR_HOST=1) and the oracle:
ragged orders (m not a multiple of the 32-pivot block or the 64-tile), an ill-conditioned S, and a
singular S (duplicate constraint) that both routes reject."""
import os
from contextlib import contextmanager

import numpy as np
import pytest

from oracle import admm
from oracle import decompose as dc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib():
    import paper_1609_06068_b200 as L
    return L


@contextmanager
def env(**kv):
    old = {k: os.environ.get(k) for k in kv}
    try:
        for k, v in kv.items():
            os.environ[k] = str(v)
        yield
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def rel_inf(g, o):
    return float(np.max(np.abs(g - o)) / max(float(np.max(np.abs(o))), 1e-300))


@pytest.mark.parametrize("l,d,h,m", [(7, 3, 3, 11), (40, 10, 5, 200), (30, 8, 6, 333), (24, 12, 8, 1000)])
def test_device_inverse_matches_host_route_and_oracle(lib, gen, l, d, h, m):
    prob = gen.block_arrow(l, d, h, m, seed=3)
    dec = dc.decompose(prob)
    st = admm.step(dec, admm.zero_state(dec), 1.0, "primal", 12)
    with env(SDP_SCHUR_HOST=1, SDP_FUSED=0):
        ref = lib.Solver(prob, form="primal", rho=1.0)
    with env(SDP_FUSED=0):
        s = lib.Solver(prob, form="primal", rho=1.0)
    assert s.info()["s_factor"] == 1 and ref.info()["s_factor"] == 1
    ref.step(12)
    s.step(12)
    for a, b in ((s.y(), ref.y()), (s.x(), ref.x()), (s.blocks("xk"), ref.blocks("xk"))):
        assert rel_inf(a, b) <= 1e-11
    for g, o in ((s.x(), st.x), (s.y(), st.y), (s.blocks("xk"), st.xk)):
        assert rel_inf(g, o) <= 1e-9
    s.close()
    ref.close()


@pytest.mark.parametrize("delta", [1e-2, 1e-3])
def test_device_inverse_ill_conditioned(lib, gen, delta):
    """Two nearly dependent constraints (cond(S) ~ 1e4 .. 1e6): 50 iterations match the oracle."""
    prob = gen.block_arrow(20, 6, 4, 150, seed=8)
    rng = np.random.default_rng(4)
    prob.a_val = prob.a_val.copy()
    prob.a_val[-1] = prob.a_val[-2] + delta * rng.uniform(-1, 1, prob.a_val.shape[1])
    dec = dc.decompose(prob)
    assert np.linalg.cond((dec.A / dec.D) @ dec.A.T) > 1e3
    st = admm.step(dec, admm.zero_state(dec), 1.0, "dual", 50)
    s = lib.Solver(prob, form="dual", rho=1.0)
    s.step(50)
    for g, o in ((s.x(), st.x), (s.y(), st.y), (s.blocks("xk"), st.xk)):
        assert rel_inf(g, o) <= 1e-9
    s.close()


@pytest.mark.parametrize("host", [0, 1])
def test_singular_schur_rejected(lib, gen, host):
    prob = gen.block_arrow(20, 6, 4, 150, seed=8)
    prob.a_val = prob.a_val.copy()
    prob.a_val[77] = prob.a_val[12]  # a repeated constraint: S singular
    with env(SDP_SCHUR_HOST=host):
        with pytest.raises(lib.SdpError, match="RANK_DEFICIENT"):
            lib.Solver(prob, form="primal", rho=1.0)
