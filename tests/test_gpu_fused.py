"""The fused persistent iteration (kernels_fused.cu): one cooperative launch per sdp_step runs every
phase of every iteration for small single-rank problems.  Parity with the oracle element by element
(same tolerance as tests/test_gpu_parity.py), agreement with the per-phase kernels, the grid
barrier at several grid sizes (1 CTA, odd counts, the full default grid), the device-side stopping
rule inside one launch, checkpoint / resume, and rho changes."""
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
    return float(np.max(np.abs(g - o)) / max(float(np.max(np.abs(o))), 1e-300)) if o.size else 0.0


def compare(st, s, form, tol=1e-9):
    fam = {"x": (s.x(), st.x), "y": (s.y(), st.y), "xk": (s.blocks("xk"), st.xk),
           "lambda": (s.blocks("lambda"), st.lam)}
    if form == "dual":
        fam["vk"] = (s.blocks("vk"), st.vk)
    errs = {k: rel_inf(g, o) for k, (g, o) in fam.items()}
    assert max(errs.values()) <= tol, errs
    return errs


def problems(gen):
    return {
        "cfg0": gen.config(0),                          # 5 cliques of 7: one CTA
        "cfg1": gen.config(1),                          # 40 cliques of 15
        "arrow_odd": gen.block_arrow(7, 3, 3, 11, seed=5),
        "mixed": gen.maxcut_er(60, 3, p=0.12),          # ragged clique orders across k <= 8 / 16 / 32
        "k30": gen.block_arrow(12, 20, 10, 40, seed=7),  # the k = 30 bucket (groups of 128)
        "theta5": gen.lovasz_theta_cycle(5),
    }


@pytest.mark.parametrize("name", ["cfg0", "cfg1", "arrow_odd", "mixed", "k30", "theta5"])
@pytest.mark.parametrize("form", ["primal", "dual"])
def test_fused_iterates_match_oracle(lib, gen, name, form):
    prob = problems(gen)[name]
    dec = dc.decompose(prob)
    if max(len(c) for c in dec.cliques) > 32:
        pytest.skip("cliques above 32: not eligible")
    iters = 70  # crosses a warm-start cold restart (every 64 iterations)
    st = admm.step(dec, admm.zero_state(dec), 1.0, form, iters, record=True)
    with env(SDP_FUSED=1):
        s = lib.Solver(prob, form=form, rho=1.0)
    assert s.info()["fused"] == 1
    s.step(iters)
    compare(st, s, form)
    h = s.history()
    o = np.array(st.history)
    assert h.shape[0] == iters
    # (residuals at the rounding floor of a solved instance: absolute 1e-13 on these normalised
    # O(1) quantities)
    assert np.allclose(h[:, 0], o[:, 1], rtol=1e-7, atol=1e-13)
    assert np.allclose(h[:, 1], o[:, 2], rtol=1e-7, atol=1e-13)
    assert np.allclose(h[:, 2], o[:, 3], rtol=1e-9, atol=1e-12)
    s.close()


def test_fused_is_default_for_small_problems(lib, gen):
    for cfg in (0, 1):
        s = lib.Solver(gen.config(cfg), form="primal", rho=1.0)
        info = s.info()
        assert info["fused"] == 1 and info["launches_per_iter"] == 1
        s.close()
    with env(SDP_FUSED=0):
        s = lib.Solver(gen.config(1), form="primal", rho=1.0)
    assert s.info()["fused"] == 0
    s.close()


@pytest.mark.parametrize("form", ["primal", "dual"])
@pytest.mark.parametrize("ctas", [1, 3, 7, 0])
def test_fused_grid_sizes_agree(lib, gen, form, ctas):
    """The grid barrier and the grid-strided work split at 1, 3, 7 CTAs and the default grid: every
    grid gives the per-phase kernels' iterates to rounding."""
    prob = gen.config(1)
    with env(SDP_FUSED=0):
        ref = lib.Solver(prob, form=form, rho=2.0)
    ref.step(40)
    kv = {"SDP_FUSED": 1}
    if ctas:
        kv["SDP_FUSED_CTAS"] = ctas
    with env(**kv):
        s = lib.Solver(prob, form=form, rho=2.0)
    assert s.info()["fused"] == 1
    s.step(40)
    for a, b in ((s.x(), ref.x()), (s.y(), ref.y()), (s.blocks("xk"), ref.blocks("xk")),
                 (s.blocks("lambda"), ref.blocks("lambda"))):
        assert rel_inf(a, b) <= 1e-10
    assert np.allclose(s.history()[:, :2], ref.history()[:, :2], rtol=1e-7, atol=1e-14)
    s.close()
    ref.close()


def test_fused_deterministic_and_call_split(lib, gen):
    """Bit-identical iterates whether 30 iterations are one launch or 30, and after reset."""
    prob = gen.config(1)
    s = lib.Solver(prob, form="primal", rho=1.0)
    s.step(30)
    a = (s.x(), s.y(), s.blocks("xk"), s.blocks("lambda"), s.history())
    s.reset()
    for i in range(30):
        s.step(1)
        if i % 7 == 3:
            s.step(0)  # an empty call must not disturb the launches' barrier counters
    b = (s.x(), s.y(), s.blocks("xk"), s.blocks("lambda"), s.history())
    for u, v in zip(a, b):
        assert np.array_equal(u, v)
    s.close()


@pytest.mark.parametrize("form,rho", [("primal", 10.0), ("dual", 0.1)])
def test_fused_solve_stops_on_device(lib, gen, form, rho):
    """sdp_solve without adaptation is one launch; the device stopping rule (reading G10) ends it at
    the oracle's stop iteration."""
    prob = gen.config(1)
    dec = dc.decompose(prob)
    st, ostatus = admm.solve(dec, rho, form, 1e-4, 3000)
    s = lib.Solver(prob, form=form, rho=rho)
    status, info = s.solve(3000, 1e-4)
    assert status == ostatus == "solved"
    assert info["iters"] == st.it
    assert abs(info["objective"] - st.objective) <= 1e-6 * max(1.0, abs(st.objective))
    # a later step continues (the stop flag is cleared)
    s.step(3)
    assert s.info()["iters"] == info["iters"] + 3
    s.close()


def test_fused_checkpoint_resume_and_rho(lib, gen):
    prob = gen.config(1)
    dec = dc.decompose(prob)
    st = admm.step(dec, admm.zero_state(dec), 1.0, "primal", 20)
    st = admm.step(dec, st, 4.0, "primal", 15)
    s = lib.Solver(prob, form="primal", rho=1.0)
    s.step(20)
    blob = s.save_state()
    s.set_rho(4.0)
    s.step(15)
    compare(st, s, "primal")
    x1 = s.x()
    t = lib.Solver(prob, form="primal", rho=1.0)
    t.load_state(blob)
    t.set_rho(4.0)
    t.step(15)
    assert np.array_equal(t.x(), x1)
    s.close()
    t.close()


def test_fused_long_run_no_capped_sweeps(lib, gen):
    """500 iterations in one launch (warm-start restarts every 64) stay finite and uncapped."""
    s = lib.Solver(gen.config(0), form="dual", rho=1.0)
    s.step(500)
    info = s.info()
    assert info["iters"] == 500 and info["jacobi_capped"] == 0
    assert np.isfinite(info["eps_p"]) and np.isfinite(info["eps_d"])
    s.close()


@pytest.mark.parametrize("name", ["scalar", "cyc5", "cyc9", "trace", "theta7", "sensor60"])
@pytest.mark.parametrize("form", ["primal", "dual"])
def test_fused_small_generators(lib, gen, name, form):
    """Degenerate and sparse-A shapes through the fused path: one 1 x 1 clique (n = m = 1), cliques of
    2 / 3 / 7, a diagonal S (max-cut), a sparse S (distance constraints on a geometric graph with
    cliques of 3..16); 40 iterations against the oracle element by element."""
    prob = {"scalar": lambda: gen.scalar_primal(), "cyc5": lambda: gen.cycle_maxcut(5),
            "cyc9": lambda: gen.cycle_maxcut(9), "trace": lambda: gen.trace_one_tridiagonal(12),
            "theta7": lambda: gen.lovasz_theta_cycle(7), "sensor60": lambda: gen.sensor_network(60, 0.3, 2)}[name]()
    dec = dc.decompose(prob)
    st = admm.step(dec, admm.zero_state(dec), 1.0, form, 40, record=True)
    with env(SDP_FUSED=1):
        s = lib.Solver(prob, form=form, rho=1.0)
    assert s.info()["fused"] == 1
    s.step(40)
    compare(st, s, form)
    h = s.history()
    o = np.array(st.history)
    assert np.allclose(h[:, 2], o[:, 3], rtol=1e-9, atol=1e-12)
    s.close()
