"""GPU tests of the C-ABI boundary and of the sharded device path (8(e)):
  * the recovered primal-dual SDP pair (Remark 1; KKT multipliers rho*y P:226,
    rho*x P:354) in both forms against oracle.admm.recovered_pair, and its duality gap;
  * PSD completion of the SDP X in the dual form (Theorem 1);
  * the caller-owned device memory (sdp_options.allocator, torch tensors);
  * the optional user pattern E;
  * the pipelined dual schedule's iteration index (no race at warm-start period);
  * the clique-sharded iteration (shard plan, partial scatter sums, owned-column GEMV,
    fix-up, residual all-reduce) run through the in-process loopback communicator at
    world = 2, 3, 4 on one GPU, element by element against the oracle.
"""
import threading

import numpy as np
import pytest

from oracle import admm
from oracle import completion
from oracle import chordal
from oracle import decompose as dc

pytestmark = pytest.mark.gpu


def rel(g, o):
    return float(np.linalg.norm(g - o) / max(np.linalg.norm(o), 1e-300))


def rel_inf(g, o):
    return float(np.max(np.abs(g - o)) / max(float(np.max(np.abs(o))), 1e-300))


@pytest.fixture(scope="module")
def lib():
    import paper_1609_06068_b200 as L
    return L


# ------------------------------------------------------------------ recovered SDP pair

@pytest.mark.parametrize("name,form,rho", [("cfg1", "primal", 10.0), ("cfg1", "dual", 0.1),
                                           ("maxcut200", "primal", 0.1), ("maxcut200", "dual", 10.0)])
def test_recovered_pair_both_forms(lib, gen, name, form, rho):
    prob = gen.config(1) if name == "cfg1" else gen.maxcut_er(200, 11)
    dec = dc.decompose(prob)
    st = admm.step(dec, admm.zero_state(dec), rho, form, 40)
    s = lib.Solver(prob, form=form, rho=rho)
    s.step(40)
    X, yhat, Z = admm.recovered_pair(dec, st, rho, form)
    Xm = dec.unsvec_pattern(X)
    for g, o in ((s.sdp_x(), Xm), (s.sdp_y(), yhat), (s.sdp_z(), Z)):
        assert rel(g, o) <= 1e-9 and rel_inf(g, o) <= 1e-9
    # A(X) = b holds exactly at every iterate in both forms (P:354 for the dual form)
    r, c = s.pattern()
    xs = np.where(r == c, s.sdp_x(), np.sqrt(2.0) * s.sdp_x())
    assert np.linalg.norm(dec.A @ xs - dec.b) <= 1e-9 * max(1.0, np.linalg.norm(dec.b))
    # at convergence: duality gap <C,X> - <b,yhat> -> 0 (Remark 1)
    status, info = s.solve(20000, 1e-5)
    assert status == "solved"
    xs = np.where(r == c, s.sdp_x(), np.sqrt(2.0) * s.sdp_x())
    gap = dec.c @ xs - dec.b @ s.sdp_y()
    assert abs(gap) <= 1e-3 * max(1.0, abs(info["objective"])), gap
    s.close()


@pytest.mark.parametrize("name", ["cfg0", "maxcut200", "theta5"])
def test_completion_dual_form(lib, gen, name):
    """sdp_complete_x on a dual-form handle completes the SDP X = -rho x (not the KKT x):
    agreement with oracle.completion of the recovered X, and PSD (Grone) after a solve."""
    prob = {"cfg0": gen.config(0), "maxcut200": gen.maxcut_er(200, 11), "theta5": gen.lovasz_theta_cycle(5)}[name]
    rho = {"cfg0": 0.1, "maxcut200": 10.0, "theta5": 1.0}[name]   # reading G11 (dual form)
    dec = dc.decompose(prob)
    s = lib.Solver(prob, form="dual", rho=rho)
    status, _ = s.solve(50000, 1e-7)
    assert status == "solved"
    adj = chordal.aggregate_adjacency(prob)
    order, later, filled = chordal.minimum_degree_elimination(adj)
    n = prob.n
    known = filled | np.eye(n, dtype=bool)
    r, c = s.pattern()
    X = np.zeros((n, n))
    xm = s.sdp_x()
    X[r, c] = xm
    X[c, r] = xm
    # separator blocks of a converged X are singular to solver accuracy: a pseudo-inverse cut well
    # above the noise (1e-6) makes the two constructions take the same rank decisions
    want = completion.complete_psd(X, known, order, later, rtol=1e-6)
    got = s.complete_x(rtol=1e-6)
    assert np.allclose(got[known], X[known], rtol=0, atol=0)
    assert np.linalg.norm(got - want) <= 1e-9 * np.linalg.norm(want)
    assert np.linalg.eigvalsh(got).min() >= -1e-5 * np.linalg.norm(got)
    assert np.trace(got) > 0
    s.close()


# ------------------------------------------------------------------ caller-owned device memory

def test_torch_allocator_owns_device_memory(lib, gen):
    import torch
    prob = gen.config(1)
    a = lib.Solver(prob, form="primal", rho=1.0)
    b = lib.Solver(prob, form="primal", rho=1.0, allocator="torch")
    live, peak = b.workspace_bytes()
    assert live > 0 and peak >= live
    assert b.allocator.bytes_held() == live       # every live device byte is a torch tensor
    before = torch.cuda.memory_allocated(0)
    assert before >= live
    a.step(30)
    b.step(30)
    for fam in ("xk", "lambda"):
        assert np.array_equal(a.blocks(fam), b.blocks(fam))
    assert np.array_equal(a.x(), b.x())
    b.close()
    assert b.allocator.bytes_held() == 0
    ks, vals = gen.psd_batch(300, seed=3)
    p1 = lib.PsdPlan(ks)
    p2 = lib.PsdPlan(ks, allocator="torch")
    assert p2.allocator.bytes_held() > 0
    assert np.array_equal(p1.project_host(vals), p2.project_host(vals))
    with pytest.raises(ValueError):
        p2.project_host(vals[:-1])
    t = torch.zeros(p2.values - 1, dtype=torch.float64, device="cuda")
    with pytest.raises(ValueError):
        p2.project(t, t)
    p1.close()
    p2.close()
    a.close()


# ------------------------------------------------------------------ user pattern E

@pytest.mark.parametrize("form", ["primal", "dual"])
def test_user_pattern_E(lib, gen, form):
    prob = gen.block_arrow(7, 3, 3, 11, seed=5)
    prob.e_row = np.array([0, 2, 5], np.int32)   # links between diagonal blocks 0-1, 0-2, 1-2
    prob.e_col = np.array([4, 7, 8], np.int32)
    dec = dc.decompose(prob)
    base = dc.decompose(gen.block_arrow(7, 3, 3, 11, seed=5))
    assert [c.tolist() for c in dec.cliques] != [c.tolist() for c in base.cliques]
    st = admm.step(dec, admm.zero_state(dec), 1.0, form, 50)
    s = lib.Solver(prob, form=form, rho=1.0)
    s.step(50)
    assert [c.tolist() for c in s.cliques()] == [c.tolist() for c in dec.cliques]
    r, c = s.pattern()
    assert np.array_equal(r, dec.coord_row) and np.array_equal(c, dec.coord_col)
    for g, o in ((s.x(), st.x), (s.y(), st.y), (s.blocks("xk"), st.xk), (s.blocks("lambda"), st.lam)):
        assert rel(g, o) <= 1e-9 and rel_inf(g, o) <= 1e-9
    s.close()


# ------------------------------------------------------------------ pipelined dual schedule

def test_cfg2_dual_pipelined_split_calls_bit_identical(lib, gen):
    """the next iteration's P_+(H1) runs concurrently with the current finalize; its
    warm/cold-start decision reads a published iteration index, so sdp_step(130) and
    sdp_step(65) + sdp_step(65) (crossing the warm-start period 64 twice) are bit-identical."""
    prob = gen.config(2)
    a = lib.Solver(prob, form="dual", rho=0.1)
    b = lib.Solver(prob, form="dual", rho=0.1)
    assert a.info()["pipelined"] == 1
    a.step(130)
    b.step(65)
    b.step(65)
    for fam in ("xk", "lambda", "vk"):
        assert np.array_equal(a.blocks(fam), b.blocks(fam)), fam
    assert np.array_equal(a.x(), b.x()) and np.array_equal(a.y(), b.y())
    assert np.array_equal(a.history(), b.history())
    a.close()
    b.close()


# ------------------------------------------------------------------ sharded path, loopback

def run_sharded(L, prob, form, rho, iters, world, streams=True):
    import torch
    grp = L.LoopbackGroup(world)
    out = [None] * world
    err = []

    def rank_main(r):
        try:
            st = torch.cuda.Stream() if streams else None
            s = L.Solver(prob, form=form, rho=rho, rank=r, world=world, comm=grp, stream=st)
            s.step(iters)
            res = {"x": s.x(), "y": s.y(), "xk": s.blocks("xk"), "lambda": s.blocks("lambda"),
                   "vk": s.blocks("vk"), "hist": s.history(), "info": s.info()}
            s.close()
            out[r] = res
        except Exception as e:  # noqa: BLE001
            err.append(repr(e))

    th = [threading.Thread(target=rank_main, args=(r,), daemon=True) for r in range(world)]
    for t in th:
        t.start()
    wait_ranks(th, err)
    grp.close()
    return out


def wait_ranks(th, err, limit=600.0):
    """Join the rank threads; a rank that raised leaves the others blocked in a collective, so
    report the first error at once instead of waiting for them."""
    import time
    t0 = time.time()
    while any(t.is_alive() for t in th) and not err and time.time() - t0 < limit:
        time.sleep(0.02)
    assert not err, err
    assert not any(t.is_alive() for t in th), "rank threads still running (deadlock?)"


SHARD_CASES = [
    ("arrow", lambda g: g.block_arrow(12, 10, 5, 60, seed=9), 2),
    ("arrow", lambda g: g.block_arrow(12, 10, 5, 60, seed=9), 4),
    ("cfg1", lambda g: g.config(1), 3),
    ("maxcut200", lambda g: g.maxcut_er(200, 11), 2),
    ("maxcut200", lambda g: g.maxcut_er(200, 11), 4),
    ("trace1", lambda g: g.trace_one_tridiagonal(12), 2),
]


@pytest.mark.parametrize("name,make,world", SHARD_CASES, ids=[f"{c[0]}-w{c[2]}" for c in SHARD_CASES])
@pytest.mark.parametrize("form", ["primal", "dual"])
def test_sharded_loopback_matches_oracle(lib, gen, name, make, world, form):
    prob = make(gen)
    rho = 1.0
    dec = dc.decompose(prob)
    st = admm.step(dec, admm.zero_state(dec), rho, form, 30, record=True)
    out = run_sharded(lib, prob, form, rho, 30, world)
    fam = {"x": st.x, "y": st.y, "xk": st.xk, "lambda": st.lam}
    if form == "dual":
        fam["vk"] = st.vk
    o = np.array(st.history)
    for r in range(world):
        for k, want in fam.items():
            g = out[r][k]
            assert rel(g, want) <= 1e-9 and rel_inf(g, want) <= 1e-9, (r, k, rel(g, want), rel_inf(g, want))
        h = out[r]["hist"]
        assert h.shape[0] == 30
        assert np.allclose(h[:, 0], o[:, 1], rtol=1e-7, atol=1e-14)
        assert np.allclose(h[:, 1], o[:, 2], rtol=1e-7, atol=1e-14)
        assert np.allclose(h[:, 2], o[:, 3], rtol=1e-9, atol=1e-12)
    # every rank reports the same (replicated) residual history
    for r in range(1, world):
        assert np.array_equal(out[r]["hist"], out[0]["hist"])


@pytest.mark.slow
@pytest.mark.parametrize("form,rho", [("primal", 10.0), ("dual", 0.1)])
def test_sharded_loopback_cfg2(lib, gen, form, rho):
    """BASELINE configs[2] (dense A, 400 cliques of 30, the multi-GPU case of SURVEY 8(e)) split
    over 2 ranks: A column-sharded by owned coordinates, 20 iterations against the oracle."""
    prob = gen.config(2)
    dec = dc.decompose(prob)
    st = admm.step(dec, admm.zero_state(dec), rho, form, 20)
    out = run_sharded(lib, prob, form, rho, 20, 2)
    for r in range(2):
        for k, want in (("x", st.x), ("y", st.y), ("xk", st.xk), ("lambda", st.lam)):
            assert rel(out[r][k], want) <= 1e-9 and rel_inf(out[r][k], want) <= 1e-9, (r, k)


def test_sharded_loopback_solve_stops_together(lib, gen):
    """sdp_solve on sharded handles: the stop flag comes from all-reduced residuals, so every
    rank stops at the oracle's iteration with the same objective."""
    import torch
    prob = gen.config(1)
    dec = dc.decompose(prob)
    st, status = admm.solve(dec, 10.0, "primal", 1e-4, 5000)
    grp = lib.LoopbackGroup(2)
    res = [None, None]

    err = []

    def rank_main(r):
        try:
            s = lib.Solver(prob, form="primal", rho=10.0, rank=r, world=2, comm=grp, stream=torch.cuda.Stream(),
                           check_every=7)
            res[r] = s.solve(5000, 1e-4)
            s.close()
        except Exception as e:  # noqa: BLE001
            err.append(repr(e))

    th = [threading.Thread(target=rank_main, args=(r,), daemon=True) for r in range(2)]
    [t.start() for t in th]
    wait_ranks(th, err)
    grp.close()
    for r in range(2):
        gstatus, info = res[r]
        assert gstatus == status and info["iters"] == st.it
        assert abs(info["objective"] - st.objective) <= 1e-6 * abs(st.objective)


# ------------------------------------------------------------------ sparse S

@pytest.mark.parametrize("form", ["primal", "dual"])
def test_sensor_network_sparse_schur(lib, gen, tmp_path, form):
    """An SDPA instance with m >= 5000 (distance constraints on a random geometric graph, written
    and read back through the SDPA reader): S = A D^-1 A^T is factorised by the sparse Cholesky
    (s_factor 2, nnz(L) << m^2), and 30 iterations match the oracle (dense KKT) element by element."""
    from paper_1609_06068_b200 import sdpa
    prob = gen.sensor_network(2000, 0.032, seed=7)
    assert prob.m >= 5000
    path = tmp_path / "sensor.dat-s"
    sdpa.write_sdpa(prob, str(path))
    data = sdpa.read_sdpa(str(path))
    dec = dc.decompose(data)
    st = admm.step(dec, admm.zero_state(dec), 1.0, form, 30, record=True)
    s = lib.Solver(data, form=form, rho=1.0)
    info = s.info()
    assert info["s_factor"] == 2 and info["nnz_l"] < prob.m * prob.m / 16
    s.step(30)
    for g, o in ((s.x(), st.x), (s.y(), st.y), (s.blocks("xk"), st.xk), (s.blocks("lambda"), st.lam)):
        assert rel(g, o) <= 1e-9 and rel_inf(g, o) <= 1e-9
    h = s.history()
    o = np.array(st.history)
    assert np.allclose(h[:, 2], o[:, 3], rtol=1e-9, atol=1e-12)
    s.close()


def test_forced_sparse_schur_subprocess():
    """SDP_SPARSE_S=1 forces the sparse factorisation on small problems (dense-ish S included):
    iterates still match the oracle."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import numpy as np, sys; sys.path.insert(0, %r)\n"
        "import paper_1609_06068_b200 as L, sdp_inputs as gen\n"
        "from oracle import admm, decompose as dc\n"
        "r = lambda g, o: float(np.max(np.abs(g - o)) / np.max(np.abs(o)))\n"
        "def coo(p):\n"
        "    m, npat = p.a_val.shape\n"
        "    p.a_con = np.repeat(np.arange(m, dtype=np.int32), npat)\n"
        "    p.a_row = np.tile(p.a_row, m); p.a_col = np.tile(p.a_col, m); p.a_val = p.a_val.reshape(-1)\n"
        "    p.a_fmt = 'coo'; return p\n"
        "for prob in (coo(gen.block_arrow(4, 3, 2, 9, seed=2)), gen.sensor_network(60, 0.3, 2),\n"
        "             gen.sensor_network(200, 0.12, 1)):\n"
        "    dec = dc.decompose(prob)\n"
        "    for form in ('primal', 'dual'):\n"
        "        st = admm.step(dec, admm.zero_state(dec), 1.0, form, 40)\n"
        "        s = L.Solver(prob, form=form, rho=1.0); assert s.info()['s_factor'] == 2, s.info()\n"
        "        s.step(40)\n"
        "        e = max(r(s.x(), st.x), r(s.y(), st.y), r(s.blocks('xk'), st.xk), r(s.blocks('lambda'), st.lam))\n"
        "        print(prob.name, form, e); assert e <= 1e-9, e\n" % root)
    env = dict(os.environ, SDP_SPARSE_S="1")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.slow
def test_sensor_network_solve_to_tolerance(lib, gen):
    """The m = 6079 SDPA-type instance solved to 1e-4 (dual form, rho = 1: 521 oracle iterations)
    through the sparse-Cholesky path: same stop iteration, objective within 1e-6 (north_star)."""
    prob = gen.sensor_network(2000, 0.032, seed=7)
    dec = dc.decompose(prob)
    st, status = admm.solve(dec, 1.0, "dual", 1e-4, 2000)
    assert status == "solved"
    s = lib.Solver(prob, form="dual", rho=1.0, check_every=7)
    assert s.info()["s_factor"] == 2
    gstatus, info = s.solve(2000, 1e-4)
    assert gstatus == status
    if info["iters"] != st.it:  # reading G19 fallback
        s.reset()
        s.step(st.it)
        info = s.info()
    assert info["iters"] == st.it
    assert abs(info["objective"] - st.objective) <= 1e-6 * abs(st.objective)
    s.close()


@pytest.mark.parametrize("delta", [1e-2, 1e-3])
def test_ill_conditioned_schur(lib, gen, delta):
    """The iteration applies the cached S^-1 = G^T G (one mat-vec) while the oracle solves with the
    Cholesky factor; both are accurate to O(cond(S) eps).  Block-arrow with two nearly dependent
    constraints (A_m = A_{m-1} + delta R): cond(S) ~ 1e4 .. 1e6, and 50 iterations still match the
    oracle to 1e-9."""
    prob = gen.block_arrow(7, 3, 3, 11, seed=5)
    rng = np.random.default_rng(9)
    prob.a_val = prob.a_val.copy()
    prob.a_val[-1] = prob.a_val[-2] + delta * rng.uniform(-1, 1, prob.a_val.shape[1])
    dec = dc.decompose(prob)
    S = (dec.A / dec.D) @ dec.A.T
    cond = np.linalg.cond(S)
    assert cond > 1e3
    for form in ("primal", "dual"):
        st = admm.step(dec, admm.zero_state(dec), 1.0, form, 50)
        s = lib.Solver(prob, form=form, rho=1.0)
        s.step(50)
        for g, o in ((s.x(), st.x), (s.y(), st.y), (s.blocks("xk"), st.xk), (s.blocks("lambda"), st.lam)):
            assert rel(g, o) <= 1e-9, (form, cond, rel(g, o))
        s.close()
