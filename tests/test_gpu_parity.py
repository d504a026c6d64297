"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same seeded inputs.  Bars (BASELINE.json north_star):
  * ADMM iterates after 50 iterations: rel. error <= 1e-9 per family
    (x; y; x_k or z_k; lambda_k; v_k), reading G23;
  * objective at the 1e-4 stopping tolerance: rel. error <= 1e-6, same stop
    iteration (reading G19);
  * batched P_+: ||P_gpu - P_oracle||_F <= 1e-11 ||X||_F per matrix (Jacobi
    stops at off(A) <= 1e-15 ||A||_F; P_+ is 1-Lipschitz).
"""
import os

import numpy as np
import pytest

from oracle import admm
from oracle import decompose as dc
from oracle import psd as opsd

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def rel(g, o):
    return float(np.linalg.norm(g - o) / max(np.linalg.norm(o), 1e-300))


@pytest.fixture(scope="module")
def lib():
    import paper_1609_06068_b200 as L
    return L


# ------------------------------------------------------------------ batched projection

def check_batch(L, ks, vals, tol=1e-11):
    plan = L.PsdPlan(ks)
    out = plan.project_host(vals)
    want = opsd.project_psd_packed_batch(ks, vals)
    off = 0
    worst = 0.0
    for k in np.asarray(ks).tolist():
        s = k * (k + 1) // 2
        X = opsd.unpack_upper(vals[off:off + s], k)
        e = np.linalg.norm(opsd.unpack_upper(out[off:off + s] - want[off:off + s], k)) / max(np.linalg.norm(X), 1e-300)
        worst = max(worst, e)
        off += s
    assert worst <= tol, worst
    plan.close()
    return out


def test_batch_all_tiers_ragged(lib, gen):
    """Every order 1..100 (all tiers, odd and even, ragged CTA tails)."""
    ks = np.array(list(range(1, 101)) * 2, dtype=np.int32)
    rng = np.random.default_rng(0)
    rng.shuffle(ks)
    vals = np.concatenate([rng.standard_normal(k * (k + 1) // 2) for k in ks])
    check_batch(lib, ks, vals)


def test_batch_cfg4_mix(lib, gen):
    ks, vals = gen.psd_batch(3000, seed=7)
    check_batch(lib, ks, vals)


def test_batch_giant_orders(lib, gen):
    rng = np.random.default_rng(1)
    ks = np.array([97, 130, 257, 400, 660], dtype=np.int32)
    vals = np.concatenate([rng.standard_normal(k * (k + 1) // 2) for k in ks])
    check_batch(lib, ks, vals)


def test_batch_special_inputs(lib):
    """PSD, NSD, zero, rank-deficient, repeated eigenvalues, SPEC hand values."""
    mats = [np.array([[2.0, 0], [0, -1]]), np.eye(2), np.array([[0.0, 1], [1, 0]]), np.zeros((5, 5)),
            np.eye(7) * -3.0]
    rng = np.random.default_rng(3)
    G = rng.standard_normal((9, 3))
    mats.append(G @ G.T)                       # rank 3
    Q, _ = np.linalg.qr(rng.standard_normal((12, 12)))
    mats.append(Q @ np.diag([1, 1, 1, -1, -1, -1, 2, 2, 0, 0, 0, -2.0]) @ Q.T)  # clusters, zeros
    ks = np.array([M.shape[0] for M in mats], dtype=np.int32)
    vals = np.concatenate([opsd.pack_upper(M) for M in mats])
    out = check_batch(lib, ks, vals, tol=1e-12)
    assert np.allclose(out[:3], [2.0, 0.0, 0.0], atol=1e-15)
    assert np.allclose(out[6:9], [0.5, 0.5, 0.5], atol=1e-15)


def test_batch_device_inplace_and_empty(lib, gen):
    import torch
    ks, vals = gen.psd_batch(500, seed=9)
    plan = lib.PsdPlan(ks)
    d = torch.from_numpy(vals).cuda()
    plan.project(d, d)  # in place
    torch.cuda.synchronize()
    want = opsd.project_psd_packed_batch(ks, vals)
    assert rel(d.cpu().numpy(), want) <= 1e-11
    empty = lib.PsdPlan(np.zeros(0, np.int32))
    assert empty.values == 0
    empty.project(0, 0)
    with pytest.raises(lib.SdpError):
        lib.PsdPlan(np.array([0], np.int32))
    with pytest.raises(lib.SdpError):
        lib.PsdPlan(np.array([2000], np.int32))


@pytest.mark.slow
def test_batch_cfg4_full_size_sampled(lib, gen):
    """BASELINE configs[4] at full size (2e5 matrices) in the bench's launch
    configuration; 3000 sampled outputs compared with the oracle one by one."""
    import torch
    ks, vals = gen.config(4)
    plan = lib.PsdPlan(ks)
    d_in = torch.from_numpy(vals).cuda()
    d_out = torch.empty_like(d_in)
    plan.project(d_in, d_out)
    out = d_out.cpu().numpy()
    offs = np.concatenate([[0], np.cumsum(ks.astype(np.int64) * (ks + 1) // 2)])
    rng = np.random.default_rng(0)
    for i in rng.choice(len(ks), 3000, replace=False):
        k = int(ks[i])
        a, b = offs[i], offs[i + 1]
        want = opsd.pack_upper(opsd.project_psd(opsd.unpack_upper(vals[a:b], k)))
        X = opsd.unpack_upper(vals[a:b], k)
        assert np.linalg.norm(opsd.unpack_upper(out[a:b] - want, k)) <= 1e-11 * np.linalg.norm(X)


# ------------------------------------------------------------------ ADMM iterates

def run_pair(L, prob, form, rho, iters, dec=None):
    dec = dec or dc.decompose(prob)
    st = admm.step(dec, admm.zero_state(dec), rho, form, iters, record=True)
    s = L.Solver(prob, form=form, rho=rho)
    s.step(iters)
    return dec, st, s


def rel_inf(g, o):
    """Element-wise error of a family: max_i |g_i - o_i| / max(max_i |o_i|, tiny)."""
    return float(np.max(np.abs(g - o)) / max(float(np.max(np.abs(o))) if o.size else 0.0, 1e-300)) if o.size else 0.0


def compare_state(dec, st, s, form, tol=1e-9):
    """Reading G23 (family 2-norms) and, element by element, every entry of every family
    within tol of the family's largest entry."""
    fam = {"x": (s.x(), st.x), "y": (s.y(), st.y), "xk": (s.blocks("xk"), st.xk),
           "lambda": (s.blocks("lambda"), st.lam)}
    if form == "dual":
        fam["vk"] = (s.blocks("vk"), st.vk)
    errs = {k: rel(g, o) for k, (g, o) in fam.items()}
    errs.update({k + "_inf": rel_inf(g, o) for k, (g, o) in fam.items()})
    assert max(errs.values()) <= tol, errs
    return errs


PROBLEMS = {
    "cfg0": lambda g: g.config(0),
    "cfg1": lambda g: g.config(1),
    "arrow_odd": lambda g: g.block_arrow(7, 3, 3, 11, seed=5),
    "maxcut200": lambda g: g.maxcut_er(200, 11),
    "trace1": lambda g: g.trace_one_tridiagonal(12),
    "theta5": lambda g: g.lovasz_theta_cycle(5),
}


@pytest.mark.parametrize("name", list(PROBLEMS))
@pytest.mark.parametrize("form", ["primal", "dual"])
def test_iterates_after_50(lib, gen, name, form):
    prob = PROBLEMS[name](gen)
    dec, st, s = run_pair(lib, prob, form, 1.0, 50)
    # same decomposition on both sides
    assert [c.tolist() for c in s.cliques()] == [c.tolist() for c in dec.cliques]
    r, c = s.pattern()
    assert np.array_equal(r, dec.coord_row) and np.array_equal(c, dec.coord_col)
    compare_state(dec, st, s, form)
    # residual history and objective per iteration
    h = s.history()
    o = np.array(st.history)
    assert h.shape[0] == 50
    assert np.allclose(h[:, 0], o[:, 1], rtol=1e-7, atol=1e-14)
    assert np.allclose(h[:, 1], o[:, 2], rtol=1e-7, atol=1e-14)
    assert np.allclose(h[:, 2], o[:, 3], rtol=1e-9, atol=1e-12)
    s.close()


@pytest.mark.parametrize("form", ["primal", "dual"])
def test_iterates_long_run_warm_start_k30(lib, gen, form):
    """Cliques of 30 (the cfg2 shape, warp-register Jacobi tier, DMMA warm start):
    130 iterations across two cold restarts."""
    prob = gen.block_arrow(12, 20, 10, 40, seed=7)
    dec, st, s = run_pair(lib, prob, form, 1.0, 130)
    assert {len(c) for c in dec.cliques} == {30}
    compare_state(dec, st, s, form)
    assert s.info()["jacobi_capped"] == 0
    s.close()


@pytest.mark.parametrize("form", ["primal", "dual"])
def test_iterates_long_run_warm_start(lib, gen, form):
    """130 iterations: the warm-started Jacobi (V_prev basis) crosses two cold
    restarts (every 64 iterations); iterates still match the oracle."""
    prob = gen.config(1)
    dec, st, s = run_pair(lib, prob, form, 1.0, 130)
    compare_state(dec, st, s, form)
    info = s.info()
    assert info["jacobi_capped"] == 0
    s.close()


def test_determinism_and_reset(lib, gen):
    prob = gen.config(1)
    s = lib.Solver(prob, form="primal", rho=1.0)
    s.step(20)
    a = (s.x(), s.blocks("xk"), s.blocks("lambda"))
    s.reset()
    s.step(20)
    b = (s.x(), s.blocks("xk"), s.blocks("lambda"))
    for u, v in zip(a, b):
        assert np.array_equal(u, v)
    s.close()


def test_set_rho_matches_oracle(lib, gen):
    prob = gen.config(0)
    dec = dc.decompose(prob)
    st = admm.step(dec, admm.zero_state(dec), 1.0, "primal", 10)
    st = admm.step(dec, st, 3.0, "primal", 10)
    s = lib.Solver(prob, form="primal", rho=1.0)
    s.step(10)
    s.set_rho(3.0)
    s.step(10)
    compare_state(dec, st, s, "primal")


def test_affine_feasibility_each_iterate(lib, gen):
    """Primal iterates satisfy A x = b (E:OptCondMinYPrimal, second block row)."""
    prob = gen.config(1)
    dec = dc.decompose(prob, factor=False)
    s = lib.Solver(prob, form="primal", rho=2.0)
    for _ in range(5):
        s.step(3)
        x = s.x()
        assert np.linalg.norm(dec.A @ x - dec.b) <= 1e-10 * np.linalg.norm(dec.b)


# ------------------------------------------------------------------ solve to tolerance

SOLVES = [
    ("cfg0", "primal", 10.0), ("cfg0", "dual", 0.1),
    ("cfg1", "primal", 10.0), ("cfg1", "dual", 0.1),
    ("maxcut200", "primal", 0.1), ("maxcut200", "dual", 10.0),
]


@pytest.mark.parametrize("name,form,rho", SOLVES)
def test_solve_objective(lib, gen, name, form, rho):
    """Stop at max(eps_p, eps_d) < 1e-4 (reading G10); same stop iteration and
    objective within 1e-6 relative (north_star)."""
    prob = PROBLEMS[name](gen)
    dec = dc.decompose(prob)
    st, status = admm.solve(dec, rho, form, 1e-4, 5000)
    s = lib.Solver(prob, form=form, rho=rho, check_every=7)
    gstatus, info = s.solve(5000, 1e-4)
    assert gstatus == status
    if info["iters"] != st.it:  # reading G19 fallback: compare at the oracle's iteration
        s.reset()
        s.step(st.it)
        info = s.info()
    assert info["iters"] == st.it
    assert abs(info["objective"] - st.objective) <= 1e-6 * abs(st.objective)
    s.close()


def test_closed_forms_on_gpu(lib, gen):
    import math
    cases = [(gen.cycle_maxcut(5), -(25 + 5 * math.sqrt(5)) / 8), (gen.lovasz_theta_cycle(5), -math.sqrt(5)),
             (gen.trace_one_tridiagonal(12), 1 - 1.4 * math.cos(math.pi / 13))]
    for prob, want in cases:
        for form in ("primal", "dual"):
            s = lib.Solver(prob, form=form, rho=1.0)
            status, info = s.solve(20000, 1e-10)
            assert status == "solved"
            assert abs(info["objective"] - want) <= 1e-8 * abs(want)


# ------------------------------------------------------------------ errors

def test_error_paths(lib, gen):
    prob = gen.trace_one_tridiagonal(5)
    bad = gen.trace_one_tridiagonal(5)
    bad.c_row = bad.c_row.copy()
    bad.c_row[0] = 99
    with pytest.raises(lib.SdpError, match="INVALID_ARG"):
        lib.Solver(bad)
    dup = gen.trace_one_tridiagonal(5)
    dup.a_con = np.concatenate([dup.a_con, np.ones_like(dup.a_con)])
    dup.a_row = np.concatenate([dup.a_row, dup.a_row])
    dup.a_col = np.concatenate([dup.a_col, dup.a_col])
    dup.a_val = np.concatenate([dup.a_val, dup.a_val])
    dup.m = 2
    dup.b = np.ones(2)
    with pytest.raises(lib.SdpError, match="RANK_DEFICIENT"):
        lib.Solver(dup)
    with pytest.raises(lib.SdpError):
        lib.Solver(prob, rho=-1.0)


# ------------------------------------------------------------------ full-size configs

@pytest.mark.slow
@pytest.mark.parametrize("form", ["primal", "dual"])
def test_cfg2_full_size_50_iterations(lib, gen, form):
    """BASELINE configs[2] (n = 8010, m = 2000, 400 cliques of 30) at full size."""
    prob = gen.config(2)
    dec, st, s = run_pair(lib, prob, form, 1.0, 50)
    compare_state(dec, st, s, form)
    s.close()


def test_cfg2_pipelined_path_checkpoint_and_layout(lib, gen, tmp_path):
    """configs[2] primal runs the pipelined iteration: a checkpoint taken
    between sdp_step calls resumes bit-identically, single steps and one multi-step call
    give the same iterates, and a blob is rejected by a handle with the canonical coordinate
    layout (SDP_PIPELINE=0)."""
    import subprocess
    import sys
    prob = gen.config(2)
    a = lib.Solver(prob, form="primal", rho=10.0)
    assert a.info()["pipelined"] == 1
    a.step(4)
    blob = a.save_state()
    a.step(3)
    b = lib.Solver(prob, form="primal", rho=10.0)
    b.load_state(blob)
    for _ in range(3):
        b.step(1)
    assert np.array_equal(a.x(), b.x()) and np.array_equal(a.y(), b.y())
    assert np.array_equal(a.blocks("xk"), b.blocks("xk"))
    assert np.array_equal(a.blocks("lambda"), b.blocks("lambda"))
    a.close()
    b.close()
    path = tmp_path / "state.bin"
    path.write_bytes(bytes(blob))
    code = (
        "import sys; sys.path.insert(0, %r)\n"
        "import paper_1609_06068_b200 as L, sdp_inputs as gen\n"
        "s = L.Solver(gen.config(2), form='primal', rho=10.0)\n"
        "assert s.info()['pipelined'] == 0\n"
        "try:\n"
        "    s.load_state(open(%r, 'rb').read())\n"
        "except L.SdpError as e:\n"
        "    print('rejected', e); sys.exit(0)\n"
        "sys.exit(3)\n" % (ROOT, str(path)))
    env = dict(os.environ, SDP_PIPELINE="0")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "rejected" in r.stdout, r.stdout + r.stderr


def test_cfg2_pipelined_settle_between_calls(lib, gen):
    """The next iteration's A is left issued at the end of every sdp_step call; reading the
    state in between (getters put the finished iteration's x / y back) and then stepping on
    gives exactly the iterates of an uninterrupted run, and the state read is the iteration
    boundary (x, y of the same iteration as the residuals)."""
    prob = gen.config(2)
    a = lib.Solver(prob, form="primal", rho=10.0)
    b = lib.Solver(prob, form="primal", rho=10.0)
    a.step(6)
    for _ in range(3):
        b.step(2)
        xb, yb = b.x(), b.y()          # settle between calls
    assert b.info()["iters"] == 6
    assert np.array_equal(a.x(), xb) and np.array_equal(a.y(), yb)
    assert np.array_equal(a.blocks("lambda"), b.blocks("lambda"))
    a.step(3)
    b.step(1)
    b.set_rho(10.0)                    # a rho change settles and rebuilds r1 (same rho: same state)
    b.step(2)
    assert np.array_equal(a.x(), b.x()) and np.array_equal(a.blocks("xk"), b.blocks("xk"))
    a.close()
    b.close()


def test_cfg2_dual_pipelined_call_patterns(lib, gen):
    """Dual form on configs[2]: sdp_step(4) and two sdp_step(2) calls (pipelined schedule) give
    bit-identical iterates; single-step calls (one-graph iteration) agree to rounding."""
    prob = gen.config(2)
    a = lib.Solver(prob, form="dual", rho=0.1)
    b = lib.Solver(prob, form="dual", rho=0.1)
    c = lib.Solver(prob, form="dual", rho=0.1)
    assert a.info()["pipelined"] == 1
    a.step(4)
    b.step(2)
    b.step(2)
    for _ in range(4):
        c.step(1)
    for fam in ("xk", "lambda", "vk"):
        assert np.array_equal(a.blocks(fam), b.blocks(fam)), fam
        assert rel(c.blocks(fam), a.blocks(fam)) <= 1e-12, fam
    assert np.array_equal(a.x(), b.x()) and np.array_equal(a.y(), b.y())
    assert np.array_equal(a.history(), b.history())
    for s_ in (a, b, c):
        s_.close()


@pytest.mark.parametrize("form,rho", [("primal", 10.0), ("dual", 0.1)])
def test_pipelined_odd_block_arrow(lib, gen, form, rho):
    """A second pipelined instance with odd sizes (330 blocks of 19, arrow width 7, m = 900):
    uneven clique halves and coordinate classes; 12 iterations against the oracle."""
    prob = gen.block_arrow(330, 19, 7, 900, seed=3)
    dec = dc.decompose(prob)
    st = admm.step(dec, admm.zero_state(dec), rho, form, 12)
    s = lib.Solver(prob, form=form, rho=rho)
    assert s.info()["pipelined"] == 1
    s.step(12)
    compare_state(dec, st, s, form)
    s.close()


def test_cfg2_unpipelined_subprocess():
    """SDP_PIPELINE=0: the one-graph iteration on configs[2] still matches the oracle."""
    import subprocess
    import sys
    code = (
        "import numpy as np, sys; sys.path.insert(0, %r)\n"
        "import paper_1609_06068_b200 as L, sdp_inputs as gen\n"
        "from oracle import admm, decompose as dc\n"
        "prob = gen.config(2); dec = dc.decompose(prob)\n"
        "st = admm.step(dec, admm.zero_state(dec), 10.0, 'primal', 12)\n"
        "s = L.Solver(prob, form='primal', rho=10.0); assert s.info()['pipelined'] == 0\n"
        "s.step(12)\n"
        "r = lambda g, o: np.linalg.norm(g - o) / np.linalg.norm(o)\n"
        "e = max(r(s.x(), st.x), r(s.y(), st.y), r(s.blocks('xk'), st.xk), r(s.blocks('lambda'), st.lam))\n"
        "print(e); assert e <= 1e-9, e\n" % ROOT)
    env = dict(os.environ, SDP_PIPELINE="0")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.slow
@pytest.mark.parametrize("form,rho", [("primal", 0.1), ("dual", 10.0)])
def test_cfg3_full_size_50_iterations(lib, gen, form, rho):
    """BASELINE configs[3] (max-cut, n = 3000, cliques up to ~650: giant tridiagonal path, QL,
    CTA and register tiers; diagonal S) at the north-star bar: 50 iterations at the G11 rho of
    each form (the giant cliques' projection inputs develop dense bands of negative
    eigenvalues: clusters beyond one vector-kernel group, cut at their largest gaps)."""
    prob = gen.config(3)
    dec = dc.decompose(prob)
    st = admm.step(dec, admm.zero_state(dec), rho, form, 50, record=True)
    s = lib.Solver(prob, form=form, rho=rho)
    s.step(50)
    assert s.info()["s_diagonal"] == 1
    compare_state(dec, st, s, form)
    h = s.history()
    o = np.array(st.history)
    assert np.allclose(h[:, 0], o[:, 1], rtol=1e-7, atol=1e-14)
    assert np.allclose(h[:, 1], o[:, 2], rtol=1e-7, atol=1e-14)
    assert np.allclose(h[:, 2], o[:, 3], rtol=1e-9, atol=1e-12)
    s.close()


@pytest.mark.slow
@pytest.mark.parametrize("form,rho", [("primal", 10.0), ("dual", 0.1)])
def test_cfg2_solve_to_tolerance(lib, gen, form, rho):
    """BASELINE configs[2] solved to max(eps_p, eps_d) < 1e-4 (reading G10) at the G11 rho
    (primal 759, dual 402 iterations): same stop iteration and objective within
    1e-6 relative (north_star; reading G19 fallback if the stop iteration differed)."""
    prob = gen.config(2)
    dec = dc.decompose(prob)
    st, status = admm.solve(dec, rho, form, 1e-4, 3000)
    assert status == "solved"
    s = lib.Solver(prob, form=form, rho=rho)
    gstatus, info = s.solve(3000, 1e-4)
    assert gstatus == status
    if info["iters"] != st.it:
        s.reset()
        s.step(st.it)
        info = s.info()
    assert info["iters"] == st.it
    assert abs(info["objective"] - st.objective) <= 1e-6 * abs(st.objective)
    # the recovered SDP pair at the stop (Remark 1): duality gap at solver accuracy
    X, yhat, _ = admm.recovered_pair(dec, st, rho, form)
    Xg, yg = s.sdp_x(), s.sdp_y()
    assert rel(Xg, dec.unsvec_pattern(X)) <= 1e-6 and rel(yg, yhat) <= 1e-6
    s.close()


@pytest.mark.parametrize("name", ["cfg0", "maxcut200", "theta5", "arrow_odd"])
def test_psd_completion_matches_oracle(lib, gen, name):
    """sdp_complete_x (Theorem 1) against oracle.completion on the same
    elimination order: agreement on and off the pattern; after a primal solve the completion
    is PSD to solver accuracy (Grone)."""
    from oracle import chordal
    from oracle import completion
    prob = PROBLEMS[name](gen)
    s = lib.Solver(prob, form="primal", rho=1.0)
    s.solve(20000, 1e-7)
    order_l = s.elimination_order()
    adj = chordal.aggregate_adjacency(prob)
    order, later, filled = chordal.minimum_degree_elimination(adj)
    assert np.array_equal(order_l, np.asarray(order))
    n = prob.n
    known = filled | np.eye(n, dtype=bool)
    r, c = s.pattern()
    X = np.zeros((n, n))
    xm = s.x_mat()
    X[r, c] = xm
    X[c, r] = xm
    # the converged blocks are singular to solver accuracy: drop eigenvalues below 1e-8 max|lambda|
    # on both sides (a kept eigenvalue at the noise level would amplify rounding by its inverse)
    want = completion.complete_psd(X, known, order, later, rtol=1e-8)
    got = s.complete_x(rtol=1e-8)
    assert np.allclose(got[known], X[known], rtol=0, atol=0)
    # an eigenvalue of a conditional block lying at the 1e-8 cutoff can be dropped on one side and
    # kept on the other (the two eigensolvers round differently): each such flip moves the
    # completion by at most the cutoff, rtol * |lambda_max|, so agreement is asserted to 5 * rtol
    assert np.linalg.norm(got - want) <= 5e-8 * np.linalg.norm(want)
    assert np.linalg.eigvalsh(got).min() >= -1e-5 * np.linalg.norm(got)
    s.close()


# ------------------------------------------------------------------ giant (block-Jacobi) tier

def test_giant_tier_iterates_warm_restarts(lib, gen):
    """Max-cut on ER(700, 4/n): cliques up to ~150 go to the giant tier
    (block Jacobi + DMMA); 70 iterations cross a cold restart of the warm start."""
    prob = gen.maxcut_er(700, 21)
    dec = dc.decompose(prob)
    assert max(len(c) for c in dec.cliques) >= 97
    for form, rho in (("primal", 0.1), ("dual", 10.0)):
        st = admm.step(dec, admm.zero_state(dec), rho, form, 70)
        s = lib.Solver(prob, form=form, rho=rho)
        s.step(70)
        compare_state(dec, st, s, form)
        assert s.info()["jacobi_capped"] == 0
        s.close()


def test_giant_tier_determinism(lib, gen):
    prob = gen.maxcut_er(700, 21)
    s = lib.Solver(prob, form="primal", rho=0.1)
    s.step(12)
    a = (s.x(), s.blocks("xk"), s.blocks("lambda"))
    s.reset()
    s.step(12)
    b = (s.x(), s.blocks("xk"), s.blocks("lambda"))
    for u, v in zip(a, b):
        assert np.array_equal(u, v)
    s.close()


def test_giant_tier_small_orders_subprocess(tmp_path):
    """SDP_GIANT_MIN=33 routes every order 33..100 through the giant tier
    (padding 33 -> 64 etc.); batch results still match the oracle."""
    import subprocess
    import sys
    code = (
        "import numpy as np, sys; sys.path.insert(0, %r)\n"
        "import paper_1609_06068_b200 as L\n"
        "from oracle import psd as opsd\n"
        "rng = np.random.default_rng(5)\n"
        "ks = np.array(list(range(30, 101)), np.int32); rng.shuffle(ks)\n"
        "vals = np.concatenate([rng.standard_normal(k*(k+1)//2) for k in ks])\n"
        "p = L.PsdPlan(ks); out = p.project_host(vals)\n"
        "want = opsd.project_psd_packed_batch(ks, vals)\n"
        "e = np.linalg.norm(out - want) / np.linalg.norm(want)\n"
        "print(e); assert e <= 1e-12, e\n" % ROOT)
    env = dict(os.environ, SDP_GIANT_MIN="33")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr


# ------------------------------------------------------------------ giant tier, tridiagonal path

def test_gtrd_batch_orders_and_structured(lib, gen):
    """Giant orders take the tridiagonal path (Householder + bisection + inverse
    iteration + WY back-transform): random orders 65..800, structured inputs
    (zero, identity, repeated / clustered eigenvalues, rank one, +-pairs; the big
    clusters go to the block-Jacobi fallback) and k = 801 (> the path's maximum,
    block Jacobi), against the oracle."""
    rng = np.random.default_rng(12)
    mats = []
    for k in (65, 130):
        mats += _structured(k, rng)
    ks = [66, 97, 128, 129, 255, 400, 631, 800, 801]
    vals = [rng.standard_normal(k * (k + 1) // 2) for k in ks]
    ks = np.array([M.shape[0] for M in mats] + ks, dtype=np.int32)
    vals = np.concatenate([opsd.pack_upper(M) for M in mats] + vals)
    check_batch(lib, ks, vals, tol=1e-12)


def test_gtrd_clusters_beyond_a_group(lib, gen):
    """Clusters larger than a vector-kernel group (cap(k) = min(128, 26000/k - 2)):
    a dense band of distinct eigenvalues is cut at its largest gaps (tridiagonal path);
    exactly repeated eigenvalues on both sides of 0 cannot be cut safely and go to the
    block-Jacobi fallback.  Both against the oracle."""
    rng = np.random.default_rng(21)
    mats = []
    k = 500                                   # cap = 50
    Q, _ = np.linalg.qr(rng.standard_normal((k, k)))
    lam = np.concatenate([np.linspace(-1.2, -1.0, 200), np.linspace(1.0, 1.5, 300)])
    mats.append((Q * lam) @ Q.T)              # bands of 200 and 300: cuts at gaps ~5e-4 ||T||
    k = 300                                   # cap = 84
    Q, _ = np.linalg.qr(rng.standard_normal((k, k)))
    lam = np.repeat([-1.0, 2.0], 150)
    mats.append((Q * lam) @ Q.T)              # two multiplicity-150 eigenvalues: fallback
    ks = np.array([M.shape[0] for M in mats], dtype=np.int32)
    vals = np.concatenate([opsd.pack_upper(M) for M in mats])
    check_batch(lib, ks, vals, tol=1e-11)


def _giant_env_batch(env_extra):
    import subprocess
    import sys
    code = (
        "import numpy as np, sys; sys.path.insert(0, %r)\n"
        "import paper_1609_06068_b200 as L\n"
        "from oracle import psd as opsd\n"
        "rng = np.random.default_rng(6)\n"
        "ks = np.array([65, 90, 150, 333, 64, 20], np.int32)\n"
        "vals = np.concatenate([rng.standard_normal(k*(k+1)//2) for k in ks])\n"
        "out = L.PsdPlan(ks).project_host(vals)\n"
        "want = opsd.project_psd_packed_batch(ks, vals)\n"
        "e = np.linalg.norm(out - want) / np.linalg.norm(want)\n"
        "print(e); assert e <= 1e-12, e\n" % ROOT)
    env = dict(os.environ, **env_extra)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr


def test_gtrd_forced_fallback_subprocess():
    """SDP_GTRD_FORCE_FALLBACK=1 marks every matrix of the tridiagonal path failed:
    the block-Jacobi kernel redoes them (GiantDev::only) in the same call."""
    _giant_env_batch({"SDP_GTRD_FORCE_FALLBACK": "1"})


@pytest.mark.parametrize("sbr_min", ["65", "200"])
def test_gtrd_two_stage_and_mixed_subprocess(sbr_min):
    """SDP_GTRD_SBR_MIN=65: every giant takes the two-stage reduction (dense -> band by blocked
    QR panels, band -> tridiagonal by bulge chasing, back-transform Q1 Q2); =200: orders below 200
    the one-stage reduction, the others the two-stage one, in the same call."""
    _giant_env_batch({"SDP_GTRD_SBR_MIN": sbr_min})


def test_gtrd_two_stage_admm_subprocess():
    """The two-stage reduction inside the ADMM iteration (max-cut, giant cliques, both forms)."""
    import subprocess
    import sys
    code = (
        "import numpy as np, sys; sys.path.insert(0, %r)\n"
        "import paper_1609_06068_b200 as L, sdp_inputs as gen\n"
        "from oracle import admm, decompose as dc\n"
        "prob = gen.maxcut_er(700, 21); dec = dc.decompose(prob)\n"
        "r = lambda g, o: float(np.max(np.abs(g - o)) / np.max(np.abs(o)))\n"
        "for form, rho in (('primal', 0.1), ('dual', 10.0)):\n"
        "    st = admm.step(dec, admm.zero_state(dec), rho, form, 30)\n"
        "    s = L.Solver(prob, form=form, rho=rho); s.step(30)\n"
        "    e = max(r(s.x(), st.x), r(s.y(), st.y), r(s.blocks('xk'), st.xk), r(s.blocks('lambda'), st.lam))\n"
        "    print(form, e); assert e <= 1e-9, e\n" % ROOT)
    env = dict(os.environ, SDP_GTRD_SBR_MIN="65")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout + r.stderr


def test_giant_block_jacobi_only_subprocess():
    """SDP_GIANT_METHOD=jacobi: the giant tier without the tridiagonal path."""
    _giant_env_batch({"SDP_GIANT_METHOD": "jacobi"})


# ------------------------------------------------------------------ tridiagonal-QL tier

def _structured(k, rng):
    """Degenerate inputs for the QL path: zero, identity, repeated / clustered
    eigenvalues, rank one, +-pairs, sparse (max-cut-like identity + few entries)."""
    Q, _ = np.linalg.qr(rng.standard_normal((k, k)))
    lam = np.repeat([2.0, -1.0, 0.0, 1.0 + 1e-9], (k + 3) // 4)[:k]
    sparse = np.eye(k)
    for _ in range(k // 4):
        i, j = rng.integers(0, k, 2)
        if i != j:
            sparse[i, j] = sparse[j, i] = rng.uniform(-0.3, 0.3)
    v = rng.standard_normal(k)
    pm = Q @ np.diag(np.concatenate([np.full(k // 2, 3.0), np.full(k - k // 2, -3.0)])) @ Q.T
    return [np.zeros((k, k)), np.eye(k), Q @ np.diag(lam) @ Q.T, np.outer(v, v), pm, sparse, -np.eye(k) * 0.5]


def test_trd_tier_batch_many(lib, gen):
    """>= 2048 matrices per size range select the tridiagonal-QL tier; random orders
    17..64 (odd and even) plus degenerate structured inputs, against the oracle."""
    rng = np.random.default_rng(11)
    mats = []
    for k in (17, 23, 32, 33, 47, 64):
        mats += _structured(k, rng)
    ks = list(rng.integers(17, 65, 4400))
    vals = [rng.standard_normal(k * (k + 1) // 2) for k in ks]
    ks = np.array([M.shape[0] for M in mats] + ks, dtype=np.int32)
    vals = np.concatenate([opsd.pack_upper(M) for M in mats] + vals)
    check_batch(lib, ks, vals, tol=1e-12)


def test_trd16_tier_batch_many(lib, gen):
    """>= 2048 matrices of order 9..16 select the KP = 16 tridiagonal-QL tier (half-warp groups in
    the tridiagonalization, eight selected eigenvectors per matrix, one warp per apply); random
    orders plus the degenerate structured inputs, against the oracle."""
    rng = np.random.default_rng(16)
    mats = []
    for k in (9, 12, 15, 16):
        mats += _structured(k, rng)
    ks = list(rng.integers(9, 17, 4400))
    vals = [rng.standard_normal(k * (k + 1) // 2) for k in ks]
    ks = np.array([M.shape[0] for M in mats] + ks, dtype=np.int32)
    vals = np.concatenate([opsd.pack_upper(M) for M in mats] + vals)
    check_batch(lib, ks, vals, tol=1e-12)


def test_trd8_tier_batch_many(lib, gen):
    """>= 2048 matrices of order 5..8 select the KP = 8 tridiagonal-QL tier (four matrices per warp in
    the tridiagonalization, at most four selected eigenvectors, one warp per apply); random orders
    plus the degenerate structured inputs, against the oracle."""
    rng = np.random.default_rng(8)
    mats = []
    for k in (5, 6, 7, 8):
        mats += _structured(k, rng)
    ks = list(rng.integers(5, 9, 4400))
    vals = [rng.standard_normal(k * (k + 1) // 2) for k in ks]
    ks = np.array([M.shape[0] for M in mats] + ks, dtype=np.int32)
    vals = np.concatenate([opsd.pack_upper(M) for M in mats] + vals)
    check_batch(lib, ks, vals, tol=1e-12)


def test_trd_tiers_inplace_and_deterministic(lib, gen):
    """Every QL tier (KP = 8, 16, 32, 64: >= 2048 matrices per size range, the halving
    tridiagonalization cascade, twisted eigenvectors): a projection in place (d_in == d_out, the
    apply epilogue reads the side-1 input where it writes) equals the out-of-place one bit for bit,
    two plans agree bit for bit, and the result matches the oracle."""
    import torch
    rng = np.random.default_rng(21)
    ks = np.concatenate([rng.integers(lo, hi + 1, 2100) for lo, hi in ((5, 8), (9, 16), (17, 32), (33, 64))])
    rng.shuffle(ks)
    ks = ks.astype(np.int32)
    vals = np.concatenate([rng.standard_normal(k * (k + 1) // 2) for k in ks])
    pa, pb = lib.PsdPlan(ks), lib.PsdPlan(ks)
    d_in = torch.from_numpy(vals).cuda()
    out_a = torch.empty_like(d_in)
    pa.project(d_in, out_a)
    out_b = torch.empty_like(d_in)
    pb.project(d_in, out_b)
    d_ip = d_in.clone()
    pa.project(d_ip, d_ip)
    torch.cuda.synchronize()
    a_, b_, ip = out_a.cpu().numpy(), out_b.cpu().numpy(), d_ip.cpu().numpy()
    assert np.array_equal(a_, b_)
    assert np.array_equal(a_, ip)
    want = opsd.project_psd_packed_batch(ks, vals)
    assert np.linalg.norm(a_ - want) <= 1e-12 * np.linalg.norm(want)
    pa.close()
    pb.close()


def test_trd_tier_admm_subprocess():
    """SDP_PSD_TIERS=trd: every clique of order 17..64 takes the QL tier inside
    the ADMM iteration (primal and dual), iterates match the oracle."""
    import subprocess
    import sys
    code = (
        "import numpy as np, sys; sys.path.insert(0, %r)\n"
        "import paper_1609_06068_b200 as L, sdp_inputs as gen\n"
        "from oracle import admm, decompose as dc\n"
        "prob = gen.maxcut_er(400, 3); dec = dc.decompose(prob)\n"
        "ks = [len(c) for c in dec.cliques]; assert sum(17 <= k <= 64 for k in ks) >= 5, ks\n"
        "for form, rho in (('primal', 0.1), ('dual', 10.0)):\n"
        "    st = admm.step(dec, admm.zero_state(dec), rho, form, 30)\n"
        "    s = L.Solver(prob, form=form, rho=rho); s.step(30)\n"
        "    r = lambda g, o: np.linalg.norm(g - o) / np.linalg.norm(o)\n"
        "    e = max(r(s.x(), st.x), r(s.blocks('xk'), st.xk), r(s.blocks('lambda'), st.lam))\n"
        "    print(form, e); assert e <= 1e-9, (form, e)\n" % ROOT)
    env = dict(os.environ, SDP_PSD_TIERS="trd")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout + r.stderr


def test_trd_tier_inline_ql_fallback_subprocess():
    """SDP_TRD_FORCE_FALLBACK=1: every matrix of the QL tier takes the checked
    fallback (QL with eigenvector accumulation inside the apply kernel); results
    still match the oracle."""
    import subprocess
    import sys
    code = (
        "import numpy as np, sys; sys.path.insert(0, %r)\n"
        "import paper_1609_06068_b200 as L\n"
        "from oracle import psd as opsd\n"
        "rng = np.random.default_rng(4)\n"
        "ks = rng.integers(5, 65, 3000).astype(np.int32)\n"
        "vals = np.concatenate([rng.standard_normal(k*(k+1)//2) for k in ks])\n"
        "out = L.PsdPlan(ks).project_host(vals)\n"
        "want = opsd.project_psd_packed_batch(ks, vals)\n"
        "e = np.linalg.norm(out - want) / np.linalg.norm(want)\n"
        "print(e); assert e <= 1e-12, e\n" % ROOT)
    env = dict(os.environ, SDP_TRD_FORCE_FALLBACK="1", SDP_PSD_TIERS="trd")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.parametrize("variant", [{"SDP_TRD_REG": "0"}, {"SDP_TRD_QLRSQ": "0"}, {"SDP_TRD_SPLIT": "0"}])
def test_trd_tier_variants_subprocess(variant):
    """The A/B variants of the QL tier kept for measurement (shared-memory
    tridiagonalization; sqrt + reciprocal QL rotations) stay correct: random orders
    17..64 plus the degenerate structured inputs, against the oracle."""
    import subprocess
    import sys
    code = (
        "import numpy as np, sys; sys.path.insert(0, %r); sys.path.insert(0, %r)\n"
        "import paper_1609_06068_b200 as L\n"
        "from oracle import psd as opsd\n"
        "from test_gpu_parity import _structured\n"
        "rng = np.random.default_rng(5)\n"
        "mats = [M for k in (5, 8, 9, 16, 17, 32, 33, 64) for M in _structured(k, rng)]\n"
        "ks = list(rng.integers(5, 65, 3000))\n"
        "vals = [rng.standard_normal(k*(k+1)//2) for k in ks]\n"
        "ks = np.array([M.shape[0] for M in mats] + ks, dtype=np.int32)\n"
        "vals = np.concatenate([opsd.pack_upper(M) for M in mats] + vals)\n"
        "out = L.PsdPlan(ks).project_host(vals)\n"
        "want = opsd.project_psd_packed_batch(ks, vals)\n"
        "e = np.linalg.norm(out - want) / np.linalg.norm(want)\n"
        "print(e); assert e <= 1e-12, e\n" % (ROOT, os.path.dirname(os.path.abspath(__file__))))
    env = dict(os.environ, SDP_PSD_TIERS="trd", **variant)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout + r.stderr


def test_trd_ql_fused_matches_tql_subprocess():
    """The QL kernel's chain with the deflation scan fused into the sweep and the operands loaded
    one rotation ahead makes tql's rotations and deflation decisions (the two differ only in where
    the compiler contracts a multiply-add): with and without it (SDP_TRD_QLFUSED=0) the QL tier's
    projections agree to 1e-13 and both match the oracle, on random orders 17..64 and the
    structured spectra (repeated, clustered, rank-deficient, sparse) that exercise early deflation
    and block ends."""
    import subprocess
    import sys
    import tempfile
    code = (
        "import numpy as np, sys; sys.path.insert(0, %r); sys.path.insert(0, %r)\n"
        "import paper_1609_06068_b200 as L\n"
        "from oracle import psd as opsd\n"
        "from test_gpu_parity import _structured\n"
        "rng = np.random.default_rng(11)\n"
        "mats = [M for k in (9, 16, 17, 24, 32, 33, 48, 64) for M in _structured(k, rng)]\n"
        "ks = list(rng.integers(9, 65, 3000))\n"
        "vals = [rng.standard_normal(k*(k+1)//2) for k in ks]\n"
        "ks = np.array([M.shape[0] for M in mats] + ks, dtype=np.int32)\n"
        "vals = np.concatenate([opsd.pack_upper(M) for M in mats] + vals)\n"
        "out = L.PsdPlan(ks).project_host(vals)\n"
        "want = opsd.project_psd_packed_batch(ks, vals)\n"
        "assert np.linalg.norm(out - want) <= 1e-12 * np.linalg.norm(want)\n"
        "np.save(sys.argv[1], out)\n" % (ROOT, os.path.dirname(os.path.abspath(__file__))))
    outs = []
    with tempfile.TemporaryDirectory() as td:
        for flag in ("1", "0"):
            f = os.path.join(td, f"o{flag}.npy")
            env = dict(os.environ, SDP_TRD_QLFUSED=flag, SDP_PSD_TIERS="trd")
            r = subprocess.run([sys.executable, "-c", code, f], env=env, capture_output=True, text=True, timeout=900)
            assert r.returncode == 0, r.stdout + r.stderr
            outs.append(np.load(f))
    assert np.linalg.norm(outs[0] - outs[1]) <= 1e-13 * np.linalg.norm(outs[1])


def test_trd_fused_eigenvectors_bit_identical_subprocess():
    """Singleton eigenvectors formed in the apply kernel's shared memory (SDP_TRD_FUSEVEC=1) are the same
    twisted factorization as k_trd_invit's (default, vectors through the workspace),
    so the projections agree bit for bit on every QL tier (orders 5..64, >= 2048 matrices per size
    range) plus the structured spectra whose clusters still go through inverse iteration; both
    match the oracle."""
    import subprocess
    import sys
    import tempfile
    code = (
        "import numpy as np, sys; sys.path.insert(0, %r); sys.path.insert(0, %r)\n"
        "import paper_1609_06068_b200 as L\n"
        "from oracle import psd as opsd\n"
        "from test_gpu_parity import _structured\n"
        "rng = np.random.default_rng(23)\n"
        "mats = [M for k in (5, 8, 9, 16, 17, 24, 32, 33, 48, 64) for M in _structured(k, rng)]\n"
        "ks = list(np.concatenate([rng.integers(lo, hi + 1, 2100) for lo, hi in ((5, 8), (9, 16), (17, 32), (33, 64))]))\n"
        "vals = [rng.standard_normal(k*(k+1)//2) for k in ks]\n"
        "ks = np.array([M.shape[0] for M in mats] + ks, dtype=np.int32)\n"
        "vals = np.concatenate([opsd.pack_upper(M) for M in mats] + vals)\n"
        "out = L.PsdPlan(ks).project_host(vals)\n"
        "want = opsd.project_psd_packed_batch(ks, vals)\n"
        "assert np.linalg.norm(out - want) <= 1e-12 * np.linalg.norm(want)\n"
        "np.save(sys.argv[1], out)\n" % (ROOT, os.path.dirname(os.path.abspath(__file__))))
    outs = []
    with tempfile.TemporaryDirectory() as td:
        # default; singletons in the apply kernel; clusters scheduled first (SDP_TRD_INVIT_ORDER=1)
        for i, extra in enumerate(({}, {"SDP_TRD_FUSEVEC": "1"}, {"SDP_TRD_INVIT_ORDER": "1"})):
            f = os.path.join(td, f"o{i}.npy")
            env = dict(os.environ, **extra)
            r = subprocess.run([sys.executable, "-c", code, f], env=env, capture_output=True, text=True, timeout=900)
            assert r.returncode == 0, r.stdout + r.stderr
            outs.append(np.load(f))
    assert np.array_equal(outs[0], outs[1])
    assert np.array_equal(outs[0], outs[2])


# ------------------------------------------------------------------ adaptive rho

@pytest.mark.parametrize("form,rho", [("primal", 1.0), ("dual", 1.0), ("primal", 50.0)])
def test_solve_adaptive_rho(lib, gen, form, rho):
    """Residual balancing inside sdp_solve (every check_every = 10 iterations,
    mu = 10, tau = 2) against the oracle's same rule: same stop iteration, same
    final rho, objective within 1e-6."""
    prob = gen.config(1)
    dec = dc.decompose(prob)
    st, status = admm.solve(dec, rho, form, 1e-4, 5000, adapt=(10.0, 2.0, 10))
    s = lib.Solver(prob, form=form, rho=rho, check_every=10, adapt_rho=True)
    gstatus, info = s.solve(5000, 1e-4)
    assert gstatus == status == "solved"
    assert info["iters"] == st.it
    assert info["rho"] == st.rho
    assert abs(info["objective"] - st.objective) <= 1e-6 * abs(st.objective)
    s.close()


@pytest.mark.parametrize("form,rho", [("primal", 1.0), ("dual", 1.0)])
def test_cfg2_solve_adaptive_rho_pipelined_handle(lib, gen, form, rho):
    """sdp_solve with residual balancing on configs[2] (a pipelined handle: the primal solve runs
    the pipelined schedule with rho changes between chunks, the dual solve the one-graph
    iteration): 40 iterations against the oracle's same rule."""
    prob = gen.config(2)
    dec = dc.decompose(prob)
    st, status = admm.solve(dec, rho, form, 1e-12, 40, adapt=(10.0, 2.0, 10))
    s = lib.Solver(prob, form=form, rho=rho, check_every=10, adapt_rho=True)
    assert s.info()["pipelined"] == 1
    gstatus, info = s.solve(40, 1e-12)
    assert gstatus == status
    assert info["iters"] == st.it == 40
    assert info["rho"] == st.rho
    compare_state(dec, st, s, form)
    s.close()


# ------------------------------------------------------------------ checkpoint / resume

@pytest.mark.parametrize("name,form", [("cfg1", "primal"), ("cfg1", "dual"), ("maxcut200", "primal"),
                                       ("arrow30", "dual")])
def test_checkpoint_resume_bit_identical(lib, gen, name, form):
    """save_state after 37 iterations, continue 29 more; a fresh handle that loads
    the blob and runs 29 iterations ends bit-identical (x, y, blocks, history,
    iteration count); the resumed run also matches the oracle."""
    prob = gen.block_arrow(12, 20, 10, 40, seed=7) if name == "arrow30" else PROBLEMS[name](gen)
    a = lib.Solver(prob, form=form, rho=1.0)
    a.step(37)
    blob = a.save_state()
    a.step(29)
    b = lib.Solver(prob, form=form, rho=1.0)
    b.load_state(blob)
    b.step(29)
    for fam in ("xk", "lambda") + (("vk",) if form == "dual" else ()):
        assert np.array_equal(a.blocks(fam), b.blocks(fam)), fam
    assert np.array_equal(a.x(), b.x()) and np.array_equal(a.y(), b.y())
    assert np.array_equal(a.history(), b.history())
    assert a.info()["iters"] == b.info()["iters"] == 66
    dec = dc.decompose(prob)
    st = admm.step(dec, admm.zero_state(dec), 1.0, form, 66)
    compare_state(dec, st, b, form)
    # a blob of another problem / form is rejected
    c = lib.Solver(gen.config(0), form=form, rho=1.0)
    with pytest.raises(lib.SdpError, match="INVALID_ARG"):
        c.load_state(blob)
    for s_ in (a, b, c):
        s_.close()


def test_two_handles_bit_identical(lib, gen):
    """Setup is deterministic too: two handles of the same problem produce
    bit-identical iterates (the dense S = A D^-1 A^T tiles write each (i, j)
    once)."""
    prob = gen.block_arrow(12, 20, 10, 40, seed=7)
    for form in ("primal", "dual"):
        a = lib.Solver(prob, form=form, rho=1.0)
        b = lib.Solver(prob, form=form, rho=1.0)
        a.step(12)
        b.step(12)
        assert np.array_equal(a.x(), b.x()) and np.array_equal(a.blocks("xk"), b.blocks("xk"))
        a.close()
        b.close()


# ------------------------------------------------------------------ SDPA input (reader part)

@pytest.mark.parametrize("fname,want", [("theta_c5.dat-s", -5 ** 0.5),
                                        ("maxcut_c5.dat-s", -(25 + 5 * 5 ** 0.5) / 8),
                                        ("mixed_blocks.dat-s", -1.5)])
def test_sdpa_golden_solves(lib, fname, want):
    from paper_1609_06068_b200 import sdpa
    p = sdpa.read_sdpa(os.path.join(ROOT, "tests", "golden", fname))
    for form in ("primal", "dual"):
        s = lib.Solver(p, form=form, rho=1.0)
        status, info = s.solve(20000, 1e-10)
        assert status == "solved"
        assert abs(info["objective"] - want) <= 1e-8 * abs(want), (form, info["objective"])
        s.close()


def test_batch_host_pinned_pipeline(lib, gen):
    """Pinned host buffers take the pipelined host path (four sub-plans, copies overlapping the
    projections): every matrix equals the oracle's projection, and the pageable path agrees."""
    import torch
    rng = np.random.default_rng(21)
    ks = rng.choice(np.array([3, 8, 13, 24], dtype=np.int32), 20000)
    offs = np.concatenate([[0], np.cumsum(ks.astype(np.int64) * (ks + 1) // 2)])
    vals = rng.standard_normal(offs[-1])
    plan = lib.PsdPlan(ks)
    hin_t = torch.empty(vals.size, dtype=torch.float64, pin_memory=True)
    hout_t = torch.empty(vals.size, dtype=torch.float64, pin_memory=True)
    hin_t.numpy()[...] = vals
    out = plan.project_host(hin_t.numpy(), hout_t.numpy()).copy()
    out2 = plan.project_host(hin_t.numpy(), hout_t.numpy()).copy()  # reuses the sub-plans
    assert np.array_equal(out, out2)
    pageable = plan.project_host(vals)
    assert np.max(np.abs(out - pageable)) <= 1e-11 * np.max(np.abs(vals))
    for i in rng.choice(len(ks), 300, replace=False):
        k = int(ks[i])
        a, b = offs[i], offs[i + 1]
        X = opsd.unpack_upper(vals[a:b], k)
        want = opsd.project_psd(X)
        assert np.linalg.norm(opsd.unpack_upper(out[a:b], k) - want) <= 1e-11 * max(np.linalg.norm(X), 1e-300)
    plan.close()
