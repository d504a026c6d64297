"""Pins for the oracle's residuals eps_p, eps_d (oracle/admm.py; reading G9).

The paper never defines eps_p / eps_d: it defers to boyd2011; the
reading taken is SPEC.md S:312.  Nothing here calls the oracle's residual code
to produce an expected value.  The pins are:
  * hand-simulated recursions on 1x1 and 2x2 problems, both forms, with
    the expected iterates and residuals derived by hand in
    tests/golden/residuals_hand.json;
  * static fixed points: a state that the iteration maps to itself has
    (eps_p, eps_d) = (0, 0);
  * a recomputation of G9 from dense n x n matrices with explicit clique
    selectors E_k (x_k = vec(E_k X E_k^T)), Frobenius norms and
    no svec / scatter / gather code of the oracle;
  * primal form: the ADMM dual-residual identity.  The x-update of Algorithm 1
    (E:OptCondMinYPrimal) is the minimiser of
    <c,x> + rho/2 sum ||x_k - H_k x + lam_k/rho||^2 on A x = b; its optimality
    condition with lam^(n) = lam^(n-1) + rho (x_k^(n) - H_k x) (E:LambdakUpdate)
    gives  C - A*(yhat) - sum_k E_k^T Lam_k^(n) E_k = -rho sum_k E_k^T (X_k^(n) - X_k^(n-1)) E_k
    with yhat = -rho y_kkt, i.e. rho ||sum H_k^T (x_k^(n) - x_k^(n-1))|| is the
    stationarity error of the recovered SDP dual (yhat, Z_k = Lam_k) -- a
    mathematical identity independent of how the oracle evaluates G9.
A dropped rho, a wrong previous-iterate convention, a wrong denominator or a
wrong svec scaling in oracle/admm.py fails at least one of these.
"""
import math

import numpy as np
import pytest

from oracle import admm
from oracle import decompose as dc
import sdp_inputs
from tests.helpers import golden


# ------------------------------------------------------------------ problems from dense matrices

def problem_from_dense(C, A_list, b, name="hand"):
    """sdp_inputs.Problem (COO, upper triangle, unscaled entries) from dense symmetric matrices."""
    C = np.asarray(C, float)
    n = C.shape[0]
    iu, ju = np.triu_indices(n)
    keep = C[iu, ju] != 0
    con, ar, ac, av = [], [], [], []
    for i, Ai in enumerate(A_list):
        Ai = np.asarray(Ai, float)
        nz = Ai[iu, ju] != 0
        con += [i] * int(nz.sum())
        ar += iu[nz].tolist()
        ac += ju[nz].tolist()
        av += Ai[iu, ju][nz].tolist()
    return sdp_inputs.Problem(
        name=name, n=n, m=len(A_list),
        c_row=iu[keep].astype(np.int32), c_col=ju[keep].astype(np.int32), c_val=C[iu, ju][keep],
        b=np.asarray(b, float), a_fmt="coo", a_con=np.array(con, np.int32),
        a_row=np.array(ar, np.int32), a_col=np.array(ac, np.int32), a_val=np.array(av, float))


# ------------------------------------------------------------------ dense helpers (test-side, independent)

def local_packed(k):
    """(row, col) of the packed upper column-major local order (reading G14)."""
    rr, cc = [], []
    for j in range(k):
        for i in range(j + 1):
            rr.append(i)
            cc.append(j)
    return np.array(rr), np.array(cc)


def block_matrix(v, k):
    """Dense k x k symmetric matrix of a clique block stored as svec (off-diagonal x sqrt 2)."""
    r, c = local_packed(k)
    M = np.zeros((k, k))
    vals = np.where(r == c, v, v / math.sqrt(2.0))
    M[r, c] = vals
    M[c, r] = vals
    return M


def pattern_matrix(dec, x):
    """Dense n x n symmetric matrix of a pattern vector (svec on the extended pattern)."""
    X = np.zeros((dec.n, dec.n))
    r, c = dec.coord_row, dec.coord_col
    vals = np.where(r == c, x, x / math.sqrt(2.0))
    X[r, c] = vals
    X[c, r] = vals
    return X


def selector(clique, n):
    """E_k: |C_k| x n, rows e_i^T for the clique's vertices in natural order."""
    E = np.zeros((len(clique), n))
    E[np.arange(len(clique)), np.asarray(clique)] = 1.0
    return E


def dense_data(prob):
    """C and A_1..A_m as dense symmetric matrices (unscaled entries)."""
    n = prob.n
    C = np.zeros((n, n))
    C[prob.c_row, prob.c_col] = prob.c_val
    C[prob.c_col, prob.c_row] = prob.c_val
    As = np.zeros((prob.m, n, n))
    if prob.a_fmt == "dense":
        for i in range(prob.m):
            As[i, prob.a_row, prob.a_col] = prob.a_val[i]
            As[i, prob.a_col, prob.a_row] = prob.a_val[i]
    else:
        As[prob.a_con, prob.a_row, prob.a_col] = prob.a_val
        As[prob.a_con, prob.a_col, prob.a_row] = prob.a_val
    return C, As


def dense_residuals(dec, prev, cur, rho, form):
    """G9 from dense matrices: eps_p, eps_d of the iteration prev -> cur."""
    n = dec.n
    X = pattern_matrix(dec, cur.x)
    sq_diff = sq_a = sq_b = 0.0
    S_diff = np.zeros((n, n))
    S_lam = np.zeros((n, n))
    for k, C in enumerate(dec.cliques):
        E = selector(C, n)
        kk = len(C)
        sl = slice(dec.offsets[k], dec.offsets[k + 1])
        Xk = block_matrix(cur.xk[sl], kk)
        Xk_prev = block_matrix(prev.xk[sl], kk)
        Lk = block_matrix(cur.lam[sl], kk)
        # primal: (x_k, H_k x); dual: (z_k, v_k)
        other = E @ X @ E.T if form == "primal" else block_matrix(cur.vk[sl], kk)
        sq_diff += np.sum((Xk - other) ** 2)
        sq_a += np.sum(Xk ** 2)
        sq_b += np.sum(other ** 2)
        S_diff += E.T @ (Xk - Xk_prev) @ E
        S_lam += E.T @ Lk @ E
    eps_p = math.sqrt(sq_diff) / max(math.sqrt(sq_a), math.sqrt(sq_b), 1.0)
    eps_d = rho * np.linalg.norm(S_diff) / max(np.linalg.norm(S_lam), 1.0)
    return eps_p, eps_d, S_diff, S_lam


# ------------------------------------------------------------------ hand-simulated recursions

@pytest.mark.parametrize("case", golden("residuals_hand.json")["cases"], ids=lambda c: c["name"])
def test_hand_simulated_recursion(case):
    P = case["problem"]
    prob = problem_from_dense(P["C"], P["A"], P["b"], name=case["name"])
    dec = dc.decompose(prob)
    assert dec.p == 1
    st = admm.zero_state(dec)
    for want in case["iters"]:
        st = admm.step(dec, st, case["rho"], case["form"], 1)
        assert st.eps_p == pytest.approx(want["eps_p"], abs=1e-14)
        assert st.eps_d == pytest.approx(want["eps_d"], abs=1e-14)
        assert st.objective == pytest.approx(want["objective"], abs=1e-13)
        assert np.allclose(st.y, want["y"], atol=1e-13)
        k = len(dec.cliques[0])
        if "x" in want:   # 1x1: svec == matrix entries
            assert np.allclose(st.x, want["x"], atol=1e-13)
            assert np.allclose(st.xk, want["xk"], atol=1e-13)
            assert np.allclose(st.lam, want["lam"], atol=1e-13)
            if "vk" in want:
                assert np.allclose(st.vk, want["vk"], atol=1e-13)
        else:
            assert np.allclose(pattern_matrix(dec, st.x), want["X"], atol=1e-13)
            assert np.allclose(block_matrix(st.xk, k), want["Xk"], atol=1e-13)
            assert np.allclose(block_matrix(st.lam, k), want["Lam"], atol=1e-13)
            if "Vk" in want:
                assert np.allclose(block_matrix(st.vk, k), want["Vk"], atol=1e-13)


# ------------------------------------------------------------------ static fixed points

def test_static_fixed_point_primal_scalar():
    """min x s.t. x = 2, x >= 0: the state x_1 = 2, lam = 0 is a fixed point of
    Algorithm 1 (x = 2 from A x = b, P+(2 - 0) = 2, lam += rho (2 - 2)); one more
    iteration from it must report (eps_p, eps_d) = (0, 0)."""
    prob = sdp_inputs.scalar_primal()
    dec = dc.decompose(prob)
    for rho in (0.3, 1.0, 7.0):
        st = admm.zero_state(dec)
        st.xk[:] = 2.0
        st2 = admm.step(dec, st, rho, "primal", 1)
        assert st2.eps_p == 0.0 and st2.eps_d == 0.0
        assert st2.xk[0] == 2.0 and st2.lam[0] == 0.0 and st2.objective == 2.0


def test_static_fixed_point_dual_scalar():
    """max 2y s.t. y + z = 1, z >= 0: z = 0, v = 0, lam = 2 (= b) is a fixed point of
    Algorithm 2 (z = P+(0 - 2/rho) = 0, x = -b/rho, v = 0 + 2/rho + x = 0, lam = -rho x = 2)."""
    prob = problem_from_dense([[1.0]], [[[1.0]]], [2.0])
    dec = dc.decompose(prob)
    for rho in (0.3, 1.0, 7.0):
        st = admm.zero_state(dec)
        st.lam[:] = 2.0
        st2 = admm.step(dec, st, rho, "dual", 1)
        assert st2.eps_p == 0.0 and st2.eps_d == 0.0
        assert st2.y[0] == pytest.approx(1.0, abs=1e-15) and st2.objective == pytest.approx(2.0, abs=1e-15)


def test_static_fixed_point_block_problem():
    """A larger exact fixed point: the 2x2 problem with X = I fixed by the constraints
    and C = I.  P+(I) = I, so x_k = H x and lam stays 0: every iteration after the first
    reports (0, 0) in the primal form."""
    A = [[[1, 0], [0, 0]], [[0, 0], [0, 1]], [[0, .5], [.5, 0]]]
    prob = problem_from_dense(np.eye(2), A, [1.0, 1.0, 0.0])
    dec = dc.decompose(prob)
    st = admm.step(dec, admm.zero_state(dec), 2.0, "primal", 1)
    for _ in range(3):
        st = admm.step(dec, st, 2.0, "primal", 1)
        assert st.eps_p == 0.0 and st.eps_d == 0.0


# ------------------------------------------------------------------ dense recomputation of G9

CASES = [
    ("cfg0", lambda: sdp_inputs.config(0), 1.0),
    ("arrow_small", lambda: sdp_inputs.block_arrow(3, 3, 2, 6, seed=4), 3.0),
    ("maxcut30", lambda: sdp_inputs.maxcut_er(30, 2), 0.5),
    ("theta5", lambda: sdp_inputs.lovasz_theta_cycle(5), 1.0),
]


@pytest.mark.parametrize("name,make,rho", CASES, ids=[c[0] for c in CASES])
@pytest.mark.parametrize("form", ["primal", "dual"])
def test_residuals_match_dense_definition(name, make, rho, form):
    prob = make()
    dec = dc.decompose(prob)
    st = admm.zero_state(dec)
    for it in range(25):
        nxt = admm.step(dec, st, rho, form, 1)
        ep, ed, _, _ = dense_residuals(dec, st, nxt, rho, form)
        assert nxt.eps_p == pytest.approx(ep, rel=1e-11, abs=1e-15), (it, nxt.eps_p, ep)
        assert nxt.eps_d == pytest.approx(ed, rel=1e-11, abs=1e-15), (it, nxt.eps_d, ed)
        st = nxt


@pytest.mark.parametrize("name,make,rho", CASES, ids=[c[0] for c in CASES])
def test_primal_dual_residual_is_stationarity_error(name, make, rho):
    """rho ||sum_k H_k^T (x_k^(n) - x_k^(n-1))|| == ||C - A*(yhat) - sum_k E_k^T Lam_k E_k||_F with
    yhat = -rho y (module docstring), every iteration, and the oracle's eps_d uses exactly it."""
    prob = make()
    dec = dc.decompose(prob)
    Cm, As = dense_data(prob)
    st = admm.zero_state(dec)
    for it in range(25):
        nxt = admm.step(dec, st, rho, "primal", 1)
        _, _, S_diff, S_lam = dense_residuals(dec, st, nxt, rho, "primal")
        yhat = -rho * nxt.y
        stat = Cm - np.tensordot(yhat, As, axes=1) - S_lam
        lhs = rho * np.linalg.norm(S_diff)
        assert np.linalg.norm(stat) == pytest.approx(lhs, rel=1e-9, abs=1e-11 * max(1.0, np.linalg.norm(Cm)))
        assert np.allclose(stat, -rho * S_diff, atol=1e-10 * max(1.0, np.linalg.norm(Cm)))
        assert nxt.eps_d * max(np.linalg.norm(S_lam), 1.0) == pytest.approx(lhs, rel=1e-11, abs=1e-14)
        st = nxt
