"""Pins for oracle/admm.py: closed-form optima, primal/dual agreement
(Remark 1, Fig. 1), invariants of every iterate, Remark 2's scaling and the
sign of E:DualMultUpdate (reading G7), Grone/Agler (Theorems 1-2)."""
import math

import numpy as np
import pytest
import scipy.sparse

from oracle import admm, chordal
from oracle import decompose as dc
from oracle.psd import project_psd
from oracle import completion
from tests.helpers import golden

OBJ = {o["cite"].split(":")[0]: o["value"] for o in golden("spec_examples.json")["objectives"]}


def closed_forms(gen):
    vals = golden("spec_examples.json")["objectives"]
    return [
        (gen.scalar_primal(), vals[0]["value"]),
        (gen.trace_one_tridiagonal(12, 1.0, -0.7), vals[2]["value"]),
        (gen.cycle_maxcut(5), -vals[3]["value"]),
        (gen.cycle_maxcut(6), -vals[4]["value"]),
        (gen.lovasz_theta_cycle(5), -vals[5]["value"]),
    ]


@pytest.mark.parametrize("form", ["primal", "dual"])
def test_closed_form_optima(gen, form):
    for prob, want in closed_forms(gen):
        dec = dc.decompose(prob)
        st, status = admm.solve(dec, 1.0, form, 1e-10, 20000)
        assert status == "solved", prob.name
        assert abs(st.objective - want) <= 1e-8 * max(1.0, abs(want)), (prob.name, st.objective, want)


def test_trace_one_equals_lambda_min(gen):
    """min <C,X> s.t. tr X = 1 is lambda_min(C) for random tridiagonal C
    (path pattern -> cliques are edges)."""
    rng = np.random.default_rng(0)
    for _ in range(3):
        n = int(rng.integers(4, 10))
        a = rng.standard_normal(n)
        bb = -0.5 - np.abs(rng.standard_normal(n - 1))   # Perron eigenvector: strictly complementary
        prob = gen.trace_one_tridiagonal(n)
        prob.c_val = np.concatenate([a, bb])
        T = np.diag(a) + np.diag(bb, 1) + np.diag(bb, -1)
        want = np.linalg.eigvalsh(T).min()
        dec = dc.decompose(prob)
        assert dec.p == n - 1
        st, status = admm.solve(dec, 10.0, "primal", 1e-9, 50000)
        assert status == "solved"
        assert abs(st.objective - want) < 1e-6


def test_invariants_every_iterate(gen):
    """Every primal iterate satisfies A x = b (E:OptCondMinYPrimal second block
    row); every dual iterate satisfies c - A^T y - sum H_k^T v_k = 0 (E:MinYblockDual);
    primal multipliers satisfy lam_k = rho P_+(-s_k): PSD and orthogonal to x_k."""
    prob = gen.block_arrow(3, 3, 2, 6, seed=11)
    dec = dc.decompose(prob)
    rho = 1.3
    st = admm.zero_state(dec)
    for _ in range(30):
        st = admm.step(dec, st, rho, "primal", 1)
        assert np.linalg.norm(dec.A @ st.x - dec.b) <= 1e-10 * np.linalg.norm(dec.b)
        for k, C in enumerate(dec.cliques):
            L = dc.smat_dense(dec.block(st.lam, k), len(C))
            Xk = dc.smat_dense(dec.block(st.xk, k), len(C))
            nrm = max(np.linalg.norm(L), 1.0)
            assert np.linalg.eigvalsh(L).min() >= -1e-12 * nrm
            assert abs(np.sum(L * Xk)) <= 1e-10 * nrm * max(np.linalg.norm(Xk), 1.0)
    st = admm.zero_state(dec)
    for _ in range(30):
        st = admm.step(dec, st, rho, "dual", 1)
        res = dec.c - dec.A.T @ st.y - dec.scatter(st.vk)
        assert np.linalg.norm(res) <= 1e-10 * np.linalg.norm(dec.c)


def test_dual_literal_equals_shortcut_and_printed_sign_fails(gen):
    """G7: E:MultUpdateDualSDP literally applied equals lam_k = -rho H_k x;
    the printed +rho H_k x does not converge to the optimum."""
    prob = gen.block_arrow(3, 3, 2, 6, seed=1)
    dec = dc.decompose(prob)
    a = admm.step(dec, admm.zero_state(dec), 1.0, "dual", 50, literal=True)
    b = admm.step(dec, admm.zero_state(dec), 1.0, "dual", 50, literal=False)
    assert np.linalg.norm(a.lam - b.lam) <= 1e-12 * np.linalg.norm(a.lam)
    assert np.linalg.norm(a.x - b.x) <= 1e-12 * np.linalg.norm(a.x)
    # with the printed sign the iteration is no longer ADMM; it stalls away from the optimum
    ref, _ = admm.solve(dec, 1.0, "primal", 1e-8, 20000)
    st = admm.zero_state(dec)
    for _ in range(1500):
        zk = admm.project_all(dec, st.vk - st.lam / 1.0)
        r1 = dec.c - dec.scatter(zk + st.lam)
        x, y = dec.solve_kkt(r1, -dec.b)
        Hx = dec.gather(x)
        st = admm.State(x=x, y=y, xk=zk, lam=+1.0 * Hx, vk=zk + st.lam + Hx)
    assert abs(dec.b @ st.y - ref.objective) > 1e-2 * abs(ref.objective)


def test_scaled_versions_first_iterate(gen):
    """Remark 2 / P:450: from zero init, x^(1) of Algorithm 1 at rho equals
    -x^(1)/rho' ... precisely x1_primal(rho) = -(1/rho) x1_dual(1/rho)."""
    prob = gen.block_arrow(4, 3, 2, 7, seed=3)
    dec = dc.decompose(prob)
    for rho in (0.5, 1.0, 10.0):
        p = admm.step(dec, admm.zero_state(dec), rho, "primal", 1)
        d = admm.step(dec, admm.zero_state(dec), 1.0 / rho, "dual", 1)
        assert np.allclose(p.x, -d.x / rho, atol=1e-14 * np.linalg.norm(p.x) + 1e-15)


@pytest.mark.parametrize("seed", [0, 1])
def test_primal_dual_dense_agree(gen, seed):
    """Remark 1 / Fig. 1: Algorithms 1 and 2 and the undecomposed p = 1 problem
    reach the same optimum; each run also carries a primal-dual pair whose
    objectives agree (duality gap -> 0)."""
    prob = gen.block_arrow(3, 3, 2, 6, seed=seed)
    dec = dc.decompose(prob)
    dense = dc.decompose(prob, dense=True)
    assert dense.p == 1
    vals = []
    for d, form, rho in [(dec, "primal", 1.0), (dec, "dual", 1.0), (dense, "primal", 1.0)]:
        st, status = admm.solve(d, rho, form, 1e-9, 30000)
        assert status == "solved"
        vals.append(st.objective)
        X, yhat, _ = admm.recovered_pair(d, st, rho, form)
        assert abs(d.c @ X - d.b @ yhat) <= 1e-6 * abs(st.objective)
    assert max(vals) - min(vals) <= 1e-6 * abs(vals[0])


def test_grone_and_agler(gen):
    """Theorem 1: the converged clique blocks admit a PSD completion of X
    (built on the clique tree); Theorem 2: Z = sum_k E_k^T Z_k E_k is PSD and
    equals C - A*(yhat) to solver accuracy."""
    prob = gen.block_arrow(3, 3, 2, 5, seed=4)
    prob2 = gen.cycle_maxcut(7)
    for pr in (prob, prob2):
        dec = dc.decompose(pr)
        st, status = admm.solve(dec, 1.0, "primal", 1e-10, 30000)
        assert status == "solved"
        # Grone: complete the partial matrix given on the extended pattern
        X = dec.dense_from_pattern(st.x)
        known = np.zeros((dec.n, dec.n), dtype=bool)
        known[dec.coord_row, dec.coord_col] = True
        known[dec.coord_col, dec.coord_row] = True
        adj = chordal.aggregate_adjacency(pr)
        order, later, filled = chordal.minimum_degree_elimination(adj)
        M = completion.complete_psd(X, known, order, later)
        assert np.allclose(M[known], X[known])
        assert np.linalg.eigvalsh(M).min() >= -1e-7 * np.linalg.norm(M)
        # Agler: Z from the multipliers (primal form: Z_k = lam_k)
        Z = np.zeros((dec.n, dec.n))
        for k, C in enumerate(dec.cliques):
            Z[np.ix_(C, C)] += dc.smat_dense(dec.block(st.lam, k), len(C))
        assert np.linalg.eigvalsh(Z).min() >= -1e-9 * np.linalg.norm(Z)
        yhat = -1.0 * st.y
        A = dec.A.toarray() if scipy.sparse.issparse(dec.A) else dec.A
        Zs = dec.c - A.T @ yhat                      # svec of C - A*(yhat) on the pattern
        assert np.linalg.norm(dec.dense_from_pattern(Zs) - Z) <= 1e-6 * np.linalg.norm(Z)


def test_projection_of_iterates_matches_definition(gen):
    """x_k^(n+1) is the Frobenius-nearest PSD matrix to smat(H_k x - lam_k/rho):
    checked by the variational inequality against random PSD competitors."""
    prob = gen.block_arrow(2, 3, 1, 3, seed=2)
    dec = dc.decompose(prob)
    st0 = admm.step(dec, admm.zero_state(dec), 1.0, "primal", 3)
    st1 = admm.step(dec, st0, 1.0, "primal", 1)
    s = dec.gather(st1.x) - st0.lam
    rng = np.random.default_rng(0)
    for k, C in enumerate(dec.cliques):
        S = dc.smat_dense(dec.block(s, k), len(C))
        P = dc.smat_dense(dec.block(st1.xk, k), len(C))
        for _ in range(10):
            G = rng.standard_normal((len(C), len(C)))
            Y = G @ G.T
            assert np.sum((S - P) * (Y - P)) <= 1e-10 * (1 + np.linalg.norm(Y))


def test_cfg0_converges_both_forms(gen):
    prob = gen.config(0)
    dec = dc.decompose(prob)
    assert dec.p == 5 and set(dec.sizes.tolist()) == {7}
    p, sp = admm.solve(dec, 1.0, "primal", 1e-6, 5000)
    d, sd = admm.solve(dec, 1.0, "dual", 1e-6, 5000)
    assert sp == sd == "solved"
    assert abs(p.objective - d.objective) <= 1e-4 * abs(p.objective)


def test_adapt_rho_rule_spec_examples():
    """Residual balancing rule (SPEC S:318-326 examples): balanced residuals leave
    rho unchanged; ||r|| = 100 ||s|| with mu = 10, tau = 2 doubles it; the mirror
    case halves it."""
    assert admm.adapt_rho(1.0, 1e-3, 1e-3) == 1.0
    assert admm.adapt_rho(1.0, 5e-3, 1e-3) == 1.0
    assert admm.adapt_rho(1.0, 100.0, 1.0, mu=10, tau=2) == 2.0
    assert admm.adapt_rho(1.0, 1.0, 100.0, mu=10, tau=2) == 0.5


def test_adaptive_rho_reaches_same_optimum(gen):
    """Adaptation changes iteration counts, not the solution: the adaptive solve
    of the tiny block-arrow problem reaches the closed/dense objective within the
    stopping tolerance, from a badly scaled rho (same objective within 1e-3)."""
    prob = gen.block_arrow(3, 3, 2, 6, seed=1)
    dec = dc.decompose(prob)
    fixed, s1 = admm.solve(dec, 1.0, "primal", 1e-6, 20000)
    adapt, s2 = admm.solve(dec, 50.0, "primal", 1e-6, 20000, adapt=(10.0, 2.0, 10))
    assert s1 == "solved" and s2 == "solved"
    assert abs(adapt.objective - fixed.objective) <= 1e-4 * abs(fixed.objective)
    assert adapt.rho != 50.0


def test_user_pattern_E(gen):
    """Optional user pattern E ("described by the graph G(V,E)"): its entries join the
    aggregate pattern even where C and every A_i vanish.  With E = all pairs the chordal
    extension is complete (p = 1, the undecomposed cone); with E = one extra edge between two
    diagonal blocks the extension and cliques change (checked against brute force) while the
    SDP optimum does not (Theorems 1-2: the decomposition is exact for any chordal pattern
    containing the aggregate one)."""
    from tests.helpers import adj_from_edges, is_chordal_bruteforce, maximal_cliques_bruteforce
    prob = gen.block_arrow(3, 3, 2, 6, seed=0)
    n = prob.n
    base = dc.decompose(prob)
    st0, status = admm.solve(base, 1.0, "primal", 1e-9, 30000)
    assert status == "solved"
    iu, ju = np.triu_indices(n, 1)
    full = gen.block_arrow(3, 3, 2, 6, seed=0)
    full.e_row, full.e_col = iu.astype(np.int32), ju.astype(np.int32)
    dfull = dc.decompose(full)
    assert dfull.p == 1 and dfull.N == n * (n + 1) // 2
    one = gen.block_arrow(3, 3, 2, 6, seed=0)
    one.e_row, one.e_col = np.array([0], np.int32), np.array([3], np.int32)   # block 0 - block 1
    done = dc.decompose(one)
    adj = chordal.aggregate_adjacency(one)
    assert adj[0, 3] and not chordal.aggregate_adjacency(prob)[0, 3]
    pat = [(int(i), int(j)) for i, j in zip(done.coord_row, done.coord_col) if i != j]
    A2 = adj_from_edges(n, pat)
    assert is_chordal_bruteforce(A2)
    assert [tuple(c.tolist()) for c in done.cliques] == maximal_cliques_bruteforce(A2)
    assert [c.tolist() for c in done.cliques] != [c.tolist() for c in base.cliques]
    for d in (dfull, done):
        st, status = admm.solve(d, 1.0, "primal", 1e-9, 30000)
        assert status == "solved"
        assert abs(st.objective - st0.objective) <= 1e-6 * abs(st0.objective)
