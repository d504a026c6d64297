"""ORACLE (test infrastructure only): Algorithm 1 and Algorithm 2.

Primal (Algorithm 1), one iteration in the paper's order:
  1. x from the KKT system E:OptCondMinYPrimal
       r1 = sum_k H_k^T (x_k + lam_k / rho) - c / rho,  r2 = b
  2. x_k = vec{ P_k [ vec^-1( H_k x - lam_k / rho ) ] }    E:XkUpdate
  3. lam_k = lam_k + rho (x_k - H_k x)                     E:LambdakUpdate
  4. residuals eps_p, eps_d                                (reading G9)

Dual (Algorithm 2, with Remark 2's ordering P:444-451: the Y-block
(projection) before the X-block):
  1. z_k = vec{ P_k [ vec^-1( v_k - lam_k / rho ) ] }      E:zkUpdate
  2. (x, y) from E:OptCondMinYDual
       r1 = c - sum_k H_k^T (z_k + lam_k / rho),  r2 = -b / rho
  3. v_k = z_k + lam_k / rho + H_k x                       E:vkEqn
  4. lam_k = lam_k + rho (z_k - v_k) = -rho H_k x          E:MultUpdateDualSDP
     (P:414-417); E:DualMultUpdate prints +rho H_k x, which
     contradicts E:vkEqn + E:MultUpdateDualSDP (reading G7: -rho H_k x).
  5. residuals

Residuals (reading G9; the paper only cites boyd2011):
  eps_p = ||stack(x_k - H_k x)|| / max(||stack x_k||, ||stack H_k x||, 1)
  eps_d = rho ||sum_k H_k^T (x_k^(n) - x_k^(n-1))|| / max(||sum_k H_k^T lam_k||, 1)
  dual form: (z_k, v_k) in place of (x_k, H_k x).  x_k^(0) is the initial
  guess (zeros, reading G12).
Objective (reading G17): primal <c, x>, dual <b, y>.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .decompose import Decomposition
from .psd import project_psd_svec


class NumericalError(Exception):
    pass


@dataclass
class State:
    """Primal: x (N), y (m), xk, lam (stacked clique svec).
    Dual:   x (N), y (m), zk -> stored in xk, vk, lam."""
    x: np.ndarray
    y: np.ndarray
    xk: np.ndarray
    lam: np.ndarray
    vk: np.ndarray
    it: int = 0
    eps_p: float = float("inf")
    eps_d: float = float("inf")
    objective: float = float("nan")
    history: list = field(default_factory=list)
    rho: float = float("nan")  # set by solve(): the penalty in force at the end


def zero_state(dec: Decomposition) -> State:
    S = int(dec.offsets[-1])
    return State(x=np.zeros(dec.N), y=np.zeros(dec.m), xk=np.zeros(S), lam=np.zeros(S),
                 vk=np.zeros(S))


def project_all(dec: Decomposition, s: np.ndarray) -> np.ndarray:
    """Apply P_k to every clique block of the stacked vector s."""
    out = np.empty_like(s)
    for k, C in enumerate(dec.cliques):
        a, b = dec.offsets[k], dec.offsets[k + 1]
        out[a:b] = project_psd_svec(s[a:b], len(C))
    return out


def primal_iteration(dec: Decomposition, st: State, rho: float) -> State:
    # 1. E:OptCondMinYPrimal
    r1 = dec.scatter(st.xk + st.lam / rho) - dec.c / rho
    x, y = dec.solve_kkt(r1, dec.b)
    # 2. E:XkUpdate
    Hx = dec.gather(x)
    xk = project_all(dec, Hx - st.lam / rho)
    # 3. E:LambdakUpdate
    lam = st.lam + rho * (xk - Hx)
    # 4. residuals (G9)
    eps_p = np.linalg.norm(xk - Hx) / max(np.linalg.norm(xk), np.linalg.norm(Hx), 1.0)
    eps_d = rho * np.linalg.norm(dec.scatter(xk - st.xk)) / max(np.linalg.norm(dec.scatter(lam)), 1.0)
    obj = float(dec.c @ x)
    if not (np.all(np.isfinite(x)) and np.all(np.isfinite(lam))):
        raise NumericalError("non-finite iterate")
    return State(x=x, y=y, xk=xk, lam=lam, vk=st.vk, it=st.it + 1, eps_p=eps_p, eps_d=eps_d,
                 objective=obj, history=st.history)


def dual_iteration(dec: Decomposition, st: State, rho: float, literal: bool = False) -> State:
    zk_old = st.xk
    # 1. E:zkUpdate
    zk = project_all(dec, st.vk - st.lam / rho)
    # 2. E:OptCondMinYDual
    r1 = dec.c - dec.scatter(zk + st.lam / rho)
    x, y = dec.solve_kkt(r1, -dec.b / rho)
    # 3. E:vkEqn
    Hx = dec.gather(x)
    vk = zk + st.lam / rho + Hx
    # 4. E:MultUpdateDualSDP (literal) or its closed form -rho H_k x (G7)
    lam = st.lam + rho * (zk - vk) if literal else -rho * Hx
    # 5. residuals
    eps_p = np.linalg.norm(zk - vk) / max(np.linalg.norm(zk), np.linalg.norm(vk), 1.0)
    eps_d = rho * np.linalg.norm(dec.scatter(zk - zk_old)) / max(np.linalg.norm(dec.scatter(lam)), 1.0)
    obj = float(dec.b @ y)
    if not (np.all(np.isfinite(x)) and np.all(np.isfinite(lam))):
        raise NumericalError("non-finite iterate")
    return State(x=x, y=y, xk=zk, lam=lam, vk=vk, it=st.it + 1, eps_p=eps_p, eps_d=eps_d,
                 objective=obj, history=st.history)


def step(dec: Decomposition, st: State, rho: float, form: str, iters: int, literal=False,
         record=False) -> State:
    """Run exactly `iters` iterations (no stopping test)."""
    for _ in range(iters):
        if form == "primal":
            st = primal_iteration(dec, st, rho)
        else:
            st = dual_iteration(dec, st, rho, literal=literal)
        if record:
            st.history.append((st.it, st.eps_p, st.eps_d, st.objective))
    return st


def adapt_rho(rho: float, eps_p: float, eps_d: float, mu: float = 10.0, tau: float = 2.0) -> float:
    """Residual balancing (Boyd et al. 2011 Sec. 3.4.1, the reference the paper cites
    for its residuals): rho <- tau rho if the primal
    residual exceeds mu times the dual one, rho <- rho / tau in the opposite case.
    The KKT matrix of E:OptCondMinYPrimal / E:OptCondMinYDual is rho-free,
    so nothing is refactorised, and the multipliers lambda_k are kept unscaled."""
    if eps_p > mu * eps_d:
        return rho * tau
    if eps_d > mu * eps_p:
        return rho / tau
    return rho


def solve(dec: Decomposition, rho: float, form: str, tol: float, max_iter: int,
          st: State = None, literal=False, adapt=None):
    """Iterate until max(eps_p, eps_d) < tol (Algorithm 1/2 line 3) or max_iter.
    adapt = (mu, tau, every): after every `every`-th iteration that did not stop,
    rho is updated by adapt_rho from that iteration's residuals.
    Returns (state, status) with status "solved" or "max_iter"; the final rho is
    st.rho."""
    st = zero_state(dec) if st is None else st
    while st.it < max_iter:
        st = step(dec, st, rho, form, 1, literal=literal)
        if max(st.eps_p, st.eps_d) < tol:
            st.rho = rho
            return st, "solved"
        if adapt is not None and st.it % adapt[2] == 0:
            rho = adapt_rho(rho, st.eps_p, st.eps_d, adapt[0], adapt[1])
    st.rho = rho
    return st, "max_iter"


def recovered_pair(dec: Decomposition, st: State, rho: float, form: str):
    """Primal-dual SDP pair carried by the iterates (Remark 1, Fig. 1).

    primal form: X = x, SDP dual yhat = -rho * y_kkt, Z blocks = lam_k
    dual form:   X = -rho * x_kkt, yhat = y_kkt,      Z blocks = z_k
    (the KKT multipliers are rho*y and rho*x)."""
    if form == "primal":
        return st.x, -rho * st.y, st.lam
    return -rho * st.x, st.y, st.xk
