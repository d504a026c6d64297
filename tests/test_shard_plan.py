"""Clique sharding on CPU.

1. Invariants of the library's shard plan (sdp_shard_plan, host-only C++).
2. A world_size-2 `gloo` run of the sharded iteration: each process holds the
   library's plan for its rank and executes, in numpy, exactly the steps the
   CUDA path runs per rank (local scatter with c at the owner, all-reduce of the
   shared-coordinate partials, column-sharded A D^-1 r1 + all-reduce, replicated
   triangular solves, A^T y on the local coordinates, local projections,
   all-reduce of the residual partials), with the library's LPT clique assignment.  The assembled
  iterates must equal the
   single-process oracle's to rounding: this checks that the plan's ownership
   and exchange sets are complete and that no partial is counted twice.
"""
import os
import socket

import numpy as np
import pytest

from oracle import admm
from oracle import decompose as dc
from oracle.psd import project_psd_svec

L = pytest.importorskip("paper_1609_06068_b200._lib", reason="libchordal_sdp.so not built")


def pattern_of(prob):
    return (np.concatenate([prob.c_row, prob.a_row]).astype(np.int32),
            np.concatenate([prob.c_col, prob.a_col]).astype(np.int32))


def problems(gen):
    return [gen.block_arrow(6, 3, 2, 7, seed=4), gen.maxcut_er(60, 3), gen.config(0)]


@pytest.mark.parametrize("world", [1, 2, 3, 4])
def test_plan_invariants(gen, world):
    for prob in problems(gen):
        dec = dc.decompose(prob, factor=False)
        r, c = pattern_of(prob)
        plans = [L.shard_plan(prob.n, r, c, world, rk) for rk in range(world)]
        crank = plans[0]["clique_rank"]
        assert crank.shape == (dec.p,) and crank.min() >= 0 and crank.max() < world
        assert len(np.unique(crank)) == world  # every rank has a clique
        # LPT on k^3 + 16: the largest rank load is within the largest clique cost of the mean
        cost = np.array([len(C) ** 3 + 16.0 for C in dec.cliques])
        loads = np.array([cost[crank == rk].sum() for rk in range(world)])
        assert loads.max() <= cost.sum() / world + cost.max() + 1e-9
        for rk, pl in enumerate(plans):
            assert np.array_equal(pl["clique_rank"], crank)
            assert np.array_equal(pl["cliques"], np.flatnonzero(crank == rk))
            assert np.array_equal(pl["shared_coords"], plans[0]["shared_coords"])
        touch = np.zeros((world, dec.N), dtype=bool)
        for rk in range(world):
            for k in np.flatnonzero(crank == rk):
                touch[rk, dec.H[k]] = True
            want = np.flatnonzero(touch[rk])
            assert np.array_equal(plans[rk]["local_coords"], want)
        owners = np.zeros(dec.N, dtype=int)
        for rk in range(world):
            loc = plans[rk]["local_coords"]
            owners[loc[plans[rk]["owned"]]] += 1
        assert np.all(owners == 1)  # every coordinate owned exactly once
        shared = np.flatnonzero(touch.sum(0) >= 2)
        assert np.array_equal(plans[0]["shared_coords"], shared)
        # the owner is the rank of the first clique containing the coordinate
        first = np.full(dec.N, -1)
        for k in range(dec.p):
            new = first[dec.H[k]] < 0
            first[dec.H[k][new]] = crank[k]
        for rk in range(world):
            loc = plans[rk]["local_coords"]
            assert np.array_equal(plans[rk]["owned"], first[loc] == rk)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _sharded_worker(rank, world, port, form, iters, out_dir):
    import torch
    import torch.distributed as dist
    import sdp_inputs as gen
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)

    def allreduce(v):
        t = torch.from_numpy(np.ascontiguousarray(v, dtype=np.float64))
        dist.all_reduce(t)
        return t.numpy()

    prob = gen.block_arrow(6, 3, 2, 7, seed=4) if os.environ.get("SHARD_PROB", "arrow") == "arrow" \
        else gen.maxcut_er(60, 3)
    dec = dc.decompose(prob)
    r, c = pattern_of(prob)
    pl = L.shard_plan(prob.n, r, c, world, rank)
    loc, owned = pl["local_coords"], pl["owned"]
    own_mask = np.zeros(dec.N, dtype=bool)
    own_mask[loc[owned]] = True
    loc_mask = np.zeros(dec.N, dtype=bool)
    loc_mask[loc] = True
    A = dec.A.toarray() if hasattr(dec.A, "toarray") else dec.A
    c_own = np.where(own_mask, dec.c, 0.0)
    rho = 1.0
    ks = [int(k) for k in pl["cliques"]]
    xk = {k: np.zeros(len(dec.H[k])) for k in ks}
    lam = {k: np.zeros(len(dec.H[k])) for k in ks}
    vk = {k: np.zeros(len(dec.H[k])) for k in ks}
    x = np.zeros(dec.N)
    y = np.zeros(dec.m)

    def scatter(form):
        # local partial sums; c enters once (owner); shared coordinates all-reduced
        sr = np.zeros(dec.N)
        sx = np.zeros(dec.N)
        sl = np.zeros(dec.N)
        for k in ks:
            np.add.at(sr, dec.H[k], xk[k] + lam[k] / rho)
            np.add.at(sx, dec.H[k], xk[k])
            np.add.at(sl, dec.H[k], lam[k])
        r1 = sr - c_own / rho if form == "primal" else c_own - sr
        sh = pl["shared_coords"]
        buf = allreduce(np.concatenate([r1[sh], sx[sh], sl[sh]]))
        r1[sh], sx[sh], sl[sh] = buf[:len(sh)], buf[len(sh):2 * len(sh)], buf[2 * len(sh):]
        return r1, sx, sl

    def kkt(r1, r2):
        rD = r1 / dec.D
        u = allreduce(A[:, own_mask] @ rD[own_mask]) - r2      # column-sharded A D^-1 r1
        t = np.linalg.solve(np.tril(dec.L), u)
        yy = np.linalg.solve(np.tril(dec.L).T, t)             # replicated triangular solves
        xx = np.zeros(dec.N)
        xx[loc_mask] = rD[loc_mask] - (A[:, loc_mask].T @ yy) / dec.D[loc_mask]
        return xx, yy

    sprev = np.zeros(dec.N)
    hist = []
    for it in range(iters):
        if form == "primal":
            r1, sx, sl = scatter("primal")
            x, y = kkt(r1, dec.b)
            p3 = np.zeros(3)
            for k in ks:
                hx = x[dec.H[k]]
                new = project_psd_svec(hx - lam[k] / rho, len(dec.cliques[k]))
                lam[k] = lam[k] + rho * (new - hx)
                xk[k] = new
                p3 += [np.sum((new - hx) ** 2), np.sum(new ** 2), np.sum(hx ** 2)]
            _, sx2, sl2 = scatter("primal")
            d2 = np.sum(((sx2 - sprev) ** 2)[own_mask])
            sprev = sx2
            red = allreduce(np.concatenate([p3, [d2, np.sum((sl2 ** 2)[own_mask]), np.sum((dec.c * x)[own_mask])]]))
            eps_p = np.sqrt(red[0]) / max(np.sqrt(red[1]), np.sqrt(red[2]), 1.0)
            eps_d = rho * np.sqrt(red[3]) / max(np.sqrt(red[4]), 1.0)
            hist.append((eps_p, eps_d, red[5]))
        else:
            zold = {k: xk[k].copy() for k in ks}
            for k in ks:
                xk[k] = project_psd_svec(vk[k] - lam[k] / rho, len(dec.cliques[k]))
            r1, sx, sl = scatter("dual")
            x, y = kkt(r1, -dec.b / rho)
            p3 = np.zeros(3)
            for k in ks:
                hx = x[dec.H[k]]
                vk[k] = xk[k] + lam[k] / rho + hx
                lam[k] = -rho * hx
                p3 += [np.sum((xk[k] - vk[k]) ** 2), np.sum(xk[k] ** 2), np.sum(vk[k] ** 2)]
            d2 = np.sum(((sx - sprev) ** 2)[own_mask])
            sprev = sx
            red = allreduce(np.concatenate([p3, [d2, np.sum(((dec.D * x) ** 2)[own_mask])]]))
            eps_p = np.sqrt(red[0]) / max(np.sqrt(red[1]), np.sqrt(red[2]), 1.0)
            eps_d = rho * np.sqrt(red[3]) / max(rho * np.sqrt(red[4]), 1.0)
            hist.append((eps_p, eps_d, float(dec.b @ y)))
    xo = allreduce(np.where(own_mask, x, 0.0))
    lam_full = np.zeros(int(dec.offsets[-1]))
    for k in ks:
        lam_full[dec.offsets[k]:dec.offsets[k + 1]] = lam[k]
    lam_full = allreduce(lam_full)
    if rank == 0:
        np.savez(os.path.join(out_dir, "shard.npz"), x=xo, y=y, lam=lam_full, hist=np.array(hist))
    dist.destroy_process_group()


@pytest.mark.parametrize("form", ["primal", "dual"])
@pytest.mark.parametrize("probname", ["arrow", "maxcut"])
def test_sharded_iteration_gloo_world2(gen, tmp_path, form, probname):
    import torch.multiprocessing as mp
    os.environ["SHARD_PROB"] = probname
    iters = 12
    mp.spawn(_sharded_worker, args=(2, _free_port(), form, iters, str(tmp_path)), nprocs=2, join=True)
    got = np.load(tmp_path / "shard.npz")
    prob = gen.block_arrow(6, 3, 2, 7, seed=4) if probname == "arrow" else gen.maxcut_er(60, 3)
    dec = dc.decompose(prob)
    st = admm.step(dec, admm.zero_state(dec), 1.0, form, iters, record=True)
    rel = lambda a, b: np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)
    assert rel(got["x"], st.x) <= 1e-12
    assert rel(got["y"], st.y) <= 1e-12
    assert rel(got["lam"], st.lam) <= 1e-12
    h = np.array(st.history)
    assert np.allclose(got["hist"][:, 0], h[:, 1], rtol=1e-10, atol=1e-15)
    assert np.allclose(got["hist"][:, 1], h[:, 2], rtol=1e-10, atol=1e-15)
    assert np.allclose(got["hist"][:, 2], h[:, 3], rtol=1e-10, atol=1e-12)
