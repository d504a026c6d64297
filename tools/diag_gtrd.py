"""Giant-tier diagnostics: accuracy (vs numpy eigh) and device time of the
tridiagonal path against the block-Jacobi path (SDP_GIANT_METHOD=jacobi) for a
list of orders, plus the cfg3 giant mix.  Usage: diag_gtrd.py [method]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1609_06068_b200 as L  # noqa: E402
import sdp_inputs as gen  # noqa: E402


def proj_np(X):
    w, V = np.linalg.eigh(X)
    return (V * np.maximum(w, 0)) @ V.T


def run(ks, mats, label):
    vals = []
    for M in mats:
        r, c = gen.packed_upper_index(M.shape[0])
        vals.append(M[r, c])
    vals = np.concatenate(vals)
    plan = L.PsdPlan(np.array(ks, np.int32))
    din = torch.from_numpy(vals).cuda()
    dout = torch.empty_like(din)
    plan.project(din, dout)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        plan.project(din, dout)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    out = dout.cpu().numpy()
    off = 0
    worst = 0.0
    for M in mats:
        k = M.shape[0]
        s = k * (k + 1) // 2
        r, c = gen.packed_upper_index(k)
        P = proj_np(M)
        e = np.linalg.norm(out[off:off + s] - P[r, c]) / max(np.linalg.norm(M), 1e-300)
        worst = max(worst, e)
        off += s
    print(f"{label}: {len(ks)} matrices, max k {max(ks)}, {ms:.3f} ms, worst rel err {worst:.2e}", flush=True)
    plan.close()


rng = np.random.default_rng(0)
quick = len(sys.argv) > 1 and sys.argv[1] == "quick"
for k in ((630,) if quick else (65, 97, 130, 257, 400, 630, 800)):
    G = rng.standard_normal((k, k))
    run([k], [0.5 * (G + G.T)], f"random k={k}")
# structured
for k in (() if quick else (65, 300)):
    Q, _ = np.linalg.qr(rng.standard_normal((k, k)))
    lam = np.repeat([2.0, -1.0, 0.0, 1.0 + 1e-9], (k + 3) // 4)[:k]
    v = rng.standard_normal(k)
    mats = [np.zeros((k, k)), np.eye(k), Q @ np.diag(lam) @ Q.T, np.outer(v, v), -np.outer(v, v), -np.eye(k)]
    run([k] * len(mats), mats, f"structured k={k}")
# cfg3 giant mix (orders of the max-cut n=3000 cliques >= 65), max-cut-like: I + sparse
ks = [66, 68, 71, 71, 73, 73, 77, 78, 79, 79, 83, 84, 86, 91, 92, 93, 96, 98, 98, 100, 105, 108, 108, 116, 119, 125,
      126, 130, 140, 154, 156, 167, 172, 178, 186, 199, 201, 205, 208, 219, 238, 239, 299, 300, 314, 324, 332, 347,
      386, 441, 441, 445, 481, 500, 501, 503, 511, 514, 595, 596, 596, 596, 596, 596, 604, 630]
mats = []
for k in ks:
    G = rng.standard_normal((k, k))
    mats.append(0.5 * (G + G.T))
run(ks, mats, "cfg3 giant mix (random)")
