"""Time the batched projection of `count` random symmetric matrices of order k
(the giant tier for k >= 65) and check it against numpy eigh.
Usage: giant_one.py k [count] [reps]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1609_06068_b200 as L  # noqa: E402
import sdp_inputs as gen  # noqa: E402

k = int(sys.argv[1])
count = int(sys.argv[2]) if len(sys.argv) > 2 else 1
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
rng = np.random.default_rng(k)
r, c = gen.packed_upper_index(k)
mats, vals = [], []
for _ in range(count):
    G = rng.standard_normal((k, k))
    X = 0.5 * (G + G.T)
    mats.append(X)
    vals.append(X[r, c])
vals = np.concatenate(vals)
plan = L.PsdPlan(np.full(count, k, np.int32))
din = torch.from_numpy(vals).cuda()
dout = torch.empty_like(din)
plan.project(din, dout)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    plan.project(din, dout)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / max(reps, 1)
out = dout.cpu().numpy()
worst = 0.0
off = 0
for X in mats:
    w, V = np.linalg.eigh(X)
    P = (V * np.maximum(w, 0)) @ V.T
    s = k * (k + 1) // 2
    worst = max(worst, np.linalg.norm(out[off:off + s] - P[r, c]) / np.linalg.norm(X[r, c]))
    off += s
print(f"k={k} count={count}: {ms:.3f} ms per batch, max rel err {worst:.2e}")
