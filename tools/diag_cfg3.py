"""Per-clique-size error of the GPU iterate against the oracle on configs[3]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1609_06068_b200 as L  # noqa: E402
import sdp_inputs as gen  # noqa: E402
from oracle import admm  # noqa: E402
from oracle import decompose as dc  # noqa: E402

n_it = int(sys.argv[1]) if len(sys.argv) > 1 else 1
prob = gen.config(3)
dec = dc.decompose(prob)
st = admm.step(dec, admm.zero_state(dec), 0.1, "primal", n_it)
s = L.Solver(prob, form="primal", rho=0.1)
s.step(n_it)
g = s.blocks("xk")
ks = np.array([len(c) for c in dec.cliques])
off = np.concatenate([[0], np.cumsum(ks * (ks + 1) // 2)])
worst = {}
for i, k in enumerate(ks):
    a, b = off[i], off[i + 1]
    e = np.linalg.norm(g[a:b] - st.xk[a:b]) / max(np.linalg.norm(st.xk[a:b]), 1e-300)
    key = "k<=16" if k <= 16 else "17-32" if k <= 32 else "33-64" if k <= 64 else "65-96" if k <= 96 else "giant"
    if e > worst.get(key, (0, 0))[0]:
        worst[key] = (e, int(k), i)
print(os.environ.get("SDP_PSD_TIERS", "default"), n_it, worst, flush=True)
bad = []
for i, k in enumerate(ks):
    a, b = off[i], off[i + 1]
    e = np.linalg.norm(g[a:b] - st.xk[a:b]) / max(np.linalg.norm(st.xk[a:b]), 1e-300)
    if e > 1e-10:
        bad.append((i, int(k), float("%.2e" % e)))
print("bad cliques:", bad[:40], "count", len(bad))
