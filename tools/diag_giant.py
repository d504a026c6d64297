"""Giant-tier batch projection on structured inputs (diagnostics)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1609_06068_b200 as L  # noqa: E402
import sdp_inputs as gen  # noqa: E402
from oracle import admm  # noqa: E402
from oracle import decompose as dc  # noqa: E402
from oracle import psd as opsd  # noqa: E402


def run(name, mats):
    ks = np.array([M.shape[0] for M in mats], np.int32)
    vals = np.concatenate([opsd.pack_upper(M) for M in mats])
    p = L.PsdPlan(ks)
    out = p.project_host(vals)
    want = opsd.project_psd_packed_batch(ks, vals)
    off = 0
    errs = []
    for k in ks:
        s = k * (k + 1) // 2
        errs.append(np.linalg.norm(opsd.unpack_upper(out[off:off + s] - want[off:off + s], k))
                    / np.linalg.norm(opsd.unpack_upper(vals[off:off + s], k)))
        off += s
    bad = [(i, int(k), "%.2e" % e) for i, (k, e) in enumerate(zip(ks, errs)) if e > 1e-12]
    print(name, "max %.2e" % max(errs), "bad", bad, flush=True)


prob = gen.config(3)
dec = dc.decompose(prob)
st = admm.step(dec, admm.zero_state(dec), 0.1, "primal", 1)
hx = dec.gather(st.x)
ks = dec.sizes
offs = np.concatenate([[0], np.cumsum(ks * (ks + 1) // 2)])
big = [i for i in np.argsort(-ks)[:int(os.environ.get("DIAG_NBIG", "4"))]]
# svec -> matrix entries (off-diagonal / sqrt 2)
mats = []
for i in big:
    k = int(ks[i])
    v = hx[offs[i]:offs[i + 1]].copy()
    r, c = gen.packed_upper_index(k)
    v = np.where(r == c, v, v / np.sqrt(2.0))
    mats.append(opsd.unpack_upper(v, k))
run("cfg3-iter1-largest", mats)
rng = np.random.default_rng(0)
for k in (200, 400, 600):
    Q, _ = np.linalg.qr(rng.standard_normal((k, k)))
    lam = 1.0 + 1e-3 * rng.standard_normal(k)
    lam[: k // 3] -= 2.0
    run(f"clustered{k}", [Q @ np.diag(lam) @ Q.T])
    M = np.eye(k)
    M[0, 1] = M[1, 0] = 0.3
    run(f"near-identity{k}", [M])
