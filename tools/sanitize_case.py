"""Small inputs for compute-sanitizer (one tool per gpurun call): every projection tier once
(batch mode), the giant tridiagonal path (k = 130, one-stage and two-stage), the QL tier (2048
matrices of order 24), and a few ADMM iterations of BASELINE configs[0] in both forms.
Usage: sanitize_case.py [batch|trd|giant|admm]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1609_06068_b200 as L  # noqa: E402
import sdp_inputs as gen  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "batch"
rng = np.random.default_rng(0)


def batch(ks):
    ks = np.asarray(ks, np.int32)
    vals = np.concatenate([rng.standard_normal(k * (k + 1) // 2) for k in ks])
    p = L.PsdPlan(ks)
    out = p.project_host(vals)
    p.close()
    assert np.all(np.isfinite(out))


if what == "batch":      # register / warp / CTA Jacobi tiers
    batch([1, 2, 5, 8, 9, 16, 17, 30, 32, 33, 40, 64])
elif what == "trd":      # tridiagonal-QL tier (>= 2048 matrices in a size range)
    batch([24] * 2048)
elif what == "giant":    # giant tier: tridiagonal path (one-stage default) and block Jacobi fallback
    batch([70, 130])
elif what == "admm":
    for form in ("primal", "dual"):
        s = L.Solver(gen.config(0), form=form, rho=1.0)
        s.step(3)
        s.info()
        s.close()
print("ok", what)
