"""Find the first iteration / array where two fresh handles differ (dual, k=30)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1609_06068_b200 as L  # noqa: E402
import sdp_inputs as gen  # noqa: E402

prob = gen.block_arrow(12, 20, 10, 40, seed=7)
form = sys.argv[1] if len(sys.argv) > 1 else "dual"
a = L.Solver(prob, form=form, rho=1.0)
b = L.Solver(prob, form=form, rho=1.0)
for it in range(1, 70):
    a.step(1)
    b.step(1)
    diffs = {}
    for nm, fa, fb in (("x", a.x(), b.x()), ("y", a.y(), b.y()), ("xk", a.blocks("xk"), b.blocks("xk")),
                       ("lam", a.blocks("lambda"), b.blocks("lambda")), ("vk", a.blocks("vk"), b.blocks("vk"))):
        if not np.array_equal(fa, fb):
            diffs[nm] = float(np.max(np.abs(fa - fb)))
    if diffs:
        print("first difference at iteration", it, diffs, "sweeps", a.info()["jacobi_sweeps"], b.info()["jacobi_sweeps"])
        break
else:
    print("identical through 69 iterations")
