"""Determinism check: same handle, reset, rerun (bitwise)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1609_06068_b200 as L  # noqa: E402
import sdp_inputs as gen  # noqa: E402

prob = gen.block_arrow(12, 20, 10, 40, seed=7)
for form in ("primal", "dual"):
    for n in (1, 2, 5, 40, 70):
        s = L.Solver(prob, form=form, rho=1.0)
        s.step(n)
        a = s.blocks("xk").copy()
        s.reset()
        s.step(n)
        b = s.blocks("xk")
        s2 = L.Solver(prob, form=form, rho=1.0)
        s2.step(n)
        c = s2.blocks("xk")
        print(form, n, "reset-equal", np.array_equal(a, b), "fresh-equal", np.array_equal(a, c),
              float(np.max(np.abs(a - c))), flush=True)
