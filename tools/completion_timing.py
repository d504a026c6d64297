"""Wall time of sdp_complete_x (host PSD completion) on configs 1 and 2 after 200 iterations."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1609_06068_b200 as L  # noqa: E402
import sdp_inputs as gen  # noqa: E402

for idx in (1, 2):
    prob = gen.config(idx)
    s = L.Solver(prob, form="primal", rho=10.0)
    s.step(200)
    t0 = time.perf_counter()
    Y = s.complete_x()
    dt = time.perf_counter() - t0
    lmin = np.linalg.eigvalsh(Y).min() if prob.n <= 2000 else float("nan")
    print(f"cfg{idx}: n={prob.n} completion {dt:.3f} s, lambda_min/||Y|| = {lmin / np.linalg.norm(Y):.2e}", flush=True)
    s.close()
