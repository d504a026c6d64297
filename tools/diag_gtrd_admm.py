"""cfg3 ADMM with SDP_GTRD_DEBUG=1: per-giant spectrum side / cluster statistics
of the tridiagonal path at a few iterations."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1609_06068_b200 as L  # noqa: E402
import sdp_inputs as gen  # noqa: E402

prob = gen.config(3)
s = L.Solver(prob, form="primal", rho=float(sys.argv[1]) if len(sys.argv) > 1 else 1.0)
for n in (1, 5, 20):
    print("=== after", n, flush=True)
    s.step(n)
