"""Event timeline of one pipelined primal iteration (SDP_PIPE_TRACE=1, no graph)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["SDP_PIPE_TRACE"] = "1"
import paper_1609_06068_b200 as L  # noqa: E402
import sdp_inputs as gen  # noqa: E402

prob = gen.config(2)
s = L.Solver(prob, form="primal", rho=10.0, use_graph=False)
for _ in range(3):
    s.step(5)
s.close()
