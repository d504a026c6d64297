"""Setup-time variance of the cfg2 e2e path: five host-to-host setups with the library's own
cudaMalloc and with the torch caching allocator (SDP_SETUP_TRACE=1 shows the phases)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1609_06068_b200 as L  # noqa: E402
import sdp_inputs as gen  # noqa: E402

prob = gen.config(2)
pp = bench.pinned_problem(prob)
for alloc in (None, "torch"):
    for rep in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        s = L.Solver(pp, form="primal", rho=10.0, allocator=alloc)
        t1 = time.perf_counter()
        s.close()
        t2 = time.perf_counter()
        print(f"allocator={alloc} rep {rep}: setup {t1 - t0:.3f} s, close {t2 - t1:.3f} s", file=sys.stderr, flush=True)
