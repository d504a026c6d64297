"""Phase trace of the giant projection tier on BASELINE configs[3] (SDP_GIANT_TRACE=1).
usage: SDP_GIANT_TRACE=1 python tools/giant_trace.py [iters]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1609_06068_b200 as L  # noqa: E402
import sdp_inputs as gen  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 4
prob = gen.config(3)
s = L.Solver(prob, form="primal", rho=0.1)
ks = np.array([len(c) for c in s.cliques()])
print("cliques", len(ks), "k>=97:", int((ks >= 97).sum()), "65..96:", int(((ks > 64) & (ks < 97)).sum()),
      "33..64:", int(((ks > 32) & (ks <= 64)).sum()), flush=True)
for i in range(iters):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s.step(1)
    torch.cuda.synchronize()
    print(f"iter {i}: {1e3 * (time.perf_counter() - t0):.2f} ms", flush=True)
print(s.info())
