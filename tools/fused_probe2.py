"""Per-phase trace of the fused iteration (SDP_FUSED_TRACE=1: CTA 0's %globaltimer marks, printed by
the library to stderr), and a step(1) loop for an ncu cold-cache duration capture.
usage: python tools/fused_probe2.py trace | steps <cfg> <fused 0/1>"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1609_06068_b200 as L  # noqa: E402
import sdp_inputs as gen  # noqa: E402

if sys.argv[1] == "trace":
    for cfg in (0, 1):
        for form in ("primal", "dual"):
            for ctas in ((None,) if cfg == 0 else (None, "74", "148")):
                os.environ["SDP_FUSED_TRACE"] = "1"
                if ctas:
                    os.environ["SDP_FUSED_CTAS"] = ctas
                else:
                    os.environ.pop("SDP_FUSED_CTAS", None)
                s = L.Solver(gen.config(cfg), form=form, rho=1.0)
                print(f"cfg{cfg} {form} ctas={ctas}", file=sys.stderr, flush=True)
                s.step(64)
                s.step(64)
                torch.cuda.synchronize()
                inf = s.info()
                print(f"  sweeps/projection {inf['jacobi_sweeps'] / (inf['iters'] * inf['p']):.2f}", file=sys.stderr)
                s.close()
elif sys.argv[1] == "long":  # one long fused launch (for an ncu source-level capture)
    if len(sys.argv) > 3:
        os.environ["SDP_FUSED"] = sys.argv[3]
    s = L.Solver(gen.config(int(sys.argv[2])), form="primal", rho=1.0)
    s.step(20)
    s.step(200)
    torch.cuda.synchronize()
    s.close()
else:
    cfg, fz = int(sys.argv[2]), sys.argv[3]
    os.environ["SDP_FUSED"] = fz
    s = L.Solver(gen.config(cfg), form="primal", rho=1.0)
    s.step(20)
    for _ in range(5):
        s.step(1)
    torch.cuda.synchronize()
    s.close()
