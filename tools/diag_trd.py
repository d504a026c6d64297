"""Per-matrix QL-tier error on the structured inputs of test_trd_tier_batch_many
(run with SDP_PSD_TIERS=trd so that single matrices take the QL tier)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1609_06068_b200 as L  # noqa: E402
from oracle import psd as opsd  # noqa: E402
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from test_gpu_parity import _structured  # noqa: E402

rng = np.random.default_rng(11)
names = ["zero", "eye", "clusters", "rank1", "pm", "sparse", "-0.5I"]
for k in (17, 23, 32, 33, 47, 64):
    for name, M in zip(names, _structured(k, rng)):
        ks = np.array([k], np.int32)
        v = opsd.pack_upper(M)
        out = L.PsdPlan(ks).project_host(v)
        want = opsd.pack_upper(opsd.project_psd(M))
        e = np.linalg.norm(opsd.unpack_upper(out - want, k)) / max(np.linalg.norm(M), 1e-300)
        if e > 1e-13:
            print(k, name, "%.2e" % e, flush=True)
print("done")
