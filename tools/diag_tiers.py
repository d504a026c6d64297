"""Per-order error of the batch projection (few matrices per order)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1609_06068_b200 as L  # noqa: E402
from oracle import psd as opsd  # noqa: E402

rng = np.random.default_rng(0)
for k in [int(a) for a in sys.argv[1:]]:
    ks = np.full(3, k, np.int32)
    vals = np.concatenate([rng.standard_normal(k * (k + 1) // 2) for _ in ks])
    out = L.PsdPlan(ks).project_host(vals)
    want = opsd.project_psd_packed_batch(ks, vals)
    print(k, "%.2e" % (np.linalg.norm(out - want) / np.linalg.norm(want)), flush=True)
