"""One structured matrix through the QL tier (SDP_PSD_TIERS=trd SDP_TRD_DEBUG=1)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402

import paper_1609_06068_b200 as L  # noqa: E402
from oracle import psd as opsd  # noqa: E402
from test_gpu_parity import _structured  # noqa: E402

want_k, want_name = int(sys.argv[1]), sys.argv[2]
names = ["zero", "eye", "clusters", "rank1", "pm", "sparse", "-0.5I"]
rng = np.random.default_rng(11)
for k in (17, 23, 32, 33, 47, 64):
    for name, M in zip(names, _structured(k, rng)):
        if k == want_k and name == want_name:
            out = L.PsdPlan(np.array([k], np.int32)).project_host(opsd.pack_upper(M))
            P = opsd.project_psd(M)
            print("err", np.linalg.norm(opsd.unpack_upper(out, k) - P) / np.linalg.norm(M))
            w = np.linalg.eigvalsh(M)
            print("eigs", w[:3], w[-3:])
            np.save("gpurun_out/diag_M.npy", M)
