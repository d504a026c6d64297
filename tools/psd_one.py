"""One batched projection of `count` matrices of order k (ncu driver)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1609_06068_b200 as L
import sdp_inputs as gen
k, count = int(sys.argv[1]), int(sys.argv[2])
ks = np.full(count, k, np.int32)
rng = np.random.default_rng(k)
G = rng.standard_normal((count, k, k)); X = 0.5 * (G + G.transpose(0, 2, 1))
r, c = gen.packed_upper_index(k)
vals = X[:, r, c].reshape(-1).copy()
plan = L.PsdPlan(ks)
din = torch.from_numpy(vals).cuda(); dout = torch.empty_like(din)
for _ in range(2):
    plan.project(din, dout)
torch.cuda.synchronize()
print("ok", k, count)
