"""Per-size timing of sdp_project_psd_batch (diagnostics for the cfg4 tiers)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1609_06068_b200 as L
import sdp_inputs as gen

res = {}
for k in ([int(x) for x in sys.argv[1].split(',')] if len(sys.argv) > 1 else (8, 16, 32, 64)):
    for count in (50000,):
        ks = np.full(count, k, np.int32)
        rng = np.random.default_rng(k)
        s = k * (k + 1) // 2
        G = rng.standard_normal((count, k, k))
        X = 0.5 * (G + G.transpose(0, 2, 1))
        r, c = gen.packed_upper_index(k)
        vals = X[:, r, c].reshape(-1).copy()
        plan = L.PsdPlan(ks)
        din = torch.from_numpy(vals).cuda(); dout = torch.empty_like(din)
        for _ in range(2): plan.project(din, dout)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); plan.project(din, dout); e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        fl = count * 10.0 * k ** 3
        res[f"k{k}"] = {"count": count, "ms": ms, "proj_per_s": count / ms * 1e3, "alg_tflops": fl / ms / 1e9}
        print(k, count, f"{ms:.2f} ms", f"{count/ms*1e3:.3e} proj/s", f"{fl/ms/1e9:.3f} TF(alg)", flush=True)
print(json.dumps(res))
