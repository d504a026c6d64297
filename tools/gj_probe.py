import sys, time
sys.path.insert(0, '.')
import paper_1609_06068_b200 as L, sdp_inputs as gen
p = gen.block_arrow(60, 12, 8, 2000, seed=3)
for _ in range(2):
    t0 = time.perf_counter(); s = L.Solver(p, form="primal", rho=1.0); t1 = time.perf_counter(); s.close()
    print("setup", t1 - t0, flush=True)
