"""Flushed single-step timing with and without the host running ahead (a long sleep kernel enqueued
first, so the GPU never waits for a launch): separates host launch latency from device time."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1609_06068_b200 as L  # noqa: E402
import sdp_inputs as gen  # noqa: E402


def loop(s, scratch, reps, ahead):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    torch.cuda.synchronize()
    if ahead:
        torch.cuda._sleep(200_000_000)  # ~0.1 s of GPU time: the host enqueues everything meanwhile
    for a, b in ev:
        scratch.fill_(1.0)
        a.record()
        s.step(1)
        b.record()
    torch.cuda.synchronize()
    t = sorted(a.elapsed_time(b) * 1e3 for a, b in ev)
    return sum(t) / reps, t[reps // 2]


scratch = torch.empty(32 << 20, dtype=torch.float64, device="cuda")
for cfg in (0, 1):
    for fz in ("1", "0"):
        os.environ["SDP_FUSED"] = fz
        s = L.Solver(gen.config(cfg), form="primal", rho=1.0, stream=torch.cuda.current_stream().cuda_stream)
        s.step(3000)  # converged state, as in the bench after its warm-up... (bench: warmup then 20000 steps)
        torch.cuda.synchronize()
        for ahead in (False, True):
            m, med = loop(s, scratch, 150, ahead)
            print(f"cfg{cfg} fused={fz} host_ahead={ahead}: mean {m:.1f} us, median {med:.1f} us", flush=True)
        inf = s.info()
        print(f"   sweeps/projection overall {inf['jacobi_sweeps'] / (inf['iters'] * inf['p']):.2f}", flush=True)
        s.close()
