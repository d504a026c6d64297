"""Where does a fused step spend its time?  per-call time of step(1) with and without an L2 flush,
and the in-kernel per-iteration time of step(n) / n, for cfg0 / cfg1 at several grid sizes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1609_06068_b200 as L  # noqa: E402
import sdp_inputs as gen  # noqa: E402


def timeit(fn, reps, flush=None):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for a, b in ev:
        if flush is not None:
            flush.fill_(1.0)
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    return sum(a.elapsed_time(b) for a, b in ev) / reps * 1e3  # us


def main():
    scratch = torch.empty(32 << 20, dtype=torch.float64, device="cuda")
    for cfg in (0, 1):
        prob = gen.config(cfg)
        for ctas in ([None, "1", "2", "4"] if cfg == 0 else [None, "16", "37", "74", "148"]):
            for fz in ("1", "0"):
                if fz == "0" and ctas is not None:
                    continue
                os.environ["SDP_FUSED"] = fz
                if ctas:
                    os.environ["SDP_FUSED_CTAS"] = ctas
                else:
                    os.environ.pop("SDP_FUSED_CTAS", None)
                s = L.Solver(prob, form="primal", rho=1.0, stream=torch.cuda.current_stream().cuda_stream)
                s.step(50)
                torch.cuda.synchronize()
                t1 = timeit(lambda: s.step(1), 300)
                t1f = timeit(lambda: s.step(1), 300, scratch)
                tn = timeit(lambda: s.step(1000), 3) / 1000
                print(f"cfg{cfg} fused={fz} ctas={ctas}: step(1) {t1:.1f} us, flushed {t1f:.1f} us, "
                      f"in-launch {tn:.2f} us/iter", flush=True)
                s.close()


if __name__ == "__main__":
    main()
