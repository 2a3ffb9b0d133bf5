"""A/B of run-time conditions for one workload: mean wall time per run (CUDA events) under
default vs side stream, device-random vs copied input, and outcome seeds. Diagnostic only."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1604_05659_b200 import Simulator  # noqa: E402
from workloads import patterns as W  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "C3"
p = W.config_pattern(wl, seed=1)
n = len(p.inputs)
x = torch.empty(2 ** n, dtype=torch.complex64, device="cuda")
g = Simulator(precision=64)
g.load(W.Pattern(list(range(n)), list(range(n)), []))
g.set_input_random(1)
g.run("eowqs", want=False)
g.get_output_device(x.data_ptr(), 64, 2 ** n)
g.close()
torch.cuda.synchronize()


def timed(s, inp, seed0, stream, runs=6):
    ts = []
    for r in range(runs + 2):
        if inp == "rand":
            s.set_input_random(1)
        else:
            s.set_input_device(x.data_ptr(), 64, 2 ** n)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        s.run("sampled", seed=seed0 + r, want=False)
        e1.record(stream)
        torch.cuda.synchronize()
        if r >= 2:
            ts.append(e0.elapsed_time(e1))
    return sum(ts) / len(ts), min(ts), max(ts)


flag_sets = [int(f) for f in sys.argv[2].split(",")] if len(sys.argv) > 2 else [0]
for fl in flag_sets:
    for stream_kind in ("default", "side"):
        st = torch.cuda.Stream() if stream_kind == "side" else torch.cuda.default_stream()
        kw = {"stream": st.cuda_stream} if stream_kind == "side" else {}
        s = Simulator(precision=64, flags=fl, **kw)
        s.load(p)
        for inp in ("rand", "copy"):
            m, lo, hi = timed(s, inp, 0, st)
            print(f"{wl} flags={fl} stream={stream_kind} input={inp}: mean {m:.2f} min {lo:.2f} max {hi:.2f} ms", flush=True)
        s.close()

if os.environ.get("AB_IDLE"):
    import time
    s = Simulator(precision=64)
    s.load(p)
    for pause in (2.0, 0.5, 0.1, 0.0, 0.0, 0.0, 2.0, 0.0):
        time.sleep(pause)
        m, lo, hi = timed(s, "rand", 0, torch.cuda.default_stream(), runs=1)
        print(f"after {pause:.1f} s idle: {m:.2f} ms", flush=True)
    s.close()
