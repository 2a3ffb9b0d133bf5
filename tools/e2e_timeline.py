"""Host timeline of the 3-context submit/wait pipeline (config 3): when each wait returns, the
device time of each run, and the step interval."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1604_05659_b200 import Simulator  # noqa: E402
from workloads import patterns as W  # noqa: E402

C = int(sys.argv[1]) if len(sys.argv) > 1 else 3
p = W.config_pattern("C3", seed=1)
N = 2 ** 28
streams = [torch.cuda.Stream() for _ in range(C)]
FL = int(sys.argv[2]) if len(sys.argv) > 2 else 0
sims = [Simulator(precision=64, stream=s.cuda_stream, flags=FL) for s in streams]
for s in sims:
    s.load(p)
h_in = torch.empty(N, dtype=torch.complex64, pin_memory=True)
h_in.normal_()
h_in /= h_in.abs().pow(2).sum().sqrt()
outs = [torch.empty(N, dtype=torch.complex64, pin_memory=True) for _ in range(C)]
busy = [False] * C
t0 = time.perf_counter()
log = []
for i in range(4 * C + 6):
    c = i % C
    if busy[c]:
        tw = time.perf_counter()
        sims[c].wait()
        log.append((i, c, tw - t0, time.perf_counter() - t0, sims[c].stats()["last_run_ms"]))
    ts = time.perf_counter()
    sims[c].submit_host(h_in.data_ptr(), 64, outs[c].data_ptr(), 64, "sampled", seed=i)
    busy[c] = True
    log[-1:] and None
for c in range(C):
    if busy[c]:
        sims[c].wait()
prev = None
for i, c, tw, tr, ms in log:
    print(f"step {i:2d} ctx {c}: wait called {1e3 * tw:8.1f} returned {1e3 * tr:8.1f} ms  run {ms:5.1f} ms"
          + (f"  interval {1e3 * (tr - prev):5.1f}" if prev else ""))
    prev = tr
