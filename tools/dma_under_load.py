"""PCIe copy time of 2 GiB page-locked H2D / D2H alone and while config-3 kernels run on another
stream (does the DMA slow down under the pass kernels' HBM traffic?)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1604_05659_b200 import Simulator  # noqa: E402
from workloads import patterns as W  # noqa: E402

n = 2 << 30
h_in = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h_out = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d_a = torch.empty(n, dtype=torch.uint8, device="cuda")
d_b = torch.empty(n, dtype=torch.uint8, device="cuda")
cs, ks = torch.cuda.Stream(), torch.cuda.Stream()
sim = Simulator(precision=64, stream=ks.cuda_stream)
sim.load(W.config_pattern("C3", seed=1))


def copies(kind):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(cs):
        e0.record(cs)
        if kind in ("h2d", "both"):
            d_a.copy_(h_in, non_blocking=True)
        if kind in ("d2h", "both"):
            h_out.copy_(d_b, non_blocking=True)
        e1.record(cs)
    return e0, e1


for kind in ("h2d", "d2h", "both"):
    for load in (False, True):
        sim.set_input_random(1)
        torch.cuda.synchronize()
        if load:
            sim.run("sampled", seed=1, want=False)  # returns after the run; start copies concurrently below
        torch.cuda.synchronize()
        # concurrent: enqueue the kernels, then the copies on another stream
        sim.set_input_random(1)
        torch.cuda.synchronize()
        import threading
        if load:
            t = threading.Thread(target=lambda: sim.run("sampled", seed=2, want=False))
            t.start()
        e0, e1 = copies(kind)
        torch.cuda.synchronize()
        if load:
            t.join()
        print(f"{kind:5s} {'under C3 kernels' if load else 'alone':17s} {e0.elapsed_time(e1):7.1f} ms", flush=True)
