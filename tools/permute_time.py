"""Time of the output permutation (state slots -> caller order) for config 3: get_output_device."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1604_05659_b200 import Simulator  # noqa: E402
from workloads import patterns as W  # noqa: E402

sim = Simulator(precision=64)
sim.load(W.config_pattern("C3", seed=1))
sim.set_input_random(1)
sim.run("sampled", seed=1, want=False)
out = torch.empty(2 ** 28, dtype=torch.complex64, device="cuda")
for r in range(4):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    sim.get_output_device(out.data_ptr(), 64, 2 ** 28)
    e1.record()
    torch.cuda.synchronize()
    print(f"get_output_device (permute 2^28 complex64): {e0.elapsed_time(e1):.2f} ms")
