"""Small runs for compute-sanitizer: tile-engine passes (complex64 width 14, complex128 width 13),
a sub-state pattern (kron_merge), sampled + EOWQS. python tools/sanitize_run.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from paper_1604_05659_b200 import Simulator  # noqa: E402
from workloads import patterns as W  # noqa: E402
from workloads.inputs import haar_state  # noqa: E402

for prec, shape in ((64, "BW:14x3"), (128, "BW:13x2")):
    p = W.config_pattern(shape, seed=1)
    s = Simulator(precision=prec, flags=1)  # no graph: every launch visible to the tools
    s.load(p)
    for mode in ("sampled", "eowqs"):
        s.set_input(haar_state(len(p.inputs), 1))
        s.run(mode, seed=3, want=False)
        out = s.get_output()
        assert abs(np.linalg.norm(out) - 1) < 1e-3
    s.close()
from test_gpu_substates import disconnected  # noqa: E402
p = disconnected()
s = Simulator(precision=128, flags=1)
s.load(p)
s.set_input(haar_state(len(p.inputs), 2))
s.run("sampled", seed=1, want=False)
s.get_output()
s.close()
print("sanitize run ok")
