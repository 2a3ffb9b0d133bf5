"""Per-pass time variation across runs (FLAG_PROFILE events): per-run sums and the passes whose
time varies most. Diagnostic only."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1604_05659_b200 import Simulator  # noqa: E402
from paper_1604_05659_b200._capi import FLAG_PROFILE  # noqa: E402
from workloads import patterns as W  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "C3"
_keep = None
if os.environ.get("PV_TORCH"):
    import torch
    torch.cuda.init()
    torch.zeros(1, device="cuda")
    if os.environ.get("PV_ALLOC"):
        _keep = torch.empty(int(os.environ["PV_ALLOC"]) << 20, dtype=torch.uint8, device="cuda")
p = W.config_pattern(wl, seed=1)
s = Simulator(precision=64, flags=FLAG_PROFILE)
s.load(p)
T = []
for r in range(int(os.environ.get("PV_RUNS", "6"))):
    s.set_input_random(1)
    s.run("sampled", seed=r % 2, want=False)
    kc, by, ms = s.launch_profile()
    T.append(np.asarray(ms, dtype=np.float64))
    print(f"run {r} seed {r % 2}: launches {len(ms)} sum {np.sum(ms):.2f} ms  last_run_ms {s.stats()['last_run_ms']:.2f}", flush=True)
T = np.array(T[1:])
spread = T.max(0) - T.min(0)
for i in np.argsort(-spread)[:12]:
    print(i, kc[i], np.round(T[:, i], 3))
