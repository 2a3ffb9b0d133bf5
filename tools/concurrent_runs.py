"""Kernel throughput of config 3 with 1, 2, 3 contexts running concurrently on their own streams
(threads; owqs_run releases the GIL): does interleaving runs cost efficiency?"""
import os
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1604_05659_b200 import Simulator  # noqa: E402
from workloads import patterns as W  # noqa: E402

p = W.config_pattern("C3", seed=1)
streams = [torch.cuda.Stream() for _ in range(3)]
sims = [Simulator(precision=64, stream=s.cuda_stream) for s in streams]
for s in sims:
    s.load(p)
    s.set_input_random(1)
    s.run("sampled", seed=1, want=False)
torch.cuda.synchronize()
R = 6
for k in (1, 2, 3):
    def work(s):
        for r in range(R):
            s.set_input_random(r)
            s.run("sampled", seed=r, want=False)
    ts = [threading.Thread(target=work, args=(sims[i],)) for i in range(k)]
    t0 = time.perf_counter()
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"{k} concurrent contexts: {1e3 * dt / (k * R):.1f} ms per run (incl. set_input_random 2.7 ms)", flush=True)
