"""Profiling driver: load a workload, run it R times through the C-ABI (for ncu / sanitizers).

python tools/prof_run.py [--workload C3] [--mode sampled] [--precision 64] [--runs 1] [--flags 0]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1604_05659_b200 import Simulator  # noqa: E402
from workloads import patterns as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="C3")
ap.add_argument("--mode", default="sampled")
ap.add_argument("--precision", type=int, default=64)
ap.add_argument("--runs", type=int, default=1)
ap.add_argument("--flags", type=int, default=0)
a = ap.parse_args()
p = W.config_pattern(a.workload, seed=1)
s = Simulator(precision=a.precision, flags=a.flags)
s.load(p)
for r in range(a.runs):
    s.set_input_random(1)
    s.run(a.mode, seed=r, want=False)
print(a.workload, a.mode, s.stats())
s.close()
