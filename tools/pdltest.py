import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
from workloads import patterns as W
from workloads.inputs import haar_state
from paper_1604_05659_b200 import Simulator
p = W.config_pattern("QFT:13")
psi = haar_state(13, 13)
for prec in (128, 64):
    s = Simulator(precision=prec)
    s.load(p)
    ok = 0
    for r in range(20):
        s.set_input(psi)
        try:
            s.run("sampled", seed=3 + r, want=False); ok += 1
        except Exception as e:
            err = str(e)[:80]
    print(os.environ.get("OWQS_NO_PDL"), os.environ.get("OWQS_PDL_NO_TRIGGER"), prec, "ok", ok, "/ 20")
    s.close()
