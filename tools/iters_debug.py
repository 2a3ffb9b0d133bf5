import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1604_05659_b200 import Simulator
from paper_1604_05659_b200._capi import FLAG_NO_GRAPH, FLAG_PROFILE
from workloads import patterns as W
from workloads.inputs import haar_state
from paper_1604_05659_b200.host import compile_host
for prec in (64, 128):
    for shape in ("BW:16x8", "BW:19x6", "QFT:14"):
        for mode in ("sampled", "eowqs"):
            p = W.config_pattern(shape, seed=3)
            s = Simulator(precision=prec, flags=FLAG_NO_GRAPH | FLAG_PROFILE)
            s.load(p)
            s.set_input(haar_state(len(p.inputs), 4))
            try:
                s.run(mode, seed=7, want=False)
                print(prec, shape, mode, "ok", flush=True)
            except Exception as e:
                print(prec, shape, mode, "FAIL", str(e)[:120], flush=True)
                hp = compile_host(p, mode, prec)
                try:
                    kc, by, ms = s.launch_profile()
                    print("  launches profiled:", len(ms))
                except Exception as e2:
                    print("  no profile", str(e2)[:80])
                print("  widths:", [st.width for st in hp.steps][:40])
                sys.exit(1)
            s.close()
