"""Per-pass timing of a workload (OWQS_FLAG_PROFILE events between launches) joined with each pass's
shape from the host compiler: group slots, butterflies on register / lane slots, reduction kind.

python tools/pass_profile.py [--workload C3] [--mode sampled] [--precision 64] [--flags 0] [--out f.json]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1604_05659_b200 import Simulator  # noqa: E402
from paper_1604_05659_b200._capi import FLAG_PROFILE  # noqa: E402
from paper_1604_05659_b200.host import compile_host  # noqa: E402
from workloads import patterns as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="C3")
ap.add_argument("--mode", default="sampled")
ap.add_argument("--precision", type=int, default=64)
ap.add_argument("--flags", type=int, default=0)
ap.add_argument("--runs", type=int, default=3)
ap.add_argument("--out", default=None)
a = ap.parse_args()
p = W.config_pattern(a.workload, seed=1)
s = Simulator(precision=a.precision, flags=a.flags | FLAG_PROFILE)
s.load(p)
best = None
for r in range(a.runs):
    s.set_input_random(1)
    s.run(a.mode, seed=r, want=False)
    kc, by, ms = s.launch_profile()
    best = ms if best is None else [min(x, y) for x, y in zip(best, ms)]
hp = compile_host(p, a.mode, a.precision, a.flags)
SB = 6 if a.precision == 64 else 5
rows = []
for i, st in enumerate(hp.steps):
    ops = [st.ops[k] for k in range(st.n_ops)]
    bf = [o for o in ops if o.type == 4]
    lane = sum(1 for o in bf if (o.a < SB and not (SB == 6 and o.a == 0)))
    rows.append({"i": i, "kind": st.kind, "kclass": int(kc[i]), "ms": float(best[i]), "gbs": float(by[i] / best[i] / 1e6) if best[i] else 0.0,
                 "khi": st.nb_hi, "n_ops": st.n_ops, "bfly": len(bf), "lane_bfly": lane, "red": st.red_kind,
                 "flush": sum(1 for o in ops if o.type == 5), "x": sum(1 for o in ops if o.type == 3)})
tot = sum(r["ms"] for r in rows)
print(f"{a.workload} {a.mode} c{a.precision}: {len(rows)} steps, {tot:.2f} ms (sum of per-launch), stats {s.stats()}")
for r in sorted(rows, key=lambda r: -r["ms"])[:25]:
    print(r)
if a.out:
    with open(a.out, "w") as f:
        json.dump({"rows": rows, "total_ms": tot}, f)
s.close()
