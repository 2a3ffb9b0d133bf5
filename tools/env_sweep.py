"""A/B of compile-time env knobs on one workload: each variant runs in its own process (the knobs are
read once per process), loads the pattern, runs W warm-up + K timed runs and prints the median and
min run time (the library's own CUDA-event time around the run's graph, stats.last_run_ms) plus
the pass count. Diagnostic only.

python tools/env_sweep.py --workload C3 --mode sampled "" "OWQS_MAX_BFLY=32" "OWQS_COEF_SRC=ptr OWQS_MAX_BFLY=30"
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import json, statistics, sys
sys.path.insert(0, %r)
from paper_1604_05659_b200 import Simulator
from workloads import patterns as W
p = W.config_pattern(%r, seed=1)
s = Simulator(precision=%d)
s.load(p)
ts = []
for r in range(%d + %d):
    s.set_input_random(1)
    s.run(%r, seed=r, want=False)
    if r >= %d:
        ts.append(s.stats()["last_run_ms"])
st = s.stats()
print("RESULT " + json.dumps({"median_ms": statistics.median(ts), "min_ms": min(ts), "passes": st["n_passes"],
                               "launches": st["n_launches"], "jit_ms": st.get("jit_ms")}))
s.close()
"""


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="C3")
    ap.add_argument("--mode", default="sampled")
    ap.add_argument("--precision", type=int, default=64)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--runs", type=int, default=7)
    ap.add_argument("variants", nargs="*", default=[""])
    a = ap.parse_args()
    for v in a.variants:
        env = dict(os.environ)
        for kv in v.split():
            k, val = kv.split("=", 1)
            env[k] = val
        code = CHILD % (ROOT, a.workload, a.precision, a.warmup, a.runs, a.mode, a.warmup)
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=900)
        line = [x for x in r.stdout.splitlines() if x.startswith("RESULT ")]
        res = json.loads(line[0][7:]) if line else {"error": (r.stderr or r.stdout)[-400:]}
        print(json.dumps({"workload": a.workload, "mode": a.mode, "variant": v or "default", **res}), flush=True)


if __name__ == "__main__":
    main()
