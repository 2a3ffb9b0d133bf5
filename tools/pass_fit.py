"""Least-squares per-pass cost model from a pass_profile.py json and the generated sources:
ms = base + a * butterflies + sum_k c_k * (transposes synchronised by barrier kind k)."""
import json
import re
import sys

import numpy as np

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_1604_05659_b200.host import jit_host  # noqa: E402
from workloads.patterns import config_pattern  # noqa: E402

wl, js = sys.argv[1], sys.argv[2]
rows = json.load(open(js))["rows"]
src = jit_host(config_pattern(wl, seed=1), "sampled", 64, sources=True)["sources"]
X, y = [], []
for r in rows:
    s = src.get(r["i"], "")
    n64 = len(re.findall(r'"r"\(64\) : "memory"', s))
    n128 = len(re.findall(r'"r"\(128\) : "memory"', s))
    nw = s.count("__syncwarp()")
    nc = len(re.findall(r"layout \d+ -> \d+", s)) - n64 - n128 - nw
    X.append([1, r["bfly"], nw, n64, n128, nc])
    y.append(r["ms"])
X, y = np.array(X, float), np.array(y)
c = np.linalg.lstsq(X, y, rcond=None)[0]
names = ["base", "bfly", "t_warp", "t_64", "t_128", "t_cta"]
print(wl, "fit:", ", ".join(f"{n} {v:.4f}" for n, v in zip(names, c)), f"rms {np.sqrt(np.mean((X @ c - y) ** 2)):.3f}")
print("totals ms:", ", ".join(f"{n} {v * X[:, i].sum():.2f}" for i, (n, v) in enumerate(zip(names, c))), f"measured {y.sum():.2f}")
print("counts:", dict(zip(names[1:], X[:, 1:].sum(0).astype(int).tolist())))
