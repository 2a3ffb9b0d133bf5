"""Fuzz the CUDA path against the oracle on seeds and shapes the test suite does not use (diagnostic;
the oracle is test infrastructure, this tool is not part of the product path).

  python tools/fuzz_parity.py --minutes 8 --seed0 1000

Each case draws a pattern family (random general D0-D3 patterns at small and direct-engine widths,
grow/shrink-heavy wide patterns at tile-engine widths, brickwork and cluster slices, measured
tails), a precision, a mode (sampled / forced / eowqs where a gflow exists) and a Haar input, runs
both sides and applies tests/parity_util.check (north-star tolerances). Prints one JSON line per
failure and a summary line."""
import argparse
import json
import os
import sys
import time
import traceback

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from parity_util import check  # noqa: E402
from paper_1604_05659_b200 import FLAG_LOOPBACK, Simulator  # noqa: E402
from paper_1604_05659_b200.owqs import OwqsError  # noqa: E402
from workloads import patterns as W  # noqa: E402
from workloads.inputs import haar_state  # noqa: E402


def draw_case(rng, seed):
    fam = rng.choice(["general", "general_big", "wide", "bw", "cl", "bwm"], p=[0.25, 0.2, 0.2, 0.15, 0.1, 0.1])
    if fam == "general":
        n_in = int(rng.integers(1, 4))
        n_total = int(rng.integers(n_in + 4, n_in + 9))
        p = W.random_general_pattern(seed, n_in=n_in, n_total=n_total, n_out=int(rng.integers(1, 4)),
                                     max_live=int(rng.integers(4, 8)))
        det = False
    elif fam == "general_big":
        n_in = int(rng.integers(5, 9))
        p = W.random_general_pattern(seed, n_in=n_in, n_total=n_in + int(rng.integers(8, 14)),
                                     n_out=int(rng.integers(2, 6)), max_live=int(rng.integers(11, 16)))
        det = False
    elif fam == "wide":
        n_in = int(rng.integers(12, 16))
        hi = int(rng.integers(n_in + 1, 19))
        p = W.wide_random_pattern(seed, n_in=n_in, width_hi=hi, rounds=int(rng.integers(1, 4)),
                                  n_out=int(rng.integers(8, n_in)))
        det = False
    elif fam == "bw":
        p = W.config_pattern(f"BW:{int(rng.integers(4, 18))}x{int(rng.integers(1, 9))}", seed=seed)
        det = True
    elif fam == "cl":
        p = W.config_pattern(f"CL:{int(rng.integers(3, 15))}x{int(rng.integers(2, 6))}", seed=seed)
        det = True
    else:
        n = int(rng.integers(8, 17))
        p = W.config_pattern(f"BWM:{n}x{int(rng.integers(2, 8))}x{int(rng.integers(1, min(n - 2, 7)))}", seed=seed)
        det = False
    return fam, p, det


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--minutes", type=float, default=5.0)
    ap.add_argument("--seed0", type=int, default=1000)
    ap.add_argument("--loopback", action="store_true",
                    help="also shard over G = 2 / 4 / 8 virtual ranks on the one device (OWQS_FLAG_LOOPBACK)")
    a = ap.parse_args()
    sims = {}

    def sim_for(prec, G):
        if (prec, G) not in sims:
            sims[(prec, G)] = (Simulator(precision=prec) if G == 1 else
                               Simulator(precision=prec, flags=FLAG_LOOPBACK, n_ranks=G))
        return sims[(prec, G)]
    t_end = time.time() + 60 * a.minutes
    n = fails = refused = unsupported = 0
    by_fam = {}
    seed = a.seed0
    while time.time() < t_end:
        seed += 1
        rng = np.random.default_rng(seed)
        fam, p, det = draw_case(rng, seed)
        prec = int(rng.choice([128, 64]))
        G = int(rng.choice([1, 2, 4, 8])) if a.loopback else 1
        while G > 1 and (1 << len(p.inputs)) < 4 * G:  # a shard holds at least 4 input amplitudes
            G //= 2
        modes = ["sampled", "forced"] + (["eowqs"] if det else [])
        mode = str(rng.choice(modes))
        psi = haar_state(len(p.inputs), seed)
        forced = rng.integers(0, 2, p.n_measure) if mode == "forced" else None
        n += 1
        by_fam[f"{fam}/G{G}"] = by_fam.get(f"{fam}/G{G}", 0) + 1
        try:
            # non-deterministic patterns: PROA's order changes per-M probabilities (R-8): joint
            # branch probability and amplitudes are compared; impossible forced branches are skipped
            check(sim_for(prec, G), p, psi, mode, seed=seed, forced=forced, same_order=None if det else False)
        except Exception as e:  # noqa: BLE001
            msg = str(e)
            if "probability" in msg and mode == "forced" and not det:
                refused += 1  # the oracle refuses an impossible forced branch
                continue
            if isinstance(e, OwqsError) and getattr(e, "status_name", "") == "OWQS_E_BRANCH" and mode == "forced" and not det:
                refused += 1
                continue
            if G > 1 and isinstance(e, OwqsError) and "constant-width" in msg:
                unsupported += 1  # documented limit (owqs.h): sharded programs have no GROW / SHRINK steps
                continue
            fails += 1
            print(json.dumps({"fail": True, "seed": seed, "family": fam, "name": p.name, "precision": prec, "mode": mode, "ranks": G,
                              "n_in": len(p.inputs), "n_measure": int(p.n_measure), "error": msg[:300],
                              "where": traceback.format_exc().splitlines()[-3][:200]}), flush=True)
    for s in sims.values():
        s.close()
    print(json.dumps({"cases": n, "failures": fails, "refused_forced_branches": refused,
                      "sharded_unsupported_grow_shrink": unsupported, "by_family": by_fam,
                      "seed0": a.seed0, "minutes": a.minutes}), flush=True)
    return 1 if fails else 0


if __name__ == "__main__":
    sys.exit(main())
