"""A fixed slice of tools/fuzz_parity.py in the GPU suite: seeded random cases over every pattern
family (random D0-D3 patterns, grow / shrink-heavy wide patterns, brickwork and cluster slices,
measured tails), both precisions, all modes, 1 / 2 / 4 / 8 (loopback) ranks, each compared with the
oracle by parity_util.check at the north-star tolerances."""
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))

from fuzz_parity import draw_case  # noqa: E402
from paper_1604_05659_b200 import FLAG_LOOPBACK, Simulator  # noqa: E402
from paper_1604_05659_b200.owqs import OwqsError  # noqa: E402
from parity_util import check  # noqa: E402
from workloads.inputs import haar_state  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed0,loopback", [(123000, False), (456000, True)])
def test_fuzz_slice_vs_oracle(require_gpu, seed0, loopback):
    sims = {}
    ran = 0
    try:
        for seed in range(seed0, seed0 + 60):
            rng = np.random.default_rng(seed)
            fam, p, det = draw_case(rng, seed)
            prec = int(rng.choice([128, 64]))
            G = int(rng.choice([1, 2, 4, 8])) if loopback else 1
            while G > 1 and (1 << len(p.inputs)) < 4 * G:
                G //= 2
            mode = str(rng.choice(["sampled", "forced"] + (["eowqs"] if det else [])))
            psi = haar_state(len(p.inputs), seed)
            forced = rng.integers(0, 2, p.n_measure) if mode == "forced" else None
            if (prec, G) not in sims:
                sims[(prec, G)] = (Simulator(precision=prec) if G == 1 else
                                   Simulator(precision=prec, flags=FLAG_LOOPBACK, n_ranks=G))
            try:
                check(sims[(prec, G)], p, psi, mode, seed=seed, forced=forced, same_order=None if det else False)
                ran += 1
            except OwqsError as e:
                if G > 1 and e.status_name == "OWQS_E_ARG" and "constant-width" in str(e):
                    continue  # documented limit (owqs.h): sharded programs have no GROW / SHRINK steps
                # an impossible forced branch of a non-deterministic pattern is refused by both sides
                assert mode == "forced" and not det and e.status_name == "OWQS_E_BRANCH", (seed, fam, str(e))
            except Exception as e:  # the oracle refuses the same kind of branch
                assert mode == "forced" and not det and "probability" in str(e), (seed, fam, prec, mode, G, str(e))
    finally:
        for s in sims.values():
            s.close()
    assert ran >= (25 if loopback else 50)
