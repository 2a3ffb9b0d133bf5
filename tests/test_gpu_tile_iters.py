"""Tile-engine passes that process several tiles per CTA (states above 2^20 tiles, e.g. complex128
at 33 bits) exercised at small widths: OWQS_TILE_MAX_BLOCKS caps the grid so each CTA loops over
2-64 tiles (end-of-tile barrier, accumulated reduction partials, per-tile remapped stores).
Oracle parity in a subprocess (the cap is read once per process)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import numpy as np, oracle
from paper_1604_05659_b200 import Simulator
from workloads import patterns as W
from workloads.inputs import haar_state
for prec, tol in ((64, 1e-4), (128, 1e-10)):
    s = Simulator(precision=prec)
    for shape in ("BW:16x8", "BW:19x6", "QFT:14"):
        p = W.config_pattern(shape, seed=3)
        psi = haar_state(len(p.inputs), 4)
        s.load(p)
        for mode in ("sampled", "eowqs"):
            s.set_input(psi)
            outc, p0 = s.run(mode, seed=7)
            ref = oracle.run(p, psi, mode=mode, seed=7) if mode == "sampled" else oracle.run(p, psi, mode="eowqs")
            if mode == "sampled":
                assert list(outc) == list(ref.outcomes), (shape, prec)
            err = float(np.max(np.abs(s.get_output() - ref.output)))
            assert err <= tol, (shape, prec, mode, err)
    s.close()
print("ok")
"""


@pytest.mark.parametrize("extra", [{"OWQS_TILE_MAX_BLOCKS": "4"},
                                   {"OWQS_TILE_G": "7", "OWQS_TILE_G128": "7"},
                                   {"OWQS_TILE_G": "5", "OWQS_TILE_MAX_BLOCKS": "8"}])
def test_tile_geometries_vs_oracle(require_gpu, extra):
    """several tiles per CTA, and the non-default tile sizes (13-bit complex64 / 12-bit complex128
    tiles with 8-warp CTAs; 11-bit complex64 tiles with 2-warp CTAs)."""
    env = dict(os.environ, PYTHONPATH=ROOT + os.pathsep + os.path.join(ROOT, "tests"), **extra)
    r = subprocess.run([sys.executable, "-c", SCRIPT], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout[-2000:] + r.stderr[-4000:]
