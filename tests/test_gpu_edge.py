"""GPU edge cases: degenerate patterns (no commands, no measurements, corrections only, spectator
qubits, permuted outputs), the tile-engine width boundary, and the largest single-GPU state of the
BASELINE configs (config 4: 2^33 complex64 = 64 GiB), checked against the oracle or, past its reach,
against invariants (norm, Eq. 13 structural probabilities, outcome independence)."""
import numpy as np
import pytest

import oracle
from paper_1604_05659_b200 import FLAG_MEASURED_NORM, Simulator
from parity_util import check, fidelity, TOL
from workloads import patterns as W
from workloads.inputs import haar_state

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", params=[128, 64])
def sim(request, require_gpu):
    s = Simulator(precision=request.param)
    yield s
    s.close()


def test_empty_pattern_is_identity(sim):
    """No commands, O = I: the output is the input (L153)."""
    for n in (1, 3, 14):
        p = W.Pattern(list(range(n)), list(range(n)), [], "empty")
        psi = haar_state(n, n)
        out, _ = check(sim, p, psi, "sampled")
        assert np.max(np.abs(out - psi)) <= TOL[sim.precision]["amp"]


def test_permuted_outputs_and_spectators(sim):
    """Outputs in another order than the inputs (bit k <-> outputs[k], reading R-10), a spectator
    input no command touches, and corrections with empty domains."""
    p = W.Pattern([0, 1, 2], [2, 0, 1], [W.E(0, 1), W.Z(2), W.X(0)], "perm")
    psi = haar_state(3, 5)
    check(sim, p, psi, "sampled")
    # wide: 15 qubits reversed, a CZ ladder, no measurement (tile engine width at complex128)
    n = 15
    cmds = [W.E(k, k + 1) for k in range(0, n - 1, 2)]
    p = W.Pattern(list(range(n)), list(reversed(range(n))), cmds, "rev")
    check(sim, p, haar_state(n, 6), "eowqs")


def test_single_j_pattern_all_branches(sim):
    """The smallest measuring pattern: J(alpha) on one qubit (N_o E_io M_i X_o), every branch."""
    p = W.j_pattern(0.7)
    psi = haar_state(1, 2)
    for br in (0, 1):
        check(sim, p, psi, "forced", forced=[br])
    check(sim, p, psi, "eowqs")


@pytest.mark.parametrize("n", [12, 13, 14])
def test_tile_engine_width_boundary(sim, n):
    """Widths around the tile engine's minimum (12 complex128 / 13 complex64): 1, 2, 4 CTAs."""
    p = W.config_pattern(f"BW:{n}x3", seed=n)
    psi = haar_state(n, n + 1)
    check(sim, p, psi, "sampled", seed=n)
    check(sim, p, psi, "eowqs")


def test_config4_full_width_invariants(require_gpu):
    """Config 4 at full size on one GPU (33 wires: 2^33 complex64 amplitudes = 64 GiB, the tile
    engine at one tile per CTA, 2^20 CTAs per pass): EOWQS keeps the norm (flow pattern: every
    structural prob0 = 1/2), a sampled run reports prob0 = 1/2 on every M and the two outputs agree
    up to the branch phase (outcome independence of a J/CZ circuit pattern)."""
    p = W.config_pattern("C4", seed=1)
    s = Simulator(precision=64)
    t = Simulator(precision=64, flags=FLAG_MEASURED_NORM)  # structural prob0 reduced on the device
    try:
        for x in (s, t):
            x.load(p)
            x.set_input_random(3)
        s.run("eowqs", want=False)
        assert abs(s.norm2() - 1.0) < 1e-3
        outc, p0 = t.run("sampled", seed=5)
        assert np.max(np.abs(p0 - 0.5)) < 1e-5
        assert abs(t.norm2() - 1.0) < 1e-5
        assert 0 < int(outc.sum()) < len(outc)  # a genuinely mixed branch
        ov = s.inner(t)
        assert 1.0 - abs(ov) ** 2 < 1e-4
    finally:
        s.close()
        t.close()
