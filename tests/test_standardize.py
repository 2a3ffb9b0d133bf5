"""Standardisation and signal shifting (standardize.cpp), checked against the
oracle on CPU: the rewritten pattern has the standard form N* E* M* C* (PAPER L93, L153), the same
outcome labels and per-measurement probabilities (Eq. 3) on every branch, and the same output up to a
branch-dependent global phase (reading R-18; the X absorption <+-phi|X = +-e^{-i phi}<+-(-phi)|).
Signal shifting relabels outcomes as s(new) = s(old) + |T|; branches are mapped accordingly."""
import numpy as np
import pytest

import oracle
from paper_1604_05659_b200.host import compile_host, standardize
from workloads import patterns as W
from workloads.inputs import haar_state

KIND_N, KIND_E, KIND_M, KIND_X, KIND_Z = 0, 1, 2, 3, 4


def assert_standard_form(orig, std):
    kinds = [c.kind for c in std.cmds]
    order = {KIND_N: 0, KIND_E: 1, KIND_M: 2, KIND_X: 3, KIND_Z: 3}
    ranks = [order[k] for k in kinds]
    assert ranks == sorted(ranks), "not N* E* M* C*"
    assert [c.q0 for c in std.cmds if c.kind == KIND_M] == orig.measured_in_given_order()
    for c in std.cmds:
        if c.kind in (KIND_X, KIND_Z):
            assert c.q0 in orig.outputs, "correction left on a non-output qubit"
    # E's (as sets) preserved
    e0 = sorted(tuple(sorted((c.q0, c.q1))) for c in orig.cmds if c.kind == KIND_E)
    e1 = sorted(tuple(sorted((c.q0, c.q1))) for c in std.cmds if c.kind == KIND_E)
    assert e0 == e1


def phase_equal(a, b, tol=1e-10):
    """a == e^{i phi} b for some phi (both normalised outputs of the same branch)."""
    ov = np.vdot(b, a)
    return abs(abs(ov) - np.linalg.norm(a) * np.linalg.norm(b)) < tol and np.allclose(
        a, (ov / abs(ov)) * b if abs(ov) > 0 else a, atol=tol)


def patterns():
    ps = [W.config_pattern("C1", seed=s) for s in range(3)]
    ps += [W.random_general_pattern(s, n_in=2, n_total=8, n_out=2) for s in range(12)]
    # (the oracle runs the standard form in its given order: every N first, so keep |V| <= ~16)
    ps += [W.cnot_pattern_eq22(), W.cnot_pattern_eq23(), W.cluster_pattern(3, 4, seed=1), W.config_pattern("QFT:2")]
    return ps


@pytest.mark.parametrize("k", range(19))
def test_standard_form_equivalent_on_every_branch(k):
    p = patterns()[k]
    std, shifts = standardize(p)
    assert not shifts
    assert_standard_form(p, std)
    psi = haar_state(len(p.inputs), 100 + k)
    rng = np.random.default_rng(k)
    for _ in range(6):
        forced = rng.integers(0, 2, p.n_measure)
        try:
            a = oracle.run(p, psi, "forced", forced=forced)
        except oracle.OracleError:
            continue  # impossible branch of a non-deterministic pattern
        b = oracle.run(std, psi, "forced", forced=forced)
        np.testing.assert_allclose(b.prob0, a.prob0, atol=1e-12)
        assert phase_equal(b.output, a.output)


@pytest.mark.parametrize("k", range(19))
def test_signal_shifting_relabels_outcomes(k):
    p = patterns()[k]
    std, shifts = standardize(p, signal_shift=True)
    assert all(not c.tdom for c in std.cmds if c.kind == KIND_M), "t-domains left after shifting"
    assert_standard_form(p, std)
    psi = haar_state(len(p.inputs), 200 + k)
    rng = np.random.default_rng(50 + k)
    m_q = p.measured_in_given_order()
    for _ in range(6):
        old = rng.integers(0, 2, p.n_measure)
        try:
            a = oracle.run(p, psi, "forced", forced=old)
        except oracle.OracleError:
            continue
        new = {}
        for i, q in enumerate(m_q):  # s(new) = s(old) + |T| over the new labels
            new[q] = (int(old[i]) + sum(new[x] for x in shifts.get(q, ()))) & 1
        b = oracle.run(std, psi, "forced", forced=[new[q] for q in m_q])
        flip = np.array([sum(new[x] for x in shifts.get(q, ())) & 1 for q in m_q])
        exp_p0 = np.where(flip == 1, 1.0 - a.prob0, a.prob0)
        np.testing.assert_allclose(b.prob0, exp_p0, atol=1e-12)
        assert phase_equal(b.output, a.output)


def test_flow_pattern_stays_deterministic():
    """A flow cluster's standard form is still deterministic: EOWQS equals every forced branch."""
    p = W.cluster_pattern(3, 4, seed=2)
    std, _ = standardize(p, signal_shift=True)
    psi = haar_state(3, 9)
    e = oracle.run(std, psi, "eowqs").output
    rng = np.random.default_rng(3)
    for _ in range(8):
        b = oracle.run(std, psi, "forced", forced=rng.integers(0, 2, p.n_measure)).output
        assert phase_equal(b, e, tol=1e-9)


@pytest.mark.parametrize("n", [3, 5, 8])
def test_proa_on_standard_form_qft(n):
    """PROA on the standard-form input the paper assumes (L153): the QFT rows of Table III keep
    m = n + 1 (L497-501), and the compiled program of the standard form has the same width."""
    std, _ = standardize(W.config_pattern(f"QFT:{n}"))
    hp = compile_host(std)
    assert hp.info["paper_m"] == n + 1
    assert hp.info["phys_bits"] <= n + 1
