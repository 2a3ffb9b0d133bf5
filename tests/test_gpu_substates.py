"""Patterns whose entanglement graph has several components run as separate sub-states (PAPER §4.1,
L155: "the separate states (called sub-states) can be saved in distinct vectors ... combined only
when the entanglement operation is applied"): each component on its own state
vector, the output assembled by the tensor-merge kernel. Checked against the oracle (one dense
vector in the given order) at both precisions, plus the memory claim (largest sub-state, not the
sum) and the fallbacks (a signal crossing components, OWQS_FLAG_ONE_STATE)."""
import numpy as np
import pytest

import oracle
from paper_1604_05659_b200 import OwqsError, Simulator
from paper_1604_05659_b200._capi import FLAG_ONE_STATE
from parity_util import TOL, fidelity
from workloads import patterns as W
from workloads.inputs import haar_state

pytestmark = pytest.mark.gpu


def fragment(p, offset, keep_inputs):
    """p with qubit ids shifted by offset; its inputs become N-prepared |+> qubits unless kept."""
    sh = lambda q: q + offset  # noqa: E731
    cmds = [W.Cmd(c.kind, sh(c.q0), sh(c.q1) if c.q1 >= 0 else -1, c.angle, tuple(map(sh, c.sdom)),
                  tuple(map(sh, c.tdom))) for c in p.cmds]
    ins = [sh(q) for q in p.inputs]
    if not keep_inputs:
        cmds = [W.N(q) for q in ins] + cmds
        ins = []
    return ins, [sh(q) for q in p.outputs], cmds


def interleave(a, b, seed):
    """merge two command lists keeping each one's order (a random given-order shuffle)."""
    rng = np.random.default_rng(seed)
    out, i, j = [], 0, 0
    while i < len(a) or j < len(b):
        if j >= len(b) or (i < len(a) and rng.random() < 0.5):
            out.append(a[i])
            i += 1
        else:
            out.append(b[j])
            j += 1
    return out


def disconnected(seed=1):
    """a 4-wire J/CZ circuit on the inputs + an input-free 3x3 flow cluster + an untouched output
    qubit; outputs interleaved across the components."""
    ci, co, cc = fragment(W.config_pattern("BW:4x3", seed=seed), 0, True)
    _, ko, kc = fragment(W.cluster_pattern(3, 3, seed=seed), 1000, False)
    lone = 2000
    outs = [co[0], ko[0], co[1], lone, ko[1], co[2], ko[2], co[3]]
    return W.Pattern(ci, outs, interleave(cc, kc, seed), "disconnected")


def check_all_modes(s, p, psi, prec, eowqs=True):
    tol = TOL[prec]
    s.load(p)
    rng = np.random.default_rng(7)
    for _ in range(3):
        forced = rng.integers(0, 2, p.n_measure)
        s.set_input(psi)
        outc, p0 = s.run("forced", forced=forced)
        ref = oracle.run(p, psi, mode="forced", forced=forced)
        out = s.get_output()
        assert list(outc) == list(forced)
        assert np.max(np.abs(out - ref.output)) <= tol["amp"]
        joint = lambda pr, oc: float(np.prod([q if b == 0 else 1 - q for q, b in zip(pr, oc)]))  # noqa: E731
        assert abs(joint(p0, outc) - joint(ref.prob0, ref.outcomes)) <= 1e-6
        if prec == 64:
            assert 1 - fidelity(out, ref.output) <= tol["fid"]
    s.set_input(psi)
    outc, _ = s.run("sampled", seed=11)
    assert list(outc) == list(oracle.run(p, psi, mode="sampled", seed=11).outcomes)
    if not eowqs:
        return
    s.set_input(psi)
    s.run("eowqs", want=False)
    ref = oracle.run(p, psi, mode="eowqs")
    assert np.max(np.abs(s.get_output() - ref.output)) <= tol["amp"]


@pytest.mark.parametrize("prec", [128, 64])
def test_disconnected_pattern_runs_as_substates(require_gpu, prec):
    p = disconnected()
    psi = haar_state(len(p.inputs), 5)
    s = Simulator(precision=prec)
    one = Simulator(precision=prec, flags=FLAG_ONE_STATE)
    try:
        check_all_modes(s, p, psi, prec)
        st = s.stats()
        assert st["n_substates"] == 3
        one.load(p)
        assert one.stats()["n_substates"] == 1
        # memory: the largest sub-state, not the whole pattern's width
        assert st["phys_bits"] < one.stats()["phys_bits"]
        # same outputs through the one-state path
        s.set_input(psi)
        s.run("forced", forced=[0] * p.n_measure)
        one.set_input(psi)
        one.run("forced", forced=[0] * p.n_measure)
        assert np.max(np.abs(s.get_output() - one.get_output())) <= TOL[prec]["amp"]
    finally:
        s.close()
        one.close()


def test_fully_measured_component_and_no_inputs(require_gpu):
    """a component with no outputs (its outcome-dependent phase is a scalar factor) and a pattern
    without inputs (every sub-state starts from the 0-qubit state)."""
    a = [W.N(10), W.N(11), W.E(10, 11), W.M(10, 0.3), W.M(11, 1.1, sdom=(10,))]
    _, ko, kc = fragment(W.cluster_pattern(2, 3, seed=3), 100, False)
    p = W.Pattern([], ko, interleave(a, kc, 2), "no-inputs")
    s = Simulator(precision=128)
    try:
        check_all_modes(s, p, np.array([1.0 + 0j]), 128, eowqs=False)
        assert s.stats()["n_substates"] == 2
        # the fully measured component has no outputs to correct: no gflow, EOWQS refused (L372)
        s.set_input(np.array([1.0 + 0j]))
        with pytest.raises(OwqsError) as e:
            s.run("eowqs")
        assert e.value.status_name == "OWQS_E_NO_GFLOW"
    finally:
        s.close()


def test_crossing_signal_keeps_one_state(require_gpu):
    """a measurement domain that references another component: executed as one state."""
    ci, co, cc = fragment(W.config_pattern("BW:3x2", seed=2), 0, True)
    kc = [W.N(500), W.N(501), W.E(500, 501), W.M(500, 0.4, sdom=(ci[0],))]
    p = W.Pattern(ci, co + [501], cc + kc, "crossing")
    s = Simulator(precision=128)
    try:
        check_all_modes(s, p, haar_state(len(ci), 3), 128)
        assert s.stats()["n_substates"] == 1
    finally:
        s.close()


def test_unsupported_calls_report_state(require_gpu):
    p = disconnected(2)
    s = Simulator(precision=128)
    try:
        s.load(p)
        with pytest.raises(OwqsError) as e:
            s.recognize()
        assert e.value.status_name == "OWQS_E_STATE"
    finally:
        s.close()
