"""Batched small-width replicas vs the oracle, per replica."""
import numpy as np
import pytest

import oracle
from paper_1604_05659_b200 import FLAG_NO_GFLOW, OwqsError, Simulator
from parity_util import TOL, fidelity
from workloads import patterns as W
from workloads.inputs import basis_state, haar_state

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", params=[128, 64])
def sim(request, require_gpu):
    s = Simulator(precision=request.param)
    yield s
    s.close()


def _assert_close(sim, out, ref):
    tol = TOL[sim.precision]
    assert np.max(np.abs(out - ref.output)) <= tol["amp"]
    if sim.precision == 64:
        assert 1 - fidelity(out, ref.output) <= tol["fid"]


def test_config1_batch_of_64(sim):
    """Config 1: 64 Haar inputs in ONE launch, sampled (per-replica seeds) and forced."""
    for circ in range(3):
        p = W.config_pattern("C1", seed=circ)
        sim.load(p)
        psis = np.stack([haar_state(3, 77 * circ + k) for k in range(64)])
        seeds = np.arange(64) + 1000 * circ
        out, oc, p0 = sim.run_batch(psis, "sampled", seeds=seeds)
        for k in range(64):
            ref = oracle.run(p, psis[k], mode="sampled", seed=int(seeds[k]))
            assert list(oc[k]) == list(ref.outcomes)
            assert np.max(np.abs(p0[k] - ref.prob0)) <= TOL[sim.precision]["prob"]
            _assert_close(sim, out[k], ref)
        forced = np.random.default_rng(circ).integers(0, 2, (64, p.n_measure))
        out, oc, p0 = sim.run_batch(psis, "forced", forced=forced)
        for k in range(64):
            ref = oracle.run(p, psis[k], mode="forced", forced=forced[k])
            assert list(oc[k]) == list(forced[k])
            _assert_close(sim, out[k], ref)
        out, _, _ = sim.run_batch(psis, "eowqs")
        for k in range(0, 64, 7):
            _assert_close(sim, out[k], oracle.run(p, psis[k], mode="eowqs"))


def test_cnot_all_inputs_and_branches(sim):
    sim.load(W.cnot_pattern_eq22())
    psis = np.stack([basis_state(2, k) for k in range(4) for _ in range(4)])
    forced = np.array([[br & 1, br >> 1] for _ in range(4) for br in range(4)], dtype=np.uint8)
    out, oc, _ = sim.run_batch(psis, "forced", forced=forced)
    for i in range(16):
        _assert_close(sim, out[i], oracle.run(W.cnot_pattern_eq22(), psis[i], mode="forced", forced=forced[i]))


@pytest.mark.parametrize("seed", range(12))
def test_random_patterns_batch(sim, seed):
    """Grow / shrink / pending E,Z / corrections inside the one-CTA program interpreter."""
    p = W.random_general_pattern(seed, n_in=2 + seed % 3, n_total=9 + seed % 4, n_out=1 + seed % 3)
    psis = np.stack([haar_state(len(p.inputs), 100 * seed + k) for k in range(8)])
    refs = [oracle.run(p, psis[k], mode="sampled", seed=k) for k in range(8)]
    forced = np.stack([r.outcomes for r in refs])
    sim.load(p)
    out, oc, p0 = sim.run_batch(psis, "forced", forced=forced)
    for k in range(8):
        _assert_close(sim, out[k], refs[k])
    s2 = Simulator(precision=sim.precision, flags=FLAG_NO_GFLOW)
    try:
        s2.load(p)
        for k in range(2):
            ref = oracle.run(p, psis[k], mode="eowqs")
            nrm = np.vdot(ref.output, ref.output).real
            if abs(nrm - 1) <= (1e-8 if sim.precision == 128 else 1e-3):
                out, _, _ = s2.run_batch(psis[k:k + 1], "eowqs")
                _assert_close(sim, out[0], ref)
            else:
                with pytest.raises(OwqsError) as e:
                    s2.run_batch(psis[k:k + 1], "eowqs")
                assert e.value.status_name == "OWQS_E_NOT_DETERMINISTIC"
    finally:
        s2.close()


def test_batch_width_limit(require_gpu):
    s = Simulator(precision=128)
    try:
        s.load(W.config_pattern("BW:14x2", seed=1))
        with pytest.raises(OwqsError) as e:
            s.run_batch(np.stack([haar_state(14, 1)]), "sampled")
        assert e.value.status_name == "OWQS_E_ARG"
    finally:
        s.close()
