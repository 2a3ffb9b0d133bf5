"""GPU parity: the CUDA path through the C-ABI vs the oracle on the same seeded inputs.

Sizes span the small-width CTA kernel (w <= 7-8), the warp-segment pass kernel with several
tiles and a ragged grid-stride tail (w = 10..16), full-size config 2 (closed form) and full-size
config 3 (invariants)."""
import math

import numpy as np
import pytest

import oracle
from paper_1604_05659_b200 import (FLAG_GIVEN_ORDER, FLAG_MEASURED_NORM, FLAG_NO_FUSE, FLAG_NO_GRAPH, FLAG_NO_JIT,
                                    OwqsError, Simulator)
from parity_util import check, fidelity, TOL
from workloads import patterns as W
from workloads.inputs import basis_state, counter_haar_state, haar_state

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", params=[128, 64])
def sim(request, require_gpu):
    s = Simulator(precision=request.param)
    yield s
    s.close()


def test_config1_64_inputs(sim):
    """Config 1: 64 Haar inputs, forced outcomes from a seed and sampled mode, several circuits."""
    for circ in range(3):
        p = W.config_pattern("C1", seed=circ)
        rng = np.random.default_rng(1000 + circ)
        for k in range(64):
            psi = haar_state(3, 10_000 * circ + k)
            forced = rng.integers(0, 2, p.n_measure)
            check(sim, p, psi, "forced", forced=forced)
            check(sim, p, psi, "sampled", seed=k)
        check(sim, p, haar_state(3, 5), "eowqs")


def test_cnot_figure8(sim):
    """Fig. 8 (L433-448): input |11>, outcomes (0, 1) -> |q4q1> = |01>; all branches = CNOT."""
    out, ref = check(sim, W.cnot_pattern_eq23(), basis_state(2, 3), "forced", forced=[0, 1])
    assert np.allclose(out, [0, 1, 0, 0], atol=TOL[sim.precision]["amp"])
    for k in range(4):
        for br in range(4):
            check(sim, W.cnot_pattern_eq22(), basis_state(2, k), "forced", forced=[br & 1, br >> 1])


@pytest.mark.parametrize("n", [4, 8, 11, 13])
def test_qft_vs_oracle(sim, n):
    p = W.config_pattern(f"QFT:{n}")
    psi = haar_state(n, n)
    check(sim, p, psi, "sampled", seed=3)
    check(sim, p, psi, "eowqs")


@pytest.mark.parametrize("flags", [0, FLAG_NO_FUSE, FLAG_NO_GRAPH, FLAG_GIVEN_ORDER | FLAG_NO_FUSE, FLAG_NO_JIT])
@pytest.mark.parametrize("shape", ["BW:12x8", "BW:15x5", "BW:16x3"])
def test_brickwork_vs_oracle(require_gpu, flags, shape):
    """Config 3/4 family at oracle-sized widths (12-16 wires: several 2^k tiles per pass). Default
    flags run the generated kernels (complex64 width >= 13: tile engine; complex128 and narrower:
    direct engine); FLAG_NO_JIT runs the ahead-of-time op-interpreting pass kernel."""
    n = int(shape[3:].split("x")[0])
    p = W.config_pattern(shape, seed=7)
    psi = haar_state(n, 21)
    for prec in (128, 64):
        s = Simulator(precision=prec, flags=flags)
        try:
            check(s, p, psi, "sampled", seed=11)
            check(s, p, psi, "forced", forced=np.random.default_rng(3).integers(0, 2, p.n_measure))
            check(s, p, psi, "eowqs")
        finally:
            s.close()


@pytest.mark.parametrize("shape", ["BW:14x6", "BW:16x4"])
def test_direct_engine_complex64_vs_oracle(require_gpu, monkeypatch, shape):
    """The direct-load generated engine on complex64 (OWQS_JIT_NO_TILE: passes of width >= 13 that
    the tile engine would run), vs the oracle; the packer keeps <= 4 group slots for it."""
    monkeypatch.setenv("OWQS_JIT_NO_TILE", "1")
    n = int(shape[3:].split("x")[0])
    p = W.config_pattern(shape, seed=5)
    psi = haar_state(n, 8)
    s = Simulator(precision=64)
    try:
        check(s, p, psi, "sampled", seed=4)
        check(s, p, psi, "eowqs")
    finally:
        s.close()


@pytest.mark.parametrize("rows,cols", [(3, 4), (9, 4), (12, 3)])
def test_flow_cluster_vs_oracle(sim, rows, cols):
    """Config 5 family (flow domains in the angles, Z/X output corrections)."""
    p = W.cluster_pattern(rows, cols, seed=rows)
    psi = haar_state(rows, 4)
    check(sim, p, psi, "sampled", seed=2)
    check(sim, p, psi, "forced", forced=np.random.default_rng(1).integers(0, 2, p.n_measure))
    check(sim, p, psi, "eowqs")


@pytest.mark.parametrize("seed", range(24))
def test_random_patterns_vs_oracle(sim, seed):
    """Random D0-D3 patterns: grow, shrink (full rho reduction), pending E/Z, corrections."""
    big = seed % 2 == 1
    p = W.random_general_pattern(seed, n_in=3 + (4 if big else 0), n_total=10 + (8 if big else 0),
                                 n_out=2 + seed % 3, max_live=12 if big else 7)
    psi = haar_state(len(p.inputs), seed)
    check(sim, p, psi, "sampled", seed=seed, same_order=False)
    ref = oracle.run(p, psi, mode="sampled", seed=seed)
    check(sim, p, psi, "forced", forced=ref.outcomes, same_order=False)
    _eowqs_check(sim, p, psi)


def _eowqs_check(sim, p, psi):
    """EOWQS on an open graph without gflow is refused (OWQS_E_NO_GFLOW, L372). With the pre-check
    off (or with a gflow), a non-deterministic command list reports OWQS_E_NOT_DETERMINISTIC unless
    the sqrt2 rescale happens to conserve the norm; the positive branch matches the oracle."""
    from paper_1604_05659_b200 import FLAG_NO_GFLOW
    from paper_1604_05659_b200.host import host_gflow
    run_sim, own = sim, False
    if not host_gflow(p)[0]:
        sim.load(p)
        sim.set_input(psi)
        with pytest.raises(OwqsError) as e:
            sim.run("eowqs")
        assert e.value.status_name == "OWQS_E_NO_GFLOW"
        run_sim, own = Simulator(precision=sim.precision, flags=FLAG_NO_GFLOW), True
    try:
        ref = oracle.run(p, psi, mode="eowqs")
        nrm = np.vdot(ref.output, ref.output).real
        tol = 1e-8 if sim.precision == 128 else 1e-3
        if abs(nrm - 1) <= tol:
            check(run_sim, p, psi, "eowqs")
            return
        run_sim.load(p)
        run_sim.set_input(psi)
        with pytest.raises(OwqsError) as e:
            run_sim.run("eowqs")
        assert e.value.status_name == "OWQS_E_NOT_DETERMINISTIC"
        out = run_sim.get_output()  # the output is still the sqrt2-scaled positive branch
        assert np.max(np.abs(out - ref.output)) <= TOL[sim.precision]["amp"] * max(1.0, np.max(np.abs(ref.output)))
    finally:
        if own:
            run_sim.close()


def test_gflow_gate_and_layers(sim):
    """owqs_gflow on the paper's patterns (L372): CNOT and config families have one, a funnel
    graph does not (EOWQS refused)."""
    sim.load(W.cnot_pattern_eq22())
    ok, layers, depth = sim.gflow()
    assert ok and depth == 2
    sim.load(W.config_pattern("CL:6x5", seed=2))
    assert sim.gflow()[0]
    bad = W.Pattern([1, 2], [3], [W.E(1, 3), W.E(2, 3), W.M(1, 0.), W.M(2, 0.)])
    sim.load(bad)
    assert not sim.gflow()[0]
    sim.set_input(haar_state(2, 1))
    with pytest.raises(OwqsError) as e:
        sim.run("eowqs")
    assert e.value.status_name == "OWQS_E_NO_GFLOW"


def test_forced_impossible_branch(sim):
    p = W.Pattern([1, 2], [2], [W.M(1, 0.0)])
    sim.load(p)
    sim.set_input(np.array([2 ** -0.5, 2 ** -0.5, 0, 0], dtype=complex))  # qubit 1 in |+>: prob1 = 0
    with pytest.raises(OwqsError) as e:
        sim.run("forced", forced=[1])
    assert e.value.status_name == "OWQS_E_BRANCH"


def test_call_order_errors(sim):
    p = W.config_pattern("C1")
    sim.load(p)
    with pytest.raises(OwqsError) as e:
        sim.run("sampled")
    assert e.value.status_name == "OWQS_E_STATE"


def test_recognize_cnot_and_circuits(sim):
    """Recognition (L33): CNOT pattern -> the CNOT matrix (control q1), random J/CZ circuits ->
    the oracle's brute-force unitary."""
    sim.load(W.cnot_pattern_eq22())
    U, err = sim.recognize()
    ref = oracle.recognize(W.cnot_pattern_eq22())
    assert np.max(np.abs(U - ref)) <= TOL[sim.precision]["amp"]
    assert err < (1e-12 if sim.precision == 128 else 1e-5)
    for seed in range(3):
        p = W.config_pattern("C1", seed=seed)
        sim.load(p)
        U, err = sim.recognize()
        assert np.max(np.abs(U - oracle.recognize(p))) <= TOL[sim.precision]["amp"]


def test_recognize_choi_matches_basis_runs(sim):
    """NEXT-3: recognition from one Choi-state run equals the per-basis-input recognition and the
    oracle's brute-force unitary (CNOT, random J/CZ circuits, a QFT, a flow cluster)."""
    pats = [W.cnot_pattern_eq22(), W.config_pattern("C1", seed=4), W.config_pattern("QFT:3"),
            W.cluster_pattern(3, 3, seed=1)]
    for p in pats:
        sim.load(p)
        U, err = sim.recognize(choi=True)
        Ub, _ = sim.recognize()
        assert np.max(np.abs(U - Ub)) <= 2 * TOL[sim.precision]["amp"]
        assert err < (1e-10 if sim.precision == 128 else 1e-4)
        if len(p.inputs) <= 3:
            assert np.max(np.abs(U - oracle.recognize(p))) <= TOL[sim.precision]["amp"]


def test_device_haar_generator(sim):
    """owqs_set_input_random follows the documented counter generator (workloads/inputs.py)."""
    n = 12
    p = W.Pattern(list(range(n)), list(range(n)), [])
    sim.load(p)
    sim.set_input_random(1234)
    sim.run("sampled")
    out = sim.get_output()
    ref = counter_haar_state(n, 1234)
    assert np.max(np.abs(out - ref)) <= (1e-13 if sim.precision == 128 else 1e-6)


def test_device_buffers_and_inner(require_gpu):
    """Device-resident input/output (torch tensors) and the device inner product."""
    import torch
    p = W.config_pattern("BW:12x4", seed=1)
    psi = haar_state(12, 2)
    a, b = Simulator(precision=128), Simulator(precision=128)
    try:
        a.load(p)
        t = torch.from_numpy(psi).cuda()
        a.set_input_device(t.data_ptr(), 128, t.numel())
        a.run("sampled", seed=1)
        o = torch.empty(2 ** 12, dtype=torch.complex128, device="cuda")
        a.get_output_device(o.data_ptr(), 128, o.numel())
        ref = oracle.run(p, psi, mode="sampled", seed=1).output
        assert np.max(np.abs(o.cpu().numpy() - ref)) < 1e-10
        b.load(p)
        b.set_input(psi)
        b.run("eowqs")
        ip = a.inner(b)
        assert abs(ip - np.vdot(ref, ref)) < 1e-10  # wild J patterns: branch independent exactly
    finally:
        a.close()
        b.close()


# ---------------------------------------------------------------- full-size configurations

@pytest.mark.parametrize("prec", [128, 64])
def test_config2_qft20_closed_form(require_gpu, prec):
    """Config 2 at full size (QFT-20, paper m 21): output = bit-reversed sqrt(N) ifft(psi) — a
    closed form independent of the oracle (textbook DFT)."""
    n = 20
    p = W.config_pattern("C2")
    psi = haar_state(n, 1)
    # structural probabilities reduced on the device (not R-13's exact 1/2): checks the norm stays 1
    s = Simulator(precision=prec, flags=FLAG_MEASURED_NORM)
    try:
        s.load(p)
        info = s.pattern_info()
        assert info["paper_m"] == 21 and info["phys_bits"] == 20
        s.set_input(psi)
        outc, p0 = s.run("sampled", seed=3)
        out = s.get_output()
    finally:
        s.close()
    f = math.sqrt(2 ** n) * np.fft.ifft(psi)
    rev = np.array([int(format(y, f"0{n}b")[::-1], 2) for y in range(2 ** n)])
    err = np.max(np.abs(out[rev] - f))
    assert err <= TOL[prec]["amp"]
    assert 1 - fidelity(out[rev], f) <= TOL[prec]["fid"]
    assert np.max(np.abs(p0 - 0.5)) <= (1e-12 if prec == 128 else 1e-6)


def test_config3_full_width_invariants(require_gpu):
    """Config 3 at full width (28 wires x 40 layers, paper m 29): prob0 = 1/2 on every M (L372,
    reduced on the device: OWQS_FLAG_MEASURED_NORM), norm 1, and outcome independence: sampled
    (c64), forced (c64) and EOWQS (c128) outputs agree to fidelity 1 - 1e-5; c128 sampled vs EOWQS
    agree to 1e-10."""
    p = W.config_pattern("C3", seed=1)
    a, b = Simulator(precision=64, flags=FLAG_MEASURED_NORM), Simulator(precision=128)
    try:
        a.load(p)
        assert a.pattern_info()["paper_m"] == 29
        a.set_input_random(7)
        outc, p0 = a.run("sampled", seed=5)
        assert np.max(np.abs(p0 - 0.5)) < 2e-6
        assert abs(a.norm2() - 1) < 1e-5
        assert 0.3 < outc.mean() < 0.7
        b.load(p)
        b.set_input_random(7)
        b.run("eowqs")
        ip = a.inner(b)
        assert 1 - abs(ip) ** 2 <= 1e-5
        a.set_input_random(7)
        a.run("forced", forced=np.random.default_rng(9).integers(0, 2, p.n_measure))
        assert 1 - abs(a.inner(b)) ** 2 <= 1e-5
        a.close()
        a = Simulator(precision=128, flags=FLAG_MEASURED_NORM)
        a.load(p)
        a.set_input_random(7)
        _, p0 = a.run("sampled", seed=5)
        assert np.max(np.abs(p0 - 0.5)) < 1e-12
        ip = a.inner(b)
        assert abs(ip - 1) < 1e-10
    finally:
        a.close()
        b.close()


def test_config5_verification_instance(require_gpu):
    """Config 5's 1-GPU verification instance (26 x 8 cluster, fp64): EOWQS equals random forced
    branches up to a global phase (outcome independence, L372) and has norm 1."""
    p = W.config_pattern("CL:26x8", seed=1)
    a, b = Simulator(precision=128, flags=FLAG_MEASURED_NORM), Simulator(precision=128)
    try:
        b.load(p)
        b.set_input_random(3)
        b.run("eowqs")
        a.load(p)
        for k in range(2):
            a.set_input_random(3)
            _, p0 = a.run("forced", forced=np.random.default_rng(k).integers(0, 2, p.n_measure))
            assert np.max(np.abs(p0 - 0.5)) < 1e-12
            assert abs(abs(a.inner(b)) - 1) < 1e-10
        a.set_input_random(3)
        a.run("sampled", seed=4)
        assert abs(abs(a.inner(b)) - 1) < 1e-10
    finally:
        a.close()
        b.close()


@pytest.mark.parametrize("k", range(8))
def test_standard_form_patterns_vs_oracle(sim, k):
    """NEXT-2: standard-form (and signal-shifted) rewrites of wild patterns run on the GPU with exact
    amplitude parity against the oracle on the same rewritten pattern (PROA on standard form)."""
    from paper_1604_05659_b200.host import standardize
    p = (W.random_general_pattern(k, n_in=2, n_total=9, n_out=2) if k < 5 else
         [W.config_pattern("C1", seed=1), W.cluster_pattern(4, 4, seed=3), W.config_pattern("QFT:2")][k - 5])
    for shift in (False, True):
        std, _ = standardize(p, signal_shift=shift)
        psi = haar_state(len(p.inputs), 60 + k)
        rng = np.random.default_rng(k)
        # random patterns are not deterministic: PROA's order changes per-M probabilities (R-8),
        # the joint branch probability and the amplitudes are compared
        order = False if k < 5 else None
        for _ in range(3):
            forced = rng.integers(0, 2, std.n_measure)
            try:
                oracle.run(std, psi, mode="forced", forced=forced)
            except oracle.OracleError as e:
                # an impossible forced branch of a non-deterministic pattern: the GPU must refuse it
                # too (complex64 may instead report a joint branch probability below its tolerance)
                assert "probability" in str(e)
                sim.load(std)
                sim.set_input(psi)
                try:
                    outc, p0 = sim.run("forced", forced=forced)
                except OwqsError as g:
                    assert g.status_name == "OWQS_E_BRANCH"
                    continue
                assert sim.precision == 64
                assert np.prod([q if b == 0 else 1 - q for q, b in zip(p0, outc)]) <= TOL[64]["prob"]
                continue
            check(sim, std, psi, "forced", forced=forced, same_order=order)
        check(sim, std, psi, "sampled", seed=k, same_order=order)
