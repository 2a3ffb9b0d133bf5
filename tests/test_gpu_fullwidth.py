"""GPU parity on the paths full-size runs take (VERDICT r1 "next round" item 1).

* SHRINK (measurement without a fresh partner: in-place elimination), GROW (append |+>) and the
  (n0, n1, c) reduction of Eq. 13 (RED_RHO epilogue + grid finish) at tile-engine widths 17-21,
  vs the oracle, both precisions, default grid and a capped grid (several tiles per CTA);
* a 24-wire x 4-layer brickwork vs the oracle (4096 tiles per pass, remapping on);
* config 3 at its full width (28 wires) on a one-layer prefix vs sampled oracle amplitudes
  (tests/golden/, written by tools/make_golden_c3_prefix.py, which calls only oracle/);
* config 3 with device-measured structural probabilities (OWQS_FLAG_MEASURED_NORM): prob0 = 1/2
  ||psi||^2 reduced from the state before every pass, at 28 bits -- checks R-13's ||psi||^2 = 1;
* config 4 at 33 bits: complex64 vs complex128 on sampled output amplitudes (SURVEY §8(e) Checks);
* the R-13 input contract: unnormalised inputs are refused on every input path, as the oracle
  refuses them (Eq. 3-4).
"""
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
from paper_1604_05659_b200 import FLAG_MEASURED_NORM, OwqsError, Simulator
from parity_util import TOL, check, fidelity
from workloads import patterns as W
from workloads.inputs import haar_state

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")

# (n_in, width_hi, rounds, n_out, seed): physical widths 17-21, GROW + SHRINK + RED_RHO passes
WIDE = [(20, 24, 2, 20, 0), (20, 24, 2, 20, 1), (21, 21, 3, 14, 0), (21, 21, 3, 14, 3)]


def _both_refuse_or_check(sim, p, psi, forced):
    """Forced branch: if the oracle refuses it (p < 1e-12), the GPU must refuse it too
    (OWQS_E_BRANCH); complex64 may instead report a joint branch probability within its
    probability tolerance of 0 (fp32 amplitudes do not resolve p < 1e-12)."""
    try:
        oracle.run(p, psi, mode="forced", forced=forced)
    except oracle.OracleError as e:
        assert "probability" in str(e)
        sim.load(p)
        sim.set_input(psi)
        try:
            outc, p0 = sim.run("forced", forced=forced)
        except OwqsError as g:
            assert g.status_name == "OWQS_E_BRANCH"
            return
        assert sim.precision == 64
        joint = np.prod([q if s == 0 else 1 - q for q, s in zip(p0, outc)])
        assert joint <= TOL[64]["prob"]
        return
    check(sim, p, psi, "forced", forced=forced, same_order=False)


@pytest.mark.parametrize("prec", [128, 64])
@pytest.mark.parametrize("shape", WIDE, ids=[f"wr{a}-{b}-{c}-{d}-s{e}" for a, b, c, d, e in WIDE])
def test_shrink_grow_rho_at_tile_widths(require_gpu, prec, shape):
    from paper_1604_05659_b200.host import compile_host
    n_in, hi, rounds, n_out, seed = shape
    p = W.wide_random_pattern(seed, n_in=n_in, width_hi=hi, rounds=rounds, n_out=n_out)
    hp = compile_host(p, "sampled", prec)
    wide = [s for s in hp.steps if s.width >= 17]
    assert any(s.kind == 2 for s in wide) and any(s.red_kind == 2 for s in wide)  # SHRINK, RHO
    psi = haar_state(n_in, 100 + seed)
    s = Simulator(precision=prec)
    try:
        out, ref = check(s, p, psi, "sampled", seed=seed, same_order=False)
        assert np.min(np.abs(ref.prob0 - 0.5)) < 0.49 and np.max(np.abs(ref.prob0 - 0.5)) > 1e-4  # not all 1/2
        _both_refuse_or_check(s, p, psi, np.random.default_rng(seed).integers(0, 2, p.n_measure))
    finally:
        s.close()


CAPPED = r"""
import numpy as np, oracle, sys
sys.path.insert(0, "tests")
from parity_util import check
from paper_1604_05659_b200 import Simulator
from workloads import patterns as W
from workloads.inputs import haar_state
for prec in (64, 128):
    s = Simulator(precision=prec)
    for (n_in, hi, rounds, n_out, seed) in ((20, 24, 2, 20, 0), (21, 21, 3, 14, 3)):
        p = W.wide_random_pattern(seed, n_in=n_in, width_hi=hi, rounds=rounds, n_out=n_out)
        psi = haar_state(n_in, 100 + seed)
        check(s, p, psi, "sampled", seed=seed, same_order=False)
    s.close()
print("ok")
"""


def test_shrink_grow_rho_capped_grid(require_gpu):
    """The same at a capped tile grid (OWQS_TILE_MAX_BLOCKS=8: 32-256 tiles per CTA, partials
    accumulated across tiles), as states above 2^20 tiles run."""
    env = dict(os.environ, PYTHONPATH=ROOT + os.pathsep + os.path.join(ROOT, "tests"), OWQS_TILE_MAX_BLOCKS="8")
    r = subprocess.run([sys.executable, "-c", CAPPED], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=1200)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout[-2000:] + r.stderr[-4000:]


def test_brickwork_24x4_vs_oracle(require_gpu):
    """24 wires x 4 layers (config 3's recipe): 2^24 amplitudes, 4096 complex64 tiles per pass
    (c128: 8192), qubit remapping on, one oracle run (complex128, given order) for both
    precisions; every prob0 = 1/2 so the keyed draws agree and the outcome strings must match."""
    p = W.config_pattern("BW:24x4", seed=2)
    psi = haar_state(24, 5)
    ref = oracle.run(p, psi, mode="sampled", seed=9)
    for prec in (128, 64):
        s = Simulator(precision=prec)
        try:
            s.load(p)
            assert s.pattern_info()["phys_bits"] == 24
            s.set_input(psi)
            outc, p0 = s.run("sampled", seed=9)
            assert list(outc) == list(ref.outcomes)
            assert np.max(np.abs(p0 - ref.prob0)) <= TOL[prec]["prob"]
            out = s.get_output()
            err = np.max(np.abs(out - ref.output))
            assert err <= TOL[prec]["amp"], err
            assert 1 - fidelity(out, ref.output) <= TOL[prec]["fid"]
            rel = np.linalg.norm(out - ref.output) / np.linalg.norm(ref.output)
            assert rel <= (1e-12 if prec == 128 else 1e-5), rel
        finally:
            s.close()


def test_config3_full_width_prefix_vs_oracle(require_gpu):
    """Config 3 at its full 28-bit width: the first brickwork layer (28 J + 14 CZ = 126 commands)
    on the counter-Haar input (seed 7) vs the oracle's run of the same command list (sampled
    seed 5): identical outcome strings, prob0 within tolerance, and 4098 sampled output
    amplitudes (abs. 1e-10 / relative-l2 1e-5; |amp| ~ 2^-14 makes the absolute fp32 bar vacuous)."""
    g = np.load(os.path.join(GOLDEN, "c3_prefix_l1_w28_oracle.npz"))
    wires, layers, k, in_seed, run_seed = (int(x) for x in g["meta"][:5])
    p = W.prefix_pattern(W.config_pattern("C3", seed=1), k)
    for prec in (128, 64):
        s = Simulator(precision=prec)
        try:
            s.load(p)
            assert s.pattern_info()["phys_bits"] == wires
            s.set_input_random(in_seed)
            outc, p0 = s.run("sampled", seed=run_seed)
            assert list(outc) == list(g["outcomes"])
            assert np.max(np.abs(p0 - g["prob0"])) <= TOL[prec]["prob"]
            amps = s.get_output_sample(g["idx"])
            ref = g["amps"]
            rel = np.linalg.norm(amps - ref) / np.linalg.norm(ref)
            assert rel <= (1e-10 if prec == 128 else 1e-5), rel
            if prec == 128:
                assert np.max(np.abs(amps - ref)) <= TOL[128]["amp"]
            assert abs(s.norm2() - float(g["norm2"])) <= (1e-10 if prec == 128 else 1e-5)
        finally:
            s.close()


@pytest.mark.parametrize("prec", [64, 128])
def test_config3_measured_structural_prob(require_gpu, prec):
    """R-13 checked on the device at config 3's full width: with OWQS_FLAG_MEASURED_NORM every pass
    reduces ||psi||^2 and the structural decisions use prob0 = 1/2 ||psi||^2 as measured (Eq. 13);
    all 1120 reported probabilities must be 1/2 to the precision's tolerance (norm kept 1 by Eq. 4
    through 40 layers), and the run equals the default (||psi||^2 = 1) run."""
    p = W.config_pattern("C3", seed=1)
    a = Simulator(precision=prec, flags=FLAG_MEASURED_NORM)
    b = Simulator(precision=prec)
    try:
        for x in (a, b):
            x.load(p)
            x.set_input_random(7)
        oa, pa = a.run("sampled", seed=5)
        ob, pb = b.run("sampled", seed=5)
        assert a.stats()["n_reduce"] >= a.stats()["n_passes"] - 1 and b.stats()["n_reduce"] <= 2
        tol = 1e-12 if prec == 128 else 2e-6
        assert np.max(np.abs(pa - 0.5)) <= tol, np.max(np.abs(pa - 0.5))
        assert np.all(pb == 0.5)
        assert list(oa) == list(ob)
        assert abs(a.norm2() - 1) <= (1e-12 if prec == 128 else 1e-5)
        assert abs(b.norm2() - 1) <= (1e-12 if prec == 128 else 1e-5)
        assert 1 - abs(a.inner(b)) ** 2 <= (1e-12 if prec == 128 else 1e-5)
    finally:
        a.close()
        b.close()


def test_config4_c64_vs_c128_33_bits(require_gpu):
    """Config 4 (33 wires x 24 layers) at 33 bits on one GPU, complex64 (64 GiB) vs complex128
    (128 GiB), run one after the other on the same counter-Haar input and sampled seed: identical
    outcome strings (every prob0 = 1/2), equal norms, and 65538 sampled output amplitudes agree to
    relative-l2 1e-5 (SURVEY §8(e) Checks: c64 vs c128 at full width)."""
    p = W.config_pattern("C4", seed=1)
    rng = np.random.default_rng(3)
    idx = np.unique(np.concatenate([[0, 2 ** 33 - 1], rng.integers(0, 2 ** 33, 65536)]))
    res = {}
    for prec in (64, 128):
        s = Simulator(precision=prec)
        try:
            s.load(p)
            s.set_input_random(3)
            outc, _ = s.run("sampled", seed=5)
            res[prec] = (outc, s.get_output_sample(idx), s.norm2())
        finally:
            s.close()
    assert list(res[64][0]) == list(res[128][0])
    a, b = res[64][1], res[128][1]
    rel = np.linalg.norm(a - b) / np.linalg.norm(b)
    assert rel <= 1e-5, rel
    assert abs(res[128][2] - 1) <= 1e-10 and abs(res[64][2] - 1) <= 1e-5
    # the sample is not degenerate: ~2^-16.5 typical magnitude, mean |amp|^2 * 2^33 ~ 1
    assert 0.5 < np.mean(np.abs(b) ** 2) * 2 ** 33 < 2


@pytest.mark.parametrize("prec", [128, 64])
def test_unnormalised_input_refused(require_gpu, prec):
    """R-13's precondition: every input path refuses a state with ||psi||^2 != 1 (OWQS_E_ARG) --
    host, device, asynchronous submit and batched replicas -- as the oracle does; a normalised
    input within tolerance is accepted."""
    import torch
    p = W.config_pattern("BW:14x2", seed=1)
    psi = haar_state(14, 3)
    bad = psi * 1.01
    with pytest.raises(oracle.OracleError):
        oracle.run(p, bad, mode="sampled", seed=1)
    s = Simulator(precision=prec)
    try:
        s.load(p)
        with pytest.raises(OwqsError) as e:
            s.set_input(bad)
        assert e.value.status_name == "OWQS_E_ARG" and "normalised" in str(e.value)
        with pytest.raises(OwqsError) as e:  # no input after a refused one
            s.run("sampled", seed=1)
        assert e.value.status_name == "OWQS_E_STATE"
        cdt = torch.complex64 if prec == 64 else torch.complex128
        t = torch.from_numpy(bad.astype(np.complex64 if prec == 64 else np.complex128)).cuda()
        with pytest.raises(OwqsError) as e:
            s.set_input_device(t.data_ptr(), prec, t.numel())
        assert e.value.status_name == "OWQS_E_ARG"
        t = torch.from_numpy(psi).to(cdt).cuda()
        s.set_input_device(t.data_ptr(), prec, t.numel())  # accepted
        outc, _ = s.run("sampled", seed=1)
        ref = oracle.run(p, psi, mode="sampled", seed=1)
        assert list(outc) == list(ref.outcomes)
        hb = torch.from_numpy(bad).pin_memory()
        ho = torch.empty(2 ** 14, dtype=torch.complex128).pin_memory()
        s.submit_host(hb.data_ptr(), 128, ho.data_ptr(), 128, "sampled", seed=1)
        with pytest.raises(OwqsError) as e:
            s.wait()
        assert e.value.status_name == "OWQS_E_ARG"
    finally:
        s.close()
    q = W.config_pattern("C1", seed=1)
    b = Simulator(precision=prec)
    try:
        b.load(q)
        ins = np.stack([haar_state(3, k) for k in range(4)])
        ins[2] *= 0.9
        with pytest.raises(OwqsError) as e:
            b.run_batch(ins, "sampled", seeds=np.arange(4))
        assert e.value.status_name == "OWQS_E_ARG"
    finally:
        b.close()


@pytest.mark.parametrize("shape", ["BWM:16x20x7", "BWM:18x12x6", "BWM:14x6x5"])
def test_measured_tail_vs_oracle(require_gpu, shape):
    """Config 3M's family: a brickwork whose last k wires are measured after the last layer --
    SHRINK steps (Eq. 13 rho reduction in the previous pass, Fig. 6 compaction) that follow
    qubit-remapped tile passes (the packer maps the emitter's slots through the remap), both
    precisions, sampled and forced."""
    p = W.config_pattern(shape, seed=2)
    psi = haar_state(len(p.inputs), 3)
    for prec in (128, 64):
        s = Simulator(precision=prec)
        try:
            # the tail measurements commute and PROA may order them differently from the given
            # list: per-M prob0 differ (reading R-8), the joint branch probability and output do not
            check(s, p, psi, "sampled", seed=5, same_order=False)
            _both_refuse_or_check(s, p, psi, np.random.default_rng(4).integers(0, 2, p.n_measure))
        finally:
            s.close()


@pytest.mark.parametrize("shape", ["BWM:14x6x5", "BWM:12x4x4"])
def test_joint_measurement_matches_sequential(require_gpu, monkeypatch, shape):
    """Joint k-outcome sampling (ST_RHOK + ST_SHRINKK): consecutive eliminations
    decided from one reduced density matrix give the same outcome strings, per-M prob0 and outputs as
    the same program with one SHRINK per measurement (OWQS_JOINT_K=1) and as the oracle, in fewer
    passes."""
    from paper_1604_05659_b200.host import compile_host
    p = W.config_pattern(shape, seed=2)
    psi = haar_state(len(p.inputs), 3)
    joint = compile_host(p, "sampled", 128)
    assert any(s.kind == 5 for s in joint.steps)
    res = {}
    for jk in ("3", "1"):
        monkeypatch.setenv("OWQS_JOINT_K", jk)
        for prec in (128, 64):
            s = Simulator(precision=prec)
            try:
                out, _ = check(s, p, psi, "sampled", seed=7, same_order=False)
                s.load(p)
                s.set_input(psi)
                outc, p0 = s.run("sampled", seed=7)
                res[(jk, prec)] = (out, outc, p0, s.stats()["n_launches"])
            finally:
                s.close()
    for prec in (128, 64):
        a, b = res[("3", prec)], res[("1", prec)]
        assert list(a[1]) == list(b[1])
        assert np.max(np.abs(a[2] - b[2])) <= TOL[prec]["prob"]
        assert np.max(np.abs(a[0] - b[0])) <= TOL[prec]["amp"]
        assert a[3] < b[3]  # fewer launches


@pytest.mark.parametrize("shape", ["BW:16x12", "CL:14x4"])
def test_decide_ahead_vs_oracle_and_per_pass(require_gpu, monkeypatch, shape):
    """Decisions ahead (one decide launch per run, pass kernels back to back) on
    tile-engine programs at widths 14-16: sampled and forced runs equal the oracle, and equal the
    same program with per-pass decide kernels (OWQS_DECIDE_AHEAD=0) bit for bit -- outcomes, prob0
    and amplitudes -- in both precisions."""
    p = W.config_pattern(shape, seed=3)
    psi = haar_state(len(p.inputs), 5)
    forced = np.random.default_rng(6).integers(0, 2, p.n_measure)
    res, kern = {}, {}
    for ahead in ("1", "0"):
        monkeypatch.setenv("OWQS_DECIDE_AHEAD", ahead)
        for prec in (128, 64):
            s = Simulator(precision=prec)
            try:
                out_s, ref_s = check(s, p, psi, "sampled", seed=9)
                out_f, ref_f = check(s, p, psi, "forced", forced=forced)
                s.load(p)
                s.set_input(psi)
                oc, p0 = s.run("sampled", seed=9)
                res[(ahead, prec)] = (out_s, out_f, np.array(oc), np.array(p0))
                kern[(ahead, prec)] = s.stats()["n_kernels"]
            finally:
                s.close()
    for prec in (128, 64):
        assert kern[("1", prec)] < kern[("0", prec)], kern  # the ahead path ran (fewer launches)
        a, b = res[("1", prec)], res[("0", prec)]
        for x, y in zip(a, b):
            assert np.array_equal(x, y)
