"""CPU tests of the C-ABI library's host side: exported symbols, validation (D0-D3), PROA
(Eq. 18 / Table I / Eq. 23 / §4.6 / Table III QFT rows) and the compiled step program, executed
by the test-side interpreter and compared with the oracle. No GPU needed."""
import json
import math
import os
import re

import numpy as np
import pytest

import oracle
from paper_1604_05659_b200 import _capi
from paper_1604_05659_b200 import FLAG_GIVEN_ORDER, FLAG_NO_FUSE, FLAG_NO_TUNE
from paper_1604_05659_b200.host import compile_host
from paper_1604_05659_b200.owqs import OwqsError, lib
from program_interp import Interp
from workloads import patterns as W
from workloads.inputs import haar_state

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def test_library_exports_every_declared_symbol():
    """Every function include/*.h declares is exported by libowqs.so (no compute calls)."""
    declared = set()
    for h in ("owqs.h", "owqs_host.h"):
        txt = open(os.path.join(ROOT, "include", h)).read()
        declared |= set(re.findall(r"^(?:owqs_status|void|const char\*)\s+(owqs_\w+)\s*\(", txt, re.M))
    L = lib()
    for name in sorted(declared):
        assert hasattr(L, name), name
    assert set(_capi.EXPORTED) | set(_capi.HOST_EXPORTED) == declared
    assert L.owqs_version().decode().startswith("owqs")


def _err(pattern):
    with pytest.raises(OwqsError) as e:
        compile_host(pattern)
    return e.value


def test_validation_rules():
    """D0-D3 (L85-91), duplicate E and E(u,u) are OWQS_E_PATTERN with the command index."""
    assert _err(W.Pattern([1], [2], [W.N(2), W.M(1, 0.0), W.E(1, 2)])).status_name == "OWQS_E_PATTERN"  # D1
    e = _err(W.Pattern([1], [2], [W.N(2), W.E(1, 2), W.M(1, 0.0, (3,)), W.M(3, 0.0)]))
    assert "D0" in str(e)
    assert "D3" in str(_err(W.Pattern([1], [1], [W.M(1, 0.0)])))
    assert "D3" in str(_err(W.Pattern([1, 2], [2], [])))  # qubit 1 never measured
    assert "duplicate E" in str(_err(W.Pattern([1, 2], [1, 2], [W.E(1, 2), W.E(2, 1)])))
    assert "single qubit" in str(_err(W.Pattern([1], [1], [W.E(1, 1)])))
    assert "N on" in str(_err(W.Pattern([1], [1], [W.N(1)])))


def test_table1_swap_order():
    """Table I (L291-301): PROA reproduces the optimised SWAP order 2, 3, 1, 4, 5, 7, peak 3."""
    g = json.load(open(os.path.join(GOLDEN, "table1_swap.json")))
    cmds = [W.E(a, b) for a, b in g["edges"]]
    cmds += [W.M(q, 0.0) for q in g["qubits"] if q not in g["outputs"]]
    p = W.Pattern([1, 2], g["outputs"], cmds, "SWAP")
    hp = compile_host(p, "sampled")
    assert hp.plan_qubits == g["table1_order"]
    assert hp.info["paper_m"] == g["peak"]


def test_eq23_cnot_reordering():
    """Eq. 22 -> Eq. 23 (L413-417): PROA measures q2 before q3."""
    hp = compile_host(W.cnot_pattern_eq22(), "sampled")
    assert hp.plan_qubits == [2, 3]
    assert hp.info["paper_m"] == 3  # Table III CNOT row: m = 3


@pytest.mark.parametrize("rows,cols", [(2, 4), (3, 5), (5, 3), (8, 4)])
def test_cluster_width_4_6(rows, cols):
    """§4.6 (L403): an N x M cluster measured column by column has m = N + 1."""
    for mode in ("sampled", "eowqs"):
        hp = compile_host(W.cluster_pattern(rows, cols, seed=1), mode)
        assert hp.info["paper_m"] == rows + 1
        assert hp.info["phys_bits"] == rows  # slot reuse keeps the array at N bits


def test_linear_cluster_width():
    """§4.6: 1D cluster state space is O(1): m = 2, one physical bit."""
    hp = compile_host(W.linear_cluster_pattern(30, seed=2))
    assert hp.info["paper_m"] == 2 and hp.info["phys_bits"] == 1


@pytest.mark.parametrize("n", [3, 5, 8])
def test_qft_width_table3(n):
    """Table III QFT rows (L497-501): m = n + 1 (marked optimal, |O| + 1)."""
    hp = compile_host(W.config_pattern(f"QFT:{n}"))
    assert hp.info["paper_m"] == n + 1
    assert hp.info["n_measure"] == 4 * n * n - 3 * n


def test_config_widths():
    """BASELINE configs: paper m and physical width of the compiled programs."""
    for name, m, phys in (("C3", 29, 28), ("C2", 21, 20), ("C5", 36, 35)):
        hp = compile_host(W.config_pattern(name), "sampled", precision=64)
        assert hp.info["paper_m"] == m, name
        assert hp.info["phys_bits"] == phys, name
        assert hp.info["n_grow"] == 0 and hp.info["n_shrink"] == 0


def _joint(prob0, outcomes):
    """Joint branch probability prod_M p(s_M | earlier) — order independent (reading R-8)."""
    return float(np.prod([p if s == 0 else 1 - p for p, s in zip(prob0, outcomes)]))


def _compare(p, psi, mode, flags=0, precision=128, seed=5, forced=None):
    prog = compile_host(p, mode, precision=precision, flags=flags)
    it = Interp(prog, mode, seed=seed, forced=forced)
    out = it.run(psi)
    assert it.err == 0
    same_order = prog.plan_qubits == p.measured_in_given_order()
    if mode == "eowqs":
        ref = oracle.run(p, psi, mode="eowqs")
    elif mode == "sampled":
        ref = oracle.run(p, psi, mode="sampled", seed=seed)
        if list(it.outcome) != list(ref.outcomes):
            # a reordered plan samples the same joint distribution in another order (R-8):
            # replay the oracle on the executor's branch
            assert not same_order
            ref = oracle.run(p, psi, mode="forced", forced=it.outcome)
    else:
        ref = oracle.run(p, psi, mode="forced", forced=forced)
    if mode != "eowqs":
        if same_order:
            assert np.allclose(it.prob0, ref.prob0, atol=1e-12, rtol=0)
        assert abs(_joint(it.prob0, it.outcome) - _joint(ref.prob0, ref.outcomes)) < 1e-12
    assert np.allclose(out, ref.output, atol=1e-10, rtol=0)
    return prog


FLAG_SETS = [0, FLAG_NO_FUSE, FLAG_GIVEN_ORDER, FLAG_GIVEN_ORDER | FLAG_NO_FUSE, FLAG_NO_TUNE]


@pytest.mark.parametrize("flags", FLAG_SETS)
@pytest.mark.parametrize("precision", [64, 128])
def test_compiled_program_vs_oracle_configs(flags, precision):
    """The scheduler's program (slot reuse, fused passes, decisions, reductions) equals the oracle
    on the config families: C1 tiny, QFT, brickwork, flow cluster, CNOT."""
    cases = [(W.config_pattern("C1", seed=s), 3) for s in range(3)]
    cases += [(W.config_pattern("QFT:4"), 4), (W.config_pattern("BW:5x4", seed=2), 5),
              (W.cluster_pattern(3, 4, seed=3), 3), (W.cnot_pattern_eq22(), 2), (W.cnot_pattern_eq23(), 2)]
    for k, (p, n) in enumerate(cases):
        psi = haar_state(n, 40 + k)
        for mode in ("sampled", "eowqs"):
            _compare(p, psi, mode, flags, precision, seed=k)
        rng = np.random.default_rng(k)
        forced = rng.integers(0, 2, p.n_measure)
        _compare(p, psi, "forced", flags, precision, forced=forced)


@pytest.mark.parametrize("seed", range(40))
def test_compiled_program_vs_oracle_random_patterns(seed):
    """Random D0-D3 patterns (non-deterministic, non-standard): exercises grow, shrink (full rho),
    pending E/Z on fresh qubits and corrections on every branch of the compiler."""
    p = W.random_general_pattern(seed, n_in=2 + seed % 2, n_total=8 + seed % 4, n_out=1 + seed % 3)
    psi = haar_state(len(p.inputs), seed)
    flags = FLAG_SETS[seed % len(FLAG_SETS)]
    prec = 64 if seed % 3 == 0 else 128
    ref = oracle.run(p, psi, mode="sampled", seed=seed)
    _compare(p, psi, "sampled", flags, prec, seed=seed)
    _compare(p, psi, "forced", flags, prec, forced=ref.outcomes)
    _compare(p, psi, "eowqs", flags, prec)


def test_random_patterns_cover_grow_and_shrink():
    grow = shrink = 0
    for seed in range(40):
        p = W.random_general_pattern(seed, n_in=2 + seed % 2, n_total=8 + seed % 4, n_out=1 + seed % 3)
        info = compile_host(p).info
        grow += info["n_grow"]
        shrink += info["n_shrink"]
    assert grow > 0 and shrink > 0


def test_substate_split_host():
    """PAPER §4.1 sub-states (owqs_host_substates): a pattern whose E graph has separate components
    runs as one state per component (inputs together), each compiled at its own width; the output
    masks partition the caller's output bits; a signal that crosses components keeps one state."""
    import sys
    import os
    sys.path.insert(0, os.path.dirname(__file__))
    from test_gpu_substates import disconnected, fragment
    from paper_1604_05659_b200.host import substates
    p = disconnected()
    parts = substates(p)
    assert len(parts) == 3
    masks = [m for m, _ in parts]
    assert sum(masks) == (1 << len(p.outputs)) - 1 and all(a & b == 0 for a in masks for b in masks if a is not b)
    # the inputs' circuit (4 wires) is sub-state 0; the cluster (3 rows) and the lone |+> follow
    assert masks[0] == 0b10100101 and masks[2] == 0b00001000
    assert [b for _, b in parts] == [4, 3, 1]
    assert max(b for _, b in parts) < compile_host(p, "sampled", 64).info["phys_bits"]
    ci, co, cc = fragment(W.config_pattern("BW:3x2", seed=2), 0, True)
    cross = W.Pattern(ci, co + [501], cc + [W.N(500), W.N(501), W.E(500, 501), W.M(500, 0.4, sdom=(ci[0],))])
    assert substates(cross) == []
    assert substates(W.config_pattern("C1", seed=1)) == []


def _tile_invariants(hp, SB=6, kmax=6):
    """Every 2x2 op of a tile-engine pass lies in its tile (segment positions or group slots), a
    pass has at most kmax group slots, and a store remap only trades a group slot of the pass with
    a segment position (complex64 keeps position 0)."""
    for i, st in enumerate(hp.steps):
        if st.kind != 0 or st.width < SB + kmax:
            continue
        grp = [st.bhi[j] for j in range(st.nb_hi)]
        assert len(grp) <= kmax, i
        for k in range(st.n_ops):
            o = st.ops[k]
            if o.type in (3, 4):
                assert o.a < SB or o.a in grp, (i, o.a, grp)
        for k in range(st.n_remap):
            assert st.remap_a[k] in grp, i
            assert (1 if SB == 6 else 0) <= st.remap_b[k] < SB, i


def test_tile_planner_pass_counts_and_invariants():
    """Tile planning (look-ahead tiles + matching store remap, wavefront pick order): config 3 in
    at most 30 passes (38 with first-come slots), config 4 in at most 21 (34), each within the
    tile-engine invariants."""
    for name, cap in (("C3", 30), ("C3W", 31), ("C4", 21)):
        hp = compile_host(W.config_pattern(name), "sampled", precision=64)
        assert hp.info["n_passes"] <= cap, (name, hp.info["n_passes"])
        assert sum(st.n_bfly for st in hp.steps) == hp.info["n_measure"]
        _tile_invariants(hp)


@pytest.mark.parametrize("shape,mode", [("BW:16x10", "sampled"), ("BW:15x12", "eowqs"), ("BW:16x8", "forced")])
def test_tile_planned_program_vs_oracle(shape, mode):
    """Programs whose passes are tile-planned and remapped (width >= 12, complex64) executed by the
    interpreter equal the oracle: the planner's remaps and pick order keep the program exact."""
    p = W.config_pattern(shape, seed=4)
    n = len(p.inputs)
    hp = compile_host(p, mode if mode != "forced" else "sampled", precision=64)
    assert any(st.n_remap > 0 for st in hp.steps)
    _tile_invariants(hp)
    psi = haar_state(n, 11)
    forced = np.random.default_rng(3).integers(0, 2, p.n_measure) if mode == "forced" else None
    _compare(p, psi, mode, 0, 64, seed=7, forced=forced)
