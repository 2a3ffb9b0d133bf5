"""Pins of the CPU oracle to facts fixed by the paper and by mathematics (not by itself).

Every test cites the passage it checks. None of these re-types the oracle's own formula: each
compares the oracle against a printed value, a closed form, a textbook matrix product, an
independently built Kronecker operator, or an invariant.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
from oracle.owqs_oracle import apply_1q, apply_2q, CZ_4x4
from workloads import patterns as W
from workloads.inputs import basis_state, haar_state

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
H = np.array([[1, 1], [1, -1]], dtype=np.complex128) / math.sqrt(2)


def J(alpha):
    """J(alpha) = H diag(1, e^{i alpha}) (BASELINE.json north_star; measurement calculus [14,15])."""
    return H @ np.diag([1, np.exp(1j * alpha)])


def kron_embed(U, pos, L):
    """Eq. 20: I (x) ... (x) U (x) ... (x) I with U on bit `pos` (bit 0 rightmost)."""
    out = np.eye(1, dtype=np.complex128)
    for p in range(L - 1, -1, -1):
        out = np.kron(out, U if p == pos else np.eye(2))
    return out


def circuit_matrix(n, gates):
    """Textbook circuit product; wire w = bit w."""
    U = np.eye(2 ** n, dtype=np.complex128)
    for g in gates:
        if g[0] == "J":
            G = kron_embed(J(g[2]), g[1], n)
        else:
            d = np.array([-1.0 if ((x >> g[1]) & 1) and ((x >> g[2]) & 1) else 1.0 for x in range(2 ** n)])
            G = np.diag(d)
        U = G @ U
    return U


def equal_up_to_phase(a, b, tol=1e-10):
    k = int(np.argmax(np.abs(b)))
    if abs(b[k]) < 1e-14:
        return np.max(np.abs(a)) < tol
    ph = a[k] / b[k]
    return abs(abs(ph) - 1) < tol and np.max(np.abs(a - ph * b)) < tol


# ------------------------------------------------------------------ conventions and operators

def test_eq8_lsb_convention():
    """Eq. 8 (L157-161): index 4 <-> |100>; X on qubit 3 (the leftmost ket letter) moves the
    |100> amplitude to index 0 — pins 'inputs[0] = qubit 1 = LSB'."""
    g = json.load(open(os.path.join(GOLDEN, "eq8_array.json")))
    psi = np.array(g["re"]) + 1j * np.array(g["im"])
    assert abs(np.linalg.norm(psi) - 1) < 1e-15  # reading R-2: the array is normalised
    for ket, (re, im) in g["kets"].items():
        assert np.isclose(psi[int(ket, 2)], (re + 1j * im) / (2 * math.sqrt(2)))
    p = W.Pattern([1, 2, 3], [1, 2, 3], [W.X(3, ())], "noop")
    assert np.allclose(oracle.run(p, psi).output, psi)
    p = W.Pattern([1, 2, 3], [1, 2, 3], [W.X(3, (2,)), W.M(4, 0.0), W.X(3, (4,))], "bad")
    with pytest.raises(oracle.OracleError):
        oracle.run(p, psi)  # D0: signal on unmeasured qubit
    # X on qubit 3 via a measured helper whose outcome is forced to 1
    p = W.Pattern([1, 2, 3, 9], [1, 2, 3], [W.M(9, 0.0), W.X(3, (9,))], "x3")
    psi9 = np.kron(np.array([0, 1]), psi)  # helper qubit 9 = bit 3 in |1> (prob of s=1 is 1/2)
    out = oracle.run(p, psi9, mode="forced", forced=[1]).output
    ref = psi[np.arange(8) ^ 4]
    assert equal_up_to_phase(out, ref, 1e-12)


def test_eq11_12_define_the_bra_and_eq13():
    """Eqs. 11-12 (L193-195): M_0 = |0><+a| = [[1,0],[0,0]] H Rz(-a), M_1 = |1><-a|. Their rows
    are the oracle's <+-a| (reading R-1) and M_i^dag M_i = P_i (Eq. 13); Eq. 5 holds."""
    rng = np.random.default_rng(0)
    for a in rng.uniform(-10, 10, 1000):
        Rz = np.diag([1, np.exp(-1j * a)])
        M0 = np.diag([1, 0]) @ H @ Rz
        M1 = np.diag([0, 1]) @ H @ Rz
        assert np.allclose(M0, np.array([[1, np.exp(-1j * a)], [0, 0]]) / math.sqrt(2), atol=1e-14)
        assert np.allclose(M1, np.array([[0, 0], [1, -np.exp(-1j * a)]]) / math.sqrt(2), atol=1e-14)
        assert np.allclose(M0[0], np.conj(oracle.plus_alpha(a)), atol=1e-14)
        assert np.allclose(M1[1], np.conj(oracle.minus_alpha(a)), atol=1e-14)
        assert np.allclose(M0.conj().T @ M0, oracle.P0_matrix(a), atol=1e-12)
        assert np.allclose(M1.conj().T @ M1, oracle.P1_matrix(a), atol=1e-12)
        assert np.allclose(M0.conj().T @ M0 + M1.conj().T @ M1, np.eye(2), atol=1e-12)


def test_eq2_resolve_angle():
    """Eq. 2 (L77): t[M^a]^s = M^{(-1)^s a + t pi}."""
    assert oracle.resolve_angle(0.3, 0, 0) == 0.3
    assert oracle.resolve_angle(0.3, 1, 0) == -0.3
    assert math.isclose(oracle.resolve_angle(0.3, 0, 1), 0.3 + math.pi)
    assert math.isclose(oracle.resolve_angle(0.3, 1, 1), -0.3 + math.pi)


@pytest.mark.parametrize("L", [1, 2, 3, 4])
def test_1q_2q_apply_vs_kronecker(L):
    """Generic apply routines vs the explicit Eq. 20 Kronecker operator, every position."""
    rng = np.random.default_rng(L)
    psi = rng.standard_normal(2 ** L) + 1j * rng.standard_normal(2 ** L)
    U = rng.standard_normal((2, 2)) + 1j * rng.standard_normal((2, 2))
    for pos in range(L):
        assert np.allclose(apply_1q(psi, L, pos, U), kron_embed(U, pos, L) @ psi, atol=1e-12)
    for u in range(L):
        for v in range(L):
            if u == v:
                continue
            # CZ through the generic 4x4 routine vs Fig. 5's reconstructed index loop (reading R-3)
            got = apply_2q(psi, L, u, v, CZ_4x4)
            hi, lo = max(u, v) + 1, min(u, v) + 1  # Fig. 5 uses 1-based u > v
            ref = psi.copy()
            for i in range(2 ** L // 4):
                j = i % 2 ** (hi - 2)
                lam = (j // 2 ** (lo - 1)) * 2 ** lo + 2 ** (lo - 1) + (j % 2 ** (lo - 1)) \
                    + (i // 2 ** (hi - 2)) * 2 ** hi + 2 ** (hi - 1)
                ref[lam] = -ref[lam]
            assert np.allclose(got, ref, atol=1e-15)
            # and the Fig. 5 loop touches exactly the indices with both bits set
            d = np.array([-1 if (x >> u) & 1 and (x >> v) & 1 else 1 for x in range(2 ** L)])
            assert np.allclose(ref, d * psi)


# ------------------------------------------------------------------ measurement

def test_worked_example_4_4_2():
    """§4.4.2 (L356-362): 3 qubits, M_2^a, outcome 0 -> psi'' = (a_k + e^{-i a} b_k)/sqrt(2 prob0),
    with psi = (a0, a1, b0, b1, a2, a3, b2, b3) (qubit 2 = bit 1), Eq. 21's compaction map."""
    rng = np.random.default_rng(7)
    for trial in range(20):
        psi = haar_state(3, 100 + trial)
        a = rng.uniform(0, 2 * math.pi)
        al = psi[[0, 1, 4, 5]]
        be = psi[[2, 3, 6, 7]]
        unnorm = al + np.exp(-1j * a) * be
        prob0 = np.sum(np.abs(unnorm) ** 2) / 2
        expected = unnorm / math.sqrt(2 * prob0)
        p = W.Pattern([1, 2, 3], [1, 3], [W.M(2, a)])
        r = oracle.run(p, psi, mode="forced", forced=[0])
        assert np.allclose(r.output, expected, atol=1e-13)
        assert math.isclose(r.prob0[0], prob0, abs_tol=1e-14)


@pytest.mark.parametrize("L", [1, 2, 3, 4])
def test_measurement_vs_generalized_operator(L):
    """Eqs. 6-7 with the Eq. 11-12 operators embedded by Eq. 20: prob_i = <psi|M^dag M|psi> and the
    post-state M psi/sqrt(prob) with the zero half removed (L217) equal the oracle's projective
    measurement + contraction, for every position and both outcomes."""
    rng = np.random.default_rng(10 + L)
    for _ in range(5):
        psi = rng.standard_normal(2 ** L) + 1j * rng.standard_normal(2 ** L)
        psi /= np.linalg.norm(psi)
        a = rng.uniform(0, 2 * math.pi)
        M0 = np.array([[1, np.exp(-1j * a)], [0, 0]]) / math.sqrt(2)
        M1 = np.array([[0, 0], [1, -np.exp(-1j * a)]]) / math.sqrt(2)
        for pos in range(L):
            ids = list(range(1, L + 1))
            outs = [q for q in ids if q != ids[pos]]
            if not outs:
                outs_present = False
            else:
                outs_present = True
            for s, Ms in ((0, M0), (1, M1)):
                Mfull = kron_embed(Ms, pos, L)
                post = Mfull @ psi
                prob = np.vdot(post, post).real
                keep = [x for x in range(2 ** L) if ((x >> pos) & 1) == s]
                expected = post[keep] / math.sqrt(prob)
                if not outs_present:
                    p = W.Pattern(ids, [], [W.M(ids[pos], a)])
                else:
                    p = W.Pattern(ids, outs, [W.M(ids[pos], a)])
                r = oracle.run(p, psi, mode="forced", forced=[s])
                assert math.isclose(r.prob0[0] if s == 0 else 1 - r.prob0[0], prob, abs_tol=1e-12)
                assert np.allclose(r.output, expected, atol=1e-12)


def test_cnot_figure8_trace():
    """Fig. 8 (L433-448): every printed intermediate state of the CNOT run of Eq. 23."""
    g = json.load(open(os.path.join(GOLDEN, "cnot_fig8.json")))
    p = W.cnot_pattern_eq23()
    psi = basis_state(2, 0b11)
    r = oracle.run(p, psi, mode="forced", forced=g["forced"], keep_trace=True)
    assert list(r.outcomes) == g["forced"]
    assert np.allclose(r.prob0, [0.5, 0.5])
    for name, st in g["substates"].items():
        if st["after_cmd"] < 0:
            continue
        _, order, amps = r.trace[st["after_cmd"]]
        # tensor the printed factors into the oracle's order
        qubits, vec = [], np.ones(1, dtype=np.complex128)
        for fq, fa in st["factors"]:
            vec = np.kron(np.array(fa, dtype=np.complex128), vec)
            qubits += fq
        assert sorted(qubits) == sorted(order), name
        from oracle.owqs_oracle import permute_to
        assert np.allclose(permute_to(vec, qubits, order), amps, atol=1e-12), name
    assert np.allclose(r.output, [0, 1, 0, 0])  # |q4q1> = |01> (L419)


def test_cnot_truth_table_all_branches():
    """Eq. 22 (L413) implements CNOT (L63, control q1) on every branch, up to a global phase
    (exactly -1 on branch (1,1), reading R-4); Eq. 23's reordering gives identical outputs."""
    cnot = np.array([[1, 0, 0, 0], [0, 1, 0, 0], [0, 0, 0, 1], [0, 0, 1, 0]])  # |c t>, c = MSB
    for k in range(4):
        q1, q2 = k & 1, k >> 1
        tgt = q2 ^ q1
        for br in range(4):
            f = [br & 1, br >> 1]
            o22 = oracle.run(W.cnot_pattern_eq22(), basis_state(2, k), mode="forced", forced=f).output
            o23 = oracle.run(W.cnot_pattern_eq23(), basis_state(2, k), mode="forced", forced=f).output
            ref = basis_state(2, q1 | (tgt << 1))
            assert equal_up_to_phase(o22, ref)
            assert np.allclose(o22, o23, atol=1e-14)
            assert np.allclose(o22, (-1 if br == 3 else 1) * ref, atol=1e-14)
            # and the same matrix as the paper's CNOT with (control, target) = (q1, q4)
            idx_ct = (q1 << 1) | q2
            out_ct = cnot[:, idx_ct]
            assert np.argmax(np.abs(out_ct)) == ((q1 << 1) | tgt)


@pytest.mark.parametrize("alpha", [0.0, 0.4, 1.3, math.pi, 5.9])
def test_j_pattern_both_branches(alpha):
    """J(alpha) = H diag(1, e^{i alpha}) = X_o^{s_i} M_i^{-alpha} E_io N_o exactly on both branches,
    with prob0 = 1/2 (BASELINE.json north_star)."""
    for k in range(2):
        for s in range(2):
            r = oracle.run(W.j_pattern(alpha), basis_state(1, k), mode="forced", forced=[s])
            assert np.allclose(r.output, J(alpha)[:, k], atol=1e-14)
            assert math.isclose(r.prob0[0], 0.5, abs_tol=1e-15)


def test_cz_pattern():
    """E_12 = CZ = diag(1,1,1,-1) (L63)."""
    U = oracle.recognize(W.cz_pattern())
    assert np.allclose(U, np.diag([1, 1, 1, -1]))


@pytest.mark.parametrize("n,seed", [(1, 1), (2, 2), (3, 3), (4, 4), (2, 5), (3, 6)])
def test_recognition_bruteforce(n, seed):
    """Recognition (L33) on <= 4 logical qubits equals the textbook circuit product exactly."""
    rng = np.random.default_rng(seed)
    while True:  # re-draw circuits that would repeat an E on one qubit pair
        gates = []
        for _ in range(4 * n + 2):
            if n > 1 and rng.uniform() < 0.3:
                a, b = rng.choice(n, 2, replace=False)
                gates.append(("CZ", int(a), int(b)))
            else:
                gates.append(("J", int(rng.integers(n)), float(rng.uniform(0, 2 * math.pi))))
        try:
            p = W.circuit_to_pattern(n, gates)
            break
        except ValueError:
            continue
    U = oracle.recognize(p)
    assert np.allclose(U, circuit_matrix(n, gates), atol=1e-12)
    assert np.allclose(U.conj().T @ U, np.eye(2 ** n), atol=1e-12)


def test_cp_decomposition_identity():
    """Reading R-12: the 8 J + 2 CZ controlled-phase realises diag(1,1,1,e^{i theta})."""
    for th in (0.3, math.pi / 2, math.pi / 8, 2.5):
        U = circuit_matrix(2, W.cp_gates(th, 0, 1))
        assert np.allclose(U, np.diag([1, 1, 1, np.exp(1j * th)]), atol=1e-13)


@pytest.mark.parametrize("n", [2, 3, 4, 5])
def test_qft_pattern_closed_form(n):
    """QFT pattern (config 2 family): out[rev(y)] = sqrt(N) ifft(psi)[y] (textbook DFT), and
    |V| = 4n^2 - 2n as in Table II's QFT rows (L465-469)."""
    p = W.config_pattern(f"QFT:{n}")
    assert len(p.qubits()) == 4 * n * n - 2 * n
    psi = haar_state(n, n)
    r = oracle.run(p, psi, mode="sampled", seed=11)
    f = math.sqrt(2 ** n) * np.fft.ifft(psi)
    rev = [int(format(y, f"0{n}b")[::-1], 2) for y in range(2 ** n)]
    assert np.allclose(r.output[rev], f, atol=1e-12)
    assert r.peak_width == n + 1  # m = n + 1 (Table III QFT rows, L497-501)
    assert np.allclose(r.prob0, 0.5, atol=1e-12)


def test_branch_independence_wild_patterns():
    """Wild J/CZ patterns: output identical (no phase) on every branch; prob0 = 1/2 (L372)."""
    p = W.config_pattern("C1", seed=3)
    psi = haar_state(3, 2)
    ref = oracle.run(p, psi, mode="eowqs").output
    rng = np.random.default_rng(5)
    for _ in range(8):
        f = rng.integers(0, 2, p.n_measure)
        r = oracle.run(p, psi, mode="forced", forced=f)
        assert np.allclose(r.output, ref, atol=1e-12)
        assert np.allclose(r.prob0, 0.5, atol=1e-12)
    for seed in range(4):
        r = oracle.run(p, psi, mode="sampled", seed=seed)
        assert np.allclose(r.output, ref, atol=1e-12)
        assert abs(np.linalg.norm(r.output) - 1) < 1e-12


@pytest.mark.parametrize("rows,cols", [(3, 4), (4, 3), (2, 5)])
def test_flow_cluster_outcome_independence(rows, cols):
    """gflow/flow patterns (L372): prob = 1/2 on every branch and all branches give one state up
    to a global phase; the EOWQS positive branch is that state with norm 1 (config 5 family)."""
    p = W.cluster_pattern(rows, cols, seed=rows * 10 + cols)
    psi = haar_state(rows, 9)
    ref = oracle.run(p, psi, mode="eowqs")
    assert abs(np.linalg.norm(ref.output) - 1) < 1e-12
    assert ref.peak_width == rows + 1  # §4.6 (L403): m = N + 1
    rng = np.random.default_rng(rows + cols)
    for _ in range(10):
        f = rng.integers(0, 2, p.n_measure)
        r = oracle.run(p, psi, mode="forced", forced=f)
        assert np.allclose(r.prob0, 0.5, atol=1e-12)
        assert equal_up_to_phase(r.output, ref.output, 1e-11)


def test_non_flow_pattern_is_not_branch_independent():
    """Negative control: dropping the corrections of a J pattern breaks determinism, and EOWQS's
    sqrt2 rescale then no longer conserves the norm when prob0 != 1/2."""
    p = W.Pattern([1], [2], [W.N(2), W.E(1, 2), W.M(1, 0.3)])
    psi = haar_state(1, 4)
    o0 = oracle.run(p, psi, mode="forced", forced=[0]).output
    o1 = oracle.run(p, psi, mode="forced", forced=[1]).output
    assert not equal_up_to_phase(o0, o1, 1e-6)
    q = W.Pattern([1, 2], [2], [W.M(1, 0.3)])
    r = oracle.run(q, haar_state(2, 8), mode="eowqs")
    assert abs(np.linalg.norm(r.output) - 1) > 1e-3


def test_sampling_statistics():
    """Fig. 6 (L387) 'rand(0,1) <= prob': the outcome-0 frequency matches the closed-form
    prob0 = |<+theta|phi>|^2 of a product input within a 4-sigma binomial band."""
    phi = np.array([0.8, 0.6 * np.exp(0.7j)])
    theta = 1.1
    p0 = abs(np.vdot(oracle.plus_alpha(theta), phi)) ** 2
    pat = W.Pattern([1, 2], [2], [W.M(1, theta)])
    psi = np.kron(np.array([1, 0]), phi)
    n = 3000
    zeros = sum(1 - int(oracle.run(pat, psi, mode="sampled", seed=s).outcomes[0]) for s in range(n))
    sigma = math.sqrt(n * p0 * (1 - p0))
    assert abs(zeros - n * p0) < 4 * sigma
    u = np.array([oracle.draw_uniform(1, k) for k in range(20000)])
    assert abs(u.mean() - 0.5) < 4 * math.sqrt(1 / 12 / 20000)
    assert u.min() >= 0 and u.max() < 1


def test_pattern_rules_rejected():
    """D1-D3 (L85-91) and the forced impossible branch (Fig. 6 division by prob)."""
    psi = haar_state(1, 1)
    with pytest.raises(oracle.OracleError):  # D1: act after measure
        oracle.run(W.Pattern([1], [2], [W.N(2), W.M(1, 0.0), W.E(1, 2)]), psi)
    with pytest.raises(oracle.OracleError):  # D3: output measured
        oracle.run(W.Pattern([1], [1], [W.M(1, 0.0)]), psi)
    with pytest.raises(oracle.OracleError):  # forced outcome with zero probability
        oracle.run(W.Pattern([1, 2], [2], [W.M(1, 0.0)]), np.array([1, 0, 0, 0.0]) * 0 + np.array([0.5 ** .5, 0.5 ** .5, 0, 0]),
                   mode="forced", forced=[1])


def test_norm_preserved_sampled_c1():
    """Norm preservation through a whole sampled run (Eq. 4 renormalises at every M)."""
    for seed in range(3):
        p = W.config_pattern("C1", seed=seed)
        r = oracle.run(p, haar_state(3, seed), mode="sampled", seed=seed)
        assert abs(np.linalg.norm(r.output) - 1) < 1e-12
        assert r.peak_width <= 5  # configs[0]: peak active width <= 5
