"""CPU oracle: plain, slow, obviously-correct complex128 execution of a 1WQC pattern.

TEST INFRASTRUCTURE. Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and
--impl reference) may import this module. It shares no code with the CUDA path.

What it computes (the "plain definition"): a dense state vector over the
live qubits, commands executed one by one in the pattern's GIVEN (execution) order, each
through an explicit 2x2 / 4x4 matrix applied by a generic index routine:
  N v      state <- (1,1)/sqrt2 (x) state                      PAPER L69 (preparation action)
  E u v    4x4 diag(1,1,1,-1) on (u, v)                         PAPER L70, L63 (CZ matrix)
  X/Z v s  2x2 Pauli iff the XOR of the outcomes in s is 1      PAPER L81, L55 (Pauli set)
  M v      theta = (-1)^s alpha + t pi                          PAPER L77 (Eq. 2)
           prob_i = <psi|P_i|psi>, P_0, P_1 of Eqs. 9-10        PAPER L105 (Eq. 3)
           outcome: sampled "rand(0,1) <= prob0" | forced | EOWQS 0   PAPER L387 (Fig. 6)
           psi <- P_i psi / sqrt(prob_i)   (EOWQS: sqrt2 P_0 psi)     PAPER L109 (Eq. 4)
           the measured qubit is now |+-theta>; its axis is removed by contracting with
           <+-theta| (qubit elimination)
Measurement-basis sign convention (reading R-1): <+-theta| = (<0| +- e^{-i theta}<1|)/sqrt2,
i.e. |+-theta> = (|0> +- e^{+i theta}|1>)/sqrt2, the reading fixed by Eqs. 9-12 and the worked
example of §4.4.2 (L358, coefficient e^{-i alpha} on the beta half).
Random draws (reading R-5): u_M = (splitmix64(seed ^ splitmix64(ord_M)) >> 11) 2^-53 with
ord_M the ordinal of the M command in the GIVEN list; outcome 0 iff u_M <= prob0.
Index convention: order[p] is the qubit owning bit p of the amplitude index (position 1 =
least significant bit, Eq. 8); inputs[0] / outputs[0] are bit 0.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from workloads.patterns import KIND_E, KIND_M, KIND_N, KIND_X, KIND_Z, Pattern

SQRT_HALF = 1.0 / math.sqrt(2.0)
PAULI_X = np.array([[0, 1], [1, 0]], dtype=np.complex128)
PAULI_Z = np.array([[1, 0], [0, -1]], dtype=np.complex128)
CZ_4x4 = np.diag([1, 1, 1, -1]).astype(np.complex128)
PLUS = np.array([SQRT_HALF, SQRT_HALF], dtype=np.complex128)  # |+>


class OracleError(RuntimeError):
    pass


# ---------------------------------------------------------------------------------------------
# Operators
# ---------------------------------------------------------------------------------------------

def resolve_angle(alpha: float, s: int, t: int) -> float:
    """Eq. 2: t[M^alpha]^s = M^{(-1)^s alpha + t pi} (sign on alpha only, R-7)."""
    return (-1.0) ** s * alpha + t * math.pi


def plus_alpha(theta: float) -> np.ndarray:
    """|+theta> = (|0> + e^{i theta}|1>)/sqrt2 (reading R-1, so that P_0 = |+><+| is Eq. 9)."""
    return np.array([SQRT_HALF, SQRT_HALF * np.exp(1j * theta)], dtype=np.complex128)


def minus_alpha(theta: float) -> np.ndarray:
    return np.array([SQRT_HALF, -SQRT_HALF * np.exp(1j * theta)], dtype=np.complex128)


def P0_matrix(theta: float) -> np.ndarray:
    """Eq. 9: P_0 = 1/2 [[1, e^{-i a}], [e^{i a}, 1]]."""
    return 0.5 * np.array([[1, np.exp(-1j * theta)], [np.exp(1j * theta), 1]], dtype=np.complex128)


def P1_matrix(theta: float) -> np.ndarray:
    """Eq. 10: P_1 = 1/2 [[1, -e^{-i a}], [-e^{i a}, 1]]."""
    return 0.5 * np.array([[1, -np.exp(-1j * theta)], [-np.exp(1j * theta), 1]], dtype=np.complex128)


def _splitmix64(x: int) -> int:
    m = (1 << 64) - 1
    z = (x + 0x9E3779B97F4A7C15) & m
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & m
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & m
    return z ^ (z >> 31)


def draw_uniform(seed: int, ord_m: int) -> float:
    """The keyed draw of reading R-5: uniform in [0, 1) for the M with given-order ordinal ord_m."""
    return (_splitmix64((seed & ((1 << 64) - 1)) ^ _splitmix64(ord_m)) >> 11) * 2.0 ** -53


# ---------------------------------------------------------------------------------------------
# Generic apply routines (a library reshape/transposition is the only "trick" used)
# ---------------------------------------------------------------------------------------------

def _as_tensor(amps: np.ndarray, L: int) -> np.ndarray:
    """View a 2^L vector as an L-axis tensor; bit p of the index is axis L-1-p."""
    return amps.reshape((2,) * L) if L > 0 else amps.reshape(())


def apply_1q(amps: np.ndarray, L: int, pos: int, U: np.ndarray) -> np.ndarray:
    """new[..., r, ...] = sum_c U[r, c] old[..., c, ...] on bit `pos`."""
    v = amps.reshape(2 ** (L - pos - 1), 2, 2 ** pos)
    out = np.empty_like(v)
    out[:, 0, :] = U[0, 0] * v[:, 0, :] + U[0, 1] * v[:, 1, :]
    out[:, 1, :] = U[1, 0] * v[:, 0, :] + U[1, 1] * v[:, 1, :]
    return out.reshape(-1)


def apply_2q(amps: np.ndarray, L: int, pa: int, pb: int, U4: np.ndarray) -> np.ndarray:
    """Generic 4x4 on bits (pa, pb); the 4x4 basis index is 2*bit_pa + bit_pb."""
    t = _as_tensor(amps, L)
    t = np.moveaxis(t, [L - 1 - pa, L - 1 - pb], [0, 1])
    shape = t.shape
    t = (U4 @ t.reshape(4, -1)).reshape(shape)
    t = np.moveaxis(t, [0, 1], [L - 1 - pa, L - 1 - pb])
    return np.ascontiguousarray(t).reshape(-1)


def contract_out(amps: np.ndarray, L: int, pos: int, bra: np.ndarray) -> np.ndarray:
    """new[j] = sum_x bra[x] * amps[insert(j, pos, x)]: removes bit `pos`."""
    v = amps.reshape(2 ** (L - pos - 1), 2, 2 ** pos)
    return (bra[0] * v[:, 0, :] + bra[1] * v[:, 1, :]).reshape(-1)


def permute_to(amps: np.ndarray, order: Sequence[int], target: Sequence[int]) -> np.ndarray:
    """Re-index so that target[k] owns bit k."""
    L = len(order)
    if L == 0:
        return amps.copy()
    t = _as_tensor(amps, L)
    # axis of qubit q in t is L-1-order.index(q); we want target[k] at axis L-1-k
    src_axes = [L - 1 - list(order).index(target[L - 1 - a]) for a in range(L)]
    return np.ascontiguousarray(np.transpose(t, src_axes)).reshape(-1)


# ---------------------------------------------------------------------------------------------
# The run
# ---------------------------------------------------------------------------------------------

@dataclass
class OracleResult:
    output: np.ndarray            # amplitudes over pattern.outputs (outputs[0] = LSB)
    outcomes: np.ndarray          # uint8 per M, indexed by the M's ordinal in the GIVEN order
    prob0: np.ndarray             # float64 per M: <psi|P_0|psi> at the moment of measurement
    peak_width: int               # largest live width reached in the given order
    trace: List[tuple] = field(default_factory=list)  # (cmd, order, amps) after every command


def _parity(outcome_of: dict, dom: Sequence[int]) -> int:
    s = 0
    for q in dom:
        if q not in outcome_of:
            raise OracleError(f"D0: signal depends on unmeasured qubit {q}")
        s ^= outcome_of[q]
    return s


def run(pattern: Pattern, input_amps: np.ndarray, mode: str = "forced", seed: int = 0,
        forced: Optional[Sequence[int]] = None, keep_trace: bool = False,
        knife_edge_override: Optional[dict] = None) -> OracleResult:
    """Execute `pattern` in its GIVEN order. mode: 'sampled' | 'forced' | 'eowqs'.

    knife_edge_override: {ord_M: outcome} replays a sampled measurement with a fixed outcome
    (reading R-5's knife-edge rule, used only by the parity harness)."""
    if mode not in ("sampled", "forced", "eowqs"):
        raise OracleError(f"bad mode {mode}")
    inputs = list(pattern.inputs)
    amps = np.asarray(input_amps, dtype=np.complex128).copy()
    if amps.shape != (2 ** len(inputs),):
        raise OracleError("input size does not match 2^|I|")
    nrm = float(np.vdot(amps, amps).real)
    if abs(nrm - 1.0) > 1e-9:
        raise OracleError(f"input not normalised (norm^2 = {nrm})")
    order: List[int] = list(inputs)
    prepared = set(inputs)
    measured: dict = {}
    n_m = pattern.n_measure
    outcomes = np.zeros(n_m, dtype=np.uint8)
    prob0 = np.zeros(n_m, dtype=np.float64)
    if mode == "forced":
        if forced is None and n_m == 0:
            forced = []
        if forced is None or len(forced) != n_m:
            raise OracleError("forced outcomes must have one bit per M")
    trace: List[tuple] = []
    peak = len(order)
    ord_m = 0

    def ensure_prepared(q: int) -> None:
        # implicit N at first use of a non-input qubit (reading R-11)
        nonlocal amps
        if q in measured:
            raise OracleError(f"D1: action on measured qubit {q}")
        if q not in prepared:
            amps = np.kron(PLUS, amps)
            order.append(q)
            prepared.add(q)

    for cmd in pattern.cmds:
        k = cmd.kind
        if k == KIND_N:
            if cmd.q0 in prepared or cmd.q0 in measured:
                raise OracleError(f"N on already prepared qubit {cmd.q0}")
            ensure_prepared(cmd.q0)
        elif k == KIND_E:
            if cmd.q0 == cmd.q1:
                raise OracleError("E on one qubit")
            ensure_prepared(cmd.q0)
            ensure_prepared(cmd.q1)
            amps = apply_2q(amps, len(order), order.index(cmd.q0), order.index(cmd.q1), CZ_4x4)
        elif k in (KIND_X, KIND_Z):
            ensure_prepared(cmd.q0)
            if _parity(measured, cmd.sdom):
                amps = apply_1q(amps, len(order), order.index(cmd.q0),
                                PAULI_X if k == KIND_X else PAULI_Z)
        elif k == KIND_M:
            v = cmd.q0
            if v in pattern.outputs:
                raise OracleError(f"D3: output {v} measured")
            ensure_prepared(v)
            L = len(order)
            pos = order.index(v)
            theta = resolve_angle(cmd.angle, _parity(measured, cmd.sdom), _parity(measured, cmd.tdom))
            P = (P0_matrix(theta), P1_matrix(theta))
            proj = [apply_1q(amps, L, pos, P[s]) for s in (0, 1)]
            p = [float(np.vdot(amps, proj[s]).real) for s in (0, 1)]
            if abs(p[0] + p[1] - float(np.vdot(amps, amps).real)) > 1e-10:
                raise OracleError("P_0 + P_1 != I")
            if mode == "sampled":
                u = draw_uniform(seed, ord_m)
                s = 0 if u <= p[0] else 1
                if knife_edge_override and ord_m in knife_edge_override:
                    s = int(knife_edge_override[ord_m])
            elif mode == "forced":
                s = int(forced[ord_m])
            else:
                s = 0
            if mode != "eowqs" and p[s] < 1e-12:
                raise OracleError(f"forced outcome {s} on M ordinal {ord_m} has probability {p[s]}")
            scale = math.sqrt(2.0) if mode == "eowqs" else 1.0 / math.sqrt(p[s])
            amps = proj[s] * scale
            ket = plus_alpha(theta) if s == 0 else minus_alpha(theta)
            other = minus_alpha(theta) if s == 0 else plus_alpha(theta)
            residual = contract_out(amps, L, pos, np.conj(other))
            if np.max(np.abs(residual), initial=0.0) > 1e-10:
                raise OracleError("measured qubit is not in the product state |+-theta>")
            amps = contract_out(amps, L, pos, np.conj(ket))
            order.pop(pos)
            measured[v] = s
            outcomes[ord_m] = s
            prob0[ord_m] = p[0]
            ord_m += 1
        else:
            raise OracleError(f"unknown command kind {k}")
        peak = max(peak, len(order))
        if keep_trace:
            trace.append((cmd, list(order), amps.copy()))

    for o in pattern.outputs:
        if o not in prepared:  # an output never touched: |+> (implicit N, reading R-11)
            ensure_prepared(o)
    if sorted(order) != sorted(pattern.outputs):
        raise OracleError(f"live qubits {order} != outputs {pattern.outputs}")
    out = permute_to(amps, order, list(pattern.outputs))
    return OracleResult(out, outcomes, prob0, peak, trace)


def recognize(pattern: Pattern) -> np.ndarray:
    """The unitary a deterministic pattern implements (the recognition problem):
    column k = EOWQS (all outcomes 0, sqrt2 per M) run on basis input |k>."""
    n_in, n_out = len(pattern.inputs), len(pattern.outputs)
    U = np.zeros((2 ** n_out, 2 ** n_in), dtype=np.complex128)
    for k in range(2 ** n_in):
        e = np.zeros(2 ** n_in, dtype=np.complex128)
        e[k] = 1.0
        U[:, k] = run(pattern, e, mode="eowqs").output
    return U
