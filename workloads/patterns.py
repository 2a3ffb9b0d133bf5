"""Pattern data model and seeded pattern generators (command lists only; no arithmetic).

A 1WQC pattern P = (V, I, O, A) (§2.2) is stored as
  inputs  : list of qubit ids, inputs[0] = least-significant bit of the input amplitude index
  outputs : list of qubit ids, outputs[0] = least-significant bit of the output index
  cmds    : list of Cmd in EXECUTION order (first element executes first). The paper writes
            patterns right-to-left (L67, "actions are applied from right to left"); every
            generator here already emits the execution order.
Commands (L69-81): N v | E u v | M v angle s_dom t_dom | X v s_dom | Z v s_dom.
Signal domains are lists of measured qubit ids whose outcomes are XOR-summed (L75-77, Eq. 2).

Non-input qubits that are used before an explicit N get an implicit N at first use
(reading R-11; the paper's own patterns omit N, e.g. Eq. 22 at L413).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Sequence, Tuple

import numpy as np

KIND_N, KIND_E, KIND_M, KIND_X, KIND_Z = 0, 1, 2, 3, 4
KIND_NAMES = {KIND_N: "N", KIND_E: "E", KIND_M: "M", KIND_X: "X", KIND_Z: "Z"}


@dataclass(frozen=True)
class Cmd:
    kind: int                 # KIND_*
    q0: int                   # target qubit (u for E)
    q1: int = -1              # second qubit (E only)
    angle: float = 0.0        # base angle alpha of Eq. 2 (M only), radians
    sdom: Tuple[int, ...] = ()  # s-signal domain (M, X, Z)
    tdom: Tuple[int, ...] = ()  # t-signal domain (M only)

    def __str__(self) -> str:  # human-readable, execution order
        k = KIND_NAMES[self.kind]
        if self.kind == KIND_N:
            return f"N{self.q0}"
        if self.kind == KIND_E:
            return f"E{self.q0},{self.q1}"
        if self.kind == KIND_M:
            return f"M{self.q0}^{self.angle:.4f}[s{list(self.sdom)} t{list(self.tdom)}]"
        return f"{k}{self.q0}^s{list(self.sdom)}"


def N(v: int) -> Cmd:
    return Cmd(KIND_N, v)


def E(u: int, v: int) -> Cmd:
    return Cmd(KIND_E, u, v)


def M(v: int, angle: float, sdom: Sequence[int] = (), tdom: Sequence[int] = ()) -> Cmd:
    return Cmd(KIND_M, v, -1, float(angle), tuple(sdom), tuple(tdom))


def X(v: int, sdom: Sequence[int] = ()) -> Cmd:
    return Cmd(KIND_X, v, -1, 0.0, tuple(sdom))


def Z(v: int, sdom: Sequence[int] = ()) -> Cmd:
    return Cmd(KIND_Z, v, -1, 0.0, tuple(sdom))


@dataclass
class Pattern:
    inputs: List[int]
    outputs: List[int]
    cmds: List[Cmd]
    name: str = ""
    meta: dict = field(default_factory=dict)

    @property
    def n_measure(self) -> int:
        return sum(1 for c in self.cmds if c.kind == KIND_M)

    def measured_in_given_order(self) -> List[int]:
        """Qubit ids of the M commands in the GIVEN order; position = the M's ordinal."""
        return [c.q0 for c in self.cmds if c.kind == KIND_M]

    def qubits(self) -> List[int]:
        seen = dict.fromkeys(self.inputs)
        for c in self.cmds:
            seen.setdefault(c.q0, None)
            if c.kind == KIND_E:
                seen.setdefault(c.q1, None)
        for o in self.outputs:
            seen.setdefault(o, None)
        return list(seen)


# --------------------------------------------------------------------------------------------
# Circuits of J(alpha) and CZ gates and their translation to patterns (reading R-12).
# J(alpha) = H diag(1, e^{i alpha}) is realised by the wild-form pattern
#     N_o  E_io  M_i^{-alpha}  X_o^{s_i}          (execution order)
# CZ(w1, w2) is E between the wires' current qubits. (BASELINE.json configs.)
# --------------------------------------------------------------------------------------------

def circuit_to_pattern(n_wires: int, gates: Sequence[tuple], name: str = "") -> Pattern:
    """gates: ('J', wire, alpha) | ('CZ', wire_a, wire_b), in time order."""
    cur = list(range(n_wires))
    nxt = n_wires
    cmds: List[Cmd] = []
    last_e = {}  # pair -> True if an E on this exact qubit pair already exists
    for g in gates:
        if g[0] == "J":
            _, w, alpha = g
            i, o = cur[w], nxt
            nxt += 1
            cmds += [N(o), E(i, o), M(i, -alpha), X(o, (i,))]
            cur[w] = o
        elif g[0] == "CZ":
            _, a, b = g
            if a == b:
                raise ValueError("CZ on one wire")
            key = (min(cur[a], cur[b]), max(cur[a], cur[b]))
            if key in last_e:
                raise ValueError(f"duplicate E on qubit pair {key}")
            last_e[key] = True
            cmds.append(E(cur[a], cur[b]))
        else:
            raise ValueError(f"unknown gate {g!r}")
    return Pattern(list(range(n_wires)), list(cur), cmds, name)


def _circuit_has_duplicate_cz(n_wires: int, gates: Sequence[tuple]) -> bool:
    try:
        circuit_to_pattern(n_wires, gates)
    except ValueError:
        return True
    return False


def random_tiny_circuit(seed: int, n_wires: int = 3, n_j: int = 12, n_cz: int = 4) -> List[tuple]:
    """Config 1: seeded random circuit of 12 J(alpha) (alpha ~ U[0, 2pi)) on uniform random wires
    and 4 CZ on uniform random distinct pairs, in a seeded shuffled order (BASELINE.json
    configs[0]). Orders that would repeat an E on one qubit pair are re-drawn."""
    rng = np.random.default_rng(seed)
    while True:
        gates = [("J", int(rng.integers(n_wires)), float(rng.uniform(0, 2 * math.pi)))
                 for _ in range(n_j)]
        for _ in range(n_cz):
            a, b = rng.choice(n_wires, size=2, replace=False)
            gates.append(("CZ", int(a), int(b)))
        order = rng.permutation(len(gates))
        gates = [gates[i] for i in order]
        if not _circuit_has_duplicate_cz(n_wires, gates):
            return gates


def cp_gates(theta: float, control: int, target: int) -> List[tuple]:
    """Controlled phase diag(1,1,1,e^{i theta}) as 8 J + 2 CZ (reading R-12):
    target J(0) CZ J(0) J(-theta/2) CZ J(0) J(theta/2) J(0); control J(theta/2) J(0)."""
    t, c = target, control
    return [("J", t, 0.0), ("CZ", c, t), ("J", t, 0.0), ("J", t, -theta / 2), ("CZ", c, t),
            ("J", t, 0.0), ("J", t, theta / 2), ("J", t, 0.0),
            ("J", c, theta / 2), ("J", c, 0.0)]


def qft_circuit(n: int) -> List[tuple]:
    """Textbook QFT without the final swaps: for wire j = n-1 .. 0: H_j = J(0), then
    CP(pi / 2^{j-k}) controlled by k for k = j-1 .. 0 (BASELINE.json configs[1]).
    Gives 4n^2 - 3n J gates, |V| = 4n^2 - 2n (PAPER Table II QFT rows, L465-469)."""
    gates: List[tuple] = []
    for j in range(n - 1, -1, -1):
        gates.append(("J", j, 0.0))
        for k in range(j - 1, -1, -1):
            gates += cp_gates(math.pi / 2 ** (j - k), k, j)
    return gates


def brickwork_circuit(n: int, depth: int, seed: int) -> List[tuple]:
    """Configs 3/4: layer l applies J(alpha_{l,w}) (alpha ~ U[0, 2pi)) on every wire, then CZ on
    nearest-neighbour pairs (w, w+1) with w = l (mod 2)."""
    rng = np.random.default_rng(seed)
    gates: List[tuple] = []
    for layer in range(depth):
        for w in range(n):
            gates.append(("J", w, float(rng.uniform(0, 2 * math.pi))))
        for w in range(layer % 2, n - 1, 2):
            gates.append(("CZ", w, w + 1))
    return gates


def prefix_pattern(pattern: Pattern, k_cmds: int) -> Pattern:
    """The first k commands of `pattern` (given order) as a pattern of their own: same inputs, the
    outputs are the qubits live after them (prepared and not measured), in order of preparation.
    Used for full-width parity on a prefix (both sides run the same command list)."""
    cmds = list(pattern.cmds[:k_cmds])
    live = list(pattern.inputs)
    for c in cmds:
        if c.kind == KIND_N:
            live.append(c.q0)
        elif c.kind == KIND_E:
            for q in (c.q0, c.q1):
                if q not in live:
                    live.append(q)  # implicit N (reading R-11)
        elif c.kind == KIND_M:
            live.remove(c.q0)
    return Pattern(list(pattern.inputs), live, cmds, pattern.name + f"[:{k_cmds}]")


def brickwork_layer_cmds(n: int, layers: int) -> int:
    """Commands in the first `layers` layers of an n-wire brickwork pattern (4 per J, 1 per CZ)."""
    return sum(4 * n + len(range(l % 2, n - 1, 2)) for l in range(layers))


# --------------------------------------------------------------------------------------------
# Patterns printed or implied by the paper
# --------------------------------------------------------------------------------------------

def j_pattern(alpha: float, i: int = 1, o: int = 2) -> Pattern:
    """X_o^{s_i} M_i^{-alpha} E_io N_o  (execution order N, E, M, X) = J(alpha)."""
    return Pattern([i], [o], [N(o), E(i, o), M(i, -alpha), X(o, (i,))], "J")


def cz_pattern() -> Pattern:
    """E_12 on I = O = {1, 2}: the CZ gate."""
    return Pattern([1, 2], [1, 2], [E(1, 2)], "CZ")


def cnot_pattern_eq22() -> Pattern:
    """Eq. 22: CNOT = ({1,2,3,4}, {1,2}, {1,4}, X_4^3 Z_4^2 Z_1^2 M_3^0 M_2^0 E_13 E_23 E_34)
    read right to left. Inputs [1, 2] (q1 = LSB), outputs [1, 4] (q1 = LSB), as in Fig. 8."""
    cmds = [E(3, 4), E(2, 3), E(1, 3), M(2, 0.0), M(3, 0.0),
            Z(1, (2,)), Z(4, (2,)), X(4, (3,))]
    return Pattern([1, 2], [1, 4], cmds, "CNOT-Eq22")


def cnot_pattern_eq23() -> Pattern:
    """Eq. 23: the PROA reordering of Eq. 22, X_4^3 Z_4^2 Z_1^2 M_3^0 E_13 E_34 M_2^0 E_23."""
    cmds = [E(2, 3), M(2, 0.0), E(3, 4), E(1, 3), M(3, 0.0),
            Z(1, (2,)), Z(4, (2,)), X(4, (3,))]
    return Pattern([1, 2], [1, 4], cmds, "CNOT-Eq23")


def linear_cluster_pattern(length: int, seed: int) -> Pattern:
    """1D cluster (PAPER §4.6): a chain of `length` J gates on one wire."""
    rng = np.random.default_rng(seed)
    gates = [("J", 0, float(rng.uniform(0, 2 * math.pi))) for _ in range(length)]
    return circuit_to_pattern(1, gates, f"chain{length}")


def cluster_pattern(rows: int, cols: int, seed: int, angles: str = "pi4noise") -> Pattern:
    """Config 5: 2D cluster rows x cols, qubit (r, c) has id c*rows + r, I = column 0, O = last
    column, grid edges. Given order is the column-by-column order of PAPER §4.6 (L403):
      for c = 0..cols-2: vertical E's of column c; then for r: N(r,c+1) E((r,c),(r,c+1)) M(r,c)
      finally vertical E's of the last column, then Z_o^{t_o} X_o^{s_o} on every output.
    Flow f(r,c) = (r,c+1) gives s_w = {(r,c-1)}, t_w = {(r+-1,c-1), (r,c-2)} (measured ones).
    Angles: k*pi/4 + eps, k ~ U{0..7}, eps ~ U[-pi/16, pi/16] (BASELINE.json configs[4])."""
    rng = np.random.default_rng(seed)

    def qid(r, c):
        return c * rows + r

    def sdom(r, c):
        return (qid(r, c - 1),) if c - 1 >= 0 else ()

    def tdom(r, c):
        t = []
        if c - 1 >= 0:
            if r - 1 >= 0:
                t.append(qid(r - 1, c - 1))
            if r + 1 < rows:
                t.append(qid(r + 1, c - 1))
        if c - 2 >= 0:
            t.append(qid(r, c - 2))
        return tuple(t)

    cmds: List[Cmd] = []
    for c in range(cols - 1):
        for r in range(rows - 1):
            cmds.append(E(qid(r, c), qid(r + 1, c)))
        for r in range(rows):
            if angles == "pi4noise":
                a = int(rng.integers(8)) * math.pi / 4 + float(rng.uniform(-math.pi / 16, math.pi / 16))
            else:
                a = float(rng.uniform(0, 2 * math.pi))
            cmds += [N(qid(r, c + 1)), E(qid(r, c), qid(r, c + 1)), M(qid(r, c), a, sdom(r, c), tdom(r, c))]
    c = cols - 1
    for r in range(rows - 1):
        cmds.append(E(qid(r, c), qid(r + 1, c)))
    for r in range(rows):
        if tdom(r, c):
            cmds.append(Z(qid(r, c), tdom(r, c)))
        if sdom(r, c):
            cmds.append(X(qid(r, c), sdom(r, c)))
    return Pattern([qid(r, 0) for r in range(rows)], [qid(r, cols - 1) for r in range(rows)], cmds,
                   f"cluster{rows}x{cols}")


# --------------------------------------------------------------------------------------------
# BASELINE.json configurations
# --------------------------------------------------------------------------------------------

def config_pattern(name: str, seed: int = 1) -> Pattern:
    """'C1' tiny (3 wires, 12 J, 4 CZ); 'C2' QFT-20; 'C3' brickwork 28x40; 'C3W' brickwork 30x40
    (width-30 companion of C3); 'C4' brickwork 33x24; 'C5' cluster 35x8.
    Names ending in a size override (e.g. 'QFT:8', 'BW:10x6', 'CL:4x5') give scaled-down
    members of the same families for parity tests."""
    if name == "C1":
        p = circuit_to_pattern(3, random_tiny_circuit(seed), "C1")
    elif name == "C2":
        p = circuit_to_pattern(20, qft_circuit(20), "C2")
    elif name == "C3":
        p = circuit_to_pattern(28, brickwork_circuit(28, 40, seed), "C3")
    elif name == "C3W":
        p = circuit_to_pattern(30, brickwork_circuit(30, 40, seed), "C3W")
    elif name == "C4":
        p = circuit_to_pattern(33, brickwork_circuit(33, 24, seed), "C4")
    elif name == "C5":
        p = cluster_pattern(35, 8, seed)
    elif name == "C3M":
        p = measured_tail(circuit_to_pattern(28, brickwork_circuit(28, 40, seed), "C3M"), 8, seed)
    elif name.startswith("BWM:"):
        n, d, k = (int(x) for x in name[4:].split("x"))
        p = measured_tail(circuit_to_pattern(n, brickwork_circuit(n, d, seed), name), k, seed)
    elif name.startswith("QFT:"):
        n = int(name[4:])
        p = circuit_to_pattern(n, qft_circuit(n), name)
    elif name.startswith("BW:"):
        n, d = (int(x) for x in name[3:].split("x"))
        p = circuit_to_pattern(n, brickwork_circuit(n, d, seed), name)
    elif name.startswith("CL:"):
        r, c = (int(x) for x in name[3:].split("x"))
        p = cluster_pattern(r, c, seed)
        p.name = name
    else:
        raise KeyError(name)
    p.meta["seed"] = seed
    return p


def measured_tail(p: Pattern, k: int, seed: int) -> Pattern:
    """Measure the last k output qubits of a circuit pattern in the XY plane (angles ~ U[0, 2pi)) after
    its last command: measurements with no fresh neighbour, so each eliminates a qubit from the state
    (SHRINK, Eq. 13 reduction, Fig. 6 compaction) -- the SHRINK-heavy workload C3M (config 3 with 8 of
    its 28 wires read out)."""
    rng = np.random.default_rng(10_000 + seed)
    tail = [M(q, float(rng.uniform(0, 2 * math.pi))) for q in p.outputs[len(p.outputs) - k:]]
    return Pattern(list(p.inputs), list(p.outputs[:len(p.outputs) - k]), list(p.cmds) + tail, p.name)


def random_general_pattern(seed: int, n_in: int = 2, n_total: int = 9, n_out: int = 2,
                           max_live: int = 7, p_corr: float = 0.3) -> Pattern:
    """A random pattern that obeys D0-D3 but is neither standard-form nor
    deterministic: interleaved N / E / M / X / Z commands with random signal domains over the
    qubits measured so far. Used to drive every branch of the scheduler (grow, shrink, pending
    E's and Z's, corrections on fresh qubits) against the oracle."""
    rng = np.random.default_rng(seed)
    qubits = list(range(n_total))
    outputs = [int(q) for q in rng.choice(qubits, size=n_out, replace=False)]
    inputs = list(range(n_in))
    prepared = set(inputs)
    measured: list = []
    edges = set()
    cmds: List[Cmd] = []

    def dom():
        if not measured or rng.uniform() < 0.4:
            return ()
        k = int(rng.integers(1, min(3, len(measured)) + 1))
        return tuple(int(x) for x in rng.choice(measured, size=k, replace=False))

    to_measure = [q for q in qubits if q not in outputs]
    guard = 0
    while to_measure and guard < 10000:
        guard += 1
        live = [q for q in prepared if q not in measured]
        unprep = [q for q in qubits if q not in prepared]
        r = rng.uniform()
        if r < 0.25 and unprep and len(live) < max_live:
            q = int(rng.choice(unprep))
            cmds.append(N(q))
            prepared.add(q)
        elif r < 0.55 and len(live) + (1 if unprep else 0) >= 2:
            pool = live + ([int(rng.choice(unprep))] if unprep and len(live) < max_live else [])
            if len(pool) < 2:
                continue
            a, b = (int(x) for x in rng.choice(pool, size=2, replace=False))
            key = (min(a, b), max(a, b))
            if key in edges:
                continue
            edges.add(key)
            cmds.append(E(a, b))
            prepared.update((a, b))
        elif r < 0.55 + p_corr * 0.5 and live:
            q = int(rng.choice(live))
            d = dom()
            if d:
                cmds.append((X if rng.uniform() < 0.5 else Z)(q, d))
        else:
            cand = [q for q in live if q in to_measure]
            if not cand:
                continue
            q = int(rng.choice(cand))
            cmds.append(M(q, float(rng.uniform(0, 2 * math.pi)), dom(), dom()))
            measured.append(q)
            to_measure.remove(q)
    # remaining non-outputs that were never prepared: prepare + measure
    for q in to_measure:
        cmds.append(M(q, float(rng.uniform(0, 2 * math.pi))))
        measured.append(q)
    live_out = [q for q in outputs]
    for q in live_out:
        d = dom()
        if d and rng.uniform() < 0.5:
            cmds.append((X if rng.uniform() < 0.5 else Z)(q, d))
    return Pattern(inputs, outputs, cmds, f"random{seed}")


def wide_random_pattern(seed: int, n_in: int = 16, width_hi: int = 20, rounds: int = 4,
                        n_out: int = 12) -> Pattern:
    """A grow/shrink-heavy random pattern (rules D0-D3) at tile-engine widths: each round prepares
    fresh qubits E-joined to two live qubits each (the state grows: GROW), entangles random live
    pairs, then measures live qubits whose neighbours are all live (no fresh partner to absorb them:
    SHRINK with the full (n0, n1, c) reduction of Eq. 13), with random angles, random s/t domains
    over earlier outcomes and random X/Z corrections. Parity-test workload for the paths the
    brickwork / cluster configs never take."""
    rng = np.random.default_rng(seed)
    live = list(range(n_in))
    nxt = n_in
    measured: List[int] = []
    edges = set()
    cmds: List[Cmd] = []
    outputs: List[int] = []

    def dom():
        if not measured or rng.uniform() < 0.3:
            return ()
        k = int(rng.integers(1, min(3, len(measured)) + 1))
        return tuple(int(x) for x in rng.choice(measured, size=k, replace=False))

    def edge(a, b):
        key = (min(a, b), max(a, b))
        if a != b and key not in edges:
            edges.add(key)
            cmds.append(E(a, b))

    for r in range(rounds):
        while len(live) < width_hi:
            q = nxt
            nxt += 1
            cmds.append(N(q))
            for a in rng.choice(live, size=2, replace=False):
                edge(int(a), q)
            live.append(q)
        for _ in range(width_hi // 2):
            a, b = (int(x) for x in rng.choice(live, size=2, replace=False))
            edge(a, b)
        for q in rng.choice(live, size=3, replace=False):
            d = dom()
            if d:
                cmds.append((X if rng.uniform() < 0.5 else Z)(int(q), d))
        last = r == rounds - 1
        k = len(live) - n_out if last else int(rng.integers(3, 6))
        cand = [q for q in live if q not in outputs]
        for q in rng.choice(cand, size=k, replace=False):
            q = int(q)
            cmds.append(M(q, float(rng.uniform(0, 2 * math.pi)), sdom=dom(), tdom=dom()))
            measured.append(q)
            live.remove(q)
    outputs = list(live)
    return Pattern(list(range(n_in)), outputs, cmds, f"WR:{seed}:{n_in}:{width_hi}")
