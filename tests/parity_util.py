"""Parity helpers shared by the GPU tests: GPU (C-ABI) vs oracle on the same seeded inputs.

Tolerances (BASELINE.json north_star): complex128 max|d amp| <= 1e-10, |d prob| <= 1e-12;
complex64 max|d amp| <= 1e-4 and 1 - fidelity <= 1e-5. Outcome strings must be identical except
at knife edges |u - prob0| < tau (tau = 1e-9 fp64, 1e-4 fp32; reading R-5), where the oracle
is replayed with the GPU's outcome.
"""
from __future__ import annotations

import numpy as np

import oracle

TOL = {128: dict(amp=1e-10, prob=1e-12, tau=1e-9, fid=1e-12), 64: dict(amp=1e-4, prob=1e-6, tau=1e-4, fid=1e-5)}


def fidelity(a, b):
    na, nb = np.linalg.norm(a), np.linalg.norm(b)
    return abs(np.vdot(a, b)) ** 2 / (na * na * nb * nb)


def joint(prob0, outcomes):
    return float(np.prod([p if s == 0 else 1 - p for p, s in zip(prob0, outcomes)]))


def gpu_run(sim, pattern, psi, mode, seed=0, forced=None):
    sim.load(pattern)
    sim.set_input(psi)
    outc, p0 = sim.run(mode, seed=seed, forced=forced)
    return sim.get_output(), outc, p0


def check(sim, pattern, psi, mode, seed=0, forced=None, same_order=None):
    """Run both sides and assert parity; returns (gpu_out, oracle_result)."""
    prec = sim.precision
    tol = TOL[prec]
    out, outc, p0 = gpu_run(sim, pattern, psi, mode, seed, forced)
    if mode == "eowqs":
        ref = oracle.run(pattern, psi, mode="eowqs")
    elif mode == "forced":
        ref = oracle.run(pattern, psi, mode="forced", forced=forced)
    else:
        ref = oracle.run(pattern, psi, mode="sampled", seed=seed)
        if list(outc) != list(ref.outcomes):
            # every disagreement must be a knife edge, or a legitimately reordered plan of a
            # non-deterministic pattern (R-8); replay the oracle on the GPU branch
            diff = [k for k in range(len(outc)) if outc[k] != ref.outcomes[k]]
            k = diff[0]
            u = oracle.draw_uniform(seed, k)
            knife = abs(u - ref.prob0[k]) < tol["tau"]
            assert knife or same_order is False, f"outcome {k} differs, u={u}, p0={ref.prob0[k]}"
            ref = oracle.run(pattern, psi, mode="forced", forced=outc)
    if mode != "eowqs" and len(p0):
        if same_order is not False:
            assert np.max(np.abs(p0 - ref.prob0)) <= tol["prob"], np.max(np.abs(p0 - ref.prob0))
        assert abs(joint(p0, outc) - joint(ref.prob0, ref.outcomes)) <= max(tol["prob"], 1e-12) * 10
    err = np.max(np.abs(out - ref.output))
    assert err <= tol["amp"], f"max |d amp| = {err}"
    if prec == 64:
        assert 1 - fidelity(out, ref.output) <= tol["fid"]
    return out, ref
