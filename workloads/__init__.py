"""Seeded synthetic workloads shared by the oracle tests, the GPU parity tests and bench.py.

This package holds NO arithmetic of the method (no state vectors, no measurement, no
probabilities). It only builds command lists (patterns) and seeded input amplitudes, so that
the oracle (`oracle/`) and the CUDA path (`paper_1604_05659_b200/`) can be driven with the
same inputs without sharing any code of the method itself.
"""
from .patterns import (  # noqa: F401
    Cmd, Pattern, N, E, M, X, Z,
    circuit_to_pattern, random_tiny_circuit, qft_circuit, brickwork_circuit,
    cluster_pattern, cnot_pattern_eq22, j_pattern, cz_pattern, linear_cluster_pattern,
    config_pattern,
)
from .inputs import haar_state, basis_state, plus_state, counter_haar_state  # noqa: F401
