"""TEST INFRASTRUCTURE ONLY — the CPU oracle for the OWQS/EOWQS hot path.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import this package. The product path (paper_1604_05659_b200) never imports it and shares
no code with it.
"""
from .owqs_oracle import (  # noqa: F401
    OracleError, OracleResult, run, recognize, draw_uniform, resolve_angle,
    P0_matrix, P1_matrix, plus_alpha, minus_alpha,
)
