"""B200-native OWQS/EOWQS array executor for one-way quantum computer patterns (arXiv:1604.05659).

The hot path lives in libowqs.so (sm_100a CUDA kernels + C++ scheduler) behind include/owqs.h;
this package is its thin Python binding. Importing it does not need a GPU; creating a
Simulator does, and fails loudly without one (there is no CPU fallback).
"""
from .owqs import Simulator, OwqsError, lib, marshal_pattern, nccl_unique_id  # noqa: F401
from ._capi import LIB_PATH, EXPORTED, FLAG_NO_GRAPH, FLAG_NO_FUSE, FLAG_GIVEN_ORDER, FLAG_NO_TUNE, FLAG_PROFILE, FLAG_LOOPBACK, FLAG_NO_GFLOW, FLAG_NO_JIT, FLAG_ONE_STATE, FLAG_MEASURED_NORM, KCLASS_NAMES  # noqa: F401

__version__ = "0.1.0"
