"""ctypes declarations of include/owqs.h (argument marshalling only; no computation here)."""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libowqs.so")

OWQS_OK = 0
STATUS_NAMES = {0: "OWQS_OK", 1: "OWQS_E_ARG", 2: "OWQS_E_PATTERN", 3: "OWQS_E_NO_GFLOW", 4: "OWQS_E_BRANCH",
                5: "OWQS_E_STATE", 6: "OWQS_E_NOMEM", 7: "OWQS_E_CUDA", 8: "OWQS_E_NCCL",
                9: "OWQS_E_NOT_DETERMINISTIC"}
MODES = {"sampled": 0, "forced": 1, "eowqs": 2}
FLAG_NO_GRAPH, FLAG_NO_FUSE, FLAG_GIVEN_ORDER, FLAG_NO_TUNE, FLAG_PROFILE, FLAG_LOOPBACK = 1, 2, 4, 8, 16, 32
FLAG_NO_GFLOW = 64
FLAG_NO_JIT = 128
FLAG_ONE_STATE = 256  # keep a disconnected pattern in one state vector (no sub-states)
FLAG_MEASURED_NORM = 512  # structural decisions from a reduced ||psi||^2 instead of 1 (DESIGN R-13)
KCLASS_NAMES = {0: "pass", 1: "small_pass", 2: "grow", 3: "shrink", 4: "reduce", 5: "swap", 6: "rhok",
                7: "shrinkk"}

# every symbol include/owqs.h declares (checked by tests/test_capi_symbols.py)
EXPORTED = ["owqs_create", "owqs_destroy", "owqs_load_pattern", "owqs_set_input", "owqs_set_input_host",
            "owqs_get_output_host", "owqs_set_input_device",
            "owqs_set_input_random", "owqs_run", "owqs_submit_host", "owqs_wait", "owqs_run_batch", "owqs_get_output", "owqs_get_output_device",
            "owqs_get_output_sample",
            "owqs_output_inner", "owqs_output_norm", "owqs_nccl_unique_id", "owqs_recognize", "owqs_recognize_choi",
            "owqs_pattern_info", "owqs_plan_order", "owqs_gflow",
            "owqs_set_proa_weights", "owqs_stats", "owqs_launch_profile", "owqs_last_error", "owqs_version"]


class owqs_cmd(C.Structure):
    _fields_ = [("kind", C.c_int32), ("q0", C.c_int32), ("q1", C.c_int32),
                ("s_off", C.c_int32), ("s_len", C.c_int32), ("t_off", C.c_int32), ("t_len", C.c_int32),
                ("reserved", C.c_int32), ("angle", C.c_double)]


class owqs_config(C.Structure):
    _fields_ = [("precision", C.c_int32), ("n_ranks", C.c_int32), ("rank", C.c_int32), ("device", C.c_int32),
                ("nccl_id", C.c_void_p), ("flags", C.c_uint32), ("reserved", C.c_int32), ("stream", C.c_void_p)]


class owqs_stats_t(C.Structure):
    _fields_ = [("n_commands", C.c_int64), ("n_measure", C.c_int64), ("paper_m", C.c_int32),
                ("phys_bits", C.c_int32), ("n_passes", C.c_int32), ("n_grow", C.c_int32),
                ("n_shrink", C.c_int32), ("n_reduce", C.c_int32), ("n_launches", C.c_int32),
                ("n_swaps", C.c_int32), ("bytes_per_run", C.c_double), ("last_run_ms", C.c_double),
                ("schedule_ms", C.c_double), ("jit_ms", C.c_double), ("n_jit_steps", C.c_double),
                ("n_kernels", C.c_double), ("n_substates", C.c_double)]


assert C.sizeof(owqs_cmd) == 40


def load_library(path: str = LIB_PATH) -> C.CDLL:
    if not os.path.exists(path):
        raise ImportError(f"libowqs.so not built ({path}); run __graft_entry__.build() or "
                          "python -m paper_1604_05659_b200._build — there is no CPU fallback")
    lib = C.CDLL(path)
    P = C.POINTER
    ctx = C.c_void_p
    sig = {
        "owqs_create": (C.c_int, [P(owqs_config), P(ctx)]),
        "owqs_destroy": (None, [ctx]),
        "owqs_load_pattern": (C.c_int, [ctx, P(C.c_int32), C.c_int32, P(C.c_int32), C.c_int32, P(owqs_cmd),
                                        C.c_int64, P(C.c_int32), C.c_int64]),
        "owqs_set_input": (C.c_int, [ctx, P(C.c_double), C.c_int64]),
        "owqs_set_input_device": (C.c_int, [ctx, C.c_void_p, C.c_int32, C.c_int64]),
        "owqs_set_input_host": (C.c_int, [ctx, C.c_void_p, C.c_int32, C.c_int64]),
        "owqs_get_output_host": (C.c_int, [ctx, C.c_void_p, C.c_int32, C.c_int64]),
        "owqs_set_input_random": (C.c_int, [ctx, C.c_uint64]),
        "owqs_run": (C.c_int, [ctx, C.c_int, C.c_uint64, P(C.c_uint8), P(C.c_uint8), P(C.c_double)]),
        "owqs_get_output": (C.c_int, [ctx, P(C.c_double), C.c_int64]),
        "owqs_submit_host": (C.c_int, [ctx, C.c_int, C.c_uint64, P(C.c_uint8), C.c_void_p, C.c_int32, C.c_int64,
                                       C.c_void_p, C.c_int32, C.c_int64]),
        "owqs_wait": (C.c_int, [ctx, P(C.c_uint8), P(C.c_double)]),
        "owqs_run_batch": (C.c_int, [ctx, C.c_int, C.c_int64, P(C.c_double), P(C.c_uint64), P(C.c_uint8),
                                     P(C.c_double), P(C.c_uint8), P(C.c_double)]),
        "owqs_get_output_device": (C.c_int, [ctx, C.c_void_p, C.c_int32, C.c_int64]),
        "owqs_get_output_sample": (C.c_int, [ctx, C.POINTER(C.c_int64), C.c_int64, C.POINTER(C.c_double)]),
        "owqs_output_inner": (C.c_int, [ctx, ctx, P(C.c_double), P(C.c_double)]),
        "owqs_output_norm": (C.c_int, [ctx, P(C.c_double)]),
        "owqs_nccl_unique_id": (C.c_int, [C.c_void_p]),
        "owqs_recognize": (C.c_int, [ctx, P(C.c_double), C.c_int64, P(C.c_double)]),
        "owqs_recognize_choi": (C.c_int, [ctx, P(C.c_double), C.c_int64, P(C.c_double)]),
        "owqs_pattern_info": (C.c_int, [ctx, P(C.c_int64), P(C.c_int32), P(C.c_int32), P(C.c_int32)]),
        "owqs_gflow": (C.c_int, [ctx, P(C.c_int32), P(C.c_int32)]),
        "owqs_plan_order": (C.c_int, [ctx, C.c_int, P(C.c_int32), P(C.c_int32), C.c_int64]),
        "owqs_set_proa_weights": (C.c_int, [ctx, C.c_double, C.c_double, C.c_double, C.c_double, C.c_int32]),
        "owqs_stats": (C.c_int, [ctx, P(owqs_stats_t)]),
        "owqs_launch_profile": (C.c_int, [ctx, P(C.c_int32), P(C.c_double), P(C.c_float), C.c_int64]),
        "owqs_last_error": (C.c_char_p, [ctx]),
        "owqs_version": (C.c_char_p, []),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return declare_host(lib)


# ---- include/owqs_host.h (host-only introspection; no CUDA calls) ------------------------------
HOST_EXPORTED = ["owqs_host_compile", "owqs_host_info_get", "owqs_host_program", "owqs_host_gflow",
                 "owqs_host_jit", "owqs_host_jit_source", "owqs_host_nvrtc_version", "owqs_host_substates", "owqs_host_standardize", "owqs_host_error",
                 "owqs_host_free"]
KMAX_HI, MAX_OPS, MAX_BFLY = 8, 128, 64


class Op(C.Structure):
    _fields_ = [("type", C.c_uint8), ("a", C.c_uint8), ("b", C.c_uint8), ("cond", C.c_uint8),
                ("sig_off", C.c_int32), ("sig_len", C.c_int32), ("m", C.c_int32)]


class StepDesc(C.Structure):
    _fields_ = [("kind", C.c_int32), ("width", C.c_int32), ("nb_hi", C.c_int32), ("bhi", C.c_int32 * KMAX_HI),
                ("n_ops", C.c_int32), ("red_kind", C.c_int32), ("red_slot", C.c_int32), ("slot", C.c_int32),
                ("shrink_m", C.c_int32), ("n_bfly", C.c_int32), ("first_uses_red", C.c_int32),
                ("first_full_rho", C.c_int32), ("pad", C.c_int32), ("ops", Op * MAX_OPS),
                ("absorb", C.c_uint64 * MAX_BFLY), ("swap_local", C.c_int32), ("swap_global", C.c_int32),
                ("n_remap", C.c_int32), ("remap_a", C.c_int32 * 6), ("remap_b", C.c_int32 * 6),
                ("jk", C.c_int32), ("jm_pos", C.c_int32 * 4), ("jm", C.c_int32 * 4), ("j_src", C.c_int8 * 64)]


class MStatic(C.Structure):
    _fields_ = [("alpha", C.c_double), ("ord", C.c_int32), ("s_off", C.c_int32), ("s_len", C.c_int32),
                ("t_off", C.c_int32), ("t_len", C.c_int32), ("reuse", C.c_int32), ("structural", C.c_int32),
                ("key", C.c_int32)]


class owqs_host_info(C.Structure):
    _fields_ = [("n_steps", C.c_int64), ("n_measure", C.c_int64), ("sig_len", C.c_int64),
                ("paper_m", C.c_int32), ("phys_bits", C.c_int32), ("in_width", C.c_int32), ("n_out", C.c_int32),
                ("step_bytes", C.c_int32), ("mstatic_bytes", C.c_int32), ("n_passes", C.c_int32),
                ("n_grow", C.c_int32), ("n_shrink", C.c_int32), ("n_reduce", C.c_int32),
                ("n_swaps", C.c_int32), ("n_global", C.c_int32), ("bytes_per_run", C.c_double)]


def declare_host(lib: C.CDLL) -> C.CDLL:
    P = C.POINTER
    h = C.c_void_p
    sig = {
        "owqs_host_compile": (C.c_int, [P(C.c_int32), C.c_int32, P(C.c_int32), C.c_int32, P(owqs_cmd), C.c_int64,
                                        P(C.c_int32), C.c_int64, C.c_int32, C.c_int32, C.c_uint32,
                                        P(C.c_double), C.c_int32, P(h)]),
        "owqs_host_info_get": (C.c_int, [h, P(owqs_host_info)]),
        "owqs_host_program": (C.c_int, [h, C.c_void_p, C.c_void_p, P(C.c_int32), P(C.c_int32), P(C.c_int32),
                                        P(C.c_int32)]),
        "owqs_host_gflow": (C.c_int, [h, P(C.c_int32), P(C.c_int32)]),
        "owqs_host_jit": (C.c_int, [h, P(C.c_int64), P(C.c_int64), P(C.c_double)]),
        "owqs_host_jit_source": (C.c_int, [h, C.c_int64, C.c_char_p, C.c_int64, P(C.c_int64)]),
        "owqs_host_nvrtc_version": (C.c_int, [P(C.c_int32), P(C.c_int32)]),
        "owqs_host_substates": (C.c_int, [h, P(C.c_int32), P(C.c_uint64), P(C.c_int32), C.c_int32]),
        "owqs_host_standardize": (C.c_int, [h, C.c_int32, P(owqs_cmd), P(C.c_int32), P(C.c_int32), P(C.c_int32),
                                            P(C.c_int64)]),
        "owqs_host_error": (C.c_char_p, [h]),
        "owqs_host_free": (None, [h]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib
