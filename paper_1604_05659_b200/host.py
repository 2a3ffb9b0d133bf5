"""Binding of include/owqs_host.h: the scheduler's output (PROA plan, compiled step program) without a
GPU. Marshalling only; the scheduler itself is C++ inside libowqs.so."""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import List, Optional, Sequence

from . import _capi
from .owqs import OwqsError, lib, marshal_pattern

MODE_IDS = _capi.MODES


@dataclass
class HostProgram:
    info: dict
    steps: List[_capi.StepDesc]
    mst: List[_capi.MStatic]
    sig: List[int]
    out_slot: List[int]
    plan_qubits: List[int]
    plan_ms: List[int]


def host_gflow(pattern):
    """(has_gflow, layers per M in given order, depth) of the pattern's open graph (no GPU)."""
    L = lib()
    i, o, arr, pool, plen = marshal_pattern(pattern.inputs, pattern.outputs, pattern.cmds)
    h = C.c_void_p()
    st = L.owqs_host_compile(i, len(pattern.inputs), o, len(pattern.outputs), arr, len(pattern.cmds), pool, plen,
                             2, 128, 0, None, 1, C.byref(h))
    try:
        if st != 0:
            msg = L.owqs_host_error(h) if h else b""
            raise OwqsError(st, msg.decode() if msg else "")
        K = pattern.n_measure
        layers = (C.c_int32 * max(1, K))()
        depth = C.c_int32()
        st = L.owqs_host_gflow(h, layers, C.byref(depth))
        return st == 0, list(layers)[:K], depth.value
    finally:
        if h:
            L.owqs_host_free(h)


def _host_handle(pattern, mode, precision, flags, weights, n_ranks):
    L = lib()
    i, o, arr, pool, plen = marshal_pattern(pattern.inputs, pattern.outputs, pattern.cmds)
    w = (C.c_double * 4)(*weights) if weights is not None else None
    h = C.c_void_p()
    st = L.owqs_host_compile(i, len(pattern.inputs), o, len(pattern.outputs), arr, len(pattern.cmds), pool, plen,
                             MODE_IDS[mode], precision, flags, w, n_ranks, C.byref(h))
    if st != 0:
        msg = L.owqs_host_error(h) if h else b""
        if h:
            L.owqs_host_free(h)
        raise OwqsError(st, msg.decode() if msg else "")
    return L, h


def substates(pattern, mode: str = "sampled", precision: int = 64, flags: int = 0):
    """Sub-states the pattern runs as (PAPER §4.1; owqs_host_substates): a list of
    (output_mask, phys_bits) per component, or [] when it stays one state vector."""
    L, h = _host_handle(pattern, mode, precision, flags, None, 1)
    try:
        n = C.c_int32(0)
        if L.owqs_host_substates(h, C.byref(n), None, None, 0) != 0:
            raise OwqsError(1, "owqs_host_substates")
        if n.value <= 1:
            return []
        masks = (C.c_uint64 * n.value)()
        bits = (C.c_int32 * n.value)()
        st = L.owqs_host_substates(h, C.byref(n), masks, bits, n.value)
        if st != 0:
            raise OwqsError(st, "owqs_host_substates")
        return [(int(masks[c]), int(bits[c])) for c in range(n.value)]
    finally:
        L.owqs_host_free(h)


def nvrtc_version():
    """(major, minor) of the NVRTC the pass-kernel generator compiles with (the build's CUDA
    toolkit, loaded by path; include/owqs_host.h owqs_host_nvrtc_version)."""
    a, b = C.c_int32(0), C.c_int32(0)
    st = lib().owqs_host_nvrtc_version(C.byref(a), C.byref(b))
    if st != 0:
        raise OwqsError(st, "NVRTC could not be loaded")
    return a.value, b.value


def jit_host(pattern, mode: str = "sampled", precision: int = 64, flags: int = 0,
             weights: Optional[Sequence[float]] = None, n_ranks: int = 1, sources: bool = False) -> dict:
    """NVRTC-compile the generated pass kernels of the compiled program (no GPU needed).
    Returns {n_kernels, n_jit_steps, compile_ms[, sources: {step: text}]}."""
    L, h = _host_handle(pattern, mode, precision, flags, weights, n_ranks)
    try:
        nk, ns, ms = C.c_int64(), C.c_int64(), C.c_double()
        st = L.owqs_host_jit(h, C.byref(nk), C.byref(ns), C.byref(ms))
        if st != 0:
            raise OwqsError(st, L.owqs_host_error(h).decode())
        out = {"n_kernels": nk.value, "n_jit_steps": ns.value, "compile_ms": ms.value}
        if sources:
            info = _capi.owqs_host_info()
            L.owqs_host_info_get(h, C.byref(info))
            srcs = {}
            for k in range(-1, info.n_steps):
                n = C.c_int64()
                L.owqs_host_jit_source(h, k, None, 0, C.byref(n))
                if n.value:
                    buf = C.create_string_buffer(n.value + 1)
                    L.owqs_host_jit_source(h, k, buf, n.value + 1, C.byref(n))
                    srcs[k] = buf.value.decode()
            out["sources"] = srcs
        return out
    finally:
        L.owqs_host_free(h)


def standardize(pattern, signal_shift: bool = False):
    """Standard form N* E* M* C* of a pattern (owqs_host_standardize).
    Returns (Pattern, shifts): shifts maps a measured qubit to its removed t-domain T (signal
    shifting: s_v(new) = s_v(old) + |T_v| over the new labels), empty without signal_shift."""
    from workloads.patterns import Cmd, Pattern
    L, h = _host_handle(pattern, "sampled", 128, 0, None, 1)
    try:
        sizes = (C.c_int64 * 4)()
        st = L.owqs_host_standardize(h, int(signal_shift), None, None, None, None, sizes)
        if st != 0:
            raise OwqsError(st, L.owqs_host_error(h).decode())
        n, plen, slen = sizes[0], sizes[1], sizes[2]
        cmds = (_capi.owqs_cmd * max(1, n))()
        pool = (C.c_int32 * max(1, plen))()
        sl = (C.c_int32 * max(2, 2 * n))()
        sp = (C.c_int32 * max(1, slen))()
        L.owqs_host_standardize(h, int(signal_shift), cmds, pool, sl, sp, sizes)
        out, shifts = [], {}
        for k in range(n):
            c = cmds[k]
            sd = tuple(pool[c.s_off + j] for j in range(c.s_len))
            td = tuple(pool[c.t_off + j] for j in range(c.t_len))
            out.append(Cmd(c.kind, c.q0, c.q1 if c.kind == 1 else -1, c.angle, sd, td))
            if sl[2 * k + 1]:
                shifts[c.q0] = tuple(sp[sl[2 * k] + j] for j in range(sl[2 * k + 1]))
        return Pattern(list(pattern.inputs), list(pattern.outputs), out, (pattern.name or "") + ":std"), shifts
    finally:
        L.owqs_host_free(h)


def compile_host(pattern, mode: str = "sampled", precision: int = 128, flags: int = 0,
                 weights: Optional[Sequence[float]] = None, n_ranks: int = 1) -> HostProgram:
    L = lib()
    i, o, arr, pool, plen = marshal_pattern(pattern.inputs, pattern.outputs, pattern.cmds)
    w = (C.c_double * 4)(*weights) if weights is not None else None
    h = C.c_void_p()
    st = L.owqs_host_compile(i, len(pattern.inputs), o, len(pattern.outputs), arr, len(pattern.cmds), pool, plen,
                             MODE_IDS[mode], precision, flags, w, n_ranks, C.byref(h))
    try:
        if st != 0:
            msg = L.owqs_host_error(h) if h else b""
            raise OwqsError(st, msg.decode() if msg else "")
        info = _capi.owqs_host_info()
        L.owqs_host_info_get(h, C.byref(info))
        assert info.step_bytes == C.sizeof(_capi.StepDesc), "StepDesc layout mismatch"
        assert info.mstatic_bytes == C.sizeof(_capi.MStatic), "MStatic layout mismatch"
        steps = (_capi.StepDesc * max(1, info.n_steps))()
        mst = (_capi.MStatic * max(1, info.n_measure))()
        sig = (C.c_int32 * max(1, info.sig_len))()
        out_slot = (C.c_int32 * max(1, info.n_out))()
        pq = (C.c_int32 * max(1, info.n_measure))()
        pm = (C.c_int32 * max(1, info.n_measure))()
        L.owqs_host_program(h, steps, mst, sig, out_slot, pq, pm)
        d = {k: getattr(info, k) for k, _ in _capi.owqs_host_info._fields_}
        K = info.n_measure
        return HostProgram(d, list(steps)[:info.n_steps], list(mst)[:K], list(sig)[:info.sig_len],
                           list(out_slot)[:info.n_out], list(pq)[:K], list(pm)[:K])
    finally:
        if h:
            L.owqs_host_free(h)
