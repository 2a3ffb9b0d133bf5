"""Thin Python binding of libowqs.so (include/owqs.h). Marshalling only: every step of the hot path
runs in the library's sm_100a kernels; there is no CPU fallback."""
from __future__ import annotations

import ctypes as C
from typing import Optional, Sequence, Tuple

import numpy as np

from . import _capi
from ._capi import MODES, STATUS_NAMES, owqs_cmd, owqs_config, owqs_stats_t

_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        _lib = _capi.load_library()
    return _lib


class OwqsError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status
        self.status_name = STATUS_NAMES.get(status, str(status))


def _i32(a: Sequence[int]):
    arr = (C.c_int32 * max(1, len(a)))(*a)
    return arr


def marshal_pattern(inputs, outputs, cmds):
    """cmds: objects with kind, q0, q1, angle, sdom, tdom (workloads.patterns.Cmd or alike)."""
    pool = []
    arr = (owqs_cmd * max(1, len(cmds)))()
    for i, c in enumerate(cmds):
        x = arr[i]
        x.kind, x.q0, x.q1 = int(c.kind), int(c.q0), int(c.q1)
        x.angle = float(c.angle)
        sd, td = tuple(getattr(c, "sdom", ()) or ()), tuple(getattr(c, "tdom", ()) or ())
        x.s_off, x.s_len = len(pool), len(sd)
        pool += [int(v) for v in sd]
        x.t_off, x.t_len = len(pool), len(td)
        pool += [int(v) for v in td]
    return _i32(inputs), _i32(outputs), arr, _i32(pool), len(pool)


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    st = lib().owqs_nccl_unique_id(buf)
    if st != 0:
        raise OwqsError(st, "ncclGetUniqueId failed")
    return buf.raw


class Simulator:
    """One owqs context (one GPU or one rank's shard, one pattern at a time)."""

    def __init__(self, precision: int = 128, device: int = 0, flags: int = 0, stream: Optional[int] = None,
                 n_ranks: int = 1, rank: int = 0, nccl_id: Optional[bytes] = None):
        """n_ranks > 1: sharded state; with flags & FLAG_LOOPBACK all shards live on
        `device` (single-GPU testing), otherwise one process per GPU over NCCL with `nccl_id`
        (128 bytes from nccl_unique_id() on one rank, broadcast by the caller)."""
        self._lib = lib()
        cfg = owqs_config()
        cfg.precision = precision
        cfg.n_ranks, cfg.rank, cfg.device = n_ranks, rank, device
        cfg.flags = flags
        cfg.stream = stream
        self._id_buf = None
        if nccl_id is not None:
            self._id_buf = C.create_string_buffer(bytes(nccl_id), 128)
            cfg.nccl_id = C.cast(self._id_buf, C.c_void_p)
        h = C.c_void_p()
        st = self._lib.owqs_create(C.byref(cfg), C.byref(h))
        if st != 0:
            why = self._lib.owqs_last_error(None)
            raise OwqsError(st, "owqs_create failed (CUDA device visible? NCCL id / rank valid?) " +
                            (why.decode() if why else ""))
        self.n_ranks, self.rank = n_ranks, rank
        self._h = h
        self.precision = precision
        self.n_in = self.n_out = 0
        self.n_measure = 0

    def close(self):
        if getattr(self, "_h", None):
            self._lib.owqs_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, st: int):
        if st != 0:
            msg = self._lib.owqs_last_error(self._h)
            raise OwqsError(st, msg.decode() if msg else "")

    # -- boundary calls ------------------------------------------------------------------------
    def load_pattern(self, inputs, outputs, cmds):
        i, o, arr, pool, plen = marshal_pattern(inputs, outputs, cmds)
        self._check(self._lib.owqs_load_pattern(self._h, i, len(inputs), o, len(outputs), arr, len(cmds), pool, plen))
        self.n_in, self.n_out = len(inputs), len(outputs)
        nm = C.c_int64()
        self._check(self._lib.owqs_pattern_info(self._h, C.byref(nm), None, None, None))
        self.n_measure = nm.value

    def load(self, pattern):
        self.load_pattern(pattern.inputs, pattern.outputs, pattern.cmds)

    def set_input(self, amps: np.ndarray):
        """Host input; complex64 arrays are passed as is (owqs_set_input_host, precision 64: half the
        PCIe bytes on a complex64 context), anything else as complex128."""
        if isinstance(amps, np.ndarray) and amps.dtype == np.complex64 and amps.flags.c_contiguous:
            self._check(self._lib.owqs_set_input_host(self._h, C.c_void_p(amps.ctypes.data), 64, amps.size))
            return
        a = np.ascontiguousarray(amps, dtype=np.complex128)
        self._check(self._lib.owqs_set_input(self._h, a.ctypes.data_as(C.POINTER(C.c_double)), a.size))

    def set_input_device(self, ptr: int, precision: int, n: int):
        self._check(self._lib.owqs_set_input_device(self._h, C.c_void_p(ptr), precision, n))

    def set_input_random(self, seed: int):
        self._check(self._lib.owqs_set_input_random(self._h, C.c_uint64(seed)))

    def run(self, mode: str = "sampled", seed: int = 0, forced: Optional[Sequence[int]] = None,
            want: bool = True) -> Tuple[Optional[np.ndarray], Optional[np.ndarray]]:
        K = self.n_measure
        f = None
        if forced is not None:
            fa = np.ascontiguousarray(np.asarray(forced, dtype=np.uint8))
            if fa.size != K:
                raise ValueError("forced must have one entry per M")
            f = fa.ctypes.data_as(C.POINTER(C.c_uint8))
        out = np.zeros(max(K, 1), dtype=np.uint8) if want else None
        p0 = np.zeros(max(K, 1), dtype=np.float64) if want else None
        st = self._lib.owqs_run(self._h, MODES[mode], C.c_uint64(seed & (2 ** 64 - 1)), f,
                                out.ctypes.data_as(C.POINTER(C.c_uint8)) if want else None,
                                p0.ctypes.data_as(C.POINTER(C.c_double)) if want else None)
        self._check(st)
        return (out[:K], p0[:K]) if want else (None, None)

    def submit_host(self, in_ptr: int, in_precision: int, out_ptr: int, out_precision: int,
                    mode: str = "sampled", seed: int = 0, forced: Optional[Sequence[int]] = None):
        """owqs_submit_host: enqueue input copy + run + output copy between PAGE-LOCKED host buffers
        (raw addresses, e.g. torch.empty(..., pin_memory=True).data_ptr()) and return at once;
        complete with wait(). in/out hold 2^n_in / 2^n_out amplitudes at precision 64 or 128."""
        f = None
        self._forced_keep = None
        if forced is not None:
            fa = np.ascontiguousarray(np.asarray(forced, dtype=np.uint8))
            if fa.size != self.n_measure:
                raise ValueError("forced must have one entry per M")
            self._forced_keep = fa
            f = fa.ctypes.data_as(C.POINTER(C.c_uint8))
        self._check(self._lib.owqs_submit_host(self._h, MODES[mode], C.c_uint64(seed & (2 ** 64 - 1)), f,
                                               C.c_void_p(in_ptr), in_precision, 2 ** self.n_in,
                                               C.c_void_p(out_ptr), out_precision, 2 ** self.n_out))

    def wait(self, want: bool = False) -> Tuple[Optional[np.ndarray], Optional[np.ndarray]]:
        """owqs_wait: complete the submitted run; (outcomes, prob0) when want."""
        K = self.n_measure
        out = np.zeros(max(K, 1), dtype=np.uint8) if want else None
        p0 = np.zeros(max(K, 1), dtype=np.float64) if want else None
        st = self._lib.owqs_wait(self._h, out.ctypes.data_as(C.POINTER(C.c_uint8)) if want else None,
                                 p0.ctypes.data_as(C.POINTER(C.c_double)) if want else None)
        self._forced_keep = None
        self._check(st)
        return (out[:K], p0[:K]) if want else (None, None)

    def run_batch(self, inputs: np.ndarray, mode: str = "sampled", seeds: Optional[Sequence[int]] = None,
                  forced: Optional[np.ndarray] = None):
        """Batched replicas: inputs [B, 2^n_in] -> (outputs [B, 2^n_out], outcomes [B, K], prob0 [B, K])."""
        x = np.ascontiguousarray(inputs, dtype=np.complex128)
        B = x.shape[0]
        K = self.n_measure
        out = np.empty((B, 2 ** self.n_out), dtype=np.complex128)
        oc = np.zeros((B, max(K, 1)), dtype=np.uint8)
        p0 = np.zeros((B, max(K, 1)), dtype=np.float64)
        sd = None
        if seeds is not None:
            sa = np.ascontiguousarray(np.asarray(seeds, dtype=np.uint64))
            sd = sa.ctypes.data_as(C.POINTER(C.c_uint64))
        fd = None
        if forced is not None:
            fa = np.ascontiguousarray(np.asarray(forced, dtype=np.uint8).reshape(B, K))
            fd = fa.ctypes.data_as(C.POINTER(C.c_uint8))
        self._check(self._lib.owqs_run_batch(self._h, MODES[mode], B, x.ctypes.data_as(C.POINTER(C.c_double)), sd, fd,
                                             out.ctypes.data_as(C.POINTER(C.c_double)),
                                             oc.ctypes.data_as(C.POINTER(C.c_uint8)),
                                             p0.ctypes.data_as(C.POINTER(C.c_double))))
        return out, oc[:, :K], p0[:, :K]

    def get_output(self, out: Optional[np.ndarray] = None) -> Optional[np.ndarray]:
        """Full output (rank 0 / single rank / loopback); None on the other ranks (collective)."""
        root = self.n_ranks == 1 or self.rank == 0
        if out is None and root:
            out = np.empty(2 ** self.n_out, dtype=np.complex128)
        if root:
            assert out.dtype in (np.complex128, np.complex64) and out.flags.c_contiguous and out.size >= 2 ** self.n_out
            prec = 64 if out.dtype == np.complex64 else 128
            self._check(self._lib.owqs_get_output_host(self._h, C.c_void_p(out.ctypes.data), prec, out.size))
            return out
        self._check(self._lib.owqs_get_output(self._h, None, 0))
        return None

    def get_output_device(self, ptr: int, precision: int, n: int):
        self._check(self._lib.owqs_get_output_device(self._h, C.c_void_p(ptr), precision, n))

    def get_output_sample(self, idx) -> np.ndarray:
        """Output amplitudes at caller-order indices idx (owqs_get_output_sample; collective)."""
        idx = np.ascontiguousarray(idx, dtype=np.int64)
        out = np.zeros(idx.size, dtype=np.complex128)
        self._check(self._lib.owqs_get_output_sample(self._h, idx.ctypes.data_as(C.POINTER(C.c_int64)), idx.size,
                                                     out.ctypes.data_as(C.POINTER(C.c_double))))
        return out

    def norm2(self) -> float:
        v = C.c_double()
        self._check(self._lib.owqs_output_norm(self._h, C.byref(v)))
        return v.value

    def inner(self, other: "Simulator") -> complex:
        re, im = C.c_double(), C.c_double()
        self._check(self._lib.owqs_output_inner(self._h, other._h, C.byref(re), C.byref(im)))
        return complex(re.value, im.value)

    def recognize(self, choi: bool = False) -> Tuple[np.ndarray, float]:
        """(U, max unitarity error). choi=True: one run on the Choi state (owqs_recognize_choi)
        instead of one run per basis input."""
        U = np.empty((2 ** self.n_in, 2 ** self.n_out), dtype=np.complex128)  # column-major storage
        err = C.c_double()
        fn = self._lib.owqs_recognize_choi if choi else self._lib.owqs_recognize
        self._check(fn(self._h, U.ctypes.data_as(C.POINTER(C.c_double)), U.size, C.byref(err)))
        return U.T.copy(), err.value

    def gflow(self):
        """(has_gflow, layers per M in given order, depth) — L372's EOWQS pre-check."""
        K = self.n_measure
        layers = (C.c_int32 * max(1, K))()
        depth = C.c_int32()
        st = self._lib.owqs_gflow(self._h, layers, C.byref(depth))
        if st not in (0, 3):
            self._check(st)
        return st == 0, list(layers)[:K], depth.value

    def pattern_info(self) -> dict:
        nm, pm, pb, npass = C.c_int64(), C.c_int32(), C.c_int32(), C.c_int32()
        self._check(self._lib.owqs_pattern_info(self._h, C.byref(nm), C.byref(pm), C.byref(pb), C.byref(npass)))
        return {"n_measure": nm.value, "paper_m": pm.value, "phys_bits": pb.value, "n_passes": npass.value}

    def plan_order(self, mode: str = "sampled") -> Tuple[list, list]:
        K = self.n_measure
        q = (C.c_int32 * max(1, K))()
        ms = (C.c_int32 * max(1, K))()
        self._check(self._lib.owqs_plan_order(self._h, MODES[mode], q, ms, K))
        return list(q)[:K], list(ms)[:K]

    def set_proa_weights(self, a: float, b: float, g: float, d: float, tune: bool = True):
        self._check(self._lib.owqs_set_proa_weights(self._h, a, b, g, d, int(tune)))

    def launch_profile(self):
        """(kclass[n], bytes[n], ms[n]) of the last run of a context created with FLAG_PROFILE."""
        n = self.stats()["n_launches"]
        kc = np.zeros(max(n, 1), dtype=np.int32)
        by = np.zeros(max(n, 1), dtype=np.float64)
        ms = np.zeros(max(n, 1), dtype=np.float32)
        self._check(self._lib.owqs_launch_profile(self._h, kc.ctypes.data_as(C.POINTER(C.c_int32)),
                                                  by.ctypes.data_as(C.POINTER(C.c_double)),
                                                  ms.ctypes.data_as(C.POINTER(C.c_float)), n))
        return kc[:n], by[:n], ms[:n]

    def stats(self) -> dict:
        s = owqs_stats_t()
        self._check(self._lib.owqs_stats(self._h, C.byref(s)))
        return {k: getattr(s, k) for k, _ in owqs_stats_t._fields_ if k != "reserved"}
