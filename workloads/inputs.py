"""Seeded input states (no arithmetic of the method).

Amplitude index convention: bit k of the index is the value of inputs[k] (inputs[0] = LSB),
matching the paper's position-1-is-least-significant layout of Eq. 8.
Arrays are complex128 numpy vectors of length 2^n.
"""
from __future__ import annotations

import numpy as np

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def haar_state(n: int, seed: int) -> np.ndarray:
    """Haar-random pure state: i.i.d. complex Gaussian amplitudes, normalised (numpy PCG64)."""
    rng = np.random.default_rng(seed)
    v = rng.standard_normal(2 ** n) + 1j * rng.standard_normal(2 ** n)
    return v / np.linalg.norm(v)


def basis_state(n: int, k: int) -> np.ndarray:
    v = np.zeros(2 ** n, dtype=np.complex128)
    v[k] = 1.0
    return v


def plus_state(n: int) -> np.ndarray:
    return np.full(2 ** n, 2.0 ** (-n / 2), dtype=np.complex128)


def _splitmix64(x: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser on uint64 arrays (wrapping arithmetic)."""
    with np.errstate(over="ignore"):
        z = (x + np.uint64(0x9E3779B97F4A7C15)) & _M64
        z = ((z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)) & _M64
        z = ((z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)) & _M64
        return z ^ (z >> np.uint64(31))


def counter_haar_raw(seed: int, idx: np.ndarray) -> np.ndarray:
    """Unnormalised counter-based complex Gaussian for amplitude indices `idx`.

    Documented generator (the device generator behind owqs_set_input_random is the same
    recipe, written independently in CUDA): key = splitmix64(seed);
      a = splitmix64(key ^ splitmix64(2 j)),  b = splitmix64(key ^ splitmix64(2 j + 1))
      u1 = ((a >> 11) + 1) 2^-53 in (0, 1],   u2 = (b >> 11) 2^-53 in [0, 1)
      amp_j = sqrt(-2 ln u1) (cos 2 pi u2 + i sin 2 pi u2)            (Box-Muller)
    The state is amp / ||amp||.
    """
    idx = np.asarray(idx, dtype=np.uint64)
    key = _splitmix64(np.array([seed], dtype=np.uint64))[0]
    a = _splitmix64(key ^ _splitmix64(np.uint64(2) * idx))
    b = _splitmix64(key ^ _splitmix64(np.uint64(2) * idx + np.uint64(1)))
    u1 = ((a >> np.uint64(11)).astype(np.float64) + 1.0) * 2.0 ** -53
    u2 = (b >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    r = np.sqrt(-2.0 * np.log(u1))
    return r * np.cos(2 * np.pi * u2) + 1j * r * np.sin(2 * np.pi * u2)


def counter_haar_state(n: int, seed: int) -> np.ndarray:
    v = counter_haar_raw(seed, np.arange(2 ** n, dtype=np.uint64))
    return v / np.linalg.norm(v)
