"""Seeded synthetic operands, host side.

Counter-based splitmix64 digits, bit-identical to the device generator
(``decmul_gpu_generate_digits``, csrc/gen.cu): key = mix(seed + G),
v_i = mix(key + (i + 1) G); digit 0 = 1 + v_0 mod 9, digit i = v_i mod 10;
mode 1 = all nines. ``mix`` is the splitmix64 finalizer of the reference's
bench.cpp:40-45. The reference itself draws bench digits from std::mt19937_64
(bench.cpp:107-116); that stream is reproduced by oracle/_ref for cross-checks.
"""
from __future__ import annotations

import numpy as np

_G = np.uint64(0x9E3779B97F4A7C15)


def _mix(z: np.ndarray) -> np.ndarray:
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def gen_digits(seed: int, n: int, mode: int = 0, chunk: int = 1 << 24) -> bytes:
    if mode == 1:
        return b"9" * n
    with np.errstate(over="ignore"):
        key = _mix(np.array([seed], dtype=np.uint64) + _G)[0]
        out = np.empty(n, dtype=np.uint8)
        for a in range(0, n, chunk):
            i = np.arange(a, min(n, a + chunk), dtype=np.uint64)
            v = _mix(key + (i + np.uint64(1)) * _G)
            d = (v % np.uint64(10)).astype(np.uint8)
            if a == 0:
                d[0] = np.uint8(1 + int(v[0] % np.uint64(9)))
            out[a: a + len(i)] = d + 48
    return out.tobytes()


def gen_digits_range(seed: int, n: int, start: int, stop: int, mode: int = 0) -> bytes:
    """Digits [start, stop) of the n-digit operand gen_digits(seed, n, mode) (counter-based:
    a slice costs only its own length)."""
    if not 0 <= start <= stop <= n:
        raise ValueError("gen_digits_range: bad range")
    if mode == 1:
        return b"9" * (stop - start)
    with np.errstate(over="ignore"):
        key = _mix(np.array([seed], dtype=np.uint64) + _G)[0]
        i = np.arange(start, stop, dtype=np.uint64)
        v = _mix(key + (i + np.uint64(1)) * _G)
        d = (v % np.uint64(10)).astype(np.uint8)
        if start == 0 and stop > 0:
            d[0] = np.uint8(1 + int(v[0] % np.uint64(9)))
    return (d + 48).tobytes()
