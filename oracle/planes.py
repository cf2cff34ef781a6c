"""TEST INFRASTRUCTURE ONLY -- seeded synthetic planes and circuits.

Plane generators use only exactly rounded arithmetic (numpy +,-,*,/ and the
PCG64 bit stream) or scalar libm calls in a Python loop, so the same seed
gives the same bytes on this container and on the GPU box (same image).
Golden fixtures additionally record the SHA-256 of every generated input so
generator drift is detected instead of silently passing.

The plane kinds mirror the value distributions the engine produces
(SURVEY.md §4 item 2): basis / Grover-like constant planes, QFT columns,
Gaussian noise, near-tie lattices, outlier-heavy and signed-zero planes.
"""
from __future__ import annotations

import hashlib
import math

import numpy as np

KINDS = ["constant", "basis", "qft", "gauss", "smooth", "outliers", "neartie", "spike",
         "negzero", "grover", "walk", "uniform"]


def _rng(seed):
    return np.random.Generator(np.random.PCG64(seed))


def _u01(rng, n):
    # (bits >> 11) * 2^-53: exactly representable, platform independent
    return (rng.integers(0, 2**63 - 1, size=n, dtype=np.int64, endpoint=False) >> 10).astype(np.float64) * 2.0**-53


def make_plane(kind: str, n: int, seed: int) -> np.ndarray:
    rng = _rng(seed)
    if kind == "constant":
        v = np.full(n, (_u01(rng, 1)[0] - 0.5) * 2.0)
    elif kind == "basis":
        v = np.zeros(n)
        v[int(rng.integers(0, n))] = 1.0
    elif kind == "qft":
        x = int(rng.integers(0, 1 << 30))
        amp = 2.0 ** -float(int(rng.integers(6, 15)))
        nn = 1 << 30
        v = np.array([amp * math.cos(2.0 * math.pi * ((x * k) % nn) / nn) for k in range(n)])
    elif kind == "gauss":
        sigma = 2.0 ** -float(int(rng.integers(3, 16)))
        u1 = _u01(rng, n) + 2.0**-54
        u2 = _u01(rng, n)
        v = np.array([sigma * math.sqrt(-2.0 * math.log(a)) * math.cos(2.0 * math.pi * b) for a, b in zip(u1, u2)])
    elif kind == "smooth":
        f1, f2 = 1.0 + 7.0 * _u01(rng, 2)
        v = np.array([0.3 * math.sin(f1 * k / n * 6.283) + 0.01 * math.cos(f2 * k / 97.0) for k in range(n)])
    elif kind == "outliers":
        v = np.array([1e-3 * math.sin(k / 13.0) for k in range(n)])
        idx = rng.integers(0, n, size=max(1, n // 16))
        v[idx] = (_u01(rng, idx.size) - 0.5) * 8.0
    elif kind == "neartie":
        # odd multiples of 2^-11 (= eb for the dyadic configs): r lands on .5
        k = rng.integers(-64, 64, size=n) * 2 + 1
        v = k.astype(np.float64) * 2.0**-11
        jit = rng.integers(0, 4, size=n)
        v = np.where(jit == 0, v + 2.0**-40, v)
    elif kind == "spike":
        v = np.zeros(n)
        v[int(rng.integers(0, n))] = (_u01(rng, 1)[0] - 0.5) * 4.0
    elif kind == "negzero":
        choice = rng.integers(0, 4, size=n)
        small = (_u01(rng, n) - 0.5) * 1e-4
        v = np.where(choice == 0, -0.0, np.where(choice == 1, 0.0, np.where(choice == 2, small, -small)))
        v[0] = -0.0
    elif kind == "grover":
        v = np.full(n, 2.0**-10)
        v[int(rng.integers(0, n))] = 3.0 * 2.0**-10
    elif kind == "walk":
        steps = (rng.integers(-3, 4, size=n).astype(np.float64)) * 1.7e-5
        v = np.cumsum(steps)
    elif kind == "uniform":
        v = (_u01(rng, n) - 0.5) * 2.0
    else:
        raise ValueError(kind)
    return np.ascontiguousarray(v, dtype=np.float64)


def sha(data) -> str:
    if isinstance(data, np.ndarray):
        data = data.tobytes()
    return hashlib.sha256(data).hexdigest()


# ----------------------------------------------------------------- circuits
def mt19937_64(seed):
    """std::mt19937_64 raw outputs (the standard fixes this sequence),
    as SURVEY.md §8(d) prescribes for seeded workloads."""
    NN, MM = 312, 156
    MATRIX_A = 0xB5026F5AA96619E9
    UM, LM = 0xFFFFFFFF80000000, 0x7FFFFFFF
    mask = (1 << 64) - 1
    mt = [0] * NN
    mt[0] = seed & mask
    for i in range(1, NN):
        mt[i] = (6364136223846793005 * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i) & mask
    idx = NN
    while True:
        if idx >= NN:
            for i in range(NN):
                x = (mt[i] & UM) | (mt[(i + 1) % NN] & LM)
                xa = x >> 1
                if x & 1:
                    xa ^= MATRIX_A
                mt[i] = mt[(i + MM) % NN] ^ xa
            idx = 0
        x = mt[idx]
        idx += 1
        x ^= (x >> 29) & 0x5555555555555555
        x ^= (x << 17) & 0x71D67FFFEDA60000
        x ^= (x << 37) & 0xFFF7EEE000000000
        x ^= x >> 43
        yield x & mask
