"""Seeded synthetic-field centers without loading any native library.

std::mt19937_64(seed) followed by std::uniform_real_distribution<double>(-0.5, 0.5), as the reference
draws its random bump centers (proj/src/problems.cpp:126-141 in 2D, :240-249 in 3D).  libstdc++'s
uniform_real_distribution calls generate_canonical<double, 53> once per draw with a 64-bit engine:
u = double(x) / 2^64, value = u * (b - a) + a.  Pure Python so that problem definitions (and the
bench's CPU reference arm, which must not map the product library) need no shared object.
"""
from __future__ import annotations

import numpy as np

_MASK = (1 << 64) - 1


class MT19937_64:
    """The 64-bit Mersenne Twister of <random> (std::mt19937_64)."""

    def __init__(self, seed: int):
        self.mt = [0] * 312
        self.mt[0] = seed & _MASK
        for i in range(1, 312):
            self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) & _MASK
        self.idx = 312

    def _twist(self):
        mt = self.mt
        for i in range(312):
            x = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % 312] & 0x7FFFFFFF)
            xa = x >> 1
            if x & 1:
                xa ^= 0xB5026F5AA96619E9
            mt[i] = mt[(i + 156) % 312] ^ xa
        self.idx = 0

    def __call__(self) -> int:
        if self.idx >= 312:
            self._twist()
        y = self.mt[self.idx]
        self.idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & _MASK


def uniform(rng: MT19937_64, a: float, b: float) -> float:
    u = float(rng()) / 18446744073709551616.0  # generate_canonical<double, 53>: one 64-bit draw
    if u >= 1.0:
        u = np.nextafter(1.0, 0.0)
    return u * (b - a) + a


def bump_centers(seed: int, n: int = 10, dim: int = 2) -> np.ndarray:
    """n x 3 centers; coordinates beyond dim are zero (problems.cpp:131-135 sets c[2] = 0 in 2D)."""
    rng = MT19937_64(seed)
    out = np.zeros((n, 3))
    for j in range(n):
        for k in range(dim):
            out[j, k] = uniform(rng, -0.5, 0.5)
    return out
