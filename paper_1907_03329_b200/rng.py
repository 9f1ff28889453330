"""Python mirror of the reference's deterministic Rng (matrix.hpp:173-213).

mt19937_64 stream with explicit bit draws: uniform = (x >> 11) * 2^-53, below(n) =
high 64 bits of x*n, Fisher-Yates shuffle from the back.  The engine reproduces the
same stream in C++ (std::mt19937_64) for its window shuffles; this class exists so
host-side callers of make_batches get bit-identical batches.
"""
from __future__ import annotations

import math

_M64 = (1 << 64) - 1


class Rng:
    _N, _M = 312, 156

    def __init__(self, seed: int):
        mt = [0] * self._N
        mt[0] = seed & _M64
        for i in range(1, self._N):
            mt[i] = (6364136223846793005 * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i) & _M64
        self._mt, self._i = mt, self._N
        self._spare = None

    def _twist(self):
        mt, N, M = self._mt, self._N, self._M
        um, lm, a = 0xFFFFFFFF80000000, 0x7FFFFFFF, 0xB5026F5AA96619E9
        for i in range(N):
            x = (mt[i] & um) | (mt[(i + 1) % N] & lm)
            xa = x >> 1
            if x & 1:
                xa ^= a
            mt[i] = mt[(i + M) % N] ^ xa
        self._i = 0

    def raw(self) -> int:
        if self._i >= self._N:
            self._twist()
        x = self._mt[self._i]
        self._i += 1
        x ^= (x >> 29) & 0x5555555555555555
        x ^= (x << 17) & 0x71D67FFFEDA60000 & _M64
        x ^= (x << 37) & 0xFFF7EEE000000000 & _M64
        x ^= x >> 43
        return x & _M64

    def uniform(self, lo: float | None = None, hi: float | None = None) -> float:
        u = (self.raw() >> 11) * 2.0 ** -53
        return u if lo is None else lo + (hi - lo) * u

    def normal(self) -> float:
        if self._spare is not None:
            s, self._spare = self._spare, None
            return s
        u1, u2 = self.uniform(), self.uniform()
        while u1 <= 1e-300:
            u1 = self.uniform()
        r = math.sqrt(-2.0 * math.log(u1))
        th = 2.0 * 3.14159265358979323846 * u2
        self._spare = r * math.sin(th)
        return r * math.cos(th)

    def below(self, n: int) -> int:
        return (self.raw() * n) >> 64

    def shuffle(self, v: list) -> None:
        for i in range(len(v), 1, -1):
            j = self.below(i)
            v[i - 1], v[j] = v[j], v[i - 1]
