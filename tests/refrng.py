"""Bit-exact restatements of the reference tests' random fixtures, so the
Python parity tests replay the SAME batches as proj/tests/test_gating.cpp and
proj/tests/acceptance.cpp (seeds 2024, 7, 11, 31, 1001-1004 ...).

* MT19937_64  -- std::mt19937_64 (the C++11 engine, default seed 5489).
* random_batch -- proj/tests/test_util.hpp:62-81.
* make_batch / make_batch2 -- test_util.hpp:44-59.
* uniform_batch -- acceptance.cpp:60-69.
"""
from __future__ import annotations

import numpy as np

from paper_2303_06182_b200.gating import Batch, TokenAssignment

_M = (1 << 64) - 1


class MT19937_64:
    n, m = 312, 156
    a = 0xB5026F5AA96619E9
    um, lm = 0xFFFFFFFF80000000, 0x7FFFFFFF

    def __init__(self, seed: int = 5489):
        self.mt = [0] * self.n
        self.mt[0] = seed & _M
        for i in range(1, self.n):
            self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) & _M
        self.i = self.n

    def _twist(self):
        mt = self.mt
        for i in range(self.n):
            x = (mt[i] & self.um) | (mt[(i + 1) % self.n] & self.lm)
            xa = x >> 1
            if x & 1:
                xa ^= self.a
            mt[i] = mt[(i + self.m) % self.n] ^ xa
        self.i = 0

    def __call__(self) -> int:
        if self.i >= self.n:
            self._twist()
        y = self.mt[self.i]
        self.i += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & _M


def random_batch(rng: MT19937_64, seq_len: int, num_experts: int, k: int) -> Batch:
    b = Batch()
    for _ in range(seq_len):
        experts = []
        while len(experts) < k:
            e = rng() % num_experts
            if e not in experts:
                experts.append(e)
        w = [1.0 + float(rng() % 1000) for _ in range(k)]
        s = 0.0
        for x in w:
            s += x
        b.tokens.append(TokenAssignment(experts, [x / s for x in w]))
    return b


def make_batch(experts, batch_id: int = 0) -> Batch:
    return Batch([TokenAssignment([e], [1.0]) for e in experts], batch_id)


def make_batch2(pairs, batch_id: int = 0) -> Batch:
    return Batch([TokenAssignment([a, b], [0.5, 0.5]) for a, b in pairs], batch_id)


def uniform_batch(S: int, E: int, k: int) -> Batch:
    return Batch([TokenAssignment([(t + j) % E for j in range(k)], [1.0 / k] * k) for t in range(S)])


def experts_array(batch: Batch) -> np.ndarray:
    return np.array([ta.experts for ta in batch.tokens], dtype=np.int32)


def weights_array(batch: Batch) -> np.ndarray:
    return np.array([ta.weights for ta in batch.tokens], dtype=np.float64)
