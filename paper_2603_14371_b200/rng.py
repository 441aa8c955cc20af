"""splitmix64 streams: the scalar generator and its counter (random-access) form.

Mirrors the reference generator ``kvweaver/rng.py:18-61`` (API: ``next_u64``,
``uniform``, ``below``, ``poisson``) so that arrivals, budgets and weights are
bit-identical to the reference.  The counter form is what the device weight-init
kernel evaluates: output *i* (0-based) of ``SplitMix64(seed)`` is
``mix(seed + (i + 1) * GAMMA)`` because the state only ever adds GAMMA
(``kvweaver/rng.py:31-36``).  That makes every draw independent, so a tensor of
2.5 M (toy) or 3.2 G (pi0.5) weights is one parallel launch instead of a Python
loop.
"""

from __future__ import annotations

import math

import numpy as np

MASK64 = (1 << 64) - 1
GAMMA = 0x9E3779B97F4A7C15
MIX1 = 0xBF58476D1CE4E5B9
MIX2 = 0x94D049BB133111EB

__all__ = ["SplitMix64", "mix64", "counter_u64", "counter_uniform", "GAMMA"]


def mix64(z: int) -> int:
    """The splitmix64 finaliser on one 64-bit word."""
    z &= MASK64
    z = ((z ^ (z >> 30)) * MIX1) & MASK64
    z = ((z ^ (z >> 27)) * MIX2) & MASK64
    return z ^ (z >> 31)


class SplitMix64:
    """Sequential generator; same outputs as ``kvweaver.rng.SplitMix64``."""

    __slots__ = ("_state",)

    def __init__(self, seed: int):
        self._state = seed & MASK64

    @property
    def state(self) -> int:
        return self._state

    def next_u64(self) -> int:
        self._state = (self._state + GAMMA) & MASK64
        return mix64(self._state)

    def uniform(self) -> float:
        # top 53 bits scaled into [0, 1)   (kvweaver/rng.py:38-40)
        return (self.next_u64() >> 11) * 2.0 ** -53

    def below(self, n: int) -> int:
        # plain modulo reduction          (kvweaver/rng.py:42-46)
        if n <= 0:
            raise ValueError(f"below() needs a positive bound, got {n}")
        return self.next_u64() % n

    def poisson(self, lam: float) -> int:
        # Knuth product method            (kvweaver/rng.py:48-61)
        if lam < 0:
            raise ValueError(f"poisson() rate must be nonnegative, got {lam}")
        if lam == 0:
            return 0
        limit = math.exp(-lam)
        n = 0
        acc = 1.0
        while True:
            acc *= self.uniform()
            if acc <= limit:
                return n
            n += 1

    def skip(self, n: int) -> None:
        """Advance the stream by n draws in O(1) (the counter form)."""
        self._state = (self._state + n * GAMMA) & MASK64


def counter_u64(seed: int, start: int, count: int) -> np.ndarray:
    """Draws ``start .. start+count-1`` of ``SplitMix64(seed)`` as uint64."""
    idx = np.arange(start + 1, start + 1 + count, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed & MASK64) + idx * np.uint64(GAMMA)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(MIX1)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(MIX2)
        z = z ^ (z >> np.uint64(31))
    return z


def counter_uniform(seed: int, start: int, count: int) -> np.ndarray:
    """``uniform()`` draws ``start ..`` as float64, bit-identical to the loop."""
    return (counter_u64(seed, start, count) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
