"""ORACLE — test infrastructure only; never imported by the product path.

Independent restatement of the reference's splitmix64 generator
(``kvweaver/rng.py:18-61``) in its counter form: draw i of ``SplitMix64(seed)``
is ``mix(seed + (i + 1) * 0x9E3779B97F4A7C15)`` (state advance by the golden
gamma, ``kvweaver/rng.py:31-36``, then the finaliser) and ``uniform()`` is the
top 53 bits times 2^-53 (``kvweaver/rng.py:38-40``).  The oracle draws its
weights, noise and images through this module rather than the product's
``paper_2603_14371_b200.rng``, so a bug there cannot hide in both; both are
pinned to the reference's golden vectors (tests/golden/rng.json,
tests/test_rng_workload.py).
"""

from __future__ import annotations

import numpy as np

_GAMMA = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def counter_u64(seed: int, start: int, count: int) -> np.ndarray:
    """Draws ``start .. start+count-1`` of SplitMix64(seed) as uint64."""
    i = np.arange(start + 1, start + 1 + count, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed % (1 << 64)) + i * _GAMMA
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def counter_uniform(seed: int, start: int, count: int) -> np.ndarray:
    """``uniform()`` draws ``start ..`` as float64 (53-bit mantissa)."""
    return (counter_u64(seed, start, count) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
