"""Normative splitmix64 stream (src/prng.py:19-53), vectorised.

The reference steps a Python int per draw.  Because the splitmix64 state is
``seed + i*GAMMA (mod 2^64)``, the i-th output is a pure function of i, so
the whole stream is one numpy pass with bit-identical values (78M draws for
the 48-block initial shape in seconds instead of minutes).
"""

from __future__ import annotations

import numpy as np

MASK64 = (1 << 64) - 1
_GAMMA = np.uint64(0x9E3779B97F4A7C15)
_MIX1 = np.uint64(0xBF58476D1CE4E5B9)
_MIX2 = np.uint64(0x94D049BB133111EB)


def _outputs(seed: int, start: int, n: int) -> np.ndarray:
    i = np.arange(start + 1, start + n + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed & MASK64) + i * _GAMMA
        z = (z ^ (z >> np.uint64(30))) * _MIX1
        z = (z ^ (z >> np.uint64(27))) * _MIX2
    return z ^ (z >> np.uint64(31))


def splitmix64(seed: int, n: int = 1) -> list:
    """First n outputs seeded with ``seed`` (src/prng.py:19-31)."""
    return [int(v) for v in _outputs(seed, 0, n)]


class Prng:
    """Stateful stream (src/prng.py:34-53)."""

    def __init__(self, seed: int):
        self._seed = seed & MASK64
        self._count = 0

    def uniform(self, shape, low: float = -1.0, high: float = 1.0) -> np.ndarray:
        """Uniform floats in [low, high) from the 24 high bits of each draw."""
        n = int(np.prod(shape)) if shape else 1
        z = _outputs(self._seed, self._count, n)
        self._count += n
        u = (z >> np.uint64(40)).astype(np.float64) / float(1 << 24)
        return (low + (high - low) * u).astype(np.float32).reshape(shape)
