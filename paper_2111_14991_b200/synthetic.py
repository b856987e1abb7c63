"""Synthetic simulation-mode search spaces (bench / test inputs).

Vectorised numpy restatement of the reference generator
/root/reference/proj/include/gridtune/synthetic.hpp:38-180 (random-rough,
rosenbrock-disc, rastrigin-box, step-plateau) and of the unrestricted
EnumeratedSpace (search_space.hpp:57-72,158-166).  Bit-exact against the
reference (tests/test_host_cpu.py pins it on golden files written by
oracle/_ref/ref_tool).  This is an input generator, not part of the hot path.
"""
from __future__ import annotations

import numpy as np

M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
GOLDEN = np.uint64(0x9E3779B97F4A7C15)


def _u64(x) -> np.uint64:
    return np.uint64(int(x) & 0xFFFFFFFFFFFFFFFF)


def splitmix64_arr(state: np.ndarray):
    """rng.hpp:12-18 over arrays; returns (new_state, output)."""
    with np.errstate(over="ignore"):
        state = state + GOLDEN
        z = state.copy()
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return state, z ^ (z >> np.uint64(31))


def splitmix64(state: int):
    s, z = splitmix64_arr(np.array([state], dtype=np.uint64))
    return int(s[0]), int(z[0])


def fnv1a64_bytes(data: bytes, h: int = 0xCBF29CE484222325) -> int:
    for c in data:
        h ^= c
        h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h


def fnv1a64_u64(v: int, h: int) -> int:
    return fnv1a64_bytes(int(v).to_bytes(8, "little"), h)


class SeedSequence:
    """rng.hpp:89-110"""

    def __init__(self, base: int):
        self.h = fnv1a64_u64(base, 0xCBF29CE484222325)

    def with_(self, x):
        if isinstance(x, str):
            self.h = fnv1a64_bytes(x.encode(), self.h)
        else:
            self.h = fnv1a64_u64(int(x), self.h)
        return self

    def seed(self) -> int:
        return splitmix64(self.h)[1]


class Rng:
    """rng.hpp:41-85 (the parts the generators and tests need)."""

    def __init__(self, seed: int):
        self.state = int(seed) & 0xFFFFFFFFFFFFFFFF

    def next_u64(self) -> int:
        self.state, z = splitmix64(self.state)
        return z

    def uniform01(self) -> float:
        return float(self.next_u64() >> 11) * 2.0 ** -53

    def uniform_below(self, n: int) -> int:
        return (self.next_u64() * int(n)) >> 64

    def normal(self) -> float:
        """Box-Muller with the pair cached (rng.hpp:67-79)."""
        import math
        if getattr(self, "_cached", None) is not None:
            v, self._cached = self._cached, None
            return v
        u1 = 1.0 - self.uniform01()
        u2 = self.uniform01()
        r = math.sqrt(-2.0 * math.log(u1))
        theta = 6.283185307179586476925286766559 * u2
        self._cached = r * math.sin(theta)
        return r * math.cos(theta)


def hash_unit(seed: int, index: np.ndarray, salt: int) -> np.ndarray:
    """synthetic.hpp:38-43"""
    with np.errstate(over="ignore"):
        s = _u64(seed) ^ _u64(0x9E3779B97F4A7C15 * (salt + 1))
        s = s ^ (index.astype(np.uint64) * np.uint64(0xD1342543DE82EF95))
    _, z = splitmix64_arr(s)
    return (z >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def grid_ranks(grid) -> np.ndarray:
    """ranks[idx, j] for every canonical index (first parameter most
    significant, search_space.hpp:57-72)."""
    grid = [int(k) for k in grid]
    total = int(np.prod(grid))
    idx = np.arange(total, dtype=np.int64)
    ranks = np.empty((total, len(grid)), dtype=np.int64)
    rem = idx.copy()
    for j in range(len(grid) - 1, -1, -1):
        ranks[:, j] = rem % grid[j]
        rem //= grid[j]
    return ranks


def grid_coords(grid, ranks=None) -> np.ndarray:
    """SearchSpace::normalize: rank / (k - 1), 0 for single-valued params."""
    if ranks is None:
        ranks = grid_ranks(grid)
    out = np.zeros(ranks.shape, dtype=np.float64)
    for j, k in enumerate(grid):
        if k > 1:
            out[:, j] = ranks[:, j].astype(np.float64) / float(k - 1)
    return out


def random_rough(grid, seed: int, invalid_fraction: float = 0.10):
    """random-rough landscape, synthetic.hpp:150-160.  Returns
    (coords [N,d], ids [N], values [N] with NaN for runtime-invalid)."""
    grid = [int(k) for k in grid]
    d = len(grid)
    total = int(np.prod(grid))
    if total > 1_000_000:
        raise ValueError("grid exceeds 1e6 points")
    ranks = grid_ranks(grid)
    coords = grid_coords(grid, ranks)
    rng = Rng(SeedSequence(seed).with_("rough-center").seed())
    center = [0.2 + 0.6 * rng.uniform01() for _ in range(d)]
    idx = np.arange(total, dtype=np.int64)
    bowl = np.zeros(total)
    for j in range(d):
        diff = coords[:, j] - center[j]
        bowl = bowl + diff * diff
    value = (1.0 + 4.0 * bowl / float(d)) + 0.5 * hash_unit(seed, idx, 1)
    invalid = hash_unit(seed, idx, 2) < invalid_fraction
    value[invalid] = np.nan
    return coords, idx.astype(np.uint64), value


def rosenbrock_disc(grid, seed: int = 0):
    """synthetic.hpp:118-126 (2-D, invalid outside the radius-1.5 disc)."""
    grid = [int(k) for k in grid]
    if len(grid) != 2:
        raise ValueError("rosenbrock-disc is two-dimensional")
    ranks = grid_ranks(grid)
    coords = grid_coords(grid, ranks)
    lo, hi = -1.5, 1.5
    x = [lo + (hi - lo) * ranks[:, j].astype(np.float64) / float(grid[j] - 1) for j in range(2)]
    invalid = x[0] * x[0] + x[1] * x[1] > 2.25
    a = 1.0 - x[0]
    b = x[1] - x[0] * x[0]
    value = 1.0 + a * a + 100.0 * b * b
    value[invalid] = np.nan
    return coords, np.arange(len(value), dtype=np.uint64), value
