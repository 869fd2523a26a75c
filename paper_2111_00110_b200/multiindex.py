"""Coefficient order shared by every grid, table and kernel.

Restates the reference's multi-index contract (``pkg/src/fc2t2/multiindex.py``):
the set ``{(n1, n2, n3): n1 + n2 + n3 <= rho}`` in graded-lexicographic order
(total order first, then lexicographic), so entry 0 is ``(0, 0, 0)`` and a
lower order is a prefix (reference ``multiindex.py:74-96``, sort key at :84).

The order is a *layout contract*: the P axis of every device grid
(``(res, res, res, C, P)`` viewed through the padded row stride) and of every
M2L / shift table follows it, and ``csrc/common.cuh`` regenerates the same
order at compile time (``MI<RHO>``).

Difference from the reference: the reference caps rho at 4 (``MAX_ORDER``,
:17, :76-77) because its root layers solve quartics in closed form.  The
expansion engine itself is rho-generic and BASELINE config 5 needs rho = 6,
so this package accepts rho up to 6; the root layers still require rho <= 4
(enforced where they are called).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from itertools import product

import numpy as np

MAX_ORDER = 6          # engine limit (reference: 4, see module docstring)
ROOT_MAX_ORDER = 4     # closed-form first-root layers need quartic line polys


class OrderError(ValueError):
    """Expansion order outside the supported range (reference multiindex.py:20-21)."""


def index_count(rho: int) -> int:
    """|{n : |n| <= rho}| in 3D (reference multiindex.py:24-26)."""
    return math.comb(rho + 3, 3)


def padded_count(rho: int) -> int:
    """Row stride of a cell's coefficient vector on the device: P rounded up
    to a multiple of 4 floats so every row is 16-byte aligned (P=35 -> 36)."""
    return (index_count(rho) + 3) // 4 * 4


def _graded_lex(rho: int) -> list[tuple[int, int, int]]:
    triples = [t for t in product(range(rho + 1), repeat=3) if sum(t) <= rho]
    triples.sort(key=lambda t: (t[0] + t[1] + t[2], t))
    return triples


@dataclass(frozen=True)
class MultiIndexTable:
    """Graded-lex multi-indices plus factorial / binomial lookups
    (field names follow reference multiindex.py:29-71)."""

    rho: int
    entries: np.ndarray        # (P, 3) int64
    factorial: np.ndarray      # 0! .. (2 rho)!
    binomial: np.ndarray       # (2 rho + 1, 2 rho + 1)
    _lookup: dict = field(repr=False, default_factory=dict)

    @property
    def size(self) -> int:
        return int(self.entries.shape[0])

    @property
    def padded_size(self) -> int:
        return padded_count(self.rho)

    def index_of(self, n) -> int:
        key = tuple(int(v) for v in n)
        if key not in self._lookup:
            raise OrderError(f"multi-index {key} exceeds total order {self.rho}")
        return self._lookup[key]

    def __contains__(self, n) -> bool:
        return tuple(int(v) for v in n) in self._lookup

    @property
    def norms(self) -> np.ndarray:
        return self.entries.sum(axis=1)

    def entry_factorial(self) -> np.ndarray:
        f = self.factorial
        return f[self.entries].prod(axis=1)

    def shift_map(self, s) -> np.ndarray:
        """Ordinal of ``entries[j] + s`` for every j, -1 if it leaves the
        table: coefficient-space differentiation (reference expansion.py:309-329)."""
        out = np.full(self.size, -1, dtype=np.int64)
        for j, n in enumerate(self.entries):
            key = (int(n[0] + s[0]), int(n[1] + s[1]), int(n[2] + s[2]))
            out[j] = self._lookup.get(key, -1)
        return out


_TABLES: dict[int, MultiIndexTable] = {}


def build_table(rho: int) -> MultiIndexTable:
    """Multi-index table of total order <= rho, 1 <= rho <= MAX_ORDER."""
    if not isinstance(rho, (int, np.integer)) or not 1 <= rho <= MAX_ORDER:
        raise OrderError(f"expansion order must be in [1, {MAX_ORDER}], got {rho}")
    rho = int(rho)
    if rho not in _TABLES:
        entries = np.array(_graded_lex(rho), dtype=np.int64)
        top = 2 * rho
        fact = np.array([math.factorial(i) for i in range(top + 1)], dtype=np.float64)
        binom = np.array([[math.comb(n, k) if k <= n else 0 for k in range(top + 1)]
                          for n in range(top + 1)], dtype=np.float64)
        lookup = {tuple(int(v) for v in e): i for i, e in enumerate(entries)}
        _TABLES[rho] = MultiIndexTable(rho, entries, fact, binom, lookup)
    return _TABLES[rho]
