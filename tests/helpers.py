"""Shared test helpers: seeded random instances in the style of the
reference's InstanceRng (tests/naive_search.hpp:73-106)."""
from __future__ import annotations

import numpy as np


def alphabet_bytes(lib, sigma: int):
    a = lib.alphabet(sigma)
    return a, np.array([b for b in range(256) if a.symbol(b) >= 0], dtype=np.uint8)


def pattern_set(rng: np.random.Generator, symbols: np.ndarray, count: int, min_len: int, max_len: int):
    """`count` distinct patterns with lengths uniform in [min_len, max_len], in
    sorted order like the reference's std::set-based generator."""
    seen = set()
    guard = 0
    while len(seen) < count and guard < 100 * count + 1000:
        guard += 1
        n = int(rng.integers(min_len, max_len + 1))
        seen.add(bytes(symbols[rng.integers(0, symbols.size, size=n)]))
    return sorted(seen)


def text(rng: np.random.Generator, symbols: np.ndarray, n: int) -> np.ndarray:
    return symbols[rng.integers(0, symbols.size, size=n)].astype(np.uint8)


def plant(t: np.ndarray, p: bytes, at: int):
    if at + len(p) <= t.size:
        t[at:at + len(p)] = np.frombuffer(p, dtype=np.uint8)


def as_tuples(arr):
    return [(int(r["start"]), int(r["length"]), int(r["pattern_id"])) for r in arr]


def same(a, b) -> bool:
    return a.shape == b.shape and bool(np.array_equal(a, b))
