"""Synthetic inputs for the five BASELINE.json configurations.

Pattern sets use MT19937 exactly as the survey specifies for variable-length
sets: len = lo + mt() % (hi - lo + 1), symbols byte_of(mt() % sigma),
duplicates rejected, loaded through hepfac_patterns_create.  Fixed-length
sweeps (config 4) use the library's own hepfac_patterns_generate with the
reference's derive_seed (bench.cpp:14-24).  Texts >= 1 GiB come from a
counter-based generator (numpy PCG64) because the reference's MT19937 corpus
generator runs at ~200 MB/s; the same buffer feeds every arm.  Plants: one
pattern occurrence per 4 KiB, round robin over the set.  The text is built
from independent 16 MiB blocks, so any global range (a rank's shard plus its
halo) can be generated on its own.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional

import numpy as np

M64 = (1 << 64) - 1

GiB = 1 << 30
MiB = 1 << 20


def derive_seed(seed: int, a: int, b: int) -> int:
    """Reference derive_seed (bench.cpp:14-24): splitmix64 finaliser."""
    x = ((seed << 32) ^ ((a * 0x9E3779B97F4A7C15) & M64) ^ ((b + 0xBF58476D1CE4E5B9) & M64)) & M64
    x ^= x >> 30
    x = (x * 0xBF58476D1CE4E5B9) & M64
    x ^= x >> 27
    x = (x * 0x94D049BB133111EB) & M64
    x ^= x >> 31
    return x & 0xFFFFFFFF


def mt19937(seed: int) -> np.random.MT19937:
    bg = np.random.MT19937(0)
    bg._legacy_seeding(seed)  # init_genrand(seed): std::mt19937 stream
    return bg


def standard_symbols(sigma: int) -> bytes:
    """Reference Alphabet::standard order (alphabet.cpp:33-63)."""
    if sigma == 4:
        return b"ACGT"
    if sigma == 256:
        return bytes(range(256))
    order = list(range(ord("a"), ord("z") + 1)) + list(range(ord("A"), ord("Z") + 1)) + \
        list(range(ord("0"), ord("9") + 1))
    order += [b for b in range(33, 127) if b not in order]
    order += [b for b in range(256) if b < 33 or b >= 127]
    return bytes(order[:sigma])


def variable_patterns(seed: int, symbols: bytes, count: int, lo: int, hi: int) -> List[bytes]:
    bg = mt19937(seed)
    sig = len(symbols)
    table = np.frombuffer(symbols, dtype=np.uint8)
    out: List[bytes] = []
    seen = set()
    buf = bg.random_raw(1 << 16).astype(np.uint64)
    pos = 0

    def draw(k):
        nonlocal buf, pos
        if pos + k > buf.size:
            buf = np.concatenate([buf[pos:], bg.random_raw(max(1 << 16, k)).astype(np.uint64)])
            pos = 0
        r = buf[pos:pos + k]
        pos += k
        return r

    while len(out) < count:
        n = lo + int(draw(1)[0]) % (hi - lo + 1)
        p = table[(draw(n) % sig).astype(np.intp)].tobytes()
        if p not in seen:
            seen.add(p)
            out.append(p)
    return out


def random_text(seed: int, symbols: bytes, nbytes: int) -> np.ndarray:
    rng = np.random.Generator(np.random.PCG64(seed))
    if len(symbols) == 256 and symbols == bytes(range(256)):
        return np.frombuffer(rng.bytes(nbytes), dtype=np.uint8).copy()
    table = np.frombuffer(symbols, dtype=np.uint8)
    out = np.empty(nbytes, dtype=np.uint8)
    step = 1 << 28
    for o in range(0, nbytes, step):
        n = min(step, nbytes - o)
        out[o:o + n] = table[rng.integers(0, len(symbols), size=n, dtype=np.uint16)]
    return out


def plant(text: np.ndarray, patterns: List[bytes], every: int = 4096, seed: int = 0, base: int = 0) -> int:
    """One occurrence per `every` bytes at seeded offsets, round robin."""
    n = text.size // every
    if n == 0 or not patterns:
        return 0
    rng = np.random.Generator(np.random.PCG64(seed ^ 0x5EED))
    offs = rng.integers(0, text.size - 64, size=n)
    for i, at in enumerate(offs.tolist()):
        p = patterns[(base + i) % len(patterns)]
        if at + len(p) <= text.size:
            text[at:at + len(p)] = np.frombuffer(p, dtype=np.uint8)
    return n


# The synthetic text of a workload is one global byte string made of
# independent 16 MiB blocks: block i is random_text(seed, i) with its own
# planted occurrences.  Any range of it can be generated on its own, so every
# rank of a sharded run builds exactly its global bytes [lo, hi) -- halo
# included -- and a one-rank scan of the same global text is the check.
BLOCK = 16 * MiB


def _block(seed: int, symbols: bytes, patterns, i: int) -> np.ndarray:
    b = random_text(seed * 7919 + 1_000_003 * i, symbols, BLOCK)
    if patterns:
        plant(b, patterns, 4096, seed + 31 * i, base=i * (BLOCK // 4096))
    return b


def text_range(seed: int, symbols: bytes, patterns, lo: int, hi: int) -> np.ndarray:
    out = np.empty(max(0, hi - lo), dtype=np.uint8)
    at = lo
    while at < hi:
        i, off = divmod(at, BLOCK)
        n = min(BLOCK - off, hi - at)
        out[at - lo:at - lo + n] = _block(seed, symbols, patterns, i)[off:off + n]
        at += n
    return out


@dataclass
class Workload:
    name: str
    sigma: int
    symbols: bytes
    patterns: Optional[List[bytes]]
    text_bytes: int
    seed: int
    gen_count: int = 0  # fixed-length sets generated by the library itself
    gen_length: int = 0

    def make_text(self, nbytes: Optional[int] = None, lo: int = 0) -> np.ndarray:
        """Bytes [lo, lo + nbytes) of the workload's global text."""
        n = self.text_bytes if nbytes is None else nbytes
        if self.patterns is None:
            # config 4's fixed-length set comes from the library's generator:
            # without it no occurrence could be planted
            raise ValueError(f"{self.name}: call build_trie(lib, workload) before make_text (plants the set)")
        return text_range(self.seed, self.symbols, self.patterns, lo, lo + n)


def config(name: str, text_bytes: Optional[int] = None, sigma: int = 256, count: int = 0) -> Workload:
    """c1..c5 of BASELINE.json (sizes overridable for tests / samples)."""
    if name == "c1":
        sy = standard_symbols(256)
        return Workload("c1", 256, sy, variable_patterns(1, sy, 1000, 4, 32), text_bytes or 16 * MiB, 1)
    if name == "c2":
        sy = b"ACGT"
        return Workload("c2", 4, sy, variable_patterns(2, sy, 10000, 8, 32), text_bytes or GiB, 2)
    if name == "c3":
        sy = standard_symbols(256)
        return Workload("c3", 256, sy, variable_patterns(3, sy, 20000, 4, 32), text_bytes or 4 * GiB, 3)
    if name == "c4":
        sy = standard_symbols(sigma)
        return Workload(f"c4-s{sigma}", sigma, sy, None, text_bytes or GiB, 4,
                        gen_count=10000, gen_length=20)
    if name == "c5":
        sy = standard_symbols(256)
        n = count or 100000
        return Workload(f"c5-n{n}", 256, sy, variable_patterns(5 + n, sy, n, 4, 32), text_bytes or 4 * GiB, 5)
    raise KeyError(name)


def build_trie(lib, w: Workload, state: str = "s1trunc"):
    """Pattern set + trie for a workload through the C ABI.

    state: 'full' | 'stage1' | 'stage2' | 's1trunc' (stage 1 truncated at
    choose_depth: the reference benchmark path, bench.cpp:199-205)."""
    a = lib.alphabet(w.sigma)
    if w.patterns is None:
        ps = lib.generate_patterns(derive_seed(42, w.sigma, w.gen_count), a, w.gen_count, w.gen_length)
        w.patterns = ps.to_list()
    else:
        ps = lib.patterns(w.patterns, a)
    t = lib.build_trie(ps)
    if state == "full":
        return t, ps
    if state == "stage2":
        return t.compress(2)[0], ps
    s1 = t.compress(1)[0]
    if state == "stage1":
        return s1, ps
    tr, noop = s1.truncate(ps.choose_depth())
    return (s1 if noop else tr), ps
