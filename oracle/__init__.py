"""Oracle package -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this package.  It is the checker, never the thing measured,
and nothing in paper_1704_02272_b200/ imports it.

Two checkers live here:
  * liboracle.so  -- plain-C restatement of the reference's match path
    (pfac_oracle.c: naive_find_all = naive_search.hpp:17-31; walk_scan =
    scan.cpp:20-119 over the canonical cells of trie.hpp:45-81);
  * _ref/libhepfac_ref.so -- the unmodified reference library compiled from
    /root/reference/proj/src by oracle/Makefile (present when it was built in
    the source container; it travels to the GPU box as a built artefact).
Both are pinned against the reference's golden vectors in tests/test_oracle.py.
"""
from __future__ import annotations

import ctypes as C
import os
import struct
from typing import List, Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
REF_LIB_PATH = os.path.join(HERE, "_ref", "libhepfac_ref.so")
MATCH_DTYPE = np.dtype([("start", "<u8"), ("length", "<u4"), ("pattern_id", "<u4")])


class _OracleTrie(C.Structure):
    _fields_ = [("cells", C.c_void_p), ("node_count", C.c_uint32), ("words", C.c_uint32),
                ("symbol_of", C.c_void_p), ("depth_limit", C.c_uint32), ("pattern_bytes", C.c_void_p),
                ("pattern_offsets", C.c_void_p), ("pattern_lengths", C.c_void_p), ("pattern_count", C.c_uint32),
                ("bucket_nodes", C.c_void_p), ("bucket_starts", C.c_void_p), ("bucket_ids", C.c_void_p),
                ("bucket_count", C.c_uint32)]


_lib = None


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise FileNotFoundError(f"{LIB_PATH} missing: run `make -C {HERE} liboracle.so`")
        _lib = C.CDLL(LIB_PATH)
        _lib.oracle_naive_find_all.restype = C.c_uint64
        _lib.oracle_naive_find_all.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p,
                                               C.c_uint32, C.c_void_p, C.c_uint64]
        _lib.oracle_walk_scan.restype = C.c_uint64
        _lib.oracle_walk_scan.argtypes = [C.POINTER(_OracleTrie), C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64]
        _lib.oracle_transition.restype = C.c_uint32
        _lib.oracle_transition.argtypes = [C.POINTER(_OracleTrie), C.c_uint32, C.c_uint8]
    return _lib


def _u8(text) -> np.ndarray:
    if isinstance(text, np.ndarray):
        return np.ascontiguousarray(text.view(np.uint8).reshape(-1))
    return np.frombuffer(bytes(text), dtype=np.uint8)


def _ptr(a: np.ndarray):
    return a.ctypes.data if a.size else None


def _dict_arrays(patterns: Sequence[bytes]):
    lens = np.array([len(p) for p in patterns], dtype=np.uint32)
    offs = np.zeros(len(patterns), dtype=np.uint64)
    if len(patterns):
        offs[1:] = np.cumsum(lens[:-1], dtype=np.uint64)
    blob = np.frombuffer(b"".join(patterns) or b"\0", dtype=np.uint8).copy()
    return blob, offs, lens


def naive_find_all(text, patterns: Sequence[bytes]) -> np.ndarray:
    """Every pattern at every offset (naive_search.hpp:17-31), sorted."""
    lib = _load()
    t = _u8(text)
    blob, offs, lens = _dict_arrays(patterns)
    n = lib.oracle_naive_find_all(_ptr(t), t.size, _ptr(blob), _ptr(offs), _ptr(lens), len(patterns), None, 0)
    out = np.empty(n, dtype=MATCH_DTYPE)
    lib.oracle_naive_find_all(_ptr(t), t.size, _ptr(blob), _ptr(offs), _ptr(lens), len(patterns),
                              _ptr(out), n)
    return out


class HtriTrie:
    """A trie in the reference's canonical layout, read from .htri bytes
    (format of trie_io.hpp:13-27; parser restates trie_io.cpp:103-166)."""

    def __init__(self, data: bytes):
        p = 0

        def take(fmt):
            nonlocal p
            v = struct.unpack_from("<" + fmt, data, p)
            p += struct.calcsize("<" + fmt)
            return v if len(v) > 1 else v[0]

        assert data[:4] == b"HTRI"
        p = 4
        version, sigma, self.node_count, self.words = take("HHIH")
        assert version == 1
        sigma = sigma or 256
        ncells = self.node_count * (self.words + 1)
        self.cells = np.frombuffer(data, dtype="<u4", count=ncells, offset=p).copy()
        p += 4 * ncells
        count = take("I")
        pats: List[Optional[bytes]] = [None] * count
        for _ in range(count):
            ln = take("H")
            s = data[p:p + ln]
            p += ln
            pats[take("I")] = s
        self.patterns = pats
        self.stage, self.depth_limit = 0, 0
        symbols = None
        if p < len(data) and data[p:p + 4] == b"HTRX":
            p += 4
            _xver, self.stage, has_lim, lim, alen = take("HBBHH")
            self.depth_limit = lim if has_lim else 0
            symbols = data[p:p + alen]
        if symbols is None:
            raise ValueError("oracle expects the HTRX trailer (tries written by hepfac_trie_save)")
        self.symbol_of = np.full(256, -1, dtype=np.int16)
        for i, b in enumerate(symbols):
            self.symbol_of[b] = i
        self.blob, self.offs, self.lens = _dict_arrays(self.patterns)
        self._struct = _OracleTrie(_ptr(self.cells), self.node_count, self.words, _ptr(self.symbol_of),
                                   self.depth_limit, _ptr(self.blob), _ptr(self.offs), _ptr(self.lens),
                                   len(self.patterns), None, None, None, 0)
        self._buckets()

    def transition(self, node: int, byte: int) -> int:
        return _load().oracle_transition(C.byref(self._struct), node, byte)

    def _buckets(self):
        # build_verification_buckets (prefix.cpp:14-31)
        d = self.depth_limit
        by_node = {}
        if d:
            for pid, pat in enumerate(self.patterns):
                if len(pat) <= d:
                    continue
                node = 0
                for i in range(d):
                    node = self.transition(node, pat[i])
                    assert node != 0xFFFFFFFF, "dictionary pattern not present in trie"
                by_node.setdefault(node, []).append(pid)
        nodes = sorted(by_node)
        self.b_nodes = np.array(nodes, dtype=np.uint32)
        starts = [0]
        ids: List[int] = []
        for nd in nodes:
            ids += sorted(by_node[nd])
            starts.append(len(ids))
        self.b_starts = np.array(starts, dtype=np.uint32)
        self.b_ids = np.array(ids or [0], dtype=np.uint32)
        s = self._struct
        s.bucket_nodes, s.bucket_starts, s.bucket_ids = _ptr(self.b_nodes), _ptr(self.b_starts), _ptr(self.b_ids)
        s.bucket_count = len(nodes)

    def scan(self, text) -> np.ndarray:
        """scan.cpp:69-119 restated (single worker)."""
        lib = _load()
        t = _u8(text)
        n = lib.oracle_walk_scan(C.byref(self._struct), _ptr(t), t.size, None, 0)
        if n == 0xFFFFFFFFFFFFFFFF:
            raise RuntimeError("terminal node spells no dictionary pattern")
        out = np.empty(n, dtype=MATCH_DTYPE)
        lib.oracle_walk_scan(C.byref(self._struct), _ptr(t), t.size, _ptr(out), n)
        return out


def walk_scan(htri_bytes: bytes, text) -> np.ndarray:
    return HtriTrie(htri_bytes).scan(text)


def ref_library():
    """The compiled reference (oracle/_ref), or None when it was not built."""
    if not os.path.exists(REF_LIB_PATH):
        return None
    from paper_1704_02272_b200.hepfac import Library
    return Library(REF_LIB_PATH)
