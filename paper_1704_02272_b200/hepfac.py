"""ctypes mirror of the hepfac C ABI (include/hepfac.h, include/hepfac_b200.h).

The same binding drives any library exporting the reference's ABI: the B200
library built in this package (the product, default) or, in tests only, the
reference library compiled from its sources into ``oracle/_ref``.  Names follow
the reference's C++ API (``build_trie``, ``merge_final_nodes``, ``compress``,
``truncate``, ``scan``, ``scan_two_stage``, ``run_throughput``; reference
include/hepfac/*.hpp) so the parity tests read like the reference's own tests.

No CPU fallback: if ``libhepfac.so`` is missing this module raises on import of
the default library, and ``scan`` fails with HEPFAC_ERR_INTERNAL when no CUDA
device is usable.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Iterable, Optional, Sequence, Union

import numpy as np

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HEPFAC_LIB") or os.path.join(PKG_DIR, "libhepfac.so")

MATCH_DTYPE = np.dtype([("start", "<u8"), ("length", "<u4"), ("pattern_id", "<u4")])
NO_NODE = 0xFFFFFFFF

STATUS = {
    0: "HEPFAC_OK",
    1: "HEPFAC_ERR_INVALID_ARG",
    2: "HEPFAC_ERR_DUPLICATE",
    3: "HEPFAC_ERR_BAD_BYTE",
    4: "HEPFAC_ERR_STATE",
    5: "HEPFAC_ERR_IO",
    6: "HEPFAC_ERR_FORMAT",
    7: "HEPFAC_ERR_NOMEM",
    8: "HEPFAC_ERR_INTERNAL",
}
OK, INVALID_ARG, DUPLICATE, BAD_BYTE, STATE, IO, FORMAT, NOMEM, INTERNAL = range(9)


class HepfacError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"{STATUS.get(status, status)}: {message}")
        self.status = status
        self.message = message


class _MemoryReport(C.Structure):
    _fields_ = [("node_count", C.c_uint64), ("bytes_per_node", C.c_uint32), ("total_bytes", C.c_uint64),
                ("sigma", C.c_uint16), ("total_mib", C.c_char * 32)]


class _CompressionStats(C.Structure):
    _fields_ = [("nodes_before", C.c_uint64), ("nodes_after_stage1", C.c_uint64),
                ("nodes_after_stage2", C.c_uint64), ("pattern_count", C.c_uint64),
                ("reduction_percent", C.c_double)]


class _ScanConfig(C.Structure):
    _fields_ = [("workers", C.c_uint32), ("chunk", C.c_uint32)]


class _Throughput(C.Structure):
    _fields_ = [("bytes", C.c_uint64), ("seconds", C.c_double), ("merge_seconds", C.c_double),
                ("gbps", C.c_double), ("workers", C.c_uint32), ("runs", C.c_uint32), ("matches", C.c_uint64)]


class _Comparison(C.Structure):
    _fields_ = [("node_count", C.c_uint64), ("sigma", C.c_uint16), ("ours_bytes", C.c_uint64),
                ("pfac_bytes", C.c_uint64), ("accw_bytes", C.c_uint64), ("gravity_bytes", C.c_uint64),
                ("ratio_pfac", C.c_double), ("ratio_accw", C.c_double), ("ratio_gravity", C.c_double)]


class _Reduction(C.Structure):
    _fields_ = [("r", C.c_uint64), ("n", C.c_uint64), ("formula_value", C.c_double),
                ("oracle_value", C.c_double), ("oracle_std_error", C.c_double), ("trials", C.c_uint64),
                ("conforms", C.c_int)]


class _ScanStats(C.Structure):
    _fields_ = [("h2d_ms", C.c_double), ("kernel_ms", C.c_double), ("d2h_ms", C.c_double),
                ("total_ms", C.c_double), ("bytes", C.c_uint64), ("matches", C.c_uint64),
                ("kernel_launches", C.c_uint32), ("chunks", C.c_uint32), ("relaunches", C.c_uint32),
                ("device", C.c_int32), ("staged", C.c_uint32)]


class _LayoutInfo(C.Structure):
    _fields_ = [(n, C.c_uint32) for n in ("node_count", "groups", "record_bytes", "filter_k", "filter_bits",
                                          "min_emit", "smem_bytes", "blocks_per_sm", "sm_count", "identity")] + \
               [(n, C.c_uint64) for n in ("filter_paths", "reach", "device_bytes", "private_terminals",
                                          "keyed_terminals")] + \
               [(n, C.c_uint32) for n in ("filter_mode", "filter_pass_ppm", "filter2_bits")]


_P = C.c_void_p
_PP = C.POINTER(C.c_void_p)
_U8P = C.POINTER(C.c_uint8)

# (name, restype, argtypes, is_b200_extension)
_PROTOTYPES = [
    ("hepfac_status_string", C.c_char_p, [C.c_int]),
    ("hepfac_version", C.c_char_p, []),
    ("hepfac_last_error", C.c_char_p, []),
    ("hepfac_alphabet_create", C.c_int, [_P, C.c_size_t, _PP]),
    ("hepfac_alphabet_standard", C.c_int, [C.c_uint16, _PP]),
    ("hepfac_alphabet_size", C.c_uint16, [_P]),
    ("hepfac_alphabet_symbol", C.c_int32, [_P, C.c_uint8]),
    ("hepfac_alphabet_destroy", None, [_P]),
    ("hepfac_patterns_create", C.c_int, [_P, _P, C.c_size_t, _P, _PP]),
    ("hepfac_patterns_generate", C.c_int, [C.c_uint32, _P, C.c_uint64, C.c_uint32, _PP]),
    ("hepfac_patterns_load", C.c_int, [C.c_char_p, _P, C.c_int, _PP]),
    ("hepfac_patterns_save", C.c_int, [_P, C.c_char_p]),
    ("hepfac_patterns_count", C.c_size_t, [_P]),
    ("hepfac_patterns_get", _P, [_P, C.c_size_t, C.POINTER(C.c_size_t)]),
    ("hepfac_patterns_unique_prefix", C.c_int, [_P, C.POINTER(C.c_uint32)]),
    ("hepfac_patterns_choose_depth", C.c_int, [_P, C.POINTER(C.c_uint32)]),
    ("hepfac_patterns_destroy", None, [_P]),
    ("hepfac_corpus_generate", C.c_int, [C.c_uint32, _P, C.c_uint64, _P]),
    ("hepfac_corpus_plant", C.c_int, [_P, C.c_uint64, _P, C.c_uint64, C.c_uint32]),
    ("hepfac_sha256", C.c_int, [_P, C.c_uint64, C.c_char_p]),
    ("hepfac_trie_build", C.c_int, [_P, _PP]),
    ("hepfac_trie_compress", C.c_int, [_P, C.c_int, _PP]),
    ("hepfac_trie_compress_stats", C.c_int, [_P, C.c_int, _PP, C.POINTER(_CompressionStats)]),
    ("hepfac_trie_truncate", C.c_int, [_P, C.c_uint32, _PP, C.POINTER(C.c_int)]),
    ("hepfac_trie_save", C.c_int, [_P, C.c_char_p]),
    ("hepfac_trie_load", C.c_int, [C.c_char_p, _PP]),
    ("hepfac_trie_destroy", None, [_P]),
    ("hepfac_trie_node_count", C.c_uint32, [_P]),
    ("hepfac_trie_sigma", C.c_uint16, [_P]),
    ("hepfac_trie_stage", C.c_int, [_P]),
    ("hepfac_trie_depth_limit", C.c_int, [_P, C.POINTER(C.c_uint32)]),
    ("hepfac_trie_transition", C.c_int, [_P, C.c_uint32, C.c_uint8, C.POINTER(C.c_uint32)]),
    ("hepfac_trie_terminal", C.c_int, [_P, C.c_uint32]),
    ("hepfac_trie_memory_report", C.c_int, [_P, C.POINTER(_MemoryReport)]),
    ("hepfac_scan", C.c_int, [_P, _P, C.c_uint64, C.POINTER(_ScanConfig), _PP]),
    ("hepfac_match_list_size", C.c_size_t, [_P]),
    ("hepfac_match_list_data", _P, [_P]),
    ("hepfac_match_list_destroy", None, [_P]),
    ("hepfac_run_throughput", C.c_int, [_P, _P, C.c_uint64, C.POINTER(_ScanConfig), C.c_uint32,
                                        C.POINTER(_Throughput)]),
    ("hepfac_string_free", None, [_P]),
    ("hepfac_compare_footprint", C.c_int, [C.c_uint64, C.c_uint16, C.POINTER(_Comparison)]),
    ("hepfac_prefix_analysis_csv", C.c_int, [_P, C.c_size_t, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                             C.POINTER(C.c_void_p)]),
    ("hepfac_trie_size_curve_csv", C.c_int, [C.c_uint16, _P, C.c_size_t, C.c_uint32, C.c_uint32,
                                             C.POINTER(C.c_void_p)]),
    ("hepfac_scaling_csv", C.c_int, [_P, C.c_size_t, _P, C.c_size_t, C.c_uint32, C.c_uint64, C.c_uint32,
                                     C.c_uint32, C.c_uint32, C.POINTER(C.c_void_p)]),
    ("hepfac_filesize_csv", C.c_int, [C.c_uint16, C.c_uint64, C.c_uint32, _P, C.c_size_t, C.c_uint32,
                                      C.c_uint32, C.c_uint32, C.POINTER(C.c_void_p)]),
    ("hepfac_reduction_estimate", C.c_int, [C.c_uint16, C.c_uint64, C.c_uint64, C.c_uint32,
                                            C.POINTER(_Reduction)]),
]

_B200_PROTOTYPES = [
    ("hepfac_b200_device_count", C.c_int, []),
    ("hepfac_b200_halo", C.c_int, [_P, C.POINTER(C.c_uint64)]),
    ("hepfac_b200_scan_shard", C.c_int, [_P, _P, C.c_uint64, C.c_uint64, C.c_uint64, _PP]),
    ("hepfac_b200_last_scan_stats", C.c_int, [C.POINTER(_ScanStats)]),
    ("hepfac_b200_session_create", C.c_int, [_P, _P, C.c_uint64, C.c_uint64, C.c_uint64, _PP]),
    ("hepfac_b200_session_kernel_ms", C.c_int, [_P, C.c_uint32, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                                C.POINTER(C.c_uint32)]),
    ("hepfac_b200_session_run", C.c_int, [_P, C.c_uint32, C.c_int, C.POINTER(C.c_double),
                                          C.POINTER(C.c_uint64)]),
    ("hepfac_b200_session_fetch", C.c_int, [_P, _PP]),
    ("hepfac_b200_session_destroy", None, [_P]),
    ("hepfac_b200_layout_info", C.c_int, [_P, C.POINTER(_LayoutInfo)]),
    ("hepfac_b200_trim", C.c_int, []),
]

ABI_SYMBOLS = [p[0] for p in _PROTOTYPES]
B200_SYMBOLS = [p[0] for p in _B200_PROTOTYPES]


def _as_u8(data) -> np.ndarray:
    if isinstance(data, np.ndarray):
        arr = data
        if arr.dtype != np.uint8:
            arr = arr.view(np.uint8)
        return np.ascontiguousarray(arr).reshape(-1)
    if isinstance(data, str):
        data = data.encode("latin-1")
    return np.frombuffer(bytes(data), dtype=np.uint8)


def _ptr(arr: np.ndarray):
    return C.c_void_p(arr.ctypes.data) if arr.size else None


class Library:
    """One loaded libhepfac-ABI shared object."""

    def __init__(self, path: str = LIB_PATH):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built: run `make -C {os.path.dirname(path)}` "
                                    "(or __graft_entry__.build()); there is no fallback implementation")
        self.path = path
        self.dll = C.CDLL(path, mode=os.RTLD_LOCAL | os.RTLD_NOW)
        for name, res, args in _PROTOTYPES:
            fn = getattr(self.dll, name)
            fn.restype, fn.argtypes = res, args
        self.is_b200 = hasattr(self.dll, "hepfac_b200_device_count")
        if self.is_b200:
            for name, res, args in _B200_PROTOTYPES:
                fn = getattr(self.dll, name, None)  # (an older build may lack a later addition)
                if fn is not None:
                    fn.restype, fn.argtypes = res, args

    # -- plumbing ---------------------------------------------------------
    def check(self, status: int):
        if status != OK:
            raise HepfacError(status, self.dll.hepfac_last_error().decode("utf-8", "replace"))

    def last_error(self) -> str:
        return self.dll.hepfac_last_error().decode("utf-8", "replace")

    def version(self) -> str:
        return self.dll.hepfac_version().decode()

    def status_string(self, s: int) -> str:
        return self.dll.hepfac_status_string(s).decode()

    # -- objects ----------------------------------------------------------
    def alphabet(self, sigma_or_symbols: Union[int, bytes, str]) -> "Alphabet":
        return Alphabet(self, sigma_or_symbols)

    def patterns(self, patterns: Sequence[Union[bytes, str]], alphabet: "Alphabet") -> "PatternSet":
        return PatternSet.create(self, patterns, alphabet)

    def generate_patterns(self, seed: int, alphabet: "Alphabet", count: int, length: int) -> "PatternSet":
        return PatternSet.generate(self, seed, alphabet, count, length)

    def load_patterns(self, path: str, alphabet: "Alphabet", hex: bool = False) -> "PatternSet":
        h = C.c_void_p()
        self.check(self.dll.hepfac_patterns_load(path.encode(), alphabet.h, int(hex), C.byref(h)))
        return PatternSet(self, h, alphabet)

    def build_trie(self, patterns: "PatternSet") -> "Trie":
        h = C.c_void_p()
        self.check(self.dll.hepfac_trie_build(patterns.h, C.byref(h)))
        return Trie(self, h)

    def load_trie(self, path: str) -> "Trie":
        h = C.c_void_p()
        self.check(self.dll.hepfac_trie_load(path.encode(), C.byref(h)))
        return Trie(self, h)

    def generate_corpus(self, seed: int, alphabet: "Alphabet", nbytes: int) -> np.ndarray:
        out = np.empty(nbytes, dtype=np.uint8)
        self.check(self.dll.hepfac_corpus_generate(seed, alphabet.h, nbytes, _ptr(out) if nbytes else
                                                   C.c_void_p(1)))
        return out

    def plant(self, corpus: np.ndarray, patterns: "PatternSet", occurrences: int, seed: int) -> None:
        assert corpus.dtype == np.uint8 and corpus.flags.c_contiguous
        self.check(self.dll.hepfac_corpus_plant(_ptr(corpus) or C.c_void_p(1), corpus.size, patterns.h,
                                                occurrences, seed))

    def sha256(self, data) -> str:
        arr = _as_u8(data)
        buf = C.create_string_buffer(65)
        self.check(self.dll.hepfac_sha256(_ptr(arr), arr.size, buf))
        return buf.value.decode()

    # -- matching ---------------------------------------------------------
    def _list(self, h, view: bool = False) -> np.ndarray:
        """The records of a match list.  view=False copies them and destroys
        the list; view=True returns a zero-copy array over the list's own
        memory (hepfac_match_list_data), which destroys the list when the
        array (and every view of it) is garbage-collected -- what a C caller
        gets, without a host copy of the records."""
        n = self.dll.hepfac_match_list_size(h)
        if view and n:
            import weakref
            buf = (C.c_uint8 * (n * MATCH_DTYPE.itemsize)).from_address(self.dll.hepfac_match_list_data(h))
            weakref.finalize(buf, self.dll.hepfac_match_list_destroy, h)
            return np.frombuffer(buf, dtype=MATCH_DTYPE)
        try:
            out = np.empty(n, dtype=MATCH_DTYPE)
            if n:
                C.memmove(out.ctypes.data, self.dll.hepfac_match_list_data(h), n * MATCH_DTYPE.itemsize)
            return out
        finally:
            self.dll.hepfac_match_list_destroy(h)

    def scan(self, trie: "Trie", text, workers: int = 0, chunk: int = 0, view: bool = False) -> np.ndarray:
        """hepfac_scan: every occurrence sorted by (start, length, pattern_id)
        (view=True: zero-copy over the library's list, see _list)."""
        arr = _as_u8(text)
        cfg = _ScanConfig(workers, chunk)
        h = C.c_void_p()
        self.check(self.dll.hepfac_scan(trie.h, _ptr(arr), arr.size, C.byref(cfg), C.byref(h)))
        return self._list(h, view)

    def scan_two_stage(self, trie: "Trie", text, workers: int = 0, chunk: int = 0) -> np.ndarray:
        """Reference scan_two_stage (scan.cpp:121-129): a scan that requires a truncated trie."""
        if trie.depth_limit() is None:
            raise HepfacError(INVALID_ARG, "two-stage scan requires a depth-truncated trie")
        return self.scan(trie, text, workers, chunk)

    def run_throughput(self, trie: "Trie", text, runs: int = 3, workers: int = 0, chunk: int = 0) -> dict:
        arr = _as_u8(text)
        cfg = _ScanConfig(workers, chunk)
        rep = _Throughput()
        self.check(self.dll.hepfac_run_throughput(trie.h, _ptr(arr), arr.size, C.byref(cfg), runs, C.byref(rep)))
        return {f: getattr(rep, f) for f, _ in _Throughput._fields_}

    # -- reports ------------------------------------------------------------
    def compare_footprint(self, node_count: int, sigma: int) -> dict:
        r = _Comparison()
        self.check(self.dll.hepfac_compare_footprint(node_count, sigma, C.byref(r)))
        return {f: getattr(r, f) for f, _ in _Comparison._fields_}

    def reduction_estimate(self, sigma: int, n: int, trials: int, seed: int) -> dict:
        r = _Reduction()
        self.check(self.dll.hepfac_reduction_estimate(sigma, n, trials, seed, C.byref(r)))
        return {f: getattr(r, f) for f, _ in _Reduction._fields_}

    # -- B200 extensions -------------------------------------------------------
    def device_count(self) -> int:
        return self.dll.hepfac_b200_device_count()

    def halo(self, trie: "Trie") -> Optional[int]:
        """Bytes of right context a shard needs; None when unbounded (a cyclic
        loaded trie: hepfac_b200_halo reports UINT64_MAX)."""
        v = C.c_uint64()
        self.check(self.dll.hepfac_b200_halo(trie.h, C.byref(v)))
        return None if v.value == (1 << 64) - 1 else v.value

    def scan_shard(self, trie: "Trie", text, offset: int, owned: int, view: bool = False) -> np.ndarray:
        arr = _as_u8(text)
        h = C.c_void_p()
        self.check(self.dll.hepfac_b200_scan_shard(trie.h, _ptr(arr), arr.size, offset, owned, C.byref(h)))
        return self._list(h, view)

    def last_scan_stats(self) -> dict:
        s = _ScanStats()
        self.check(self.dll.hepfac_b200_last_scan_stats(C.byref(s)))
        return {f: getattr(s, f) for f, _ in _ScanStats._fields_}

    def trim(self) -> None:
        """hepfac_b200_trim: free pooled workspaces and pinned blocks."""
        self.check(self.dll.hepfac_b200_trim())

    def layout_info(self, trie: "Trie") -> dict:
        s = _LayoutInfo()
        self.check(self.dll.hepfac_b200_layout_info(trie.h, C.byref(s)))
        return {f: getattr(s, f) for f, _ in _LayoutInfo._fields_}

    def session(self, trie: "Trie", text, offset: int = 0, owned: Optional[int] = None) -> "Session":
        return Session(self, trie, text, offset, owned)


class Alphabet:
    def __init__(self, lib: Library, spec):
        self.lib, self.h = lib, C.c_void_p()
        if isinstance(spec, int):
            lib.check(lib.dll.hepfac_alphabet_standard(spec, C.byref(self.h)))
        else:
            arr = _as_u8(spec)
            lib.check(lib.dll.hepfac_alphabet_create(_ptr(arr) or C.c_void_p(1), arr.size, C.byref(self.h)))

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.dll.hepfac_alphabet_destroy(self.h)
            self.h = None

    def size(self) -> int:
        return self.lib.dll.hepfac_alphabet_size(self.h)

    def symbol(self, byte: int) -> int:
        return self.lib.dll.hepfac_alphabet_symbol(self.h, byte)


class PatternSet:
    def __init__(self, lib: Library, h, alphabet: Alphabet):
        self.lib, self.h, self.alphabet = lib, h, alphabet

    @classmethod
    def create(cls, lib: Library, patterns: Sequence[Union[bytes, str]], alphabet: Alphabet) -> "PatternSet":
        raw = [p.encode("latin-1") if isinstance(p, str) else bytes(p) for p in patterns]
        bufs = [C.create_string_buffer(p, len(p)) for p in raw]
        ptrs = (C.c_void_p * max(1, len(raw)))(*[C.cast(b, C.c_void_p) for b in bufs])
        lens = (C.c_size_t * max(1, len(raw)))(*[len(p) for p in raw])
        h = C.c_void_p()
        lib.check(lib.dll.hepfac_patterns_create(ptrs, lens, len(raw), alphabet.h, C.byref(h)))
        return cls(lib, h, alphabet)

    @classmethod
    def generate(cls, lib: Library, seed: int, alphabet: Alphabet, count: int, length: int) -> "PatternSet":
        h = C.c_void_p()
        lib.check(lib.dll.hepfac_patterns_generate(seed, alphabet.h, count, length, C.byref(h)))
        return cls(lib, h, alphabet)

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.dll.hepfac_patterns_destroy(self.h)
            self.h = None

    def count(self) -> int:
        return self.lib.dll.hepfac_patterns_count(self.h)

    def get(self, i: int) -> bytes:
        n = C.c_size_t()
        p = self.lib.dll.hepfac_patterns_get(self.h, i, C.byref(n))
        if not p:
            raise IndexError(i)
        return C.string_at(p, n.value)

    def to_list(self):
        return [self.get(i) for i in range(self.count())]

    def save(self, path: str):
        self.lib.check(self.lib.dll.hepfac_patterns_save(self.h, path.encode()))

    def unique_prefix(self) -> int:
        v = C.c_uint32()
        self.lib.check(self.lib.dll.hepfac_patterns_unique_prefix(self.h, C.byref(v)))
        return v.value

    def choose_depth(self) -> int:
        v = C.c_uint32()
        self.lib.check(self.lib.dll.hepfac_patterns_choose_depth(self.h, C.byref(v)))
        return v.value


@dataclass
class CompressionStats:
    nodes_before: int
    nodes_after_stage1: int
    nodes_after_stage2: int
    pattern_count: int
    reduction_percent: float


class Trie:
    def __init__(self, lib: Library, h):
        self.lib, self.h = lib, h

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.dll.hepfac_trie_destroy(self.h)
            self.h = None

    def node_count(self) -> int:
        return self.lib.dll.hepfac_trie_node_count(self.h)

    def sigma(self) -> int:
        return self.lib.dll.hepfac_trie_sigma(self.h)

    def stage(self) -> int:
        return self.lib.dll.hepfac_trie_stage(self.h)

    def depth_limit(self) -> Optional[int]:
        d = C.c_uint32()
        return d.value if self.lib.dll.hepfac_trie_depth_limit(self.h, C.byref(d)) else None

    def transition(self, node: int, byte: int) -> int:
        v = C.c_uint32()
        self.lib.check(self.lib.dll.hepfac_trie_transition(self.h, node, byte, C.byref(v)))
        return v.value

    def terminal(self, node: int) -> bool:
        return bool(self.lib.dll.hepfac_trie_terminal(self.h, node))

    def memory_report(self) -> dict:
        r = _MemoryReport()
        self.lib.check(self.lib.dll.hepfac_trie_memory_report(self.h, C.byref(r)))
        return {"node_count": r.node_count, "bytes_per_node": r.bytes_per_node, "total_bytes": r.total_bytes,
                "sigma": r.sigma, "total_mib": r.total_mib.decode()}

    def compress(self, stages: int = 2):
        st = _CompressionStats()
        h = C.c_void_p()
        self.lib.check(self.lib.dll.hepfac_trie_compress_stats(self.h, stages, C.byref(h), C.byref(st)))
        return Trie(self.lib, h), CompressionStats(st.nodes_before, st.nodes_after_stage1, st.nodes_after_stage2,
                                                   st.pattern_count, st.reduction_percent)

    def merge_final_nodes(self):
        return self.compress(1)

    def truncate(self, depth: int):
        h = C.c_void_p()
        noop = C.c_int(-1)
        self.lib.check(self.lib.dll.hepfac_trie_truncate(self.h, depth, C.byref(h), C.byref(noop)))
        return Trie(self.lib, h), bool(noop.value)

    def save(self, path: str):
        self.lib.check(self.lib.dll.hepfac_trie_save(self.h, path.encode()))

    def save_bytes(self) -> bytes:
        import tempfile
        with tempfile.TemporaryDirectory() as d:
            p = os.path.join(d, "t.htri")
            self.save(p)
            with open(p, "rb") as f:
                return f.read()


class Session:
    """Device-resident benchmark session (hepfac_b200_session_*)."""

    def __init__(self, lib: Library, trie: Trie, text, offset: int = 0, owned: Optional[int] = None):
        self.lib, self.trie = lib, trie
        arr = _as_u8(text)
        self.h = C.c_void_p()
        owned = arr.size if owned is None else owned
        lib.check(lib.dll.hepfac_b200_session_create(trie.h, _ptr(arr), arr.size, offset, owned, C.byref(self.h)))
        self.bytes, self.owned = arr.size, owned

    def run(self, iterations: int, flush_l2: bool = False):
        ms = (C.c_double * max(1, iterations))()
        m = C.c_uint64()
        self.lib.check(self.lib.dll.hepfac_b200_session_run(self.h, iterations, int(flush_l2), ms, C.byref(m)))
        return list(ms)[:iterations], m.value

    def kernel_ms(self, iterations: int):
        """Per-kernel device ms of the last run: (first pass, second pass, kernels per scan)."""
        a = (C.c_double * max(1, iterations))()
        b = (C.c_double * max(1, iterations))()
        k = C.c_uint32()
        self.lib.check(self.lib.dll.hepfac_b200_session_kernel_ms(self.h, iterations, a, b, C.byref(k)))
        return list(a)[:iterations], list(b)[:iterations], k.value

    def fetch(self) -> np.ndarray:
        h = C.c_void_p()
        self.lib.check(self.lib.dll.hepfac_b200_session_fetch(self.h, C.byref(h)))
        return self.lib._list(h)

    def close(self):
        if getattr(self, "h", None):
            self.lib.dll.hepfac_b200_session_destroy(self.h)
            self.h = None

    __del__ = close


_default: Optional[Library] = None


def lib() -> Library:
    """The product library (built in-tree); raises if it was not built."""
    global _default
    if _default is None:
        _default = Library(LIB_PATH)
    return _default
