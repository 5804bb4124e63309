"""B200-native PFAC matcher (arXiv 1704.02272) behind the reference's C ABI.

The product is ``libhepfac.so`` (csrc/: host trie compiler + sm_100a CUDA
engine); ``hepfac`` is its ctypes mirror.
"""
from .hepfac import (ABI_SYMBOLS, B200_SYMBOLS, MATCH_DTYPE, HepfacError, Library, lib)  # noqa: F401

__all__ = ["ABI_SYMBOLS", "B200_SYMBOLS", "MATCH_DTYPE", "HepfacError", "Library", "lib"]
