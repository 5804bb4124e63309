#!/usr/bin/env python
"""Small scans covering every kernel form, for compute-sanitizer runs
(scripts/sanitize.sh): the fused one-pass kernel (byte keys, single-probe and
pair filters), the two-pass pipeline (pair filter pass, queue and in-lane
forms, + the cooperative walking pass), the packed-symbol pipeline (pack +
symbol filter + walking pass), the streamed path (several chunks, pinned
staging, per-chunk D2H) and the device-resident session.  Each result is
checked against the C oracle, so a run that passes the sanitizer also passed
parity.  Usage: python scripts/sanitize_cases.py [case ...]"""
import os
import sys
import zlib

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle  # noqa: E402
from helpers import pattern_set, plant, text  # noqa: E402
from paper_1704_02272_b200 import hepfac, workloads  # noqa: E402

lib = hepfac.lib()


def instance(sigma, count, lo, hi, nbytes, seed):
    rng = np.random.default_rng(seed)
    syms = np.frombuffer(workloads.standard_symbols(sigma), dtype=np.uint8)
    pats = pattern_set(rng, syms, count, lo, hi)
    tx = text(rng, syms, nbytes)
    for i in range(0, tx.size - 64, 997):
        plant(tx, pats[i % len(pats)], i)
    return pats, tx


def run(name, sigma, count, lo, hi, nbytes, stages=1, depth=None, env=None, session=False):
    for k, v in (env or {}).items():
        os.environ[k] = v
    try:
        pats, tx = instance(sigma, count, lo, hi, nbytes, zlib.crc32(name.encode()) & 0xFFFF)
        t = lib.build_trie(lib.patterns(pats, lib.alphabet(sigma)))
        if stages:
            t, _ = t.compress(stages)
        if depth:
            t, _ = t.truncate(depth)
        want = oracle.naive_find_all(tx, pats)
        if session:
            s = lib.session(t, tx)
            s.run(2)
            got = s.fetch()
            s.close()
        else:
            got = lib.scan(t, tx)
        info = lib.layout_info(t)
        ok = got.shape == want.shape and bool(np.array_equal(got, want))
        print(f"{name}: filter_mode {info['filter_mode']} launches {lib.last_scan_stats()['kernel_launches']} "
              f"matches {got.size} {'ok' if ok else 'MISMATCH'}", flush=True)
        if not ok:
            raise SystemExit(1)
    finally:
        for k in (env or {}):
            os.environ.pop(k, None)


CASES = {
    "fused_pair": lambda: run("fused_pair", 256, 300, 4, 20, 1 << 20),
    "fused_single": lambda: run("fused_single", 20, 300, 6, 20, 1 << 20, env={"HEPFAC_FILTER_MODE": "single"}),
    "fused_dna": lambda: run("fused_dna", 4, 300, 8, 20, 1 << 20, stages=2),
    "two_pass_pair": lambda: run("two_pass_pair", 256, 300, 4, 20, 1 << 20, depth=4,
                                 env={"HEPFAC_PIPELINE_MIN_MIB": "0"}),
    "two_pass_pair_l2": lambda: run("two_pass_pair_l2", 256, 30000, 4, 24, 1 << 16,
                                    env={"HEPFAC_PIPELINE_MIN_MIB": "0"}),
    "two_pass_l2": lambda: run("two_pass_l2", 256, 300, 4, 20, 1 << 20, env={"HEPFAC_PIPELINE_MIN_MIB": "0",
                                                                            "HEPFAC_FILTER_MODE": "l2"}),
    "symbol": lambda: run("symbol", 4, 200, 12, 24, 1 << 20, stages=2),
    "streamed": lambda: run("streamed", 256, 300, 4, 40, 3 << 20, stages=2, env={"HEPFAC_CHUNK_MIB": "1"}),
    "session": lambda: run("session", 256, 300, 4, 20, 1 << 20, session=True,
                           env={"HEPFAC_PIPELINE_MIN_MIB": "0"}),
}

if __name__ == "__main__":
    for c in sys.argv[1:] or list(CASES):
        CASES[c]()
