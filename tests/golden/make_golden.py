#!/usr/bin/env python
"""Generates the golden fixtures in this directory by running the UNMODIFIED
reference library (compiled from /root/reference/proj/src into oracle/_ref by
oracle/Makefile).  Run in the source container:

    make -C oracle ref && python tests/golden/make_golden.py

Outputs
  tries.json  -- per seeded pattern set: node counts and SHA-256 of the .htri
                 bytes for stage 0/1/2 and truncations (trie compiler parity)
  scans.npz   -- seeded instances (patterns, text, trie state) with the
                 reference hepfac_scan result (match-path parity)
  config4.json-- config-4 sweep (10k x len 20, derive_seed(42, sigma, 10000)):
                 node counts, reduction %, choose_depth
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle  # noqa: E402
from helpers import pattern_set, plant, text  # noqa: E402
from paper_1704_02272_b200 import workloads  # noqa: E402


def instances():
    """(name, sigma, patterns, text, state) -- small, seeded."""
    out = []
    rng = np.random.default_rng(777)
    for i, sigma in enumerate([2, 4, 20, 52, 64, 128, 256, 4, 52, 256, 256, 4]):
        R = oracle.ref_library()
        a = R.alphabet(sigma)
        syms = np.array([b for b in range(256) if a.symbol(b) >= 0], dtype=np.uint8)
        lo, hi = (1, 6) if i % 3 == 0 else (2, 20)
        pats = pattern_set(rng, syms, int(rng.integers(5, 150)), lo, hi)
        tx = text(rng, syms, int(rng.integers(2000, 20000)))
        for k in range(len(pats)):
            plant(tx, pats[k], int(rng.integers(0, tx.size)))
        state = ["full", "stage1", "stage2", "trunc1", "trunc2", "trunc5", "s1trunc3"][i % 7]
        out.append((f"inst{i}_s{sigma}_{state}", sigma, pats, tx, state))
    return out


def make_trie(lib, sigma, pats, state):
    a = lib.alphabet(sigma)
    t = lib.build_trie(lib.patterns(pats, a))
    if state == "stage1":
        return t.compress(1)[0]
    if state == "stage2":
        return t.compress(2)[0]
    if state.startswith("trunc"):
        tr, noop = t.truncate(int(state[5:]))
        return tr
    if state.startswith("s1trunc"):
        tr, noop = t.compress(1)[0].truncate(int(state[7:]))
        return tr
    return t


def main():
    R = oracle.ref_library()
    assert R is not None, "build oracle/_ref first (make -C oracle ref)"

    # trie compiler fixtures
    tries = []
    rng = np.random.default_rng(4242)
    for sigma in (2, 4, 20, 52, 128, 256):
        a = R.alphabet(sigma)
        syms = np.array([b for b in range(256) if a.symbol(b) >= 0], dtype=np.uint8)
        for rep in range(3):
            pats = pattern_set(rng, syms, int(rng.integers(20, 400)), 1 + rep, 8 + 6 * rep)
            rec = {"sigma": sigma, "patterns": [p.hex() for p in pats], "tries": {}}
            for state in ("full", "stage1", "stage2", "trunc1", "trunc3", "s1trunc2", "s1trunc4"):
                try:
                    t = make_trie(R, sigma, pats, state)
                except Exception as e:  # e.g. truncation no-op collisions
                    rec["tries"][state] = {"error": str(e)}
                    continue
                b = t.save_bytes()
                rec["tries"][state] = {"nodes": t.node_count(), "sha256": hashlib.sha256(b).hexdigest(),
                                       "bytes": len(b)}
            tries.append(rec)
    with open(os.path.join(HERE, "tries.json"), "w") as f:
        json.dump(tries, f, indent=0)

    # match-path fixtures
    arrays = {}
    meta = []
    for name, sigma, pats, tx, state in instances():
        t = make_trie(R, sigma, pats, state)
        res = R.scan(t, tx, workers=3, chunk=1009)
        arrays[name + "/text"] = tx
        arrays[name + "/pat_blob"] = np.frombuffer(b"".join(pats), dtype=np.uint8)
        arrays[name + "/pat_len"] = np.array([len(p) for p in pats], dtype=np.uint32)
        arrays[name + "/matches"] = res
        meta.append({"name": name, "sigma": sigma, "state": state, "matches": int(res.size)})
    np.savez_compressed(os.path.join(HERE, "scans.npz"), **arrays)
    with open(os.path.join(HERE, "scans.json"), "w") as f:
        json.dump(meta, f, indent=1)

    # config-4 sweep (node counts are deterministic API outputs)
    c4 = []
    for sigma in (2, 4, 20, 64, 128, 256):
        a = R.alphabet(sigma)
        ps = R.generate_patterns(workloads.derive_seed(42, sigma, 10000), a, 10000, 20)
        t = R.build_trie(ps)
        s2, st = t.compress(2)
        mem = s2.memory_report()
        c4.append({"sigma": sigma, "nodes": st.nodes_before, "stage1": st.nodes_after_stage1,
                   "stage2": st.nodes_after_stage2, "reduction_percent": st.reduction_percent,
                   "choose_depth": ps.choose_depth(), "bytes_per_node": mem["bytes_per_node"],
                   "stage2_total_bytes": mem["total_bytes"],
                   "first_pattern": ps.get(0).hex(), "last_pattern": ps.get(9999).hex()})
    with open(os.path.join(HERE, "config4.json"), "w") as f:
        json.dump(c4, f, indent=1)
    print("wrote", len(tries), "trie fixtures,", len(meta), "scan fixtures, config4", [r["stage2"] for r in c4])


if __name__ == "__main__":
    main()
