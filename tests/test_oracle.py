"""Pins the oracle before it is trusted (CPU only): the C restatement
(oracle/pfac_oracle.c) against the reference's golden vectors, the committed
fixtures made by running the reference, and the compiled reference itself."""
import os

import numpy as np
import pytest

import oracle
from helpers import as_tuples, pattern_set, plant, same, text

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def htri(lib, pats, sigma=256, stages=0, depth=None):
    t = lib.build_trie(lib.patterns(pats, lib.alphabet(sigma)))
    if stages:
        t = t.compress(stages)[0]
    if depth:
        t = t.truncate(depth)[0]
    return t.save_bytes()


def test_known_answers(lib):
    kat = [(2, 2, 2), (2, 6, 0), (10, 6, 1), (18, 2, 2)]  # test_capi.cpp:81-96
    pats = [b"ABCXYZ", b"DEFXYZ", b"AB"]
    txt = b"xxABCXYZ--DEFXYZ++ABq"
    assert as_tuples(oracle.naive_find_all(txt, pats)) == kat
    for stages in (0, 1, 2):
        assert as_tuples(oracle.walk_scan(htri(lib, pats, stages=stages), txt)) == kat
    assert as_tuples(oracle.walk_scan(htri(lib, pats, depth=2), txt)) == kat
    # test_scan.cpp:19-41, 90-101
    assert as_tuples(oracle.walk_scan(htri(lib, [b"AB"]), b"XABY")) == [(1, 2, 0)]
    assert as_tuples(oracle.walk_scan(htri(lib, [b"AB", b"ABC"]), b"ABC")) == [(0, 2, 0), (0, 3, 1)]
    hits = oracle.walk_scan(htri(lib, [b"ABAB"]), b"AB" * 50)
    assert list(hits["start"]) == list(range(0, 97, 2))


def test_oracle_transition_matches_library(lib):
    pats = [b"AB", b"AD", b"C"]
    tr = oracle.HtriTrie(htri(lib, pats))
    t = lib.build_trie(lib.patterns(pats, lib.alphabet(256)))
    for node in range(t.node_count()):
        for byte in range(256):
            assert tr.transition(node, byte) == t.transition(node, byte)


def test_golden_scan_fixtures_naive_and_walk(lib):
    z = np.load(os.path.join(GOLDEN, "scans.npz"))
    names = sorted({k.split("/")[0] for k in z.files})
    assert len(names) >= 12
    for name in names:
        tx = z[name + "/text"]
        blob, lens = z[name + "/pat_blob"].tobytes(), z[name + "/pat_len"]
        offs = np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(int)
        pats = [blob[o:o + n] for o, n in zip(offs, lens)]
        want = z[name + "/matches"]
        assert same(oracle.naive_find_all(tx, pats), want), name
        sigma = int(name.split("_s")[1].split("_")[0])
        state = name.split("_")[-1]
        t = lib.build_trie(lib.patterns(pats, lib.alphabet(sigma)))
        if state == "stage1":
            t = t.compress(1)[0]
        elif state == "stage2":
            t = t.compress(2)[0]
        elif state.startswith("trunc"):
            t = t.truncate(int(state[5:]))[0]
        elif state.startswith("s1trunc"):
            t = t.compress(1)[0].truncate(int(state[7:]))[0]
        assert same(oracle.walk_scan(t.save_bytes(), tx), want), name


@pytest.mark.parametrize("sigma", [4, 52, 256])
def test_oracles_equal_reference_scan(lib, ref, sigma):
    # acceptance.cpp:101-150 in miniature: every trie state, reference scan as truth
    rng = np.random.default_rng(sigma + 99)
    a = ref.alphabet(sigma)
    syms = np.array([b for b in range(256) if a.symbol(b) >= 0], dtype=np.uint8)
    for rep in range(8):
        pats = pattern_set(rng, syms, int(rng.integers(1, 120)), 2, 20)
        tx = text(rng, syms, int(rng.integers(1024, 16384)))
        for k in range(len(pats) // 3 + 1):
            plant(tx, pats[int(rng.integers(0, len(pats)))], int(rng.integers(0, tx.size)))
        want = oracle.naive_find_all(tx, pats)
        t = ref.build_trie(ref.patterns(pats, a))
        assert same(ref.scan(t, tx, workers=2, chunk=1009), want)
        for tt in (t, t.compress(1)[0], t.compress(2)[0]):
            assert same(oracle.walk_scan(tt.save_bytes(), tx), want)
        for d in (1, 2, 5, 8):
            tr, noop = t.truncate(d)
            if noop:
                continue
            assert same(ref.scan(tr, tx, workers=2, chunk=1009), want)
            assert same(oracle.walk_scan(tr.save_bytes(), tx), want)


def test_oracle_reports_foreign_terminal(lib):
    # A terminal spelling no dictionary pattern is the reference's logic_error
    # (scan.cpp:34); hand-edit a .htri so "AB"'s dictionary entry says "AC".
    b = bytearray(htri(lib, [b"AB"]))
    i = b.index(b"AB", 4)
    b[i + 1] = ord("C")
    with pytest.raises(RuntimeError):
        oracle.walk_scan(bytes(b), b"xxAByy")
