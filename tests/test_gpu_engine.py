"""GPU engine behaviour behind hepfac_scan: how host text reaches the device
(pageable text through the pinned staging ring, pinned text and device
pointers copied directly), the overlapped per-chunk D2H into pinned match
lists, kernel attributes shared between tries, pool trimming, run_throughput
on tries that cannot match, and the stronger .htri validation.

The bar is the same as test_gpu_parity.py: bit-exact hepfac_match_t arrays
against the oracle (naive_find_all, reference naive_search.hpp:17-31).
"""
import struct

import numpy as np
import pytest

import oracle
from helpers import pattern_set, plant, same, text

pytestmark = pytest.mark.gpu


def build(lib, pats, sigma=256, stages=0, depth=None):
    a = lib.alphabet(sigma)
    t = lib.build_trie(lib.patterns(pats, a))
    if stages:
        t, _ = t.compress(stages)
    if depth is not None:
        t, _ = t.truncate(depth)
    return t


def dense_instance(seed, sigma=256, mib=5, count=400, lo=4, hi=24, every=61):
    """A text with many planted matches (so match lists exceed the 1 MiB
    pinned-list threshold) and occurrences straddling 1 MiB chunk seams."""
    rng = np.random.default_rng(seed)
    _, syms = alphabet_bytes_np(sigma)
    pats = pattern_set(rng, syms, count, lo, hi)
    tx = text(rng, syms, mib * (1 << 20) + 777)
    for i in range(0, tx.size - 64, every):
        plant(tx, pats[i % len(pats)], i)
    for c in range(1 << 20, tx.size, 1 << 20):
        p = pats[c % len(pats)]
        plant(tx, p, c - len(p) // 2)
    return pats, tx


def alphabet_bytes_np(sigma):
    from paper_1704_02272_b200 import workloads
    return None, np.frombuffer(workloads.standard_symbols(sigma), dtype=np.uint8).copy()


@pytest.mark.parametrize("two_pass", [False, True])
def test_pageable_pinned_and_device_inputs_agree(gpu, monkeypatch, two_pass):
    # hepfac_scan borrows any host pointer (reference capi.cpp:393-401; the
    # reference CLI passes a pageable std::vector, hepfac_cli.cpp:247-255).
    # Pageable text goes through the pinned staging ring, pinned text is
    # copied directly, and a device pointer (UVA) is read in place; 1 MiB
    # chunks give many seams and per-chunk D2H of the records.
    import torch

    if two_pass:
        monkeypatch.setenv("HEPFAC_PIPELINE_MIN_MIB", "0")
    monkeypatch.setenv("HEPFAC_CHUNK_MIB", "1")
    pats, tx = dense_instance(5)
    t = build(gpu, pats, 256, 2)
    want = oracle.naive_find_all(tx, pats)
    assert want.size * 16 > (1 << 20)  # the list is pinned-pool backed

    got = gpu.scan(t, tx)  # numpy array: pageable
    st = gpu.last_scan_stats()
    assert st["staged"] == 1 and st["chunks"] == 6
    assert same(got, want)

    pinned = torch.empty(tx.size, dtype=torch.uint8, pin_memory=True)
    pinned.numpy()[:] = tx
    got = gpu.scan(t, pinned.numpy())
    assert gpu.last_scan_stats()["staged"] == 0
    assert same(got, want)

    dev = torch.from_numpy(tx).cuda()
    torch.cuda.synchronize()
    from paper_1704_02272_b200 import hepfac as H
    import ctypes as C
    h = C.c_void_p()
    cfg = H._ScanConfig(0, 0)
    gpu.check(gpu.dll.hepfac_scan(t.h, C.c_void_p(dev.data_ptr()), tx.size, C.byref(cfg), C.byref(h)))
    assert gpu.last_scan_stats()["staged"] == 0
    assert same(gpu._list(h), want)


def test_many_small_pageable_scans(gpu, monkeypatch):
    # Each staging piece is one batch of the host copy pool (helpers spin
    # between pieces, then sleep); hundreds of short scans with 1 MiB pieces
    # exercise the hand-off between the caller and the helpers.
    monkeypatch.setenv("HEPFAC_STAGE_MIB", "1")
    rng = np.random.default_rng(31)
    syms = np.arange(256, dtype=np.uint8)
    pats = pattern_set(rng, syms, 300, 4, 16)
    t = build(gpu, pats, 256, 1)
    tx = text(rng, syms, (5 << 20) + 13)
    for i in range(0, tx.size - 64, 4099):
        plant(tx, pats[i % len(pats)], i)
    want = oracle.naive_find_all(tx, pats)
    for k in range(300):
        n = tx.size - 4096 * (k % 7)
        got = gpu.scan(t, tx[:n])
        assert gpu.last_scan_stats()["staged"] == 1
        assert same(got, want[want["start"] + want["length"] <= n])


def test_match_list_growth_and_reuse(gpu, monkeypatch):
    # The host list is reserved from the first chunks' record rate and grown
    # when a later chunk outruns it; repeated scans reuse pooled pinned blocks.
    monkeypatch.setenv("HEPFAC_CHUNK_MIB", "1")
    rng = np.random.default_rng(9)
    syms = np.frombuffer(b"ACGT", dtype=np.uint8)
    pats = pattern_set(rng, syms, 200, 3, 9)
    tx = text(rng, syms, 4 * (1 << 20) + 99)
    tx[: 1 << 20] = ord("N")  # chunk 0: no matches (outside the alphabet), later chunks: many
    t = build(gpu, pats, 4)
    want = oracle.naive_find_all(tx, pats)
    for _ in range(3):
        assert same(gpu.scan(t, tx), want)
    gpu.trim()
    assert same(gpu.scan(t, tx), want)


def test_kernel_smem_cap_survives_smaller_trie(gpu):
    # the dynamic shared-memory cap is a property of the
    # kernel function, shared by every trie with the same kernel choice.
    # Big trie (2^20-bit filter), then a small one, then the big one again.
    rng = np.random.default_rng(77)
    syms = np.arange(256, dtype=np.uint8)
    big_p = pattern_set(rng, syms, 20000, 4, 32)
    small_p = pattern_set(rng, syms, 40, 4, 32)
    big, small = build(gpu, big_p, 256, 1), build(gpu, small_p, 256, 1)
    assert gpu.layout_info(big)["smem_bytes"] > gpu.layout_info(small)["smem_bytes"]
    tx = text(rng, syms, 3 << 20)
    for i in range(0, tx.size - 64, 1021):
        plant(tx, (big_p if i % 2 else small_p)[i % 40], i)
    wb, ws = oracle.naive_find_all(tx, big_p), oracle.naive_find_all(tx, small_p)
    assert same(gpu.scan(big, tx), wb)
    assert same(gpu.scan(small, tx), ws)
    assert same(gpu.scan(big, tx), wb)


def test_run_throughput_times_unmatchable_trie(gpu):
    # The reference always times its runs (bench.cpp:64-76); a trie whose
    # shortest pattern is longer than the text still reports seconds > 0.
    t = build(gpu, [b"ABCDEFGHIJ"])
    rep = gpu.run_throughput(t, b"ABC" * 3, runs=3)
    assert rep["seconds"] > 0 and rep["matches"] == 0 and rep["gbps"] > 0


def test_htri_child_run_past_node_array_is_format_error(gpu, tmp_path):
    # The format checks only offset < node_count (reference
    # trie_io.cpp:155-159).  A root whose child run starts at the last node
    # passes that check but would send walks past the node array; the GPU
    # image builder refuses it: HEPFAC_ERR_FORMAT, no device fault, and the
    # library keeps working afterwards.
    from paper_1704_02272_b200 import hepfac as H
    t = build(gpu, [b"AB", b"XYZW"])
    raw = bytearray(t.save_bytes())
    assert raw[:4] == b"HTRI"
    _, sigma, n, words = struct.unpack_from("<HHIH", raw, 4)
    stride = 4 * (words + 1)
    root_off = 14 + 4 * words  # node 0's offset word
    (cell,) = struct.unpack_from("<I", raw, root_off)
    assert cell & 0x7FFFFFFF == 1  # children of the root start at node 1
    struct.pack_into("<I", raw, root_off, (cell & 0x80000000) | (n - 1))
    p = str(tmp_path / "bad.htri")
    open(p, "wb").write(bytes(raw))
    bad = gpu.load_trie(p)  # the format itself accepts it, like the reference
    assert bad.node_count() == n and stride > 0
    with pytest.raises(H.HepfacError) as e:
        gpu.scan(bad, b"xxAByyXYZW")
    assert e.value.status == H.FORMAT and "child run" in e.value.message
    assert gpu.scan(t, b"xxAByyXYZW").size == 2


def test_output_invariant_across_engine_configurations(gpu, monkeypatch):
    # The reference asserts byte-identical output for every worker count and
    # chunk size (acceptance.cpp:274-332, test_scan.cpp:43-56).  Here the
    # same list must come out of every engine configuration: one-pass fused
    # kernel or two-pass pipeline (or pair tries kept on the fused kernel), 1 MiB or
    # 64 MiB chunks, one device or three shards, and any scan config.
    pats, tx = dense_instance(21, mib=3, every=509)
    t = build(gpu, pats, 256, 1, 5)
    want = oracle.naive_find_all(tx, pats)
    combos = [{}, {"HEPFAC_PIPELINE_MIN_MIB": "0"}, {"HEPFAC_PIPELINE_MIN_MIB": "0", "HEPFAC_PAIR_PIPELINE": "0"},
              {"HEPFAC_CHUNK_MIB": "1"}, {"HEPFAC_CHUNK_MIB": "1", "HEPFAC_PIPELINE_MIN_MIB": "0"},
              {"HEPFAC_DEVICES": "0,0,0"}, {"HEPFAC_DEVICES": "0,0", "HEPFAC_PIPELINE_MIN_MIB": "0"}]
    keys = {k for c in combos for k in c}
    for c in combos:
        for k in keys:
            monkeypatch.delenv(k, raising=False)
        for k, v in c.items():
            monkeypatch.setenv(k, v)
        for workers, chunk in ((0, 0), (1, 1), (8, 4096)):
            got = gpu.scan(t, tx, workers=workers, chunk=chunk)
            assert got.tobytes() == want.tobytes(), (c, workers, chunk)
