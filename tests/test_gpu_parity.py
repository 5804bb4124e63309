"""GPU parity: hepfac_scan (sm_100a kernel, called through the C ABI) against
the oracles.  Bar: bit-exact hepfac_match_t arrays.

Cases follow the reference's own tests: test_capi.cpp:30-100 (end-to-end KAT),
test_scan.cpp:19-143 (single offsets, nesting, brute-force equality, unit
boundaries, periodic overlaps, two-stage), acceptance.cpp:101-150 (criteria 3
and 4: random instances, all trie states, truncation depths {1,2,5,8}).
"""
import os

import numpy as np
import pytest

import oracle
from helpers import alphabet_bytes, as_tuples, pattern_set, plant, same, text

pytestmark = pytest.mark.gpu


def build(lib, pats, sigma=256, stages=0, depth=None):
    a = lib.alphabet(sigma)
    t = lib.build_trie(lib.patterns(pats, a))
    if stages:
        t, _ = t.compress(stages)
    if depth is not None:
        t, noop = t.truncate(depth)
    return t


def test_capi_end_to_end_known_answer(gpu, tmp_path):
    # test_capi.cpp:30-100: stage-2 trie, saved, loaded, scanned.
    t = build(gpu, [b"ABCXYZ", b"DEFXYZ", b"AB"], stages=2)
    path = str(tmp_path / "t.htri")
    t.save(path)
    loaded = gpu.load_trie(path)
    assert loaded.node_count() == 9 and loaded.stage() == 2
    got = gpu.scan(loaded, b"xxABCXYZ--DEFXYZ++ABq", workers=2, chunk=8)
    assert as_tuples(got) == [(2, 2, 2), (2, 6, 0), (10, 6, 1), (18, 2, 2)]


def test_single_offsets_and_nesting(gpu):
    # test_scan.cpp:19-41
    assert as_tuples(gpu.scan(build(gpu, [b"AB"]), b"XABY")) == [(1, 2, 0)]
    assert as_tuples(gpu.scan(build(gpu, [b"AB", b"ABC"]), b"ABC")) == [(0, 2, 0), (0, 3, 1)]
    assert gpu.scan(build(gpu, [b"ACG"]), b"xyzxyzxyz").size == 0


def test_periodic_overlaps(gpu):
    # test_scan.cpp:90-101
    s = b"AB" * 50
    hits = gpu.scan(build(gpu, [b"ABAB"]), s)
    assert hits.size == (len(s) - 4) // 2 + 1
    assert list(hits["start"]) == [2 * i for i in range(hits.size)]


def test_empty_and_tiny_texts(gpu):
    t = build(gpu, [b"ABC", b"Q"])
    assert gpu.scan(t, b"").size == 0
    assert as_tuples(gpu.scan(t, b"Q")) == [(0, 1, 1)]
    assert gpu.scan(t, b"AB").size == 0
    assert as_tuples(gpu.scan(t, b"ABC")) == [(0, 3, 0)]


@pytest.mark.parametrize("two_pass", [False, True])
@pytest.mark.parametrize("sigma", [2, 4, 20, 52, 64, 128, 256])
def test_random_instances_all_states(gpu, monkeypatch, sigma, two_pass):
    # acceptance criteria 3 + 4 shape: random sets, planted + boundary copies.
    # two_pass: pair-filter tries on the two-pass pipeline even for small texts
    if two_pass:
        monkeypatch.setenv("HEPFAC_PIPELINE_MIN_MIB", "0")
    rng = np.random.default_rng(1000 + sigma)
    a, syms = alphabet_bytes(gpu, sigma)
    for rep in range(6):
        n = int(rng.integers(1, 200))
        pats = pattern_set(rng, syms, n, 2, 20)
        n = len(pats)
        tl = int(rng.integers(1024, 64 * 1024))
        tx = text(rng, syms, tl)
        for _ in range(n // 4 + 1):
            plant(tx, pats[int(rng.integers(0, n))], int(rng.integers(0, tl)))
        for c in range(4096 - 7, tl, 4096):  # astride kernel tile boundaries
            p = pats[int(rng.integers(0, n))]
            plant(tx, p, max(0, c - len(p) // 2))
        want = oracle.naive_find_all(tx, pats)
        full = build(gpu, pats, sigma)
        assert same(gpu.scan(full, tx), want), ("stage0", sigma, rep)
        s1, _ = full.compress(1)
        s2, _ = full.compress(2)
        assert same(gpu.scan(s1, tx), want), ("stage1", sigma, rep)
        assert same(gpu.scan(s2, tx), want), ("stage2", sigma, rep)
        for d in (1, 2, 5, 8):
            for base in (full, s1):
                tr, noop = base.truncate(d)
                if noop:
                    continue
                assert same(gpu.scan(tr, tx), want), ("trunc", d, sigma, rep)


def test_matches_walk_oracle_and_reference(gpu, ref):
    # Same trie bytes through three engines: GPU, C restatement, reference.
    rng = np.random.default_rng(5)
    a, syms = alphabet_bytes(gpu, 52)
    pats = pattern_set(rng, syms, 80, 6, 20)
    tx = text(rng, syms, 32768)
    for i in range(0, len(pats), 3):
        plant(tx, pats[i], int(rng.integers(0, 32000)))
    t = build(gpu, pats, 52, stages=1)
    tr, _ = t.truncate(5)
    ra = ref.alphabet(52)
    rt, _ = ref.build_trie(ref.patterns(pats, ra)).compress(1)
    rtr, _ = rt.truncate(5)
    assert tr.save_bytes() == rtr.save_bytes()
    want = ref.scan(rtr, tx, workers=2, chunk=512)
    assert same(oracle.walk_scan(tr.save_bytes(), tx), want)
    assert same(gpu.scan(tr, tx), want)


def test_long_patterns_beyond_shared_halo(gpu):
    # walks and verifications that read past the 64-byte shared-memory halo
    rng = np.random.default_rng(11)
    syms = np.arange(256, dtype=np.uint8)
    pats = [bytes(rng.integers(0, 256, size=n, dtype=np.uint8)) for n in (70, 150, 300, 1000, 5000)]
    pats.append(pats[0][:40])
    tx = text(rng, syms, 200000)
    for i, p in enumerate(pats):
        for k in range(3):
            plant(tx, p, 30000 * i + 9000 * k + 4095 - 17 * i)
    want = oracle.naive_find_all(tx, pats)
    assert want.size >= 15
    for stages, depth in ((0, None), (1, None), (2, None), (0, 3), (1, 33)):
        assert same(gpu.scan(build(gpu, pats, 256, stages, depth), tx), want), (stages, depth)


def test_bytes_outside_alphabet_kill_walks(gpu):
    pats = [b"ACGT", b"GATTACA", b"CC"]
    tx = b"ACGTxACGTNNGATTACACCxC" * 50
    want = oracle.naive_find_all(tx, pats)
    for stages in (0, 1, 2):
        assert same(gpu.scan(build(gpu, pats, 4, stages), tx), want)


def test_permuted_byte_alphabet(gpu):
    sym = bytes(np.random.default_rng(3).permutation(256).astype(np.uint8))
    a = gpu.alphabet(sym)
    rng = np.random.default_rng(4)
    pats = pattern_set(rng, np.arange(256, dtype=np.uint8), 100, 1, 6)
    t = gpu.build_trie(gpu.patterns(pats, a))
    tx = rng.integers(0, 256, size=200000, dtype=np.uint8)
    assert same(gpu.scan(t, tx), oracle.naive_find_all(tx, pats))


def test_dense_nested_matches_overflow_capacity(gpu):
    # every offset reports up to 32 nested patterns: forces the exact-size re-run
    pats = [b"A" * k for k in range(1, 33)]
    tx = b"A" * 300000
    got = gpu.scan(build(gpu, pats, 256), tx)
    n = len(tx)
    assert got.size == sum(n - k + 1 for k in range(1, 33))
    assert same(got, oracle.naive_find_all(tx, pats))
    assert gpu.last_scan_stats()["relaunches"] in (0, 1)


def test_text_sizes_around_tiles(gpu):
    rng = np.random.default_rng(9)
    syms = np.frombuffer(b"ACGT", dtype=np.uint8)
    pats = pattern_set(rng, syms, 300, 3, 9)
    t = build(gpu, pats, 4, 1)
    for n in (1, 2, 3, 15, 16, 17, 4095, 4096, 4097, 8191, 8192, 8193, 4096 * 37 + 5):
        tx = text(rng, syms, n)
        assert same(gpu.scan(t, tx), oracle.naive_find_all(tx, pats)), n


@pytest.mark.parametrize("two_pass", [False, True])
def test_shards_concatenate_to_full_scan(gpu, monkeypatch, two_pass):
    if two_pass:
        monkeypatch.setenv("HEPFAC_PIPELINE_MIN_MIB", "0")
    rng = np.random.default_rng(21)
    syms = np.arange(256, dtype=np.uint8)
    pats = pattern_set(rng, syms, 500, 2, 24)
    tx = text(rng, syms, 1 << 18)
    for i, p in enumerate(pats):
        plant(tx, p, (i * 523) % (tx.size - 30))
    t = build(gpu, pats, 256, 2)
    full = gpu.scan(t, tx)
    halo = gpu.halo(t)
    assert halo == 23
    N = tx.size
    for shards in (2, 3, 8):
        parts = []
        for g in range(shards):
            lo, hi = g * N // shards, (g + 1) * N // shards
            end = min(N, hi + halo)
            parts.append(gpu.scan_shard(t, tx[lo:end], lo, hi - lo))
        assert same(np.concatenate(parts), full), shards


def test_run_throughput_report(gpu):
    rng = np.random.default_rng(2)
    syms = np.arange(256, dtype=np.uint8)
    pats = pattern_set(rng, syms, 1000, 4, 32)
    tx = text(rng, syms, 1 << 22)
    t = build(gpu, pats, 256, 2)
    rep = gpu.run_throughput(t, tx, runs=3, workers=5)
    assert rep["bytes"] == tx.size and rep["runs"] == 3 and rep["workers"] == 5
    assert rep["seconds"] > 0 and rep["gbps"] > 0
    assert rep["matches"] == gpu.scan(t, tx).size


@pytest.mark.parametrize("two_pass", [False, True])
def test_session_device_resident(gpu, monkeypatch, two_pass):
    if two_pass:
        monkeypatch.setenv("HEPFAC_PIPELINE_MIN_MIB", "0")
    rng = np.random.default_rng(8)
    syms = np.arange(256, dtype=np.uint8)
    pats = pattern_set(rng, syms, 2000, 4, 32)
    tx = text(rng, syms, 1 << 21)
    for i, p in enumerate(pats):
        plant(tx, p, (i * 1009) % (tx.size - 40))
    t = build(gpu, pats, 256, 2)
    s = gpu.session(t, tx)
    ms, m = s.run(3)
    assert len(ms) == 3 and all(x > 0 for x in ms)
    first, second, kernels = s.kernel_ms(3)
    assert kernels == (2 if two_pass else 1)
    assert all(abs(f + g - x) < 1e-3 for f, g, x in zip(first, second, ms))
    assert all(g > 0 for g in second) if two_pass else all(g == 0 for g in second)
    assert same(s.fetch(), oracle.naive_find_all(tx, pats))
    s.close()


def test_config1_against_reference(gpu, ref):
    # BASELINE config 1: 1,000 byte patterns len 4-32, 16 MiB, 1 plant / 4 KiB.
    rng = np.random.default_rng(20240601)
    syms = np.arange(256, dtype=np.uint8)
    pats = pattern_set(rng, syms, 1000, 4, 32)
    tx = text(rng, syms, 16 << 20)
    for i in range(4096):
        p = pats[i % len(pats)]
        plant(tx, p, int(rng.integers(0, tx.size - len(p))))
    ra = ref.alphabet(256)
    rt, _ = ref.build_trie(ref.patterns(pats, ra)).compress(2)
    want = ref.scan(rt, tx, workers=os.cpu_count() or 1)
    t = build(gpu, pats, 256, 2)
    assert same(gpu.scan(t, tx), want)
    assert want.size >= 4000


def test_golden_fixtures(gpu):
    # tests/golden/scans.npz: reference hepfac_scan results on seeded instances
    from test_oracle import GOLDEN
    z = np.load(os.path.join(GOLDEN, "scans.npz"))
    for name in sorted({k.split("/")[0] for k in z.files}):
        tx = z[name + "/text"]
        blob, lens = z[name + "/pat_blob"].tobytes(), z[name + "/pat_len"]
        offs = np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(int)
        pats = [blob[o:o + n] for o, n in zip(offs, lens)]
        sigma = int(name.split("_s")[1].split("_")[0])
        state = name.split("_")[-1]
        t = gpu.build_trie(gpu.patterns(pats, gpu.alphabet(sigma)))
        if state == "stage1":
            t = t.compress(1)[0]
        elif state == "stage2":
            t = t.compress(2)[0]
        elif state.startswith("trunc"):
            t = t.truncate(int(state[5:]))[0]
        elif state.startswith("s1trunc"):
            t = t.compress(1)[0].truncate(int(state[7:]))[0]
        assert same(gpu.scan(t, tx), z[name + "/matches"]), name


def test_foreign_terminal_is_reported(gpu, tmp_path):
    # reference: logic_error "terminal node spells no dictionary pattern"
    # (scan.cpp:34) -> HEPFAC_ERR_INTERNAL through capi.cpp:39-64
    from paper_1704_02272_b200 import hepfac as H
    a = gpu.alphabet(256)
    t, _ = gpu.build_trie(gpu.patterns([b"AB", b"XYZW"], a)).compress(1)
    b = bytearray(t.save_bytes())
    i = b.index(b"AB", 4)
    b[i + 1] = ord("C")
    p = str(tmp_path / "bad.htri")
    open(p, "wb").write(bytes(b))
    bad = gpu.load_trie(p)
    with pytest.raises(H.HepfacError) as e:
        gpu.scan(bad, b"xxAByy")
    assert e.value.status == H.INTERNAL and "spells no dictionary pattern" in e.value.message
    assert gpu.scan(bad, b"xxXYZWyy").size == 1


@pytest.mark.parametrize("two_pass", [False, True])
@pytest.mark.parametrize("sigma,stages,depth", [(256, 2, None), (4, 1, 5), (256, 0, 3)])
def test_streamed_scan_equals_resident(gpu, monkeypatch, sigma, stages, depth, two_pass):
    # hepfac_scan streams texts longer than two chunks (H2D of chunk c+1 under
    # the kernel of chunk c, device-side running output base); 1 MiB chunks
    # force many chunk seams, planted matches straddle them.
    if two_pass:
        monkeypatch.setenv("HEPFAC_PIPELINE_MIN_MIB", "0")
    rng = np.random.default_rng(sigma + 7)
    a, syms = alphabet_bytes(gpu, sigma)
    pats = pattern_set(rng, syms, 300, 4, 40)
    tx = text(rng, syms, 5 * (1 << 20) + 12345)
    for c in range(1 << 20, tx.size, 1 << 20):
        for i in range(6):
            p = pats[int(rng.integers(0, len(pats)))]
            plant(tx, p, c - len(p) + 1 + i * 3)
    for i in range(0, tx.size - 64, 4099):
        plant(tx, pats[i % len(pats)], i)
    t = build(gpu, pats, sigma, stages, depth)
    want = oracle.naive_find_all(tx, pats)
    monkeypatch.setenv("HEPFAC_CHUNK_MIB", "1")
    got = gpu.scan(t, tx)
    st = gpu.last_scan_stats()
    assert st["chunks"] == 6
    assert same(got, want)
    monkeypatch.setenv("HEPFAC_CHUNK_MIB", "64")
    assert same(gpu.scan(t, tx), want)
    # one 64 MiB chunk; the pageable text is staged through the pinned ring
    # in pieces (2 MiB here, and HEPFAC_STAGE_MIB=1: six pieces)
    st = gpu.last_scan_stats()
    assert st["staged"] and st["chunks"] == 1
    monkeypatch.setenv("HEPFAC_STAGE_MIB", "1")
    assert same(gpu.scan(t, tx), want)


@pytest.mark.parametrize("stages,depth", [(1, 4), (2, None)])
@pytest.mark.parametrize("mode,code", [("pair", 2), ("l2", 4)])
def test_pair_pipeline_all_starts_pass(gpu, monkeypatch, stages, depth, mode, code):
    # Every start of a run of 'A's passes both filter levels and the prefix
    # recheck: exercises the filter pass's per-chunk fallback (a step with more
    # candidates than its queue), candidate-region overflow and re-run, and
    # walk units with more candidates than a warp queue.  Both two-pass filter
    # forms: pair probes, and the single probe + L2 bitmap.
    monkeypatch.setenv("HEPFAC_FILTER_MODE", mode)
    monkeypatch.setenv("HEPFAC_PIPELINE_MIN_MIB", "0")
    rng = np.random.default_rng(31)
    syms = np.arange(256, dtype=np.uint8)
    pats = pattern_set(rng, syms, 1000, 4, 24)
    pats = sorted(set(pats) | {b"AAAA", b"AAAAB", b"AAAAAAAA", b"AAAAAAAAAAAAAAAAAAAAAAAAAAAAAA"})
    t = build(gpu, pats, 256, stages, depth)
    assert gpu.layout_info(t)["filter_mode"] == code
    tx = np.frombuffer(b"A" * 400000, dtype=np.uint8).copy()
    tx[123456:123456 + 4096] = text(rng, syms, 4096)
    for i, p in enumerate(pats[:200]):
        plant(tx, p, 200000 + i * 97)
    got = gpu.scan(t, tx)
    assert same(got, oracle.naive_find_all(tx, pats))


@pytest.mark.parametrize("count,lo", [(30000, 4), (60000, 5)])
def test_pair_filter_with_l2_level(gpu, ref, monkeypatch, count, lo):
    # Pair tries whose pair survivors are dense (c5 100k: 3.6% of starts)
    # get an L2-resident third level that the filter pass tests on its
    # survivors (two bits per key); k = 4 and k = 5 (8-byte key reads from
    # the staged step).  The walking pass then skips its own L2 probe.
    monkeypatch.setenv("HEPFAC_PIPELINE_MIN_MIB", "0")
    rng = np.random.default_rng(count + lo)
    a, syms = alphabet_bytes(gpu, 256)
    pats = pattern_set(rng, syms, count, lo, 24)
    tx = text(rng, syms, (1 << 21) + 77)
    for i in range(0, tx.size - 40, 977):
        plant(tx, pats[i % len(pats)], i)
    # (the naive oracle is O(text x patterns): the compiled reference instead)
    want = ref.scan(ref.build_trie(ref.patterns(pats, ref.alphabet(256))), tx, workers=os.cpu_count())
    assert want.size > 2000
    for stages, depth in ((1, 6), (2, None)):
        t = build(gpu, pats, 256, stages, depth)
        info = gpu.layout_info(t)
        assert info["filter_mode"] == 2 and info["filter2_bits"] > 0
        assert same(gpu.scan(t, tx), want)


@pytest.mark.parametrize("sigma,lo", [(20, 5), (64, 4), (256, 4), (256, 7)])
@pytest.mark.parametrize("stages,depth", [(0, None), (1, 6), (2, None)])
def test_l2_filter_pipeline_random(gpu, monkeypatch, sigma, lo, stages, depth):
    # The single probe + L2 bitmap filter pass (filter mode 4, chosen by the
    # image builder when the shared-memory level saturates: c5 at 1M
    # patterns) on random instances, k = 4 and k in 5..8, every trie state.
    monkeypatch.setenv("HEPFAC_FILTER_MODE", "l2")
    monkeypatch.setenv("HEPFAC_PIPELINE_MIN_MIB", "0")
    rng = np.random.default_rng(sigma * 13 + lo + stages)
    a, syms = alphabet_bytes(gpu, sigma)
    pats = pattern_set(rng, syms, 1500, lo, 30)
    t = build(gpu, pats, sigma, stages, depth)
    assert gpu.layout_info(t)["filter_mode"] == 4
    tx = text(rng, syms, (1 << 21) + 333)
    for i in range(0, tx.size - 40, 1499):
        plant(tx, pats[i % len(pats)], i)
    assert same(gpu.scan(t, tx), oracle.naive_find_all(tx, pats))


@pytest.mark.parametrize("ext", ["1", "0"])
@pytest.mark.parametrize("two_pass", [False, True])
@pytest.mark.parametrize("sigma,depth", [(4, 8), (20, 5), (256, 4)])
def test_depth_limit_buckets(gpu, monkeypatch, sigma, depth, two_pass, ext):
    # Walks that start at the depth limit (filter_k == limit) emit from the
    # jump slot; with HEPFAC_JUMP_EXT the bucket's first entry and its next 16
    # bytes come from the slot's extension.  Buckets of 1..6 entries, lengths
    # from the limit to 40 past it (compares beyond the inline 16 bytes),
    # near misses in the last byte, and copies overhanging the text end.
    monkeypatch.setenv("HEPFAC_JUMP_EXT", ext)
    if two_pass:
        monkeypatch.setenv("HEPFAC_PIPELINE_MIN_MIB", "0")
    rng = np.random.default_rng(500 + sigma + depth)
    a, syms = alphabet_bytes(gpu, sigma)
    pats = set()
    for _ in range(60):
        head = bytes(syms[rng.integers(0, syms.size, size=depth)])
        if rng.random() < 0.3:
            pats.add(head)
        body = bytes(syms[rng.integers(0, syms.size, size=40)])
        for _ in range(int(rng.integers(1, 7))):
            n = int(rng.integers(1, 41))
            tail = bytearray(body[:n])
            tail[-1] = int(syms[rng.integers(0, syms.size)])
            pats.add(head + bytes(tail))
    pats = sorted(pats)
    t = build(gpu, pats, sigma, 1, depth)
    assert gpu.layout_info(t)["filter_k"] == depth
    tx = text(rng, syms, 200000)
    for i, p in enumerate(pats):
        at = int(rng.integers(0, tx.size - 64))
        plant(tx, p, at)
        miss = bytearray(p)
        miss[-1] = int(syms[(np.searchsorted(syms, miss[-1]) + 1) % syms.size])
        plant(tx, bytes(miss), int(rng.integers(0, tx.size - 64)))
    longest = max(pats, key=len)
    tx[-(len(longest) - 1):] = np.frombuffer(longest[:-1], dtype=np.uint8)
    assert same(gpu.scan(t, tx), oracle.naive_find_all(tx, pats))


@pytest.mark.parametrize("sigma", [2, 4])
def test_symbol_key_mode(gpu, sigma):
    # small alphabets with long shortest patterns: filter and jump keys are
    # packed symbols (filter_mode 3) -- every trie state, text sizes around the
    # packed-word and tile boundaries, bytes outside the alphabet
    rng = np.random.default_rng(50 + sigma)
    a, syms = alphabet_bytes(gpu, sigma)
    pats = pattern_set(rng, syms, 400, 10, 24)
    full = build(gpu, pats, sigma)
    assert gpu.layout_info(full)["filter_mode"] == 3
    s1, _ = full.compress(1)
    s2, _ = full.compress(2)
    tries = [full, s1, s2] + [tr for tr, noop in (s1.truncate(d) for d in (10, 12, 16)) if not noop]
    for n in (1, 9, 31, 33, 8191, 8193, 70001):
        tx = text(rng, syms, n)
        for i in range(0, max(1, n - 30), 97):
            plant(tx, pats[i % len(pats)], i)
        if n > 100:
            tx[50] = 0xFF  # outside every standard alphabet
            tx[n // 2] = 0x00
        want = oracle.naive_find_all(tx, pats)
        for t in tries:
            assert same(gpu.scan(t, tx), want), (sigma, n, t.stage(), t.depth_limit())


@pytest.mark.parametrize("sigma", [2, 4])
def test_symbol_key_aliased_bytes(gpu, sigma):
    # Bytes outside the alphabet pack as symbol 0, so a start whose first k
    # bytes hold one can produce a real jump key.  The walk must still reject
    # it: inline lists by comparing bytes from byte 0, longer lists (several
    # patterns sharing the key) by the byte-wise symbol check.  Patterns up to
    # 40 bytes also take the inline compare past its 24 stored bytes.
    rng = np.random.default_rng(90 + sigma)
    a, syms = alphabet_bytes(gpu, sigma)
    pats = set(pattern_set(rng, syms, 300, 17, 40))
    for _ in range(20):  # keys shared by 3-5 patterns
        head = bytes(syms[rng.integers(0, syms.size, size=16)])
        for _ in range(int(rng.integers(3, 6))):
            pats.add(head + bytes(syms[rng.integers(0, syms.size, size=int(rng.integers(1, 20)))]))
    pats = sorted(pats)
    full = build(gpu, pats, sigma)
    assert gpu.layout_info(full)["filter_mode"] == 3
    s1, _ = full.compress(1)
    tries = [full, s1, full.compress(2)[0], s1.truncate(16)[0]]
    tx = text(rng, syms, 1 << 18)
    at = 0
    for p in pats:
        for bad in (0xFF, 0x00):
            q = bytearray(p)
            zeros = [j for j in range(min(16, len(q))) if q[j] == syms[0]]
            if zeros:
                q[zeros[int(rng.integers(0, len(zeros)))]] = bad
            plant(tx, bytes(q), at)
            at += len(q) + 3
        plant(tx, p, at)
        at += len(p) + 3
    assert at < tx.size
    want = oracle.naive_find_all(tx, pats)
    for t in tries:
        assert same(gpu.scan(t, tx), want), (sigma, t.stage(), t.depth_limit())


def test_symbol_key_mode_streamed(gpu, monkeypatch):
    rng = np.random.default_rng(77)
    a, syms = alphabet_bytes(gpu, 4)
    pats = pattern_set(rng, syms, 300, 12, 30)
    t, _ = build(gpu, pats, 4).compress(1)
    t, _ = t.truncate(12)
    tx = text(rng, syms, 3 * (1 << 20) + 777)
    for c in range(1 << 20, tx.size, 1 << 20):
        p = pats[c % len(pats)]
        plant(tx, p, c - len(p) // 2)
    monkeypatch.setenv("HEPFAC_CHUNK_MIB", "1")
    assert same(gpu.scan(t, tx), oracle.naive_find_all(tx, pats))


def test_config3_full_size_against_reference(gpu, ref):
    # BASELINE config 3 at its bench size per GPU (4 GiB of text, 20k
    # signatures, the benchmark trie), device-resident through the two-pass
    # pipeline and through the streamed hepfac_scan path, against the
    # compiled reference on all host threads: identical arrays.  Offsets past
    # 2^32 are exercised by a 4.5 GiB text.
    from paper_1704_02272_b200 import workloads
    w = workloads.config("c3")
    tx = w.make_text((4 << 30) + (512 << 20))
    t, _ = workloads.build_trie(gpu, w, "s1trunc")
    rt, _ = workloads.build_trie(ref, w, "s1trunc")
    want = ref.scan(rt, tx, workers=os.cpu_count())
    s = gpu.session(t, tx)
    s.run(1)
    assert s.kernel_ms(1)[2] == 2
    assert same(s.fetch(), want)
    s.close()
    assert same(gpu.scan(t, tx), want)
    assert want.size > 1_000_000 and int(want["start"][-1]) >= (1 << 32)


@pytest.mark.parametrize("state", ["s1trunc", "stage2"])
def test_config2_full_size_against_reference(gpu, ref, state):
    # BASELINE config 2 at full size: DNA, 10k patterns len 8-32, 1 GiB genome
    # (8.3 M matches), identical to the compiled reference.
    from paper_1704_02272_b200 import workloads
    w = workloads.config("c2")
    tx = w.make_text(1 << 30)
    t, _ = workloads.build_trie(gpu, w, state)
    rt, _ = workloads.build_trie(ref, w, state)
    want = ref.scan(rt, tx, workers=os.cpu_count())
    assert want.size > 8_000_000
    assert same(gpu.scan(t, tx), want)


@pytest.mark.parametrize("devices", ["0,0,0", "all", "0,0"])
def test_multi_device_scan(gpu, monkeypatch, devices):
    # HEPFAC_DEVICES: one hepfac_scan shards its text into contiguous start
    # ranges with halos, one host thread per shard (a device may repeat, so a
    # one-GPU box exercises the sharded path), lists concatenated in order.
    rng = np.random.default_rng(61)
    syms = np.arange(256, dtype=np.uint8)
    pats = pattern_set(rng, syms, 800, 3, 40)
    tx = text(rng, syms, 50 * (1 << 20) + 4321)
    for i in range(0, tx.size - 64, 65537):
        plant(tx, pats[i % len(pats)], i)
    for g in range(1, 4):  # straddle the shard seams of 2 and 3 shards
        for c in (tx.size * g // 3, tx.size * g // 2):
            p = pats[(c + g) % len(pats)]
            plant(tx, p, c - len(p) // 2)
    t = build(gpu, pats, 256, 2)
    want = gpu.scan(t, tx)
    monkeypatch.setenv("HEPFAC_DEVICES", devices)
    got = gpu.scan(t, tx)
    assert same(got, want)
    from paper_1704_02272_b200 import hepfac as H
    monkeypatch.setenv("HEPFAC_DEVICES", "9")
    with pytest.raises(H.HepfacError):
        gpu.scan(t, tx)


def test_concurrent_scans_share_one_trie(gpu):
    # hepfac.h:4-8 / SURVEY 8(b): handles are shared read-only across threads
    # and hepfac_scan may run concurrently on one trie (ctypes drops the GIL
    # during the call).  Eight threads, two tries (one truncated, so both
    # kernel paths and both jump-table forms run at once), distinct texts.
    import threading

    rng = np.random.default_rng(123)
    a, syms = alphabet_bytes(gpu, 256)
    pats = pattern_set(rng, syms, 500, 4, 20)
    full = build(gpu, pats, 256, 2)
    trunc = build(gpu, pats, 256, 1, 4)
    texts = []
    for i in range(8):
        tx = text(rng, syms, int(rng.integers(1 << 16, 1 << 20)))
        for j in range(0, tx.size - 32, 997):
            plant(tx, pats[(i * 31 + j) % len(pats)], j)
        texts.append(tx)
    wants = [oracle.naive_find_all(tx, pats) for tx in texts]
    results, errors = [None] * 8, []

    def work(i):
        try:
            for _ in range(3):
                got = gpu.scan(full if i % 2 else trunc, texts[i])
                if not same(got, wants[i]):
                    results[i] = False
                    return
            results[i] = True
        except Exception as e:  # surfaced below
            errors.append(e)

    threads = [threading.Thread(target=work, args=(i,)) for i in range(8)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    assert not errors, errors
    assert all(results), results


@pytest.mark.parametrize("alphabet", [b"ACGT", b"acgt", b"AC", b"XYZ"])
@pytest.mark.parametrize("stages,depth", [(0, None), (1, 5), (2, None), (1, 9)])
def test_direct_index_small_alphabet(gpu, monkeypatch, alphabet, stages, depth):
    # Filter mode 5 (sigma <= 4, every pattern 8..32 symbols): exact
    # shared-memory tables and 2-bit compares instead of trie walks.  Shared
    # 8-symbol prefixes, nested patterns, bytes outside the alphabet inside
    # occurrences, and patterns overhanging the text end; compared with the
    # oracle and with the byte-key path (HEPFAC_DNA=0).
    rng = np.random.default_rng(len(alphabet) * 7 + stages + (depth or 0))
    a = gpu.alphabet(alphabet.decode())
    syms = np.frombuffer(alphabet, dtype=np.uint8)
    pats = set(pattern_set(rng, syms, 600, 8, 32))
    base = bytes(syms[rng.integers(0, syms.size, size=32)])
    pats |= {base[:n] for n in (8, 9, 12, 20, 32)}  # nested, one 8-symbol prefix
    pats = sorted(pats)
    t = gpu.build_trie(gpu.patterns(pats, a))
    if stages:
        t, _ = t.compress(stages)
    if depth:
        t, _ = t.truncate(depth)
    assert gpu.layout_info(t)["filter_mode"] == 5
    tx = text(rng, syms, (1 << 20) + 4097)
    for i in range(0, tx.size - 40, 613):
        plant(tx, pats[i % len(pats)], i)
    for i in range(3000, tx.size - 40, 50021):
        plant(tx, base, i)
        tx[i + 10] = ord("N")  # kills the 12-, 20- and 32-symbol occurrences
    plant(tx, base, tx.size - 20)  # 8, 9, 12 fit; 20 and 32 overhang the end
    want = oracle.naive_find_all(tx, pats)
    got = gpu.scan(t, tx)
    assert same(got, want)
    monkeypatch.setenv("HEPFAC_DNA", "0")
    t2 = gpu.build_trie(gpu.patterns(pats, a))
    assert gpu.layout_info(t2)["filter_mode"] != 5
    assert same(gpu.scan(t2, tx), want)


def test_direct_index_tiny_and_ragged_texts(gpu):
    # The direct-index path at the text end: every text length 0..96 and a
    # few ragged ones past the pack pass's 32-byte blocks, with occurrences
    # that end exactly at the last byte, overhang it, or contain a byte
    # outside the alphabet.
    rng = np.random.default_rng(2024)
    a = gpu.alphabet("ACGT")
    syms = np.frombuffer(b"ACGT", dtype=np.uint8)
    pats = sorted(set(pattern_set(rng, syms, 300, 8, 32)) | {b"ACGTACGT", b"ACGTACGTA", b"ACGTACGTAC"})
    t = gpu.build_trie(gpu.patterns(pats, a))
    assert gpu.layout_info(t)["filter_mode"] == 5
    for n in list(range(0, 97)) + [127, 128, 129, 4095, 4097, 65535]:
        tx = text(rng, syms, n)
        if n >= 10:
            plant(tx, b"ACGTACGTAC", n - 10)  # ends at the last byte
        if n >= 9:
            plant(tx, pats[n % len(pats)][: 9], n - 9)
        if n > 40 and n % 3 == 0:
            tx[n // 2] = ord("N")
        assert same(gpu.scan(t, tx), oracle.naive_find_all(tx, pats)), n
