"""The CLI's build/match path (tools/hepfac_b200_cli.cpp) against the
reference library: the reference CLI's `build` writes the .htri of
hepfac_trie_build [+ compress] (hepfac_cli.cpp:156-193) and `match` prints
hepfac_scan's records as "start\\tlength\\tid" lines (hepfac_cli.cpp:234-279).
The reference CLI itself does not build here (CLI11 is not vendored), so its
outputs are reproduced through the compiled reference library."""
from __future__ import annotations

import json
import os
import subprocess

import numpy as np
import pytest

from helpers import alphabet_bytes, pattern_set, plant, text

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_1704_02272_b200", "hepfac_b200_cli")


def run(*args, **kw):
    return subprocess.run([CLI, *args], capture_output=True, **kw)


def write_patterns(path, pats):
    with open(path, "wb") as f:
        f.write(b"".join(p + b"\n" for p in pats))


def lines_of(arr) -> bytes:
    return b"".join(b"%d\t%d\t%d\n" % (int(r["start"]), int(r["length"]), int(r["pattern_id"])) for r in arr)


def test_cli_usage_and_errors(tmp_path):
    assert os.access(CLI, os.X_OK), "hepfac_b200_cli not built (make -C paper_1704_02272_b200)"
    r = run()
    assert r.returncode == 1 and b"usage" in r.stderr
    assert run("frobnicate").returncode == 1
    assert run("build", "--bogus", "1").returncode == 1
    assert run("build", "--patterns", str(tmp_path / "missing.txt"), "--out", str(tmp_path / "t.htri")).returncode == 2
    assert run("match", "--trie", str(tmp_path / "missing.htri"), "--input", "/dev/null").returncode == 2


@pytest.mark.parametrize("stages", [0, 1, 2])
def test_cli_build_equals_reference(tmp_path, lib, ref, stages):
    rng = np.random.default_rng(40 + stages)
    _, sym = alphabet_bytes(lib, 52)
    pats = pattern_set(rng, sym, 200, 3, 12)
    pf = tmp_path / "p.txt"
    write_patterns(pf, pats)
    out = tmp_path / "ours.htri"
    r = run("build", "--patterns", str(pf), "--compress", str(stages), "--out", str(out))
    assert r.returncode == 0, r.stderr
    report = json.loads(r.stdout)
    rt = ref.build_trie(ref.load_patterns(str(pf), ref.alphabet(52)))
    if stages:
        rt, st = rt.compress(stages)
        assert report["compression"]["nodes_after_stage2"] == st.nodes_after_stage2
    assert open(out, "rb").read() == rt.save_bytes()
    assert report["memory"]["node_count"] == rt.node_count()
    assert report["trie"] == str(out)


@pytest.mark.gpu
@pytest.mark.parametrize("depth", [0, 3])
def test_cli_match_equals_reference(tmp_path, gpu, ref, depth):
    rng = np.random.default_rng(7 + depth)
    _, sym = alphabet_bytes(gpu, 256)
    pats = [p for p in pattern_set(rng, sym, 300, 2, 10) if b"\n" not in p and b"\r" not in p]
    t = text(rng, sym, 1 << 18)
    for i, p in enumerate(pats):
        plant(t, p, (i * 977) % (t.size - 16))
    pf, tf, inp = tmp_path / "p.txt", tmp_path / "t.htri", tmp_path / "in.bin"
    write_patterns(pf, pats)
    inp.write_bytes(t.tobytes())
    # the benchmark trie for --depth is stage 1 (a tail-merged trie cannot be truncated)
    stages = "1" if depth else "2"
    assert run("build", "--patterns", str(pf), "--sigma", "256", "--compress", stages, "--out", str(tf)).returncode == 0
    args = ["match", "--trie", str(tf), "--input", str(inp)] + (["--depth", str(depth)] if depth else [])
    r = run(*args)
    assert r.returncode == 0, r.stderr
    rt = ref.load_trie(str(tf))
    if depth:
        rt, _ = rt.truncate(depth)
    want = ref.scan(rt, t, workers=os.cpu_count())
    assert r.stdout == lines_of(want)
    summary = json.loads(r.stderr.decode().strip().splitlines()[-1])
    assert summary["matches"] == want.size and summary["bytes"] == t.size
    # --out writes the same bytes
    out = tmp_path / "m.txt"
    assert run(*args, "--out", str(out)).returncode == 0
    assert out.read_bytes() == r.stdout


@pytest.mark.gpu
def test_cli_match_truncate_stage2_is_invalid(tmp_path, gpu):
    pf, tf, inp = tmp_path / "p.txt", tmp_path / "t.htri", tmp_path / "in.bin"
    write_patterns(pf, [b"abcd", b"abce", b"xbcd"])
    inp.write_bytes(b"zzabcdzz")
    assert run("build", "--patterns", str(pf), "--compress", "2", "--out", str(tf)).returncode == 0
    r = run("match", "--trie", str(tf), "--input", str(inp), "--depth", "2")
    assert r.returncode == 1 and b"truncate" in r.stderr
