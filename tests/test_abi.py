"""The drop-in boundary: libhepfac.so loads, exports exactly the functions the
headers declare (the reference's 46 + the hepfac_b200_* additions), and keeps
the reference's error conventions (test_capi.cpp:102-143).  CPU only."""
import os
import re
import subprocess

import pytest

from paper_1704_02272_b200 import hepfac as H

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared(header):
    src = open(os.path.join(ROOT, "include", header)).read()
    return set(re.findall(r"\b(hepfac_\w+)\s*\(", src))


def exported(path):
    out = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True, text=True, check=True).stdout
    return {line.split()[-1] for line in out.splitlines() if " T " in line and line.split()[-1].startswith("hepfac_")}


def test_exports_match_headers(lib):
    decl = declared("hepfac.h") | declared("hepfac_b200.h")
    exp = exported(lib.path)
    assert decl == exp, (decl ^ exp)
    assert len(declared("hepfac.h")) == 46


def test_reference_abi_is_a_subset(lib, ref):
    # Every symbol the reference library exports is exported by ours.
    assert exported(ref.path) <= exported(lib.path)
    assert exported(ref.path) == declared("hepfac.h")


def test_binding_covers_every_symbol(lib):
    assert set(H.ABI_SYMBOLS) == declared("hepfac.h")
    assert set(H.B200_SYMBOLS) == declared("hepfac_b200.h")


def test_no_foreign_symbols_exported(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", lib.path], capture_output=True, text=True).stdout
    names = [line.split()[-1] for line in out.splitlines() if line.split()[1] in "TDBVW"]
    assert names and all(n.startswith("hepfac_") for n in names), names[:5]


def test_status_strings_and_version(lib):
    assert lib.status_string(H.OK) == "ok"
    assert lib.status_string(H.INTERNAL) == "internal error"
    assert lib.version() == "1.0.0"


def test_error_codes(lib):
    a = lib.alphabet(4)
    with pytest.raises(H.HepfacError) as e:
        lib.patterns([b"ACG", b"ACG"], a)
    assert e.value.status == H.DUPLICATE
    with pytest.raises(H.HepfacError) as e:
        lib.patterns([b"AB"], a)
    assert e.value.status == H.BAD_BYTE and "0x42" in e.value.message
    assert lib.dll.hepfac_trie_build(None, None) == H.INVALID_ARG
    assert lib.last_error() == "null argument"
    assert lib.dll.hepfac_alphabet_standard(4, None) == H.INVALID_ARG
    with pytest.raises(H.HepfacError) as e:
        lib.load_trie("does_not_exist.htri")
    assert e.value.status == H.IO
    t = lib.build_trie(lib.generate_patterns(1, a, 10, 8))
    t2, _ = t.compress(2)
    with pytest.raises(H.HepfacError) as e:
        t2.compress(1)
    assert e.value.status == H.STATE


def test_last_error_is_thread_local(lib):
    # capi.cpp:37, 138-141: each thread reads the message of its own last
    # failure, whatever other threads did in between.
    import threading

    a = lib.alphabet(4)
    step = threading.Barrier(2)
    seen = {}

    def first():
        assert lib.dll.hepfac_trie_build(None, None) == H.INVALID_ARG
        step.wait()  # the other thread fails differently
        step.wait()
        seen["first"] = lib.last_error()

    def second():
        step.wait()
        with pytest.raises(H.HepfacError):
            lib.patterns([b"AB"], a)
        seen["second"] = lib.last_error()
        step.wait()

    ts = [threading.Thread(target=first), threading.Thread(target=second)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert seen["first"] == "null argument"
    assert "0x42" in seen["second"]


def test_out_untouched_on_failure(lib):
    import ctypes as C
    a = lib.alphabet(4)
    bufs = [C.create_string_buffer(b"ACG", 3)] * 2
    ptrs = (C.c_void_p * 2)(*[C.cast(b, C.c_void_p) for b in bufs])
    lens = (C.c_size_t * 2)(3, 3)
    out = C.c_void_p(0x1234)
    assert lib.dll.hepfac_patterns_create(ptrs, lens, 2, a.h, C.byref(out)) == H.DUPLICATE
    assert out.value == 0x1234


def test_scan_argument_checks(lib):
    a = lib.alphabet(256)
    t = lib.build_trie(lib.patterns([b"AB"], a))
    import ctypes as C
    out = C.c_void_p()
    # text may be NULL only when bytes == 0 (capi.cpp:395-396)
    assert lib.dll.hepfac_scan(t.h, None, 5, None, C.byref(out)) == H.INVALID_ARG
    assert lib.dll.hepfac_scan(None, None, 0, None, C.byref(out)) == H.INVALID_ARG


@pytest.mark.skipif(H.lib().device_count() > 0, reason="checks the no-GPU failure mode")
def test_no_cpu_fallback_without_gpu(lib):
    a = lib.alphabet(256)
    t = lib.build_trie(lib.patterns([b"AB"], a))
    with pytest.raises(H.HepfacError) as e:
        lib.scan(t, b"xxABxx")
    assert e.value.status == H.INTERNAL and "no CUDA device" in e.value.message
    # empty texts never touch the device (reference returns an empty list)
    assert lib.scan(t, b"").size == 0


def test_kernels_are_sm100a(lib):
    # The engine ships SASS for sm_100a only (no PTX/JIT, no other archs).
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lib.path], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    assert all("sm_100a" in line for line in out.splitlines() if ".cubin" in line)
