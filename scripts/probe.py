#!/usr/bin/env python
"""Throughput probe over the BASELINE configs (device-resident sessions).

Prints one JSON line per (config, trie state): layout of the GPU image,
mean/min kernel ms, Gbps and GB/s of the text stream, match count.  Used for
tuning; bench.py is the contract measurement.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1704_02272_b200 import hepfac, workloads  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c1,c2,c3,c4:2,c4:4,c4:20,c4:64,c4:128,c4:256,c5:1000,c5:10000,c5:100000")
    ap.add_argument("--bytes", type=int, default=1 << 30)
    ap.add_argument("--states", default="s1trunc,stage2")
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--check", action="store_true", help="compare with the compiled reference on 16 MiB")
    ap.add_argument("--full-check", action="store_true",
                    help="compare the whole text's match array with the compiled reference (memcmp + SHA-256)")
    args = ap.parse_args()
    lib = hepfac.lib()
    for spec in args.configs.split(","):
        name, _, arg = spec.partition(":")
        kw = {}
        if name == "c4":
            kw["sigma"] = int(arg)
        if name == "c5":
            kw["count"] = int(arg)
        t0 = time.perf_counter()
        w = workloads.config(name, **kw)
        nbytes = args.bytes if name != "c1" else 16 << 20
        workloads.build_trie(lib, w, "full")  # c4: the library generates the set; make_text plants it
        text = w.make_text(nbytes)
        gen_s = time.perf_counter() - t0
        for state in args.states.split(","):
            t1 = time.perf_counter()
            trie, ps = workloads.build_trie(lib, w, state)
            build_s = time.perf_counter() - t1
            info = lib.layout_info(trie)
            s = lib.session(trie, text)
            s.run(3)
            ms, m = s.run(args.iters)
            s.close()
            mean = sum(ms) / len(ms)
            rec = {"config": spec, "state": state, "bytes": nbytes, "mean_ms": round(mean, 4),
                   "min_ms": round(min(ms), 4), "gbps": round(nbytes * 8 / mean / 1e6, 2),
                   "GBps": round(nbytes / mean / 1e6, 1), "matches": m, "nodes": trie.node_count(),
                   "depth_limit": trie.depth_limit(), "gen_s": round(gen_s, 1), "build_s": round(build_s, 2),
                   "layout": {k: info[k] for k in ("record_bytes", "filter_k", "filter_bits", "filter_paths",
                                                   "min_emit", "smem_bytes", "blocks_per_sm", "reach",
                                                   "keyed_terminals", "private_terminals", "filter_mode", "filter_pass_ppm")}}
            if args.check:
                import oracle
                ref = oracle.ref_library()
                sub = text[: 16 << 20]
                rt, _ = workloads.build_trie(ref, w, state)
                want = ref.scan(rt, sub, workers=os.cpu_count())
                got = lib.scan(trie, sub)
                rec["parity_16MiB"] = bool(got.shape == want.shape and (got == want).all())
            if args.full_check:
                import hashlib

                import oracle
                ref = oracle.ref_library()
                rt, _ = workloads.build_trie(ref, w, state)
                t2 = time.perf_counter()
                want = ref.scan(rt, text, workers=os.cpu_count())
                ref_s = time.perf_counter() - t2
                got = lib.scan(trie, text)
                rec["parity_full"] = {
                    "equal": bool(got.shape == want.shape and got.tobytes() == want.tobytes()),
                    "matches": int(got.size), "ref_matches": int(want.size),
                    "sha256": hashlib.sha256(got.tobytes()).hexdigest(),
                    "ref_sha256": hashlib.sha256(want.tobytes()).hexdigest(),
                    "ref_scan_s": round(ref_s, 2), "ref_workers": os.cpu_count()}
            print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
