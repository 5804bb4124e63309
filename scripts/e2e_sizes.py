#!/usr/bin/env python
"""hepfac_scan end-to-end throughput by text size, pageable vs pinned host
text (tuning aid for the staging ring; bench.py is the contract).  One JSON
line per (config, size, memory)."""
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
    ap.add_argument("--configs", default="c3,c2")
    ap.add_argument("--mib", default="16,64,256,1024")
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    import torch
    lib = hepfac.lib()
    for spec in args.configs.split(","):
        w = workloads.config(spec)
        trie, _ = workloads.build_trie(lib, w, "s1trunc")
        big = max(int(m) for m in args.mib.split(",")) << 20
        text = w.make_text(big)
        pinned = torch.empty(big, dtype=torch.uint8, pin_memory=True).numpy()
        pinned[:] = text
        for mib in map(int, args.mib.split(",")):
            n = mib << 20
            for kind, buf in (("pageable", text[:n]), ("pinned", pinned[:n])):
                r = lib.scan(trie, buf, view=True)
                r = None
                ts = []
                for _ in range(args.reps):
                    t0 = time.perf_counter()
                    r = lib.scan(trie, buf, view=True)
                    ts.append(time.perf_counter() - t0)
                    r = None
                best = min(ts)
                print(json.dumps({"config": spec, "mib": mib, "memory": kind, "gbps": round(n * 8 / best / 1e9, 1),
                                  "ms": round(best * 1e3, 3), "spin_us": os.environ.get("HEPFAC_COPY_SPIN_US")}),
                      flush=True)


if __name__ == "__main__":
    main()
