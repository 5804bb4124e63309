#!/usr/bin/env python
"""One-line summary of a bench.py JSON line (and its reference arm)."""
import json
import sys


def last_json(path):
    try:
        lines = [l for l in open(path) if l.startswith("{")]
        return json.loads(lines[-1]) if lines else None
    except OSError:
        return None


b = last_json(sys.argv[1])
r = last_json(sys.argv[2]) if len(sys.argv) > 2 else None
if not b:
    print("no result")
    sys.exit(0)
rf = b.get("roofline", {})
cb = b.get("cpu_baseline", {})
parts = [f"value {b['value']:.0f} Gbps", f"frac {rf.get('frac')}", f"e2e {b['e2e']['value']:.0f}",
         f"e2e_pageable {b.get('e2e_pageable', {}).get('value', 0):.0f}",
         f"matches {b['config'].get('matches_per_gpu')}", f"cpu {cb.get('value')} ({cb.get('cores')} cores)"]
if r:
    parts.append(f"ref_arm {r.get('value')}")
print(", ".join(parts))
