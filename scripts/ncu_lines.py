#!/usr/bin/env python
"""Per-source-line instruction and stall-sample shares of one kernel from an
ncu report, by mapping its SASS page onto nvdisasm line info of the same
cubin (the report's own CUDA source page needs the box's source paths).
usage: ncu_lines.py REPORT.ncu-rep OBJECT.o MANGLED_KERNEL_NAME [top]"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

rep, obj, fun = sys.argv[1:4]
obj = os.path.abspath(obj)
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
with tempfile.TemporaryDirectory() as d:
    subprocess.run(["cuobjdump", "-xelf", "all", obj], cwd=d, check=True, capture_output=True)
    cubin = subprocess.run("ls *.cubin", shell=True, cwd=d, capture_output=True, text=True).stdout.split()[0]
    sass = subprocess.run(["nvdisasm", "--print-line-info", cubin], cwd=d, capture_output=True, text=True).stdout
lines = sass.split("\n")
st = [i for i, l in enumerate(lines) if l.startswith(".text." + fun + ":")][0]
cur, where = None, {}
for l in lines[st + 1:]:
    if l.startswith(".text.") or l.startswith("//----"):
        break
    g = re.match(r'\s*//## File "([^"]+)", line (\d+)', l)
    if g:
        cur = (g.group(1).split("/")[-1], int(g.group(2)))
        continue
    g = re.match(r"\s*/\*([0-9a-f]{4,5})\*/", l)
    if g:
        where[int(g.group(1), 16) // 16] = cur
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
h, rows = r[1], r[2:]
iw, ie = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
E, W = collections.Counter(), collections.Counter()
for i, x in enumerate(rows):
    E[where.get(i)] += int(x[ie])
    W[where.get(i)] += int(x[iw])
te, tw = sum(E.values()), sum(W.values())
print(f"{len(rows)} SASS ({len(where)} mapped), {te} warp instructions, {tw} stall samples")
order = sys.argv[5] if len(sys.argv) > 5 else "inst"
for k, v in (W if order == "stall" else E).most_common(top):
    v = E[k]
    print(f"{k}: inst {100 * v / te:5.1f}%  stall {100 * W[k] / tw:5.1f}%")
