#!/usr/bin/env python
"""Per-instruction stall hot spots of one kernel in an ncu report.
    python scripts/ncu_src.py <report.ncu-rep> <kernel-regex> [top]"""
import csv
import subprocess
import sys
from collections import Counter

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kern,
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
si, wi, ei = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
data = []
seen = set()
for r in rows[2:]:
    if len(r) <= max(si, wi, ei) or r[0] == "Address":
        continue
    key = (r[0], r[si])
    if key in seen:
        continue
    seen.add(key)
    try:
        data.append((int(r[wi] or 0), int(r[ei] or 0), r[si]))
    except ValueError:
        pass
tot = sum(d[0] for d in data) or 1
toti = sum(d[1] for d in data) or 1
print(f"samples {tot}  warp-instructions {toti}  static instructions {len(data)}")
c = Counter()
for d in data:
    toks = d[2].split()
    op = toks[1] if toks and toks[0].startswith("@") else (toks[0] if toks else "?")
    c[op.split(".")[0]] += d[1]
print("mix:", ", ".join(f"{k} {100 * v / toti:.1f}%" for k, v in c.most_common(14)))
for d in sorted(data, reverse=True)[:top]:
    print(f"{d[0]:6d} {100 * d[0] / tot:5.1f}% {d[1]:9d}  {d[2][:100]}")
