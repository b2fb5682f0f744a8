#!/usr/bin/env python
"""Per CUDA-source-line instruction counts and stall samples of one kernel.
    python scripts/ncu_lines.py <report.ncu-rep> <kernel-regex> [top]"""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kern,
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = [i for i, r in enumerate(rows) if len(r) > 3 and r[0] == "Line No"][0]
h = rows[hi]
wi, ei = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
lines, tot, toti = [], 0, 0
for r in rows[hi + 1:]:
    if len(r) <= ei or r[2] != "-":
        continue
    try:
        w, e = int(r[wi] or 0), int(r[ei] or 0)
    except ValueError:
        continue
    lines.append((e, w, r[0], r[1][:95]))
    tot += w
    toti += e
print(f"warp-instructions {toti}  stall samples {tot}")
for e, w, ln, src in sorted(lines, reverse=True)[:top]:
    print(f"{e:10d} {100 * e / max(toti, 1):5.1f}%  stall {100 * w / max(tot, 1):5.1f}%  L{ln}: {src}")
