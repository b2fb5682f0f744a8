#!/usr/bin/env python
"""Summarise ncu outputs brought back in gpurun_out/ into profiles/.

    python scripts/ncu_summary.py <tag> [gpurun_out]

Writes
  profiles/<tag>_launches.md   per-kernel device time and share of the step
                               (from the --metrics gpu__time_duration.sum list)
  profiles/<tag>_kernels.md    key --set full metrics per captured kernel
  profiles/ncu_traffic.json    dram read+write bytes per launch (for bench.py)
"""
import csv
import glob
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram % peak"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % peak"),
    ("sm__inst_executed.sum", "instructions"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
    ("launch__registers_per_thread", "registers"),
    ("l1tex__t_sector_hit_rate.pct", "L1 hit %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("smsp__sass_thread_inst_executed_op_ffma_pred_on.sum", "FFMA thread-inst"),
    ("smsp__sass_thread_inst_executed_op_fadd_pred_on.sum", "FADD thread-inst"),
    ("smsp__sass_thread_inst_executed_op_fmul_pred_on.sum", "FMUL thread-inst"),
]


def short(name):
    n = name.split("(")[0]
    return n.replace("void ", "").replace("sg::", "")


def launches(tag, out):
    path = os.path.join(out, "launches.csv")
    if not os.path.exists(path):
        return
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = defaultdict(list)
    for r in rows[hi + 1:]:
        if len(r) > vi:
            v = float(r[vi].replace(",", ""))
            if r[ui] == "us":
                v *= 1e3
            elif r[ui] == "ms":
                v *= 1e6
            agg[short(r[ki])].append(v)
    ours = {k: v for k, v in agg.items() if "at::" not in k}
    tot = sum(sum(v) for v in ours.values())
    lines = [f"# {tag}: ncu launch list (`--metrics gpu__time_duration.sum --clock-control none`)",
             "", "Cold-cache, serialised launches of `bench.py --steps 1 --warmup 1` (2 steps);",
             "shares are of our kernels' summed device time (torch's L2-flush fill excluded).", "",
             "| kernel | launches | total µs | avg µs | share |", "|---|---:|---:|---:|---:|"]
    for k, v in sorted(ours.items(), key=lambda x: -sum(x[1])):
        lines.append(f"| `{k}` | {len(v)} | {sum(v) / 1e3:.1f} | {sum(v) / len(v) / 1e3:.2f} | "
                     f"{100 * sum(v) / tot:.1f}% |")
    open(os.path.join(ROOT, "profiles", f"{tag}_launches.md"), "w").write("\n".join(lines) + "\n")


def reports(tag, out):
    traffic_path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    lines = [f"# {tag}: ncu --set full summaries", ""]
    for rep in sorted(glob.glob(os.path.join(out, "*.ncu-rep"))):
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout
        rows = list(csv.reader(raw.splitlines()))
        if len(rows) < 3:
            continue
        h = rows[0]
        col = {k: h.index(k) for k, _ in KEYS if k in h}
        units = rows[1]
        ki = h.index("Kernel Name")
        for r in rows[2:]:
            name = short(r[ki])
            lines.append(f"## `{name}` ({os.path.basename(rep)})")
            lines.append("")
            for k, label in KEYS:
                if k in col:
                    lines.append(f"- {label}: {r[col[k]]} {units[col[k]]}")
            lines.append("")
            try:
                rd = float(r[col["dram__bytes_read.sum"]].replace(",", ""))
                wr = float(r[col["dram__bytes_write.sum"]].replace(",", ""))
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
                b = rd * scale.get(units[col["dram__bytes_read.sum"]], 1) + \
                    wr * scale.get(units[col["dram__bytes_write.sum"]], 1)
                base = name.split("<")[0]
                cfg = "C3" if "c3" in os.path.basename(rep) else "C2"
                traffic.setdefault(cfg, {})[base] = b
            except Exception:
                pass
    open(os.path.join(ROOT, "profiles", f"{tag}_kernels.md"), "w").write("\n".join(lines) + "\n")
    json.dump(traffic, open(traffic_path, "w"), indent=1)


if __name__ == "__main__":
    tag = sys.argv[1]
    out = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "gpurun_out")
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    launches(tag, out)
    reports(tag, out)
