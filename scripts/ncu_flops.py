#!/usr/bin/env python
"""Per-kernel executed arithmetic from an ncu --metrics CSV -> profiles/ncu_flops.json
(read by bench.py for the ALU rooflines of the fp64 build kernels and the
executed-FMA fraction of K7).

    python scripts/ncu_flops.py CONFIG gpurun_out/flops_CONFIG.csv [...more CONFIG CSV pairs]

Per kernel (short name, launches averaged): us (gpu__time_duration), thread-level
DFMA / DADD / DMUL / FFMA / FADD / FMUL (and the paired FFMA2 / FADD2 / FMUL2)
instruction counts, DRAM bytes.
"""
import csv
import json
import os
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
MET = {
    "gpu__time_duration.sum": "us",
    "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum": "dfma",
    "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum": "dadd",
    "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum": "dmul",
    "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum": "ffma",
    "smsp__sass_thread_inst_executed_op_fadd_pred_on.sum": "fadd",
    "smsp__sass_thread_inst_executed_op_fmul_pred_on.sum": "fmul",
    # paired FP32 (sm_100): each thread instruction is two lane operations
    "smsp__sass_thread_inst_executed_op_ffma2_pred_on.sum": "ffma2",
    "smsp__sass_thread_inst_executed_op_fadd2_pred_on.sum": "fadd2",
    "smsp__sass_thread_inst_executed_op_fmul2_pred_on.sum": "fmul2",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
}
SCALE = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3,
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def short(name):
    n = name.split("(")[0].replace("void ", "").replace("sg::", "")
    return n.split("<")[0]


def parse(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, ii = h.index("Kernel Name"), h.index("ID")
    mi, ui, vi = h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
    per = defaultdict(dict)  # launch id -> metrics
    names = {}
    for r in rows[hi + 1:]:
        if len(r) <= vi or r[mi] not in MET:
            continue
        v = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1.0)
        per[r[ii]][MET[r[mi]]] = v
        names[r[ii]] = short(r[ki])
    agg = defaultdict(lambda: defaultdict(list))
    for lid, m in per.items():
        for k, v in m.items():
            agg[names[lid]][k].append(v)
    return {n: {k: sum(v) / len(v) for k, v in m.items()} | {"launches": len(m["us"])}
            for n, m in agg.items() if "us" in m}


def main():
    out_path = os.path.join(ROOT, "profiles", "ncu_flops.json")
    data = json.load(open(out_path)) if os.path.exists(out_path) else {}
    args = sys.argv[1:]
    for cfg, path in zip(args[::2], args[1::2]):
        data[cfg] = parse(path)
    json.dump(data, open(out_path, "w"), indent=1, sort_keys=True)
    print(json.dumps(data, indent=1))


if __name__ == "__main__":
    main()
