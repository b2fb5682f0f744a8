#!/usr/bin/env python
"""Table-1 workloads of the paper on the GPU.

The shelled sphere (centre 0.5, r 0.3 / 0.31) at "resolution 1/1024" read as
dx = 1/1024 (reading R-19): 256^3 background cells, 579,128 packages,
37,064,192 active data points.  "Sequential" adds a constant to every active
value (sg_table1 op 0), "Stencil" applies the 7-point Laplacian to every active
value into a second buffer (op 1).  Prints one JSON line with device times
(CUDA events, median of 20 after 5 warm-ups) beside the paper's CPU numbers
(context only: CPU, unit not stated; read as ms under R-19).
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads as W  # noqa: E402
from paper_2512_11473_b200 import build, sg  # noqa: E402


def run(name):
    w = W.config(name)
    g = sg.Grid(w)
    n_act = (g.info["n_pkg"] - 2) * 64
    res = {}
    for op, name in ((0, "sequential"), (1, "stencil")):
        ts = []
        for it in range(25):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.table1(op, 1e-6)
            e1.record()
            torch.cuda.synchronize()
            if it >= 5:
                ts.append(e0.elapsed_time(e1))
        ms = float(np.median(ts))
        bytes_ = n_act * (8 if op == 0 else 8 + 108 / 64)
        res[name] = {"ms": ms, "points_per_s": n_act / (ms * 1e-3),
                     "algorithmic_GBps": bytes_ / (ms * 1e-3) / 1e9}
    g.close()
    return n_act, res


def main():
    build.build()
    n_act, res = run("T1")
    # SURVEY 8(f) NEXT-1 also asks for C5 (the paper shell + 8 small shells,
    # dx = 1/4096, 970.7 M active points)
    n5, res5 = run("C5")
    out = {"workload": "Table-1 shelled sphere, dx = 1/1024 (R-19), fp32",
           "active_points": n_act, "gpu": torch.cuda.get_device_name(0), **res,
           "C5": {"workload": "C5 multi-shell scene, dx = 1/4096, fp32", "active_points": n5,
                  **res5},
           "paper_table1_cpu_context": {"sequential_1thread": 22.948, "sequential_4threads": 7.429,
                                        "stencil_1thread": 59.972, "stencil_4threads": 21.378,
                                        "source": "PAPER.md P:614-617 (CPU, units not stated)"}}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
