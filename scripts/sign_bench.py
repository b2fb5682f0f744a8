"""Timing of the NEXT-3 sign-consistency correction (sg_sign_correct) on the
leaky variants of C2 / C3 (workloads.leaky: SG_LEAK balls inside, across and
outside the body).  One JSON line per config on stdout.

python scripts/sign_bench.py [C2 C3 ...]
"""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
import workloads as W  # noqa: E402
from paper_2512_11473_b200 import sg  # noqa: E402


def run(name, reps=5):
    w = W.leaky(W.config(name))
    stream = torch.cuda.current_stream()
    g = sg.Grid(w, stream=stream)
    info = g.info
    for _ in range(2):
        sw = g.sign_correct(stream=stream)
    torch.cuda.synchronize()
    ms = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        sw = g.sign_correct(stream=stream)
        e1.record(stream)
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    t = sorted(ms)[len(ms) // 2]
    ncell = w.n[0] * w.n[1] * w.n[2]
    return {"config": w.name, "cells": ncell, "active_points": (info["n_pkg"] - 2) * 64,
            "sweeps": {"coarse": sw[0], "refined": sw[1]}, "ms": t, "ms_all": ms,
            "cell_sweeps_per_s": ncell * sw[0] / (t * 1e-3),
            "note": "median of reps; includes the host convergence reads (one per batch of "
                    "sweeps) and the table / phi rewrite"}


if __name__ == "__main__":
    names = sys.argv[1:] or ["C2", "C3"]
    for n in names:
        print(json.dumps(run(n)), flush=True)
