"""Timing of the NEXT-3 small-feature cleaning (sg_clean, threshold 0.4,
max 5 rounds of K + marking + 20 reinit sweeps) on a fresh grid per rep.
One JSON line per workload on stdout.

python scripts/clean_bench.py [C2 FIN128 ...]
"""
import json
import sys

import torch

sys.path.insert(0, ".")
import workloads as W  # noqa: E402
from paper_2512_11473_b200 import sg  # noqa: E402


def workload(name):
    if name.startswith("FIN"):
        return W.fins(int(name[3:]), dtype="f32")
    return W.config(name)


def run(name, reps=3):
    w = workload(name)
    stream = torch.cuda.current_stream()
    res = []
    for k in range(reps + 1):
        g = sg.Grid(w, stream=stream)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        rounds, mods = g.clean(threshold=0.4, stream=stream)
        e1.record(stream)
        torch.cuda.synchronize()
        if k:  # first rep warms up
            res.append(e0.elapsed_time(e1))
        n_pkg = g.info["n_pkg"]
        g.close()
    t = sorted(res)[len(res) // 2]
    pts = (n_pkg - 2) * 64
    return {"config": w.name, "active_points": pts, "rounds": rounds, "raised": mods, "ms": t,
            "ms_per_round": t / max(1, rounds + (1 if rounds < 5 else 0)),
            "note": "median; a round = K (SG_KINT) + marking + host count read + 20 reinit "
                    "sweeps (the last, raising round excluded from the reinit)"}


if __name__ == "__main__":
    for n in sys.argv[1:] or ["C2", "FIN128"]:
        print(json.dumps(run(n)), flush=True)
