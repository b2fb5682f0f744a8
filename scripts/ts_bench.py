"""Two-sweep reinit micro-benchmark: per-call reinit(20) time on a built grid
(plan cached) and the first-call cost (plan build), for the given configs.
Run with SG_TSWEEP=1 for the two-sweep tiles (default: single sweeps)."""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
import workloads as W  # noqa: E402
from paper_2512_11473_b200 import sg  # noqa: E402

torch.cuda.init()
for name in sys.argv[1:] or ["C2", "C3"]:
    w = W.config(name)
    g = sg.Grid(w)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    g.reinit(2)
    torch.cuda.synchronize()
    first = time.perf_counter() - t0
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    g.reinit(20)  # graph capture
    ts = []
    for _ in range(7):
        torch.cuda.synchronize()
        ev[0].record()
        g.reinit(20)
        ev[1].record()
        torch.cuda.synchronize()
        ts.append(ev[0].elapsed_time(ev[1]))
    ts.sort()
    print(json.dumps({"config": name, "first_reinit2_ms": first * 1e3, "reinit20_ms": ts[len(ts) // 2],
                      "per_sweep_us": ts[len(ts) // 2] / 20 * 1e3, "n_pkg": g.info["n_pkg"]}), flush=True)
    del g
