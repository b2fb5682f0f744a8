#!/usr/bin/env python
"""NEXT-2 measurement: SPH relaxation steps of the C4 particle set (19.45 M
lattice particles, dp = dx) against the C2 prism level set, 1 GPU.  Prints
one JSON line: ms per relaxation step (device events, median of 10 after 3
warm-ups) and particle updates per second."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workloads as W  # noqa: E402
from paper_2512_11473_b200 import build, sg  # noqa: E402


def main():
    build.build()
    w = W.config("C2")
    g = sg.Grid(w)
    g.reinit(20).gradient(sg.SG_GRAD | sg.SG_KINT)
    pos = torch.from_numpy(W.lattice_particles(w, seed=0)).cuda()
    ts = []
    for it in range(13):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.relax(pos, dp=w.dx, steps=1)
        e1.record()
        torch.cuda.synchronize()
        if it >= 3:
            ts.append(e0.elapsed_time(e1))
    ms = float(np.median(ts))
    phi, _ = g.probe(pos, want_grad=False)
    print(json.dumps({"workload": "C4 particles relaxing against the C2 prism (dp = dx, h = 1.3 dp)",
                      "particles": int(pos.shape[0]), "ms_per_step": ms,
                      "particle_updates_per_s": pos.shape[0] / (ms * 1e-3),
                      "max_phi_after": float(phi.max()), "gpu": torch.cuda.get_device_name(0)}))


if __name__ == "__main__":
    main()
