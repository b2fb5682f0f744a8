"""A small pass over every C-ABI entry point for compute-sanitizer
(memcheck / racecheck / synccheck; scripts/sanitize.sh): C1 fp64 and a random
fp32 scene through build, reinit (single sweep and the cached multi-sweep
graph), gradient (separate and fused K6+K7), probe (device and host buffers),
Table-1 ops, relaxation, sign correction of a leaky sphere, cleaning, a mesh
build, a refined layer, and a 3-rank partitioned grid over the in-process
communicator (exchanges, K9 binning).  Prints "sanitize_run ok"."""
import os
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2512_11473_b200 import sg  # noqa: E402

ALL = sg.SG_GRAD | sg.SG_NORMAL | sg.SG_KINT


def single(w):
    dt = torch.float64 if w.dtype == "f64" else torch.float32
    g = sg.Grid(w)
    g.reinit(1).reinit(6)
    g.gradient(sg.SG_GRAD | sg.SG_NORMAL).gradient(sg.SG_KINT).gradient(ALL)
    pos = torch.from_numpy(W.random_positions(w, 5000, seed=1)).to(dt)
    phi, grad = g.probe(pos.cuda())
    hphi, hgrad = g.probe(pos.pin_memory())
    assert torch.equal(phi.cpu(), hphi)
    g.table1(1).table1(0, 0.1)
    g.gradient(sg.SG_GRAD | sg.SG_KINT)
    g.relax(pos[:2000].cuda().contiguous(), dp=w.dx, steps=1)
    torch.cuda.synchronize()
    g.close()


def main():
    single(W.config("C1"))
    single(W.random_scene(3, 20, dtype="f32"))
    lk = sg.Grid(W.leaky(W.config("C1")))
    lk.sign_correct()
    lk.clean(max_rounds=2)
    lk.close()
    m = W.Workload("ico", (16, 16, 16), 1.0 / 16, dtype="f32", mesh=W.icosphere(2))
    gm = sg.Grid(m)
    gr = gm.refined()
    gr.reinit(2)
    gr.close()
    gm.close()
    # partitioned grid, 3 ranks in one process
    w = W.config("C1")
    comms = sg.Comm.local(3)
    pos = torch.from_numpy(W.random_positions(w, 6000, seed=2)).cuda()
    errs = []

    def rank(r):
        try:
            st = torch.cuda.Stream()
            g = sg.Grid(w, comm=comms[r], stream=st)
            g.reinit(9, stream=st).gradient(ALL, stream=st)
            g.probe(pos[2000 * r:2000 * (r + 1)].contiguous(), stream=st)
            st.synchronize()
            g.close()
        except Exception as e:  # noqa: BLE001
            errs.append(e)
    ts = [threading.Thread(target=rank, args=(r,)) for r in range(3)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=600)
    for c in comms:
        c.close()
    assert not errs, errs
    torch.cuda.synchronize()
    print("sanitize_run ok")


if __name__ == "__main__":
    main()
