"""Try the NCCL communicator with 2 processes on ONE GPU (NCCL normally
refuses two ranks on one device; if it does, the result says so).  When it
runs, the partitioned C2 grid + probe must equal the plain grid bitwise.

    python scripts/nccl_two_ranks.py  -> one JSON line
"""
import json
import os
import socket
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def worker(rank, world, port, q):
    try:
        import numpy as np
        import torch
        import torch.distributed as dist
        import workloads as W
        from paper_2512_11473_b200 import sg
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        comm = sg.Comm.nccl()
        w = W.config("C2")
        g = sg.Grid(w, comm=comm).reinit(20, w.cfl).gradient(sg.SG_GRAD | sg.SG_NORMAL | sg.SG_KINT)
        pos = W.lattice_particles(w, seed=0)[::5]
        n = pos.shape[0]
        a, b = n * rank // world, n * (rank + 1) // world
        phi, grad = g.probe(torch.from_numpy(pos[a:b].copy()).cuda())
        ref = sg.Grid(w).reinit(20, w.cfl).gradient(sg.SG_GRAD | sg.SG_NORMAL | sg.SG_KINT)
        rphi, rgrad = ref.probe(torch.from_numpy(pos[a:b].copy()).cuda())
        info = g.info
        lo, hi = info["own_lo"], info["own_hi"]
        ga, gb = lo - 2 + info["id_base"], hi - 2 + info["id_base"]
        ok = (torch.equal(phi, rphi) and torch.equal(grad, rgrad)
              and torch.equal(g.view("phi")[lo:hi], ref.view("phi")[ga:gb])
              and torch.equal(g.view("kint")[lo:hi], ref.view("kint")[ga:gb]))
        q.put({"rank": rank, "ok": bool(ok), "own": [ga, gb]})
        g.close()
        comm.close()
        dist.destroy_process_group()
    except Exception as e:  # noqa: BLE001
        q.put({"rank": rank, "ok": False, "error": f"{type(e).__name__}: {e}"[:500]})


def main():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = []
    for _ in ps:
        try:
            res.append(q.get(timeout=240))
        except Exception:
            res.append({"ok": False, "error": "timeout"})
    for p in ps:
        p.join(timeout=30)
        if p.is_alive():
            p.kill()
    print(json.dumps({"nccl_two_ranks_one_gpu": res}))


if __name__ == "__main__":
    main()
