"""Host side of the multi-GPU z-slab partition at world size 2 and 3 over the
gloo backend on CPU (no GPU): every rank derives its plan with the library's
host function (sg_slab_plan, the function the partitioned build calls after
its all-gather) from per-plane counts it computes and all-gathers itself, as
the build does; the plans of all ranks are then checked against each other
and against the oracle's global tables: owned ranges tile the global id
range, each rank's ghost planes are exactly its neighbours' boundary planes
(global ids and cells), and one grouped send/recv over the plan's ranges
(driven by the test, the role NCCL plays inside libsg) refreshes every ghost
package with the owner's values."""
import os
import socket

import numpy as np
import pytest

import workloads as W


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, q):
    try:
        import torch
        import torch.distributed as dist
        from oracle.oracle import Oracle
        from paper_2512_11473_b200 import slab
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        w = W.config(name) if name in W.CONFIGS else W.random_scene(3, 24)
        t = Oracle(w).build_tables()
        nz = w.n[2]
        # the build's count pass: this rank's uniform plane range, all-gathered
        lo, hi = rank * nz // world, (rank + 1) * nz // world
        mine = torch.from_numpy(t.plane_count[lo:hi].copy())
        maxper = -(-nz // world)
        buf = torch.zeros(maxper, dtype=torch.int64)
        buf[:hi - lo] = mine
        parts = [torch.zeros(maxper, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(parts, buf)
        counts = np.concatenate([parts[r][:(r + 1) * nz // world - r * nz // world].numpy()
                                 for r in range(world)])
        p = slab.plan(counts, world, rank)
        gl = lambda l: l - 2 + p.id_base  # noqa: E731
        # global package values: id-dependent pattern (64 per package)
        gvals = (np.arange(t.n_pkg)[:, None] * 64 + np.arange(64)[None, :]).astype(np.float32)
        loc = torch.full((p.n_pkg, 64), float("nan"))
        loc[p.own_lo:p.own_hi] = torch.from_numpy(gvals[gl(p.own_lo):gl(p.own_hi)])
        loc[:2] = torch.from_numpy(gvals[:2])
        ops = []
        flat = loc.reshape(-1)

        def sl(r):
            return flat[r[0] * 64:r[1] * 64]
        for peer, send, recv in ((rank - 1, p.send_lo, p.recv_lo), (rank + 1, p.send_hi, p.recv_hi)):
            if 0 <= peer < world:
                if send[1] > send[0]:
                    ops.append(dist.P2POp(dist.isend, sl(send), peer))
                if recv[1] > recv[0]:
                    ops.append(dist.P2POp(dist.irecv, sl(recv), peer))
        if ops:
            for h in dist.batch_isend_irecv(ops):
                h.wait()
        exp = gvals[[0, 1] + [gl(i) for i in range(2, p.n_pkg)]]
        ok = np.array_equal(loc.numpy(), exp)
        spans = [None] * world
        dist.all_gather_object(spans, (gl(p.own_lo), gl(p.own_hi)))
        tiled = spans[0][0] == 2 and spans[-1][1] == t.n_pkg and all(
            a[1] == b[0] for a, b in zip(spans, spans[1:]))
        # ghost planes hold exactly the neighbours' boundary planes (cells)
        meta_ok = True
        for (a, b), z in ((p.recv_lo, p.z_lo - 1), (p.recv_hi, p.z_hi)):
            if b > a:
                zs = t.meta_cell[[gl(i) for i in range(a, b)]] // (w.n[0] * w.n[1])
                meta_ok &= bool(np.all(zs == z))
        plans = [None] * world
        dist.all_gather_object(plans, (p.cuts, p.id_base, p.z_lo, p.z_hi))
        same_cuts = all(pl[0] == p.cuts for pl in plans)
        q.put((rank, bool(ok), bool(tiled), bool(meta_ok), bool(same_cuts)))
        dist.destroy_process_group()
    except Exception:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, False, False, False, traceback.format_exc()))


@pytest.mark.parametrize("world,name", [(2, "C1"), (3, "C1"), (2, "rand"), (3, "C2")])
def test_slab_plan_and_halo_gloo(world, name):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for r in res:
        assert r[1] and r[2] and r[3] and r[4], r


def test_plan_id_base_and_cuts():
    from oracle.oracle import Oracle
    from paper_2512_11473_b200 import slab
    t = Oracle(W.config("C2")).build_tables()
    for world in (2, 4, 8):
        plans = [slab.plan(t.plane_count, world, r) for r in range(world)]
        assert plans[0].z_lo == 0 and plans[-1].z_hi == 128
        for a, b in zip(plans, plans[1:]):
            assert a.z_hi == b.z_lo
        for p in plans:
            # id_base = 2 + packages below the first stored plane
            assert p.id_base == 2 + int(t.plane_count[:p.zs_lo].sum())
            assert p.zs_lo == max(0, p.z_lo - 1) and p.zs_hi == min(128, p.z_hi + 1)
