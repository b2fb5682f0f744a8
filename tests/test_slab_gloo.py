"""Multi-GPU z-slab plan and halo exchange, exercised on CPU with the gloo
backend at world size 2 and 3 (no GPU): the plan's global id bases and halo
ranges are checked against the oracle's global tables, and one grouped
send/recv refreshes every ghost package with the owner's values."""
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


def _local_plane_first(t, p, nx_ny):
    """local first id of every stored plane (+ end) from the oracle tables"""
    pf = []
    for z in range(p.zs_lo, p.zs_hi + 1):
        g = 2 + int(t.plane_count[:z].sum())  # global first id of plane z
        pf.append(g - p.id_base + 2)
    return pf


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
        o = Oracle(w)
        t = o.build_tables()
        p = slab.plan(t.plane_count, world, rank)
        # the slab's stored packages are one contiguous global id range
        pf = _local_plane_first(t, p, w.n[0] * w.n[1])
        halo = slab.halo_ranges(p, pf)
        n_local = pf[-1]
        # global package values: id-dependent pattern (64 per package)
        gvals = (np.arange(t.n_pkg)[:, None] * 64 + np.arange(64)[None, :]).astype(np.float32)
        loc = torch.full((n_local, 64), float("nan"))
        own_lo, own_hi = pf[p.z_lo - p.zs_lo], pf[p.z_hi - p.zs_lo]
        gl = lambda l: l - 2 + p.id_base  # noqa: E731
        loc[own_lo:own_hi] = torch.from_numpy(gvals[gl(own_lo):gl(own_hi)])
        loc[:2] = torch.from_numpy(gvals[:2])
        slab.exchange(loc, halo, rank, world, 64)
        exp = gvals[[0, 1] + [gl(i) for i in range(2, n_local)]]
        ok = np.array_equal(loc.numpy(), exp)
        # the owned ranges of all ranks tile the global id range exactly
        spans = [None] * world
        dist.all_gather_object(spans, (gl(own_lo), gl(own_hi)))
        tiled = spans[0][0] == 2 and spans[-1][1] == t.n_pkg and all(
            a[1] == b[0] for a, b in zip(spans, spans[1:]))
        # ghost planes hold exactly the neighbours' boundary planes
        meta_ok = True
        for (a, b) in (halo.recv_lo, halo.recv_hi):
            if b > a:
                zs = t.meta_cell[[gl(i) for i in range(a, b)]] // (w.n[0] * w.n[1])
                meta_ok &= len(set(zs.tolist())) == 1 and zs[0] in (p.z_lo - 1, p.z_hi)
        q.put((rank, bool(ok), bool(tiled), bool(meta_ok), p.cuts))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, False, False, False, traceback.format_exc()))


@pytest.mark.parametrize("world,name", [(2, "C1"), (3, "C1"), (2, "rand")])
def test_slab_halo_exchange_gloo(world, name):
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
        assert r[1] and r[2] and r[3], r


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
