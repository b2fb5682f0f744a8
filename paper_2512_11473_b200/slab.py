"""Multi-GPU z-slab partition of the sparse grid (north_star: "Packages are
partitioned across the 8xB200 box in z-slabs of the background grid, with
NCCL halo exchange of boundary packages ... each reinitialization iteration
and particles binned to their owning rank").

Plan (host logic, no device compute here):
  1. every rank counts active packages per background plane of a uniform
     z-range (sg_plane_counts), the counts are all-gathered;
  2. balanced cuts (sg_balanced_cuts): rank r owns planes [cuts[r], cuts[r+1]);
  3. global ids follow the linear cell order (z slowest, R-1), so a rank's
     stored planes [z_lo-1, z_hi+1) are ONE contiguous global id range
     starting at id_base = 2 + (packages in planes < z_lo-1);
  4. halos are whole background planes = contiguous local id ranges: the
     first owned plane goes to rank r-1's ghost-above plane, the last owned
     plane to rank r+1's ghost-below plane.  No packing, no index remap.

Per reinit sweep each rank updates its owned packages (sg_reinit(g, 1)) and
then refreshes the ghost packages of the new current phi buffer with one
grouped send/recv (torch.distributed P2P over NCCL; any backend works for
the host-side tests).  Jacobi sweeps are order-independent, so P-GPU results
are bitwise identical to 1 GPU.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class SlabPlan:
    rank: int
    world: int
    cuts: list          # [world + 1] plane cuts
    z_lo: int
    z_hi: int
    zs_lo: int          # stored planes (owned + ghosts inside the domain)
    zs_hi: int
    id_base: int        # global id of local id 2


def plan(counts, world: int, rank: int, cuts=None) -> SlabPlan:
    """counts: per-plane package counts of the whole domain (len nz)."""
    counts = np.asarray(counts, dtype=np.int64)
    nz = counts.size
    if cuts is None:
        from .sg import sg_balanced_cuts
        cuts = sg_balanced_cuts(counts, world)
    z_lo, z_hi = cuts[rank], cuts[rank + 1]
    zs_lo, zs_hi = max(0, z_lo - 1), min(nz, z_hi + 1)
    id_base = 2 + int(counts[:zs_lo].sum())
    return SlabPlan(rank, world, list(cuts), z_lo, z_hi, zs_lo, zs_hi, id_base)


@dataclass
class Halo:
    """Local id ranges [a, b) of the four halo pieces of one rank."""
    send_lo: tuple   # first owned plane -> rank - 1
    send_hi: tuple   # last owned plane  -> rank + 1
    recv_lo: tuple   # ghost plane below <- rank - 1
    recv_hi: tuple   # ghost plane above <- rank + 1


def halo_ranges(p: SlabPlan, plane_first) -> Halo:
    """plane_first: local first id of every stored plane (+ end), i.e. the
    SG_VIEW_PLANE_FIRST array of the rank's grid."""
    pf = [int(v) for v in plane_first]

    def rng(z):  # local id range of stored plane z
        i = z - p.zs_lo
        return (pf[i], pf[i + 1])

    none = (0, 0)
    has_lo, has_hi = p.rank > 0, p.rank < p.world - 1
    return Halo(send_lo=rng(p.z_lo) if has_lo else none,
                send_hi=rng(p.z_hi - 1) if has_hi else none,
                recv_lo=rng(p.z_lo - 1) if has_lo else none,
                recv_hi=rng(p.z_hi) if has_hi else none)


def exchange(field, halo: Halo, rank: int, world: int, per_pkg: int, group=None):
    """Refresh the ghost packages of `field` (a tensor whose first dimension
    is the local package id, flattened to [n_pkg * per_pkg] or shaped
    [n_pkg, ...]) with one grouped send/recv."""
    import torch.distributed as dist
    flat = field.reshape(-1)
    ops = []

    def sl(r):
        return flat[r[0] * per_pkg:r[1] * per_pkg]

    if rank > 0:
        ops.append(dist.P2POp(dist.isend, sl(halo.send_lo), rank - 1, group))
        ops.append(dist.P2POp(dist.irecv, sl(halo.recv_lo), rank - 1, group))
    if rank < world - 1:
        ops.append(dist.P2POp(dist.isend, sl(halo.send_hi), rank + 1, group))
        ops.append(dist.P2POp(dist.irecv, sl(halo.recv_hi), rank + 1, group))
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()


def owner_mask(pos, w, p: SlabPlan):
    """Particles whose containing background plane this rank owns (the
    binning rule of the probe: OOB on every other rank)."""
    import torch
    cz = torch.floor((pos[:, 2].double() - w.lower[2]) / w.cell)
    return (cz >= p.z_lo) & (cz < p.z_hi)


class SlabGrid:
    """One rank's slab of the global grid plus its halo plan."""

    def __init__(self, w, world: int, rank: int, group=None, stream=None):
        import torch
        import torch.distributed as dist
        from . import sg
        self.w, self.world, self.rank, self.group = w, world, rank, group
        nz = w.n[2]
        desc, geom, keep = sg.make_desc(w)
        # 1. per-plane counts of a uniform z range, all-gathered
        lo, hi = rank * nz // world, (rank + 1) * nz // world
        cnt = torch.zeros(max(1, hi - lo), dtype=torch.int64, device="cuda")
        sg.sg_plane_counts(desc, geom, lo, hi, cnt.data_ptr(), stream)
        parts = [torch.zeros(max(1, (r + 1) * nz // world - r * nz // world), dtype=torch.int64,
                             device="cuda") for r in range(world)]
        dist.all_gather(parts, cnt, group=group)
        counts = torch.cat([p[:(r + 1) * nz // world - r * nz // world]
                            for r, p in enumerate(parts)]).cpu().numpy()
        self.counts = counts
        # 2-3. cuts and id base
        self.plan = plan(counts, world, rank)
        self.grid = sg.Grid(w, slab=(self.plan.z_lo, self.plan.z_hi, self.plan.id_base),
                            stream=stream)
        pf = self.grid.view("plane_first").cpu().numpy()
        self.halo = halo_ranges(self.plan, pf)

    def exchange(self, name: str):
        per = {"phi": 64, "kint": 64, "grad": 256}.get(name, 192)
        exchange(self.grid.view(name), self.halo, self.rank, self.world, per, self.group)

    # sweeps between two ghost exchanges: the ghost plane is 4 data points
    # deep, so up to 4 sweeps over owned + ghost packages keep the owned ones
    # exact (include/sg.h sg_reinit_halo; SURVEY 8(e) ghost reuse)
    GHOST_SWEEPS = 4

    def reinit(self, iters: int, cfl: float, stream=None, per_exchange: int | None = None):
        from . import sg
        k = self.GHOST_SWEEPS if per_exchange is None else per_exchange
        done = 0
        while done < iters:
            m = min(k, iters - done)
            if k == 1:
                sg.sg_reinit(self.grid.handle, 1, cfl, stream)
            else:
                sg.sg_reinit_halo(self.grid.handle, m, cfl, stream)
            self.exchange("phi")
            done += m

    def gradient(self, fields: int, h_ratio: float, stream=None):
        from . import sg
        sg.sg_gradient(self.grid.handle, fields, h_ratio, stream)
        if fields & sg.SG_GRAD:
            self.exchange("grad")

    def close(self):
        self.grid.close()


def bench_slab(args, w, rank, world, local):
    """bench.py body for z-slab runs (torchrun, one rank per GPU; also usable
    at world size 1 with --slab to exercise the path): each rank owns a slab,
    reinit sweeps exchange ghost planes over NCCL, particles are binned to the
    owner rank.  Times are device events, max over ranks."""
    import json

    import torch
    import torch.distributed as dist

    import workloads as W
    from . import sg
    from bench import METRIC, UNIT, REINIT_ITERS, ClockSampler, L2Flush, peaks, workload_name

    if not dist.is_initialized():
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    stream = torch.cuda.current_stream()
    npdt = np.float32 if w.dtype == "f32" else np.float64
    pos_np = (W.lattice_particles(w, seed=0, order=args.order, dtype=npdt) if w.particles
              else np.zeros((0, 3), dtype=npdt))
    flush = L2Flush("cuda")
    fields = sg.SG_GRAD | sg.SG_NORMAL | sg.SG_KINT

    # particles binned to their owner rank (input preparation, untimed)
    s0 = SlabGrid(w, world, rank, stream=stream)
    d_pos_all = torch.from_numpy(pos_np).cuda()
    d_pos = d_pos_all[owner_mask(d_pos_all, w, s0.plan)].contiguous()
    del d_pos_all
    n_local = int(d_pos.shape[0])
    info0 = s0.grid.info
    n_pkg_local = info0["own_hi"] - info0["own_lo"]
    s0.close()
    d_phi = torch.empty(n_local, dtype=d_pos.dtype, device="cuda")
    d_grad = torch.empty((n_local, 3), dtype=d_pos.dtype, device="cuda")
    h_pos = d_pos.cpu().pin_memory()
    h_phi = torch.empty(n_local, dtype=d_pos.dtype).pin_memory()
    h_grad = torch.empty((n_local, 3), dtype=d_pos.dtype).pin_memory()

    def full_step(ev, host=False):
        ev[0].record(stream)
        s = SlabGrid(w, world, rank, stream=stream)
        ev[1].record(stream)
        s.reinit(REINIT_ITERS, w.cfl, stream)
        ev[2].record(stream)
        s.gradient(fields, w.h_ratio, stream)
        ev[3].record(stream)
        if n_local:
            if host:
                sg.sg_probe(s.grid.handle, n_local, h_pos.data_ptr(), h_phi.data_ptr(),
                            h_grad.data_ptr(), None, stream)
            else:
                sg.sg_probe(s.grid.handle, n_local, d_pos.data_ptr(), d_phi.data_ptr(),
                            d_grad.data_ptr(), None, stream)
        ev[4].record(stream)
        return s

    def mk():
        return [torch.cuda.Event(enable_timing=True) for _ in range(5)]

    def timed(host):
        st = []
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            dist.barrier()
            ev = mk()
            s = full_step(ev, host)
            torch.cuda.synchronize()
            t = torch.tensor([ev[i].elapsed_time(ev[i + 1]) for i in range(4)], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            st.append(t.cpu().numpy())
            s.close()
        return np.array(st)

    for _ in range(args.warmup):
        flush.zero_()
        full_step(mk()).close()
    torch.cuda.synchronize()
    l0 = sg.sg_launch_count()
    with ClockSampler(local) as clk:
        st = timed(False)
    launches = sg.sg_launch_count() - l0
    e2e = None
    if not args.no_e2e and n_local:
        et = timed(True)
    tot = torch.tensor([n_pkg_local, n_local], dtype=torch.int64, device="cuda")
    dist.all_reduce(tot)
    n_act = int(tot[0].item()) * 64
    n_part = int(tot[1].item())
    ms = float(st.sum(1).mean())
    updates = n_act * (REINIT_ITERS + 1)
    if not args.no_e2e and n_local:
        e_ms = float(et.sum(1).mean())
        e2e = {"value": updates / (e_ms * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": int(n_part * 3 * h_pos.element_size()),
               "d2h_bytes_per_step": int(n_part * 4 * h_pos.element_size()),
               "ms_per_step": e_ms}
    reinit_ms = float(st[:, 1].mean()) / REINIT_ITERS
    esz = 4 if w.dtype == "f32" else 8
    bpc = 2 * esz + 108 / 64
    hbm, src = peaks()
    # per-GPU achieved bandwidth of the sweep (incl. the ghost exchange)
    achieved = bpc * n_act / world / (reinit_ms * 1e-3) / 1e9
    if rank == 0:
        out = {"metric": METRIC, "value": updates / (ms * 1e-3), "unit": UNIT,
               "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
               "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
               "dtype": w.dtype, "data": "synthetic",
               "config": {"workload": workload_name(w, n_part, args.order) +
                          f", z-slab partitioned over {world} GPUs, NCCL ghost planes every "
                          f"{SlabGrid.GHOST_SWEEPS} sweeps",
                          "active_cells": n_act, "particles": n_part,
                          "parallelism": f"zslab{world}",
                          "l2": "flushed between steps (512 MiB write + 256 MiB read of another buffer, outside the timed events)"},
               "probes_per_s": n_part / (ms * 1e-3),
               "stages": {n: {"ms": float(st[:, i].mean())} for i, n in
                          enumerate(["build", "reinit", "gradient", "probe"])},
               "e2e": e2e, "gpu_launches": int(launches),
               "roofline": {"kernel": "k_reinit<float> + ghost exchange", "bound": "hbm",
                            "achieved": achieved, "peak": hbm, "peak_source": src,
                            "unit": "GB/s", "frac": achieved / hbm, "traffic": None,
                            "note": "per GPU, sweep time max over ranks incl. NCCL exchange"},
               "clocks": clk.summary()}
        print(json.dumps(out), flush=True)
    dist.destroy_process_group()
