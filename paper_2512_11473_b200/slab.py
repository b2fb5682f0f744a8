"""Multi-GPU z-slab partition (north_star: "Packages are partitioned across the
8xB200 box in z-slabs of the background grid, with NCCL halo exchange of
boundary packages over NVLink each reinitialization iteration and particles
binned to their owning rank").

Everything happens in libsg (include/sg.h): the plan (sg_slab_plan: balanced
cuts of the all-gathered per-plane package counts, contiguous global id
ranges, halo ranges), the partitioned build (sg_build_ex with a
communicator), the ghost exchanges inside sg_reinit / sg_gradient (grouped
NCCL send/recv of whole background planes, overlapped with the interior
sweep) and the particle binning + all-to-all inside sg_probe.  This module
only wires a communicator to a grid and runs the bench body.
"""
from __future__ import annotations

from types import SimpleNamespace


def plan(counts, world: int, rank: int) -> SimpleNamespace:
    """The library's plan of `rank` (sg_slab_plan) with attribute access;
    `cuts` holds every rank's plane cuts."""
    from .sg import sg_slab_plan
    p, cuts = sg_slab_plan(counts, world, rank)
    return SimpleNamespace(rank=rank, world=world, cuts=cuts, **p)


class SlabGrid:
    """One rank's slab of a partitioned grid (collective calls)."""

    def __init__(self, w, comm, stream=None, allocator=None):
        from . import sg
        self.comm = comm
        self.grid = sg.Grid(w, comm=comm, stream=stream, allocator=allocator)

    @property
    def info(self) -> dict:
        return self.grid.info

    def reinit(self, iters: int, cfl: float, stream=None):
        self.grid.reinit(iters, cfl, stream)
        return self

    def gradient(self, fields: int, h_ratio: float, stream=None):
        self.grid.gradient(fields, h_ratio, stream)
        return self

    def probe(self, pos, want_grad: bool = True, stream=None):
        return self.grid.probe(pos, want_grad=want_grad, stream=stream)

    def close(self):
        self.grid.close()


def share(n: int, world: int, rank: int) -> tuple:
    """[a, b): the index range of a particle array rank `rank` holds before
    binning (contiguous shares, as a loader hands them out)."""
    return n * rank // world, n * (rank + 1) // world


def bench_slab(args, w, rank, world, local):
    """bench.py body under torchrun (one rank per GPU): each rank builds its
    slab through the NCCL communicator, reinitialises (ghost exchange every 4
    sweeps, overlapped with the interior), computes grad / normal / K / G,
    and probes its contiguous share of the particles (binned to the owners
    and returned in order inside sg_probe).  Device-event times, max over
    ranks."""
    import json

    import numpy as np
    import torch
    import torch.distributed as dist

    import workloads as W  # noqa: F401
    from . import sg
    from bench import (METRIC, UNIT, REINIT_ITERS, ClockSampler, L2Flush, peaks, workload_name,
                       SWEEP_BYTES_SURVEY)

    if not dist.is_initialized():
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    stream = torch.cuda.current_stream()
    comm = sg.Comm.nccl()
    # every rank generates the workload's particle set on its device and keeps
    # a contiguous 1/world share (as a loader would hand them out); sg_probe
    # bins them to their owners
    full = W.particles(w, seed=0, order=args.order, device="cuda")
    n_all = int(full.shape[0])
    a, b = share(n_all, world, rank)
    d_pos = full[a:b].contiguous()
    del full
    flush = L2Flush("cuda")
    fields = sg.SG_GRAD | sg.SG_NORMAL | sg.SG_KINT
    n_local = int(d_pos.shape[0])
    if w.name == "C5":
        args.no_e2e = True  # 25 GB of pinned staging per step; the e2e headline is C2's
    d_phi = torch.empty(n_local, dtype=d_pos.dtype, device="cuda")
    d_grad = torch.empty((n_local, 3), dtype=d_pos.dtype, device="cuda")
    h_pos = d_pos.cpu().pin_memory() if not args.no_e2e else None
    h_phi = torch.empty(n_local, dtype=d_pos.dtype).pin_memory() if not args.no_e2e else None
    h_grad = torch.empty((n_local, 3), dtype=d_pos.dtype).pin_memory() if not args.no_e2e else None

    def full_step(ev, host=False):
        ev[0].record(stream)
        s = SlabGrid(w, comm, stream=stream)
        ev[1].record(stream)
        s.reinit(REINIT_ITERS, w.cfl, stream)
        ev[2].record(stream)
        s.gradient(fields, w.h_ratio, stream)
        ev[3].record(stream)
        if w.particles:
            if host:
                h2 = h_pos.to("cuda", non_blocking=True)
                p, g = s.grid.probe(h2, stream=stream)
                h_phi.copy_(p, non_blocking=True)
                h_grad.copy_(g, non_blocking=True)
            else:
                sg.sg_probe(s.grid.handle, n_local, d_pos.data_ptr() if n_local else 0,
                            d_phi.data_ptr() if n_local else 0,
                            d_grad.data_ptr() if n_local else 0, None, stream)
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
    s0 = SlabGrid(w, comm, stream=stream)
    info0 = s0.info
    n_pkg_local = info0["own_hi"] - info0["own_lo"]
    s0.close()
    l0 = sg.sg_launch_count()
    with ClockSampler(local) as clk:
        st = timed(False)
    launches = sg.sg_launch_count() - l0
    e2e = None
    if not args.no_e2e and w.particles:
        et = timed(True)
    comm.check()  # an asynchronous NCCL error fails the run instead of printing a number
    tot = torch.tensor([n_pkg_local], dtype=torch.int64, device="cuda")
    dist.all_reduce(tot)
    n_act = int(tot[0].item()) * 64
    med = np.median(st.sum(1))
    ms = float(med)
    updates = n_act * (REINIT_ITERS + 1)
    if e2e is None and not args.no_e2e and w.particles:
        e_ms = float(np.median(et.sum(1)))
        esz = 4 if w.dtype == "f32" else 8
        e2e = {"value": updates / (e_ms * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": int(n_all * 3 * esz),
               "d2h_bytes_per_step": int(n_all * 4 * esz),
               "ms_per_step": e_ms, "note": "per-step H2D of every rank's particle share, "
                                            "D2H of phi and grad, summed over ranks"}
    reinit_ms = float(np.median(st[:, 1])) / REINIT_ITERS
    esz = 4 if w.dtype == "f32" else 8
    bpc = SWEEP_BYTES_SURVEY(esz)
    hbm, src = peaks()
    # per-GPU achieved bandwidth of the sweep (incl. the ghost exchange)
    achieved = bpc * n_act / world / (reinit_ms * 1e-3) / 1e9
    if rank == 0:
        out = {"metric": METRIC, "value": updates / (ms * 1e-3), "unit": UNIT,
               "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
               "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
               "dtype": w.dtype, "data": "synthetic",
               "config": {"workload": workload_name(w, n_all, args.order) +
                          f", z-slab partitioned over {world} GPUs (libsg NCCL communicator: "
                          f"ghost planes every 4 sweeps overlapped with the interior sweep, "
                          f"particles binned to their owners inside sg_probe)",
                          "active_cells": n_act, "particles": n_all,
                          "parallelism": f"zslab{world}",
                          "l2": "flushed between steps (512 MiB write + 256 MiB read of another buffer, outside the timed events)",
                          "statistic": "median over the timed steps"},
               "probes_per_s": n_all / (ms * 1e-3),
               "stages": {n: {"ms": float(np.median(st[:, i]))} for i, n in
                          enumerate(["build", "reinit", "gradient", "probe"])},
               "e2e": e2e, "gpu_launches": int(launches),
               "roofline": {"kernel": "k_sweep<float> + ghost exchange", "bound": "hbm",
                            "achieved": achieved, "peak": hbm, "peak_source": src,
                            "unit": "GB/s", "frac": achieved / hbm, "traffic": None,
                            "bytes_per_cell": bpc,
                            "note": "per GPU, SURVEY 8(d) bytes per point, sweep time max over "
                                    "ranks incl. the NCCL exchange"},
               "clocks": clk.summary()}
        print(json.dumps(out), flush=True)
    comm.close()
    dist.destroy_process_group()
