#!/usr/bin/env python
"""Benchmark of the sparse-grid hot path (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config C2] [--order lattice|shuffled] [--no-cpu-baseline]

One STEP = one pass of the whole hot path over one synthetic batch
 on the workload BASELINE.json's metric is quoted
on (configs[1], "C2": extruded prism, 512^3 effective, fp32), with the
configs[3] particle set ("C4": ~19.45 M jittered lattice particles inside the
prism) as the probe batch:
    sg_build (tag, compaction, neighbour table, initial phi)
    sg_reinit (20 Godunov sweeps)
    sg_gradient (grad + normal + kernel integrals)
    sg_probe (phi and grad phi at every particle)
sg_gradient(SG_GRAD | SG_NORMAL | SG_KINT) runs the gradient / normal (K6)
and kernel-integral (K7) work in one kernel, K6 warps beside K7 warps.
(--kint-stream: K7 as a separate call on a second, low-priority stream
overlapping K6 and the probe on the step's high-priority stream -- the same
step time on C2.)
value = active data points updated by the reinit + gradient sweeps per second
of whole step (21 sweeps x 8.58 M active points), i.e. BASELINE's
"active cells updated/s (reinit+gradient)"; probes/s and per-stage numbers are
reported beside it.  Inputs are resident in HBM before timing; L2 is flushed
(a 512 MiB write, then a 256 MiB read of another buffer so the flush's dirty
lines are written back before the step) between timed steps, outside the
timed events.

e2e: the same step through the C-ABI with HOST buffers: particle positions
from pinned host memory, probe results back to pinned host memory (the
library stages them in pipelined chunks) inside the timed region.

--impl reference: the CPU oracle (oracle/, fp64, dense) as it stands, on
this host's cores, each step a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402

METRIC = "active cells updated/s (reinit+gradient) & particle probes/s; % of HBM peak, 1/2/4/8 GPU"
UNIT = "cell-updates/s"
REINIT_ITERS = 20
FALLBACK_HBM_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback


def SWEEP_BYTES_SURVEY(esz):
    """SURVEY 8(d) algorithmic bytes per point of a reinit sweep: phi in +
    phi out + the package's 108 B neighbour row over its 64 points."""
    return 2 * esz + 108 / 64


def SWEEP_BYTES_FACE(esz):
    """what k_sweep actually needs: phi in + out + the 32 B face row (the six
    face slots of the neighbour row)"""
    return 2 * esz + 32 / 64


def profile_json(name):
    try:
        with open(os.path.join(ROOT, "profiles", name)) as f:
            return json.load(f)
    except Exception:
        return None


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=30)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="C2")
    p.add_argument("--order", default="lattice", choices=["lattice", "shuffled"])
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-kernel-roofline", action="store_true",
                   help="skip the per-kernel roofline timings after the timed steps "
                        "(e.g. under ncu, so the launch list is the steps only)")
    p.add_argument("--kint-stream", action="store_true",
                   help="kernel integrals as a separate call on a second, low-priority "
                        "stream overlapping gradient and probe (default: one sg_gradient "
                        "call, K6 and K7 in one kernel)")
    p.add_argument("--slab", action="store_true",
                   help="z-slab path (NCCL) even at one rank (exercises the multi-GPU code)")
    p.add_argument("--no-c3-anchor", action="store_true",
                   help="skip the C3 sub-record (the HBM-bound reinit anchor)")
    return p.parse_args()


def rank_info():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


class L2Flush:
    """Between timed steps: write a 512 MiB buffer (evicts the working set),
    then read a separate 256 MiB one, so the flush's own dirty lines are
    written back before the next timed step instead of inside it (outside
    the timed events; stream-ordered, no host sync)."""

    def __init__(self, device):
        import torch
        self.w = torch.empty(512 << 20, dtype=torch.uint8, device=device)
        self.r = torch.zeros(256 << 20, dtype=torch.uint8, device=device)

    def zero_(self):  # drop-in for the former buffer.zero_() calls
        self.w.zero_()
        self.r.max()
        return self


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            mp = json.load(f)
        return float(mp["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def ncu_traffic(kernel: str, config: str):
    """dram read+write bytes per launch from a committed ncu --set full
    capture (profiles/ncu_traffic.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            t = json.load(f)
        return t.get(config, {}).get(kernel)
    except Exception:
        return None


# --------------------------------------------------------------- clocks ----

class ClockSampler:
    """SM clock and throttle reasons sampled every 5 ms through NVML while the
    timed region runs (nvidia-smi's clocks line, at a finer period)."""
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, device: int, period: float = 0.005):
        self.device, self.period = device, period
        self.sm, self.mx, self.reasons = [], [], set()
        self._stop = threading.Event()
        self.nv = None

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.nv = nv
            self.h = nv.nvmlDeviceGetHandleByIndex(self.device)
            self.max_sm = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
            get = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                getattr(nv, "nvmlDeviceGetCurrentClocksThrottleReasons")
            self._reasons = get
            # the first NVML queries of a process can be slow and hold driver
            # locks: take one sample before the timed region starts
            self._sample()
            self.sm.clear()
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        except Exception:
            self.nv = None
        return self

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            self._sample()
            time.sleep(self.period)

    def _sample(self):
        nv = self.nv
        try:
            self.sm.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
            r = self._reasons(self.h)
            for bit, name in self.REASONS.items():
                if r & bit:
                    self.reasons.add(name)
        except Exception:
            pass

    def __exit__(self, *a):
        self._stop.set()
        if self.nv is not None:
            self.t.join(timeout=2)

    def summary(self):
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(self.sm)), "sm_max_mhz": float(self.max_sm),
                "reasons": sorted(self.reasons), "samples": len(self.sm),
                "sm_mhz_min": float(min(self.sm))}


# ------------------------------------------------------------ our arm ------

def workload_name(w, n_part, order):
    eff = 4 * w.n[0]
    desc = {"C1": "sphere r=0.3", "C2": "extruded prism", "C3": "torus+box union",
            "C5": "thin-shell multi-body scene", "T1": "Table-1 shelled sphere"}.get(w.name, w.name)
    s = (f"{w.name}: {desc} {eff}^3 effective ({w.n[0]}^3 cells x 4^3), {w.dtype}, "
         f"reinit {REINIT_ITERS} + grad/normal/kernel-integral")
    if n_part:
        what = "C4 probe" if w.name == "C2" else "probe of the shell-wall lattice"
        s += f" + {what} of {n_part} particles ({order} order)"
    return s


def run_config(w, n_pkg, n_part, order, world):
    """The `config` object of the JSON line (shared by both arms)."""
    return {"workload": workload_name(w, n_part, order),
            "n_packages": n_pkg - 2, "active_cells": (n_pkg - 2) * 64, "particles": n_part,
            "l2": "flushed between steps (512 MiB write + 256 MiB read of another buffer, "
                  "outside the timed events)",
            "parallelism": f"zslab{world}" if world > 1 else "1 GPU"}


def kernel_rooflines(sg, w, stream, flush, d_pos, n_part, probe_ms, reinit_ms, hbm):
    """Roofline of each hot-path kernel on its own (SURVEY 8(d) units): the
    reinit sweep and the probe from the timed steps, the gradient/normal (K6)
    and kernel-integral (K7) kernels -- concurrent inside a step -- timed
    apart here on one grid (10 launches each, L2 flushed before each,
    CUDA events on the launching stream)."""
    import torch
    esz = 4 if w.dtype == "f32" else 8
    g = sg.Grid(w, stream=stream).reinit(REINIT_ITERS, w.cfl, stream=stream)
    n_act = (g.info["n_pkg"] - 2) * 64

    def timed(fn, reps=10):
        ts = []
        for _ in range(reps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn()
            b.record(stream)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        return float(np.median(ts))

    t_grad = timed(lambda: g.gradient(sg.SG_GRAD | sg.SG_NORMAL, w.h_ratio, stream=stream))
    t_kint = timed(lambda: g.gradient(sg.SG_KINT, w.h_ratio, stream=stream))
    t_both = timed(lambda: g.gradient(sg.SG_GRAD | sg.SG_NORMAL | sg.SG_KINT, w.h_ratio,
                                      stream=stream))
    clock_ghz = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["sm_max_mhz"]) \
        / 1e3 if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 1.965
    sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    fma_peak = sms * 128 * clock_ghz * 1e9  # FP32 FMA lanes x clock (B200_PROFILING.md units)

    def hbm_entry(name, bytes_, ms, note, layout_bytes=None):
        a = bytes_ / (ms * 1e-3) / 1e9
        e = {"kernel": name, "bound": "hbm", "us": ms * 1e3, "alg_bytes": bytes_,
             "achieved": a, "unit": "GB/s", "peak": hbm, "frac": a / hbm,
             "frac_nominal_8tbs": a / 8000.0, "note": note}
        if layout_bytes:
            al = layout_bytes / (ms * 1e-3) / 1e9
            e.update({"layout_bytes": layout_bytes, "achieved_layout": al, "frac_layout": al / hbm})
        return e

    out = [hbm_entry("k_sweep (reinit, per sweep)", SWEEP_BYTES_SURVEY(esz) * n_act, reinit_ms,
                     "SURVEY 8(d): phi in + out + 108 B neighbour row per package; layout: the "
                     "32 B face row the kernel reads", SWEEP_BYTES_FACE(esz) * n_act)]
    out.append(hbm_entry("k_gradient (grad + normal)", (4 * esz + 108 / 64 + 3 * esz) * n_act, t_grad,
                         "SURVEY 8(d): b + 3b + 1.69 + 12 (normals) per point; layout: phi + face "
                         "row in, (phi, grad) interleaved (16 B) + normal out",
                         (esz + 32 / 64 + 7 * esz) * n_act))
    fmas = 324.0 * n_act  # 81 taps x (K, Gx, Gy, Gz), direct form
    ke = {"kernel": "k_kint (kernel integrals)", "bound": "alu", "us": t_kint * 1e3,
          "alg_fma": fmas, "achieved": fmas / (t_kint * 1e-3) / 1e12, "unit": "TFMA/s",
          "peak": fma_peak / 1e12, "frac": None,
          "frac_direct_form": fmas / (t_kint * 1e-3) / fma_peak,
          "note": "rate of direct-form FMAs (81 taps x 4 per point) against SMs x 128 FP32 lanes x "
                  "max SM clock; above 1 where the kernel executes fewer FMAs than the direct form "
                  "(sign butterfly, paired FFMA2, closed form on uniform rows) -- the executed "
                  "fraction is the ncu entry below"}
    out.append(ke)
    fl = (profile_json("ncu_flops.json") or {}).get(w.name, {}).get("k_kint")
    if fl:
        # the step's fused K6+K7 kernel as ncu counted it: executed FP32
        # FFMA + FADD + FMUL thread instructions per launch over the ncu
        # duration of the same launch (cold cache, serialised)
        ex = fl["ffma"] + fl["fadd"] + fl["fmul"] + 2 * (fl.get("ffma2", 0.0) + fl.get("fadd2", 0.0) +
                                                         fl.get("fmul2", 0.0))
        ex_peak = (profile_json("alu_peaks.json") or {}).get("fp32_tflops", 2 * fma_peak / 1e12) / 2
        out.append({"kernel": "k_kint<..., K6 fused> executed FP32 work (ncu)", "bound": "alu",
                    "us": fl["us"], "executed_fp32_inst": ex,
                    "achieved": ex / (fl["us"] * 1e-6) / 1e12, "unit": "T inst/s",
                    "peak": ex_peak, "frac": ex / (fl["us"] * 1e-6) / 1e12 / ex_peak,
                    "peak_source": "profiles/alu_peaks.json fp32 FMA/s (measured)",
                    "note": "profiles/ncu_flops.json: FFMA+FADD+FMUL thread instructions + 2 x the "
                            "paired FFMA2/FADD2/FMUL2 ones (FP32 lane operations); one per FP32 "
                            "lane-cycle"})
    out.append({"kernel": "k_kint<..., K6 fused> (gradient + normal + kernel integrals)",
                "bound": "alu", "us": t_both * 1e3,
                "note": "one kernel: K6 warps beside K7 warps; compare with the two above"})
    if probe_ms:
        # the probe alone (inside the step it overlaps the kernel integrals)
        o_phi = torch.empty(n_part, dtype=d_pos.dtype, device=d_pos.device)
        o_grad = torch.empty((n_part, 3), dtype=d_pos.dtype, device=d_pos.device)
        probe_ms = timed(lambda: sg.sg_probe(g.handle, n_part, d_pos.data_ptr(), o_phi.data_ptr(),
                                             o_grad.data_ptr(), None, stream))
        del o_phi, o_grad
        # 12 B position in, 16 B (phi, grad) out, 4 B background entry per probe,
        # plus every touched package's (phi, grad) vectors and neighbour row once
        with torch.no_grad():
            inv = torch.tensor(1.0 / w.cell, dtype=d_pos.dtype, device=d_pos.device)
            c = torch.clamp((d_pos * inv).floor().long(), min=0)
            c[:, 0].clamp_(max=w.n[0] - 1)
            c[:, 1].clamp_(max=w.n[1] - 1)
            c[:, 2].clamp_(max=w.n[2] - 1)
            bg = g.view("bg").view(torch.int32).long()
            ids = bg[c[:, 0] + w.n[0] * (c[:, 1] + w.n[1] * c[:, 2])]
            touched = int(torch.unique(ids[ids >= 2]).numel())
        pb = 32.0 * n_part + touched * (64 * 4 * esz + 108)
        out.append(hbm_entry("k_probe", pb, probe_ms,
                             f"32 B per probe + {touched} touched packages x "
                             f"({64 * 4 * esz} B + 108 B nb row)"))
    g.close()
    # build kernels: fp64 ALU rooflines from ncu counts of the same launch
    # (profiles/ncu_flops.json: thread-level DFMA/DADD/DMUL and the kernel's
    # ncu duration, cold cache and serialised -- a share, not a step time)
    alu = profile_json("alu_peaks.json") or {}
    fp64_peak = alu.get("fp64_tflops") or sms * 64 * 2 * clock_ghz / 1e3
    for name, fl in sorted(((profile_json("ncu_flops.json") or {}).get(w.name) or {}).items()):
        if not name.startswith(("k_phi_init", "k_tag")):
            continue
        dflop = 2 * fl["dfma"] + fl["dadd"] + fl["dmul"]
        a = dflop / (fl["us"] * 1e-6) / 1e12
        out.append({"kernel": name, "bound": "alu", "us": fl["us"], "dflop": dflop,
                    "achieved": a, "unit": "TFLOP/s (fp64)", "peak": fp64_peak,
                    "frac": a / fp64_peak,
                    "peak_source": "profiles/alu_peaks.json (measured DFMA chain)" if
                    alu.get("fp64_tflops") else "SMs x 64 FP64 lanes x 2 x max SM clock",
                    "note": "executed fp64 flops (2 DFMA + DADD + DMUL) from ncu over the ncu "
                            "kernel time"})
    return out


def run_ours(args, rank, world, local):
    import torch
    import torch.distributed as dist
    from paper_2512_11473_b200 import build as B
    from paper_2512_11473_b200 import sg

    B.build()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    w = W.config(args.config)
    if world > 1 or args.slab:
        from paper_2512_11473_b200 import slab as SL
        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29533")
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        return SL.bench_slab(args, w, rank, world, local)
    # the step's stream: high priority (see the K7 side stream below)
    stream = torch.cuda.Stream(device=dev, priority=-1)
    torch.cuda.set_stream(stream)

    # the workload's particle set, generated on the device (C4 on C2: the
    # prism lattice; C5: the shell-wall lattice); C3 has none (no probe stage)
    d_pos = W.particles(w, seed=0, order=args.order, device=dev)
    n_part = int(d_pos.shape[0])
    if n_part == 0 or w.name == "C5":
        # C5's e2e would stage 25 GB through pinned host memory per step;
        # the e2e headline is C2's
        args.no_e2e = True
    d_phi = torch.empty(n_part, dtype=d_pos.dtype, device=dev)
    d_grad = torch.empty((n_part, 3), dtype=d_pos.dtype, device=dev)
    d_oob = torch.zeros(1, dtype=torch.int64, device=dev)
    flush = L2Flush(dev)
    fields = sg.SG_GRAD | sg.SG_NORMAL | sg.SG_KINT

    # --kint-stream: K7 (kernel integrals) only needs the final phi and nothing
    # downstream in the step reads K / G, so it can run on a second,
    # low-priority stream forked after the reinit and joined at the end of the
    # step while K6 and the probe run on the high-priority step stream
    side = torch.cuda.Stream(device=dev, priority=0)
    fork, join = torch.cuda.Event(), torch.cuda.Event()

    def step(ev, host=None):
        ev[0].record(stream)
        g = sg.Grid(w, stream=stream)
        ev[1].record(stream)
        g.reinit(REINIT_ITERS, w.cfl, stream=stream)
        ev[2].record(stream)
        if not args.kint_stream:
            g.gradient(fields, w.h_ratio, stream=stream)
        else:
            fork.record(stream)
            side.wait_event(fork)
            g.gradient(sg.SG_KINT, w.h_ratio, stream=side)
            g.gradient(sg.SG_GRAD | sg.SG_NORMAL, w.h_ratio, stream=stream)
        ev[3].record(stream)
        if n_part == 0:
            pass
        elif host is None:
            sg.sg_probe(g.handle, n_part, d_pos.data_ptr(), d_phi.data_ptr(), d_grad.data_ptr(),
                        d_oob.data_ptr(), stream)
        else:
            hp, hphi, hgrad = host
            sg.sg_probe(g.handle, n_part, hp.data_ptr(), hphi.data_ptr(), hgrad.data_ptr(),
                        d_oob.data_ptr(), stream)
        if args.kint_stream:
            join.record(side)
            stream.wait_event(join)
        ev[4].record(stream)
        info = g.info
        g.close_async(stream)
        return info

    def mk():
        return [torch.cuda.Event(enable_timing=True) for _ in range(5)]

    for _ in range(args.warmup):
        flush.zero_()
        step(mk())
    torch.cuda.synchronize()

    evs = [mk() for _ in range(args.steps)]
    l0 = sg.sg_launch_count()
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        t_wall = time.perf_counter()
        for k in range(args.steps):
            flush.zero_()
            info = step(evs[k])
        torch.cuda.synchronize()
        t_wall = time.perf_counter() - t_wall
    launches = sg.sg_launch_count() - l0
    st = np.array([[evs[k][i].elapsed_time(evs[k][i + 1]) for i in range(4)]
                   for k in range(args.steps)])  # ms per stage
    step_ms = st.sum(1)
    ms = float(np.median(step_ms))  # median over the timed steps
    n_pkg = info["n_pkg"]
    n_act = (n_pkg - 2) * 64
    updates = n_act * (REINIT_ITERS + 1)
    value = updates / (ms * 1e-3)

    # e2e: host buffers through the C-ABI
    e2e = None
    if not args.no_e2e:
        hp = d_pos.cpu().pin_memory()
        hphi = torch.empty(n_part, dtype=hp.dtype).pin_memory()
        hgrad = torch.empty((n_part, 3), dtype=hp.dtype).pin_memory()
        for _ in range(max(1, args.warmup // 2)):
            flush.zero_()
            step(mk(), (hp, hphi, hgrad))
        torch.cuda.synchronize()
        e_ms = []
        for _ in range(args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            ev = mk()
            step(ev, (hp, hphi, hgrad))
            torch.cuda.synchronize()
            e_ms.append(ev[0].elapsed_time(ev[4]))
        e_ms = float(np.median(e_ms))
        e2e = {"value": updates / (e_ms * 1e-3), "unit": UNIT,
               "h2d_bytes_per_step": int(hp.numel() * hp.element_size()),
               "d2h_bytes_per_step": int((hphi.numel() + hgrad.numel()) * hphi.element_size()),
               "ms_per_step": e_ms, "probes_per_s": n_part / (e_ms * 1e-3)}

    # roofline of the dominant kernel (k_sweep: 20 launches per step)
    esz = 4 if w.dtype == "f32" else 8
    reinit_ms = float(np.median(st[:, 1])) / REINIT_ITERS
    # algorithmic bytes: SURVEY 8(d)'s 2b + 108/64 per point (phi in/out, the
    # neighbour row); the kernel itself reads the 32 B face row (8.5 B at
    # fp32), reported beside it
    bytes_per_cell = SWEEP_BYTES_SURVEY(esz)
    alg_bytes = bytes_per_cell * n_act
    hbm, peak_src = peaks()
    achieved = alg_bytes / (reinit_ms * 1e-3) / 1e9
    achieved_face = SWEEP_BYTES_FACE(esz) * n_act / (reinit_ms * 1e-3) / 1e9
    stage_names = ["build", "reinit", "gradient", "probe"]
    stages = {n: {"ms": float(np.median(st[:, i]))} for i, n in enumerate(stage_names)}
    stages["build"]["note"] = ("every step builds the grid anew (all build kernels run); from the "
                               "second build of the same input the arena is sized from the previous "
                               "build's package count and the count read back is checked after the "
                               "build's work is queued (include/sg.h sg_build; SG_BUILD_HINT=0 "
                               "synchronises mid-build instead)")
    stages["reinit"]["ms_per_sweep"] = reinit_ms
    stages["reinit"]["cells_per_s"] = n_act / (reinit_ms * 1e-3)
    stages["probe"]["probes_per_s"] = n_part / max(stages["probe"]["ms"] * 1e-3, 1e-12)
    if not args.kint_stream:
        stages["gradient"]["note"] = ("grad+normal (K6) and kernel integrals (K7): one "
                                      "sg_gradient call, one kernel (K6 warps beside K7 warps)")
    else:
        stages["gradient"]["note"] = ("grad+normal (K6); the kernel integrals (K7) run on a "
                                      "second stream from here to the end of the step")
        stages["probe"]["note"] = "probe (if any), concurrent with K7, then the join of K7"
    stages["reinit_plus_gradient_cells_per_s"] = n_act * (REINIT_ITERS + 1) / (
        (np.median(st[:, 1]) + np.median(st[:, 2])) * 1e-3)
    clocks = clk.summary()
    kernels = None if args.no_kernel_roofline else kernel_rooflines(
        sg, w, stream, flush, d_pos, n_part, float(np.median(st[:, 3])) if n_part else None,
        reinit_ms, hbm)
    c3 = None
    if not args.no_c3_anchor and w.name != "C3":
        c3 = c3_anchor(sg, stream, flush, hbm)
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": w.dtype, "data": "synthetic",
        "config": run_config(w, n_pkg, n_part, args.order, world),
        "probes_per_s": n_part / (ms * 1e-3),
        "stages": stages,
        "step_ms_min_max": [float(step_ms.min()), float(step_ms.max())],
        "e2e": e2e,
        "gpu_launches": int(launches),
        "gpu_launches_per_step": launches / args.steps,
        "wall_s": t_wall,
        "roofline": {"kernel": "k_sweep<float, ReinitOp<float>> (reinit sweep)", "bound": "hbm", "achieved": achieved,
                     "peak": hbm, "peak_source": peak_src, "unit": "GB/s", "frac": achieved / hbm,
                     "bytes_per_cell": bytes_per_cell, "cells_per_launch": n_act,
                     "bytes_definition": "SURVEY 8(d): 2b + 108/64 per active point",
                     "achieved_face_bytes": achieved_face, "frac_face_bytes": achieved_face / hbm,
                     "bytes_per_cell_face": SWEEP_BYTES_FACE(esz),
                     "peak_nominal": 8000.0, "frac_nominal": achieved / 8000.0,
                     "traffic": ncu_traffic("k_sweep", w.name),
                     "note": (f"algorithmic bytes per sweep {alg_bytes / 1e6:.0f} MB; on C2 the "
                              "double-buffered working set is below the 126 MB L2 and ncu's DRAM "
                              "bytes per sweep (traffic) are about half of it, so this is not an "
                              "HBM number -- the HBM anchor is c3_anchor (profiles/README.md)")},
        "c3_anchor": c3,
        "clocks": clocks,
        "kernels": kernels,
        "gpu_name": torch.cuda.get_device_name(local),
    }
    if not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(w, n_act)
    print(json.dumps(out), flush=True)


def c3_anchor(sg, stream, flush, hbm, steps=5, warmup=2):
    """C3 (2048^3 effective, 103.9 M active points, 847 MB of DRAM per sweep
    in ncu): the configuration whose reinit sweep streams from HBM -- the
    roofline anchor beside the headline C2 line.  Build + 20 sweeps per step,
    CUDA events on the step's stream, median over the steps."""
    import torch
    w = W.config("C3")
    esz = 4
    ts = []
    for k in range(warmup + steps):
        flush.zero_()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        ev[0].record(stream)
        g = sg.Grid(w, stream=stream)
        ev[1].record(stream)
        g.reinit(REINIT_ITERS, w.cfl, stream=stream)
        ev[2].record(stream)
        torch.cuda.synchronize()
        n_act = (g.info["n_pkg"] - 2) * 64
        g.close_async(stream)
        if k >= warmup:
            ts.append((ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2])))
    ts = np.array(ts)
    sweep_ms = float(np.median(ts[:, 1])) / REINIT_ITERS
    a = SWEEP_BYTES_SURVEY(esz) * n_act / (sweep_ms * 1e-3) / 1e9
    af = SWEEP_BYTES_FACE(esz) * n_act / (sweep_ms * 1e-3) / 1e9
    tr = ncu_traffic("k_sweep", "C3")
    return {"workload": "C3: torus+box union 2048^3 effective (512^3 cells x 4^3), f32, "
                        "build + reinit 20", "active_cells": n_act, "steps": steps,
            "build_ms": float(np.median(ts[:, 0])), "sweep_us": sweep_ms * 1e3,
            "cells_per_s": n_act / (sweep_ms * 1e-3),
            "roofline": {"kernel": "k_sweep<float>", "bound": "hbm", "achieved": a, "peak": hbm,
                         "unit": "GB/s", "frac": a / hbm, "bytes_per_cell": SWEEP_BYTES_SURVEY(esz),
                         "achieved_face_bytes": af, "frac_face_bytes": af / hbm,
                         "frac_nominal": a / 8000.0, "traffic": tr,
                         "traffic_per_cell": tr / n_act if tr else None,
                         "dram_achieved": tr / (sweep_ms * 1e-3) / 1e9 if tr else None}}


# ------------------------------------------------------ oracle timing ------

def oracle_sample(w, budget_s: float = 12.0):
    """Time the oracle's reinit + gradient sweeps on the dense fp64 grid of
    the workload (tables and initial phi built beforehand, untimed)."""
    from oracle import oracle as O
    O.build()
    threads = len(os.sched_getaffinity(0))
    O.set_threads(threads)
    o = O.Oracle(w)
    t = o.build_tables()
    phi = o.phi_dense()
    n_act = (t.n_pkg - 2) * 64
    sweeps, t0 = 0, time.perf_counter()
    while True:
        phi = o.reinit_step(phi, w.cfl)
        sweeps += 1
        if time.perf_counter() - t0 > budget_s * 0.7 or sweeps >= REINIT_ITERS:
            break
    o.gradient(phi)
    dt = time.perf_counter() - t0
    cores = O.get_threads()
    # the same oracle on one thread ("also run with 1 thread"),
    # one reinit sweep
    O.set_threads(1)
    t1 = time.perf_counter()
    o.reinit_step(phi, w.cfl)
    dt1 = time.perf_counter() - t1
    O.set_threads(threads)
    return {"value": n_act * (sweeps + 1) / dt, "unit": UNIT, "cores": cores,
            "kind": "oracle",
            "sample": f"{sweeps} reinit sweeps + 1 gradient/normal sweep of the dense fp64 oracle "
                      f"on {w.name} ({n_act} active points each); tables and initial phi built "
                      f"beforehand (untimed); {dt:.1f} s",
            "single_thread": {"value": n_act / dt1, "unit": UNIT, "cores": 1,
                              "sample": f"1 reinit sweep on one thread, {dt1:.1f} s"}}


def oracle_window_sample(name="C3", planes=8, budget_s=8.0, xy_box=None):
    """The oracle on a z-window of a configuration whose dense grid does not
    fit (C3: 69 GB per fp64 field): `planes` background planes around the
    heaviest plane plus a margin of ceil(20/4) + 1 planes per side, the whole
    x-y extent; reinit sweeps timed, throughput per active
    point of the box (every one is updated by each sweep)."""
    from oracle import oracle as O
    O.build()
    threads = len(os.sched_getaffinity(0))
    O.set_threads(threads)
    w = W.config(name)
    full = O.Oracle(w)
    t = full.build_tables()
    zc = int(np.argmax(t.plane_count))
    margin = -(-REINIT_ITERS // 4) + 1
    z0 = max(0, zc - planes // 2 - margin)
    z1 = min(w.n[2], z0 + planes + 2 * margin)
    if xy_box is None:
        x0, y0, x1, y1 = 0, 0, w.n[0], w.n[1]
    else:
        # a box in x-y too (C5: a whole 4096^2 plane is 17 M fine points per
        # layer): xy_box = (nx, ny) cells around the densest row of the
        # heaviest plane
        bx, by = xy_box
        pl = t.bg.reshape(w.n[2], w.n[1], w.n[0])[zc] >= 2
        yc = int(np.argmax(pl.sum(axis=1)))
        xs = np.nonzero(pl[yc])[0]
        xc = int(np.median(xs)) if xs.size else w.n[0] // 2
        x0 = max(0, min(w.n[0] - bx, xc - bx // 2))
        y0 = max(0, min(w.n[1] - by, yc - by // 2))
        x1, y1 = x0 + bx, y0 + by
    o = O.Oracle(w, ((x0, y0, z0), (x1, y1, z1)))
    o.tables = t
    phi = o.phi_dense()
    bg3 = t.bg.reshape(w.n[2], w.n[1], w.n[0])[z0:z1, y0:y1, x0:x1]
    n_act = int(np.count_nonzero(bg3 >= 2)) * 64
    sweeps, t0 = 0, time.perf_counter()
    while True:
        phi = o.reinit_step(phi, w.cfl)
        sweeps += 1
        if time.perf_counter() - t0 > budget_s or sweeps >= REINIT_ITERS:
            break
    dt = time.perf_counter() - t0
    return {"config": name, "value": n_act * sweeps / dt, "unit": UNIT, "cores": O.get_threads(),
            "sample": f"{sweeps} reinit sweeps of the dense fp64 oracle on the window "
                      f"z [{z0}, {z1}) x [{x0}, {x1}) y [{y0}, {y1}) of {name} (heaviest plane "
                      f"{zc}, {planes} planes + {margin}-plane margins; {n_act} active points "
                      f"in the box); tables and initial phi untimed; {dt:.1f} s"}


def cpu_baseline(w, n_act):
    try:
        out = oracle_sample(w)
    except Exception as e:  # never fail the bench line on the baseline
        return {"value": None, "unit": UNIT, "cores": None, "kind": "oracle",
                "sample": f"failed: {e}"}
    out["windows"] = []
    for name, kw in (("C3", {}), ("C5", {"xy_box": (128, 48)})):
        try:
            out["windows"].append(oracle_window_sample(name, **kw))
        except Exception as e:
            out["windows"].append({"config": name, "value": None, "sample": f"failed: {e}"})
    return out


def run_reference(args, rank, world):
    if rank != 0:
        return
    w = W.config(args.config)
    from oracle import oracle as O
    O.build()
    threads = len(os.sched_getaffinity(0))
    O.set_threads(threads)
    o = O.Oracle(w)
    t = o.build_tables()
    phi0 = o.phi_dense()
    n_act = (t.n_pkg - 2) * 64
    sweeps = 2

    def step():
        phi = phi0
        for _ in range(sweeps):
            phi = o.reinit_step(phi, w.cfl)
        o.gradient(phi)

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = (time.perf_counter() - t0) / args.steps
    value = n_act * (sweeps + 1) / dt
    sample = (f"{sweeps} reinit sweeps + 1 gradient/normal sweep of the dense fp64 oracle on "
              f"{w.name} per step ({n_act} active points per sweep); tables/init untimed; the "
              f"GPU step also builds the grid, runs {REINIT_ITERS} sweeps and probes")
    n_part = 0
    if w.particles:  # the same particle set the GPU arm probes (count only)
        npdt = np.float32 if w.dtype == "f32" else np.float64
        n_part = int(W.lattice_particles(w, seed=0, order=args.order, dtype=npdt).shape[0])
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3,
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic",
           "config": run_config(w, t.n_pkg, n_part, args.order, world),
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": O.get_threads(),
                            "kind": "oracle", "sample": sample},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def main():
    args = parse()
    rank, world, local = rank_info()
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    run_ours(args, rank, world, local)


if __name__ == "__main__":
    main()
