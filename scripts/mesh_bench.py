"""Build time of triangle-mesh geometries (NEXT-4): icospheres at the C2
resolution (128^3 cells x 4^3), fp32.  One JSON line per mesh.

python scripts/mesh_bench.py [levels ...]
"""
import json
import sys

import torch

sys.path.insert(0, ".")
import workloads as W  # noqa: E402
from paper_2512_11473_b200 import sg  # noqa: E402


def run(level, n=128, reps=5):
    w = W.mesh_workload(f"ico{level}", W.icosphere(level, rot=0.4), n, "f32")
    stream = torch.cuda.current_stream()
    ms = []
    for k in range(reps + 2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        g = sg.Grid(w, stream=stream)
        e1.record(stream)
        torch.cuda.synchronize()
        if k >= 2:
            ms.append(e0.elapsed_time(e1))
        info = g.info
        g.close()
    t = sorted(ms)[len(ms) // 2]
    return {"mesh": f"icosphere level {level}", "triangles": w.mesh.n_tris, "grid": f"{n}^3 cells",
            "active_points": (info["n_pkg"] - 2) * 64, "build_ms": t, "ms_all": ms,
            "note": "sg_build incl. mesh upload, pseudonormals (host), binning, tagging, sign "
                    "flood, compaction, neighbours, initial phi"}


def run_chain(level, n0=16, layers=3, reps=5):
    """Multi-resolution: build the n0^3 layer, then refine `layers` times
    (NEXT-4, sg_build_refined); timed over the whole chain."""
    w = W.mesh_workload(f"ico{level}", W.icosphere(level, rot=0.4), n0, "f32")
    stream = torch.cuda.current_stream()
    ms = []
    for k in range(reps + 2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        gs = [sg.Grid(w, stream=stream)]
        for _ in range(layers):
            gs.append(gs[-1].refined(stream=stream))
        e1.record(stream)
        torch.cuda.synchronize()
        if k >= 2:
            ms.append(e0.elapsed_time(e1))
        info = gs[-1].info
        for g in gs:
            g.close()
    t = sorted(ms)[len(ms) // 2]
    return {"mesh": f"icosphere level {level}", "triangles": w.mesh.n_tris,
            "chain": f"{n0}^3 -> {n0 * 2 ** layers}^3 ({layers + 1} layers)",
            "active_points_finest": (info["n_pkg"] - 2) * 64, "build_ms": t, "ms_all": ms}


if __name__ == "__main__":
    args = sys.argv[1:]
    if args and args[0] == "chain":
        for lv in [int(a) for a in args[1:]] or [5]:
            print(json.dumps(run_chain(lv)), flush=True)
    else:
        for lv in [int(a) for a in args] or [4, 5, 6]:
            print(json.dumps(run(lv)), flush=True)
