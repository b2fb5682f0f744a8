"""Host-side timing of repeated sg_build calls (diagnoses build stalls).

python scripts/diag_build.py [CONFIG] [N]
"""
import sys
import time

import torch

sys.path.insert(0, ".")
import workloads  # noqa: E402
from paper_2512_11473_b200 import sg  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 12
w = workloads.CONFIGS[cfg]
stream = torch.cuda.current_stream()


def pool_stats():
    try:
        from cuda.bindings import runtime as rt
    except ImportError:
        from cuda import cudart as rt
    _, pool = rt.cudaDeviceGetDefaultMemPool(0)
    out = {}
    for name in ("cudaMemPoolAttrReservedMemCurrent", "cudaMemPoolAttrUsedMemCurrent",
                 "cudaMemPoolAttrReleaseThreshold"):
        _, v = rt.cudaMemPoolGetAttribute(pool, getattr(rt.cudaMemPoolAttr, name))
        out[name[16:]] = int(v) >> 20
    return out


flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for i in range(n):
    flush.zero_()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(stream)
    g = sg.Grid(w, stream=stream)
    t1 = time.perf_counter()
    e1.record(stream)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    g.close_async(stream)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"{i:2d} host build {1e3 * (t1 - t0):8.2f} ms  to sync {1e3 * (t2 - t0):8.2f} ms  "
          f"events {e0.elapsed_time(e1):8.2f} ms  close {1e3 * (t3 - t2):7.2f} ms  pool(MiB) "
          f"{pool_stats()}", flush=True)
