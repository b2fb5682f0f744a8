"""Host-buffer probe (C4 particles on C2) timing for one setting of the
staging overrides (SG_PROBE_CHUNK / SG_PROBE_RING / SG_PROBE_DOWN1 in env);
also the full e2e step (build + reinit 20 + gradient + host probe)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2512_11473_b200 import sg  # noqa: E402

w = W.config("C2")
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
g = sg.Grid(w, stream=st)
g.reinit(20, stream=st).gradient(sg.SG_GRAD | sg.SG_NORMAL | sg.SG_KINT, stream=st)
pos = W.particles(w, device="cuda")
n = pos.shape[0]
hp = pos.cpu().pin_memory()
hphi = torch.empty(n).pin_memory()
hgrad = torch.empty((n, 3)).pin_memory()
ts = []
for rep in range(6):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sg.sg_probe(g.handle, n, hp.data_ptr(), hphi.data_ptr(), hgrad.data_ptr(), None, st)
    torch.cuda.synchronize()
    ts.append((time.perf_counter() - t0) * 1e3)
steps = []
for rep in range(5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    g2 = sg.Grid(w, stream=st)
    g2.reinit(20, stream=st).gradient(sg.SG_GRAD | sg.SG_NORMAL | sg.SG_KINT, stream=st)
    sg.sg_probe(g2.handle, n, hp.data_ptr(), hphi.data_ptr(), hgrad.data_ptr(), None, st)
    torch.cuda.synchronize()
    steps.append((time.perf_counter() - t0) * 1e3)
    del g2
env = {k: os.environ.get(k) for k in ("SG_PROBE_CHUNK", "SG_PROBE_RING", "SG_PROBE_DOWN1")}
print(json.dumps({"env": env, "probe_host_ms": float(np.median(ts[1:])), "step_ms": float(np.median(steps[1:]))}))
