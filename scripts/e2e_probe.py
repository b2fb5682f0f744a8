import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, time, json, workloads as W
from paper_2512_11473_b200 import sg
w = W.config("C2"); st = torch.cuda.Stream(); torch.cuda.set_stream(st)
g = sg.Grid(w, stream=st); g.reinit(20, stream=st).gradient(sg.SG_GRAD|sg.SG_NORMAL|sg.SG_KINT, stream=st)
pos = W.particles(w, device="cuda"); n = pos.shape[0]
hp = pos.cpu().pin_memory(); hphi = torch.empty(n).pin_memory(); hgrad = torch.empty((n,3)).pin_memory()
res = {}
for rep in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(st)
    sg.sg_probe(g.handle, n, hp.data_ptr(), hphi.data_ptr(), hgrad.data_ptr(), None, st)
    b.record(st); torch.cuda.synchronize()
    res[f"probe_host_only_{rep}"] = (a.elapsed_time(b), (time.perf_counter()-t0)*1e3)
print(json.dumps(res))
