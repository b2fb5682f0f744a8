"""C5 reinit sweep in isolation: reinit(20) repeated on one built grid, with
NVML SM clocks sampled around it (is the step's sweep rate set by the power
cap or by the sweep itself?)."""
import json
import sys
import threading
import time

import torch

sys.path.insert(0, ".")
import workloads as W  # noqa: E402
from paper_2512_11473_b200 import sg  # noqa: E402

import pynvml as nv  # noqa: E402

nv.nvmlInit()
h = nv.nvmlDeviceGetHandleByIndex(0)
clk, stop = [], threading.Event()


def samp():
    while not stop.is_set():
        clk.append(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
        time.sleep(0.005)


name = sys.argv[1] if len(sys.argv) > 1 else "C5"
w = W.config(name)
g = sg.Grid(w)
g.reinit(20)
torch.cuda.synchronize()
t = threading.Thread(target=samp, daemon=True)
t.start()
res = []
for rep in range(8):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.reinit(20)
    b.record()
    torch.cuda.synchronize()
    res.append(a.elapsed_time(b) / 20 * 1e3)
stop.set()
t.join()
clk.sort()
print(json.dumps({"config": name, "sweep_us": res, "sm_mhz_median": clk[len(clk) // 2] if clk else None,
                  "sm_mhz_min": clk[0] if clk else None, "n_pkg": g.info["n_pkg"]}))
