"""Pinned host <-> device copy bandwidth (one direction, and both at once on
two streams), the bound of bench.py's e2e number (C4: 233 MB up, 311 MB down)."""
import json
import torch

up = 233453232
dn = 311270976
h_up = torch.empty(up, dtype=torch.uint8).pin_memory()
h_dn = torch.empty(dn, dtype=torch.uint8).pin_memory()
d_up = torch.empty(up, dtype=torch.uint8, device="cuda")
d_dn = torch.empty(dn, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d_up.copy_(h_up, non_blocking=True)
    with torch.cuda.stream(s2):
        h_dn.copy_(d_dn, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


ta = t(lambda: d_up.copy_(h_up, non_blocking=True))
tb = t(lambda: h_dn.copy_(d_dn, non_blocking=True))
tc = t(both)
print(json.dumps({"h2d_ms": ta, "h2d_gbs": up / ta / 1e6, "d2h_ms": tb, "d2h_gbs": dn / tb / 1e6,
                  "both_ms": tc}))
