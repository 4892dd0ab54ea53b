"""Pinned host<->device copy bandwidth (the e2e floor): 2 GB H2D, 0.67 GB D2H, and both at once."""
import json
import torch

h = torch.empty(2013265920, dtype=torch.uint8).pin_memory()
d = torch.empty_like(h, device="cuda")
ho = torch.empty(671088640, dtype=torch.uint8).pin_memory()
do = torch.empty_like(ho, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def both():
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        ho.copy_(do, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


h2d = t(lambda: d.copy_(h, non_blocking=True))
d2h = t(lambda: ho.copy_(do, non_blocking=True))
print(json.dumps({"h2d_ms": h2d, "h2d_GBps": h.numel() / h2d / 1e6, "d2h_ms": d2h, "d2h_GBps": ho.numel() / d2h / 1e6,
                  "both_ms": t(both)}))
