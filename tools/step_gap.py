"""Where does a bench step go? Per-step CUDA events around stages vs the
back-to-back loop time (cfg3 by default)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2605_04569_b200 as P
from paper_2605_04569_b200 import _native as N
from bench import _call_with_events

H, L = 40, 32768
q, k, v = (torch.randn(1, H, 2 * L, 128, device="cuda").to(torch.bfloat16) for _ in range(3))
prep = P.prepare(q, k, v, P.IclLayout(L, L), P.IsaConfig())
for _ in range(3):
    prep()
torch.cuda.synchronize()
n = 10
evs = [[torch.cuda.Event(enable_timing=True) for _ in range(6)] for _ in range(n)]
structs = []
for i in range(n):
    s = N.IsaEvents()
    for j, e in enumerate(evs[i]):
        e.record()
        s.ev[j] = e.cuda_event
    structs.append(s)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for i in range(n):
    _call_with_events(prep, structs[i], 0)
b.record()
torch.cuda.synchronize()
tot = a.elapsed_time(b) / n
inner = sum(evs[i][0].elapsed_time(evs[i][5]) for i in range(n)) / n
gaps = [evs[i][5].elapsed_time(evs[i + 1][0]) for i in range(n - 1)]
a.record()
for i in range(n):
    prep()
b.record()
torch.cuda.synchronize()
names = ("coarse", "select", "split", "exact", "taylor")
in_loop = {nm: sum(evs[i][j].elapsed_time(evs[i][j + 1]) for i in range(1, n)) / (n - 1) for j, nm in enumerate(names)}
iso = {nm: 0.0 for nm in names}
for r in range(3):  # isolated calls (synchronize before each)
    torch.cuda.synchronize()
    _call_with_events(prep, structs[0], 0)
    torch.cuda.synchronize()
    for j, nm in enumerate(names):
        iso[nm] += evs[0][j].elapsed_time(evs[0][j + 1]) / 3
print(json.dumps({"loop_ms_per_step_with_events": tot, "ev0_to_ev5_ms": inner, "gap_between_steps_ms": gaps,
                  "loop_ms_per_step_plain": a.elapsed_time(b) / n, "stages_in_loop": in_loop,
                  "stages_isolated": iso}))
