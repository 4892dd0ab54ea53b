"""Kernel timeline of one prepared isa_forward at cfg3 (bench inputs) under the torch
profiler: start / end of every kernel longer than argv[1] us (default 100)."""
import sys, torch
sys.path.insert(0, ".")
import bench
import paper_2605_04569_b200 as P
from torch.profiler import ProfilerActivity, profile
q, k, v = bench.synth_qkv(list(range(40)), 65536, 128, "cuda")
prep = P.prepare(q, k, v, P.IclLayout(32768, 32768), P.IsaConfig())
for _ in range(3):
    prep()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as pr:
    prep()
    torch.cuda.synchronize()
ev = sorted((e for e in pr.events() if e.device_type.name == "CUDA"), key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
for e in ev:
    if (e.time_range.end - e.time_range.start) > float(sys.argv[1] if len(sys.argv) > 1 else 100):
        print(f"{(e.time_range.start - t0)/1e3:8.3f} -> {(e.time_range.end - t0)/1e3:8.3f} ms  {e.name[:60]}")
