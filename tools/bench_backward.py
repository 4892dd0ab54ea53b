"""isa_backward at cfg3 (H=40, 32K+32K, D=128, bf16) on one B200: total time
(forward recompute + gradients) and the backward-only part, CUDA events.
FLOP convention: backward = 2.5 x the forward's algorithmic FLOPs (FA
convention: 5 GEMMs vs 2; our two-kernel scheme recomputes S and dP once more,
so it executes 7/2 x); reported as algorithmic TFLOP/s."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2605_04569_b200 as P

args = [a for a in sys.argv[1:] if not a.startswith("--")]
H = int(args[0]) if len(args) > 0 else 40
L = int(args[1]) if len(args) > 1 else 32768
q, k, v, do = (torch.randn(1, H, 2 * L, 128, device="cuda").to(torch.bfloat16) for _ in range(4))
icl, cfg = P.IclLayout(L, L), P.IsaConfig()
P.isa_backward(q, k, v, icl, cfg, do)
prep = P.prepare(q, k, v, icl, cfg)
prep()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(2):
    P.isa_backward(q, k, v, icl, cfg, do)
b.record()
torch.cuda.synchronize()
bwd = a.elapsed_time(b) / 2
a.record()
for _ in range(2):
    prep()
b.record()
torch.cuda.synchronize()
fwd = a.elapsed_time(b) / 2
f = P.IsaDims.derive(q.shape, icl, cfg).flops()
fl = 2.5 * (f.exact_mas + f.taylor_mas)
print(json.dumps({"workload": f"isa_backward H={H} {L}+{L} D=128 bf16", "backward_total_ms": bwd, "forward_ms": fwd,
                  "gradient_kernels_ms": bwd - fwd, "alg_tflops_gradients": fl / (bwd - fwd) / 1e9}))
if "--kernels" in sys.argv:  # per-kernel device times of one backward (CUPTI via torch.profiler)
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as pr:
        P.isa_backward(q, k, v, icl, cfg, do)
        torch.cuda.synchronize()
    rows = {}
    for e in pr.events():
        if e.device_type.name == "CUDA":
            r = rows.setdefault(e.name[:60], [0, 0.0])
            r[0] += 1
            r[1] += e.device_time_total / 1e3 if hasattr(e, "device_time_total") else e.cuda_time_total / 1e3
    for name, (n, ms) in sorted(rows.items(), key=lambda x: -x[1][1])[:14]:
        print(f"{ms:9.3f} ms  x{n:<3d} {name}")
if "--gaps" in sys.argv:  # idle device time between consecutive kernels of one backward (3 calls)
    from torch.profiler import ProfilerActivity, profile
    for rep in range(3):
        with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as pr:
            P.isa_backward(q, k, v, icl, cfg, do)
            torch.cuda.synchronize()
        ev = sorted((e for e in pr.events() if e.device_type.name == "CUDA"), key=lambda e: e.time_range.start)
        print(f"call {rep}: span {(ev[-1].time_range.end - ev[0].time_range.start) / 1e3:.3f} ms")
    prev = None
    for e in ev:
        if prev is not None and e.time_range.start - prev.time_range.end > 50:
            print(f"gap {(e.time_range.start - prev.time_range.end) / 1e3:8.3f} ms  after {prev.name[:50]}  before {e.name[:50]}")
        prev = e
    print(f"span {(ev[-1].time_range.end - ev[0].time_range.start) / 1e3:.3f} ms, busy "
          f"{sum(e.time_range.end - e.time_range.start for e in ev) / 1e3:.3f} ms")
if "--host" in sys.argv:  # host-side cost of one call: wall clock vs CUDA events, synchronized on both sides
    import time
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        a.record()
        P.isa_backward(q, k, v, icl, cfg, do)
        b.record()
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        print(f"call wall {1e3 * (t1 - t0):.2f} ms, events {a.elapsed_time(b):.2f} ms")
    import cProfile, pstats
    pr = cProfile.Profile()
    pr.enable()
    P.isa_backward(q, k, v, icl, cfg, do)
    torch.cuda.synchronize()
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(12)
