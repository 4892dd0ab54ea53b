"""Taylor-branch kernel choice at cfg3 (iid / clustered inputs): per-launch
CUDA-event times of the Taylor grid with every head forced to K7 (union tiles)
or K7T (transposed) and with the automatic per-head pick, alternated in one
loop (same clocks). python tools/ab_pick.py [iid|clustered] [steps]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_04569_b200 as P  # noqa: E402
from paper_2605_04569_b200 import _native as N  # noqa: E402

L = 32768
kind = sys.argv[1] if len(sys.argv) > 1 else "iid"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
if kind == "iid":
    import bench

    q, k, v = bench.synth_qkv(list(range(40)), 2 * L, 128, torch.device("cuda", 0))
else:
    from paper_2605_04569_b200.workload import WorkloadSpec, generate

    qn, kn, vn, _ = generate(WorkloadSpec(kind="clustered", heads=40, seq_len=2 * L, dim=128))
    q, k, v = (torch.from_numpy(x).cuda().to(torch.bfloat16) for x in (qn, kn, vn))
modes = {"auto": 0, "k7": N.FLAG_TAYLOR_K7, "k7t": N.FLAG_TAYLOR_K7T}
preps = {}
for m, f in modes.items():
    preps[m] = P.prepare(q, k, v, P.IclLayout(L, L), P.IsaConfig())
    preps[m].inp.knobs.flags |= f
res = {m: [] for m in modes}
for it in range(steps + 1):
    for m, pr in preps.items():
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
        es = N.IsaEvents()
        for i, e in enumerate(evs):
            e.record()
            es.ev[i] = e.cuda_event
        import ctypes

        from paper_2605_04569_b200.pipeline import _ptr

        inp = pr.inp
        N.check(N.load().isa_forward(ctypes.byref(inp.shape), ctypes.byref(inp.knobs), _ptr(inp.q), _ptr(inp.k),
                                     _ptr(inp.v), _ptr(pr.out), _ptr(pr.ws), pr.nbytes, None, None, _ptr(pr.err),
                                     ctypes.byref(es), torch.cuda.current_stream().cuda_stream))
        torch.cuda.synchronize()
        if it:
            res[m].append((evs[4].elapsed_time(evs[5]), evs[0].elapsed_time(evs[5])))
out = {m: {"taylor_ms": sum(x[0] for x in v_) / len(v_), "layer_ms": sum(x[1] for x in v_) / len(v_)}
       for m, v_ in res.items()}
d = (preps["k7"].out.float() - preps["k7t"].out.float()).abs().max().item()
print(json.dumps({"kind": kind, **out, "max_abs_k7_vs_k7t": d}))
