"""Taylor-branch kernel choice (ISA_TAYLOR_PICK = auto / 7 / 7t) on iid and clustered cfg3 inputs:
time per isa_forward (prepared, 10 back-to-back calls) and the per-head picks."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2605_04569_b200 as P

L = 32768
kind = sys.argv[1] if len(sys.argv) > 1 else "iid"
torch.manual_seed(0)
if kind == "iid":
    q, k, v = (torch.randn(1, 40, 2 * L, 128, device="cuda").to(torch.bfloat16) for _ in range(3))
else:
    from paper_2605_04569_b200.workload import WorkloadSpec, generate
    qn, kn, vn, _ = generate(WorkloadSpec(kind="clustered", heads=40, seq_len=2 * L, dim=128))
    q, k, v = (torch.from_numpy(x).cuda().to(torch.bfloat16) for x in (qn, kn, vn))
prep = P.prepare(q, k, v, P.IclLayout(L, L), P.IsaConfig())
prep(); torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(10):
    prep()
b.record(); torch.cuda.synchronize()
print(json.dumps({"kind": kind, "pick_env": os.environ.get("ISA_TAYLOR_PICK", "auto"), "ms": a.elapsed_time(b) / 10}))
torch.save(prep.out[0, :4].cpu(), f"/tmp/pick_{kind}_{os.environ.get('ISA_TAYLOR_PICK', 'auto')}.pt")
