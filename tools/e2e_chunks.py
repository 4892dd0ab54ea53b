"""e2e (pinned host in/out through isa_forward) vs heads_per_chunk at cfg3."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2605_04569_b200 as P
H, L = 40, 32768
g = torch.Generator(device="cuda").manual_seed(0)
q, k, v = (torch.randn(1, H, 2 * L, 128, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
qh, kh, vh = (t.cpu().pin_memory() for t in (q, k, v))
outh = torch.empty(q.shape, dtype=q.dtype, pin_memory=True)
icl, cfg = P.IclLayout(L, L), P.IsaConfig()
res = {}
for hpc in (0, 1, 2, 3, 4, 5, 8, 10):
    f = lambda: P.isa_forward(qh, kh, vh, icl, cfg, collect_trace=False, out=outh, heads_per_chunk=hpc)
    f(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(3):
        f()
    b.record(); torch.cuda.synchronize()
    res[hpc] = round(a.elapsed_time(b) / 3, 2)
print(json.dumps(res))
