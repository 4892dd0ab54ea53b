import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2605_04569_b200 as P
torch.manual_seed(0)
L = 32768
q, k, v = (torch.randn(1, 40, 2 * L, 128, device="cuda").to(torch.bfloat16) for _ in range(3))
icl, cfg = P.IclLayout(L, L), P.IsaConfig()
res = {}
for sep in (0, 1, 0, 1):
    prep = P.prepare(q, k, v, icl, cfg, separate_branches=bool(sep))
    prep(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        prep()
    b.record(); torch.cuda.synchronize()
    res.setdefault("sep" if sep else "fused", []).append(round(a.elapsed_time(b) / 10, 3))
    if sep == 0:
        o0 = prep.out.clone()
    else:
        print("max diff fused vs separate", (prep.out.float() - o0.float()).abs().max().item())
print(res)
