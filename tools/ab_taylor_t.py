import os, sys, torch, numpy as np
sys.path.insert(0, os.getcwd())
import paper_2605_04569_b200 as P
from paper_2605_04569_b200 import _native as N
if os.environ.get("ISA_LIB"):  # A/B a variant build of the library
    N.load(os.environ["ISA_LIB"])
torch.manual_seed(0)
L = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
q, k, v = (torch.randn(1, 40, 2 * L, 128, device="cuda").to(torch.bfloat16) for _ in range(3))
icl, cfg = P.IclLayout(L, L), P.IsaConfig()
out, _ = P.isa_forward(q, k, v, icl, cfg, collect_trace=False)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(5):
    P.isa_forward(q, k, v, icl, cfg, collect_trace=False, out=out)
b.record(); torch.cuda.synchronize()
print(os.environ.get("ISA_LIB", ""), os.environ.get("ISA_TAYLOR_T", "default"), "ms", a.elapsed_time(b) / 5)
tag = os.path.basename(os.environ.get("ISA_LIB", "")) or os.environ.get("ISA_TAYLOR_T", "d")
torch.save(out[0, :4].cpu(), f"/tmp/out_{tag}.pt")
