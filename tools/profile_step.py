"""One warm ISA layer call for ncu captures: python tools/profile_step.py [heads] [l_src] [l_ctx]"""
import sys
import torch
sys.path.insert(0, ".")
import paper_2605_04569_b200 as P

H = int(sys.argv[1]) if len(sys.argv) > 1 else 8
ls = int(sys.argv[2]) if len(sys.argv) > 2 else 32768
lc = int(sys.argv[3]) if len(sys.argv) > 3 else 32768
torch.manual_seed(0)
q, k, v = (torch.randn(1, H, ls + lc, 128, device="cuda").to(torch.bfloat16) for _ in range(3))
prep = P.prepare(q, k, v, P.IclLayout(ls, lc), P.IsaConfig(), separate_branches='--separate' in sys.argv)
for _ in range(2):
    prep()
torch.cuda.synchronize()
if "--dense" in sys.argv:
    P.dense_attention(q, k, v)
    torch.cuda.synchronize()
print("done")
