"""One decoupled-RoPE call at the cfg5 activation shape for ncu: (1,40,100000,128) bf16."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2605_04569_b200 as P

x = torch.randn(1, 100000, 40, 128, device="cuda").to(torch.bfloat16)
out = torch.empty_like(x)
icl = P.IclLayout(50000, 50000)
for _ in range(2):
    P.apply_decoupled_rope(x.permute(0, 2, 1, 3), icl, out=out.permute(0, 2, 1, 3))
torch.cuda.synchronize()
print("done")
