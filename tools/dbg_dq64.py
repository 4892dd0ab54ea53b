import torch, numpy as np, sys
sys.path.insert(0, '.')
import paper_2605_04569_b200 as P
for (S, D) in ((700, 64), (700, 128), (768, 64), (1024, 64), (704, 64)):
    g = torch.Generator(device='cuda').manual_seed(0)
    q, k, v, do = (torch.randn(1, 2, S, D, device='cuda', generator=g).to(torch.bfloat16) for _ in range(4))
    gr = P.full_attention_backward(q, k, v, None, do)
    dq = gr.dq.float()
    bad = ~torch.isfinite(dq)
    print(S, D, "nan dq:", int(bad.sum()), "rows:", torch.nonzero(bad.any(-1))[:, 2].unique().tolist()[:20],
          "cols:", torch.nonzero(bad.any(2))[:, 2].unique().tolist()[:70], "dk nan", int((~torch.isfinite(gr.dk.float())).sum()))
