import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2605_04569_b200 as P
L = 32768
torch.manual_seed(0)
q, k, v = (torch.randn(1, 40, 2 * L, 128, device="cuda").to(torch.bfloat16) for _ in range(3))
icl, cfg = P.IclLayout(L, L), P.IsaConfig()
r = P.isa_routing(q, k, v, icl, cfg)
torch.cuda.synchronize()
print(os.environ.get("ISA_COARSE_N64", "0"), [x.cpu().numpy().sum() for x in (r.selection.indices, r.split.sharp, r.mask.indices)])
torch.save({"sel": r.selection.indices.cpu(), "sharp": r.split.sharp.cpu(), "mask": r.mask.indices.cpu(), "sh": r.split.sharpness.cpu()}, f"/tmp/route_{os.environ.get('ISA_COARSE_N64','0')}.pt")
