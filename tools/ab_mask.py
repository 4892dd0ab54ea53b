"""Routing run (cfg3, seeded) with an optional variant library (ISA_LIB): saves the block mask for comparison."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_04569_b200 import _native as N
if os.environ.get("ISA_LIB"):
    N.load(os.environ["ISA_LIB"])
import paper_2605_04569_b200 as P
torch.manual_seed(0)
L = 32768
q, k, v = (torch.randn(1, 40, 2 * L, 128, device="cuda").to(torch.bfloat16) for _ in range(3))
r = P.isa_routing(q, k, v, P.IclLayout(L, L), P.IsaConfig())
torch.cuda.synchronize()
torch.save(r.mask.indices.cpu(), "/tmp/mk_" + os.path.basename(os.environ.get("ISA_LIB", "d")) + ".pt")
