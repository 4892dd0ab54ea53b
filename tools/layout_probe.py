"""ISA layer time vs Q/K/V memory layout at the cfg5 shape (one B200):
contiguous (B,H,S,D) vs (B,S,H,D) views vs V inside a packed (B,S,3,H,D) QKV buffer."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2605_04569_b200 as P

L = int(sys.argv[1]) if len(sys.argv) > 1 else 50000
H, D, S = 40, 128, 2 * L
icl, cfg = P.IclLayout(L, L), P.IsaConfig(strict=(L % 64 == 0))
qkv = torch.randn(1, S, 3, H, D, device="cuda").to(torch.bfloat16)
bshd = [qkv[:, :, i].contiguous() for i in range(3)]
bhsd = [t.permute(0, 2, 1, 3).contiguous() for t in bshd]
out_bhsd = torch.empty(1, H, S, D, device="cuda", dtype=torch.bfloat16)
out_bshd = torch.empty(1, S, H, D, device="cuda", dtype=torch.bfloat16)

def t(fn, reps=3):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps

res = {
    "bhsd_in_bhsd_out": t(lambda: P.isa_forward(*bhsd, icl, cfg, collect_trace=False, validate=False, out=out_bhsd)),
    "bshd_in_bshd_out": t(lambda: P.isa_forward(*(x.permute(0, 2, 1, 3) for x in bshd), icl, cfg, collect_trace=False,
                                                validate=False, out=out_bshd.permute(0, 2, 1, 3))),
    "packed_qkv_in": t(lambda: P.isa_forward(*(qkv[:, :, i].permute(0, 2, 1, 3) for i in range(3)), icl, cfg,
                                             collect_trace=False, validate=False, out=out_bshd.permute(0, 2, 1, 3))),
}
print(json.dumps(res))
