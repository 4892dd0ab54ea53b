"""Small-shape cases for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): every shipped kernel family once — routing (pool, fp64 coarse,
saliency, ranks, sharpness, mask, plan, pick), the D = 128 K6 + K7T / K7
Taylor launches (forced both ways), the fused grid, D = 64 K6 + K7, dense K8,
pinned routing, the gamma residual, decoupled RoPE and the backward.

    compute-sanitizer --tool memcheck python tools/sanitize_cases.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_04569_b200 as P  # noqa: E402
from paper_2605_04569_b200 import _native as N  # noqa: E402


def qkv(H, S, D, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return tuple(torch.randn((1, H, S, D), generator=g, device="cuda").to(torch.bfloat16) for _ in range(3))


def backward_cases():
    """Backward kernels (dK/dV exact + centroid modes, dQ) on ragged, D = 64 and odd-block shapes."""
    q, k, v = qkv(2, 4096, 128, 1)
    P.isa_backward(q, k, v, P.IclLayout(2048, 2048), P.IsaConfig(), torch.randn_like(q))
    q2, k2, v2 = qkv(1, 1500, 128, 4)
    P.isa_backward(q2, k2, v2, P.IclLayout(900, 600), P.IsaConfig(strict=False, gamma=0.05), torch.randn_like(q2))
    q3, k3, v3 = qkv(2, 2048, 64, 5)
    P.isa_backward(q3, k3, v3, P.IclLayout(1024, 1024), P.IsaConfig(alpha_f=0.75), torch.randn_like(q3))
    q4, k4, v4 = qkv(1, 700, 64, 6)
    P.full_attention_backward(q4, k4, v4, None, torch.randn_like(q4))
    torch.cuda.synchronize()


def main():
    if "--backward" in sys.argv:
        backward_cases()
        print("sanitize backward cases done")
        return
    q, k, v = qkv(2, 4096, 128, 1)
    icl = P.IclLayout(2048, 2048)
    out, tr = P.isa_forward(q, k, v, icl, P.IsaConfig())
    for mode in ("k7", "k7t"):
        P.isa_forward(q, k, v, icl, P.IsaConfig(), taylor_kernel=mode)
    prep = P.prepare(q, k, v, icl, P.IsaConfig())
    prep.inp.knobs.flags |= N.FLAG_FUSED_GRID
    prep()
    r = P.isa_routing(q, k, v, icl, P.IsaConfig())
    P.isa_forward_with_routing(q, k, v, icl, P.IsaConfig(), r)
    P.isa_forward(q, k, v, icl, P.IsaConfig(gamma=0.5))
    q2, k2, v2 = qkv(1, 2100, 128, 2)
    P.isa_forward(q2, k2, v2, P.IclLayout(1000, 1100), P.IsaConfig(strict=False))
    q3, k3, v3 = qkv(2, 4096, 64, 3)
    P.isa_forward(q3, k3, v3, icl, P.IsaConfig())
    P.dense_attention(q, k, v)
    P.apply_decoupled_rope(q, icl)
    backward_cases()
    print("sanitize cases done")


if __name__ == "__main__":
    main()
