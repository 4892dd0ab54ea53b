"""Taylor (K7) efficiency vs input structure at cfg3 (H=40, 32K+32K, D=128):
i.i.d. N(0,1) (bench inputs) vs the reference's `clustered` workload model
(workload.py:85-97: clusters of 256 tokens, queries aimed at a random
cluster's key centre), generated on the GPU with torch (same distribution,
not the reference's Philox stream). Separate-branch launches, CUDA events.
Also reports the mean union length per Q-tile pair (the K7 exact stream)."""
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2605_04569_b200 as P
from paper_2605_04569_b200 import _native as N


def clustered(H, S, D, g, cluster_noise=0.25):
    n = max(1, S // 256)
    run = -(-S // n)
    member = torch.clamp(torch.arange(S, device="cuda") // run, max=n - 1)
    kc = torch.randn(H, n, D, device="cuda", generator=g)
    vc = torch.randn(H, n, D, device="cuda", generator=g)
    k = kc[:, member] + cluster_noise * torch.randn(H, S, D, device="cuda", generator=g)
    v = vc[:, member] + cluster_noise * torch.randn(H, S, D, device="cuda", generator=g)
    target = torch.randint(0, n, (H, n), device="cuda", generator=g)
    tau = torch.rand(H, n, device="cuda", generator=g) * 2.25 + 0.25
    tgt = torch.gather(target, 1, member[None].expand(H, S))
    q = tau[:, member, None] * torch.gather(kc, 1, tgt[..., None].expand(H, S, D)) + 0.5 * torch.randn(
        H, S, D, device="cuda", generator=g)
    return [x[None].to(torch.bfloat16) for x in (q, k, v)]


def run(q, k, v, icl, cfg):
    from bench import _call_with_events  # noqa: E402

    prep = P.prepare(q, k, v, icl, cfg, separate_branches=True)
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
    st = N.IsaEvents()
    for i, e in enumerate(evs):
        e.record()
        st.ev[i] = e.cuda_event
    for _ in range(2):
        _call_with_events(prep, st, 1)
    torch.cuda.synchronize()
    ex = ta = 0.0
    for _ in range(3):
        _call_with_events(prep, st, 1)
        torch.cuda.synchronize()
        ex += evs[3].elapsed_time(evs[4]) / 3
        ta += evs[4].elapsed_time(evs[5]) / 3
    _, tr = P.isa_forward(q, k, v, icl, cfg)
    mask = tr.mask.indices[0]  # (H, n_flat, k)
    Hh, nf, kk = mask.shape
    pairs = mask[:, : nf // 2 * 2].reshape(Hh, nf // 2, 2 * kk)
    union = torch.stack([torch.unique(pairs[h, i]).numel() * torch.ones(()) for h in range(min(Hh, 4))
                         for i in range(pairs.shape[1])]).mean().item()
    return ex, ta, union, kk


def main():
    H, L, D = 40, 32768, 128
    icl, cfg = P.IclLayout(L, L), P.IsaConfig()
    d = P.IsaDims.derive((1, H, 2 * L, D), icl, cfg)
    f_taylor = (4 * 64 * 64 * D * d.n_flat * d.k + 4 * 64 * D * d.n_flat * (d.t_new - d.k)) * H
    g = torch.Generator(device="cuda").manual_seed(0)
    out = {}
    for kind in ("iid", "clustered"):
        if kind == "iid":
            q, k, v = (torch.randn(1, H, 2 * L, D, device="cuda", generator=g).to(torch.bfloat16) for _ in range(3))
        else:
            q, k, v = clustered(H, 2 * L, D, g)
        ex, ta, union, kk = run(q, k, v, icl, cfg)
        out[kind] = {"exact_ms": ex, "taylor_ms": ta, "taylor_alg_tflops": f_taylor / ta / 1e9,
                     "mean_union_blocks_per_pair": union, "exact_blocks_per_block": kk,
                     "union_efficiency": 2 * kk / union}
        del q, k, v
        torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
