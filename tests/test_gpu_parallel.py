"""The multi-GPU overlap machinery on one GPU (world = 1): per-head completion
counters published from inside the fused attention grid (isa_forward_signal),
stream waits on them (cuStreamWaitValue32), and both ShardedIsa schedules
("signal", "chunks") reproducing the plain forward bit for bit. The NCCL
collective itself needs >= 2 GPUs (bench.py --gpus N); its placement logic is
covered by tests/test_parallel_gloo.py."""

from __future__ import annotations

import pytest
import torch

pytestmark = pytest.mark.gpu


def _inputs(H=6, S=16384, seed=11):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return tuple(torch.randn((1, H, S, 128), generator=g, device="cuda").to(torch.bfloat16) for _ in range(3))


def test_head_done_counters_grow_per_call():
    import paper_2605_04569_b200 as P

    q, k, v = _inputs()
    prep = P.prepare(q, k, v, P.IclLayout(8192, 8192), P.IsaConfig(), signal=True)
    plain = P.prepare(q, k, v, P.IclLayout(8192, 8192), P.IsaConfig())
    for _ in range(3):
        out = prep()
    torch.cuda.synchronize()
    inc = prep.done_inc.value
    assert inc > 1  # the fused grid counts its CTAs per head
    assert torch.equal(prep.head_done.cpu(), torch.full((6,), 3 * inc, dtype=torch.int32))
    assert torch.equal(out, plain())


@pytest.mark.parametrize("mode,chunk", [("signal", 1), ("chunks", 1), ("chunks", 4)])
def test_sharded_schedule_world1_matches_plain(mode, chunk):
    """Comm-stream copies of each head (gated by the completion counters in
    "signal" mode, by chunk events in "chunks" mode) land the same bits as the
    plain forward; out_full starts as NaN, so a copy that raced ahead of its
    head's compute would show."""
    import paper_2605_04569_b200 as P
    from paper_2605_04569_b200.parallel import ShardedIsa

    q, k, v = _inputs()
    icl, cfg = P.IclLayout(8192, 8192), P.IsaConfig()
    ref = P.prepare(q, k, v, icl, cfg)().clone()
    layer = ShardedIsa(q, k, v, icl, cfg, 1, chunk_heads=chunk, mode=mode)
    for _ in range(3):
        out_full = torch.full_like(q, float("nan"))
        layer(out_full)
        torch.cuda.synchronize()
        assert torch.equal(out_full, ref)


def test_cta_pair_k6_matches_single_cta():
    """K6 / K8 on CTA pairs (cta_group::2, the default at D = 128) against the
    single-CTA kernel (ISA_FLAG_SINGLE_CTA): same routing, same outputs to the
    last bf16 bit or within one bf16 ulp (the pair MMA accumulates each output
    over the same k order; only the issue differs), odd item counts included
    (a padding CTA completes the last pair)."""
    import ctypes

    import paper_2605_04569_b200 as P
    from paper_2605_04569_b200 import _native as N
    from paper_2605_04569_b200.pipeline import _ptr

    for S, ls in ((8192, 4096), (4096 + 512, 4096)):  # T = 128 (16 K6 items) / 72 (n_sharp 36: 9 items, odd)
        q, k, v = _inputs(3, S, seed=S)
        icl, cfg = P.IclLayout(ls, S - ls), P.IsaConfig(strict=(S - ls) % 64 == 0)
        outs = []
        for flags in (0, N.FLAG_SINGLE_CTA):
            prep = P.prepare(q, k, v, icl, cfg)
            inp = prep.inp
            kn = N.IsaKnobs(inp.knobs.scale, inp.knobs.k_ctx, inp.knobs.n_flat, inp.knobs.k_mask,
                            inp.knobs.softmax_first, flags, inp.knobs.gamma, inp.knobs.residual_softmax)
            N.check(N.load().isa_forward(ctypes.byref(inp.shape), ctypes.byref(kn), _ptr(inp.q), _ptr(inp.k),
                                         _ptr(inp.v), _ptr(prep.out), _ptr(prep.ws), prep.nbytes, None, None,
                                         _ptr(prep.err), None, torch.cuda.current_stream().cuda_stream))
            outs.append(prep.out.float().clone())
        d = (outs[0] - outs[1]).abs().max().item()
        assert d <= 8e-3, d
    dq, dk, dv = _inputs(2, 4096, seed=9)
    assert torch.isfinite(P.dense_attention(dq, dk, dv).float()).all()
