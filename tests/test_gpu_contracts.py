"""Pinned-routing index contracts (isa_forward_with_routing, isa_backward with
routing=): the reference raises on bad index lists (tensor.py:120-133
BlockIndexError / ContractError via gather_blocks; taylor.py:80-84
ContractError for the Taylor mask). The device check reports them through the
error word; the clamped index narrowing keeps every kernel in bounds on the way."""

from __future__ import annotations

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _setup():
    import paper_2605_04569_b200 as P

    g = torch.Generator(device="cuda").manual_seed(7)
    q, k, v = (torch.randn((1, 2, 4096, 128), generator=g, device="cuda").to(torch.bfloat16) for _ in range(3))
    icl, cfg = P.IclLayout(2048, 2048), P.IsaConfig()
    r = P.isa_routing(q, k, v, icl, cfg)
    return P, (q, k, v, icl, cfg), r


def _numpy_routing(r):
    from paper_2605_04569_b200.types import BlockMask, IsaRouting, SelectionIndex, SharpnessSplit

    sel = r.selection.numpy().copy()
    sharp, flat = r.split.sharp.cpu().numpy().copy(), r.split.flat.cpu().numpy().copy()
    mask = r.mask.numpy().copy()
    return sel, sharp, flat, mask, lambda s, a, b, m: IsaRouting(
        SelectionIndex(s, r.selection.num_context_blocks), SharpnessSplit(a, b, r.split.sharpness.cpu().numpy()),
        BlockMask(m, r.mask.num_key_blocks))


def test_valid_pinned_routing_passes():
    P, args, r = _setup()
    out = P.isa_forward_with_routing(*args, r)
    ref, _ = P.isa_forward(*args)
    assert torch.equal(out, ref)


@pytest.mark.parametrize("what,exc", [
    ("sel_range", "BlockIndexError"),
    ("sel_negative", "BlockIndexError"),
    ("sel_order", "ContractError"),
    ("split_range", "BlockIndexError"),
    ("split_overlap", "ContractError"),
    ("mask_range", "ContractError"),
    ("mask_order", "ContractError"),
])
def test_bad_pinned_routing_raises(what, exc):
    from paper_2605_04569_b200 import errors

    P, args, r = _setup()
    sel, sharp, flat, mask, make = _numpy_routing(r)
    if what == "sel_range":
        sel[0, 1, -1] = 10_000
    elif what == "sel_negative":
        sel[0, 0, 0] = -3
    elif what == "sel_order":
        sel[0, 0, [0, 1]] = sel[0, 0, [1, 0]]
    elif what == "split_range":
        flat[0, 0, -1] = 64  # T = 64 query blocks
    elif what == "split_overlap":
        flat[0, 1, 0] = sharp[0, 1, 0]
        flat[0, 1] = np.sort(flat[0, 1])
    elif what == "mask_range":
        mask[0, 0, 3, -1] = 1 << 20
    elif what == "mask_order":
        mask[0, 1, 2, 0] = mask[0, 1, 2, -1]
    with pytest.raises(getattr(errors, exc)):
        P.isa_forward_with_routing(*args, make(sel, sharp, flat, mask))
    # the device is still healthy: a valid call afterwards works
    out = P.isa_forward_with_routing(*args, r)
    assert torch.isfinite(out.float()).all()


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two GPUs in one process")
def test_two_devices_one_process():
    """The dynamic shared-memory opt-in is per device context (ensure_smem):
    a call on cuda:1 after one on cuda:0 must launch."""
    import paper_2605_04569_b200 as P

    outs = []
    for dev in (0, 1):
        g = torch.Generator(device=f"cuda:{dev}").manual_seed(3)
        q, k, v = (torch.randn((1, 1, 2048, 128), generator=g, device=f"cuda:{dev}").to(torch.bfloat16)
                   for _ in range(3))
        with torch.cuda.device(dev):
            out, _ = P.isa_forward(q, k, v, P.IclLayout(1024, 1024), P.IsaConfig())
        outs.append(out.cpu())
    assert torch.equal(outs[0], outs[1])
