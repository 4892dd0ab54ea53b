"""Block-layout utilities (reference tensor.py:25-36, 67-75, 122-190): same
results and error classes as the reference's definitions, for numpy and torch
inputs (pure data movement; CPU)."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from paper_2605_04569_b200.blocks import concat_seq, ensure_tensor4, gather_blocks, pad_to_blocks, scatter_blocks
from paper_2605_04569_b200.errors import BlockIndexError, ContractError, InputError, LayoutError
from paper_2605_04569_b200.types import BlockLayout


def test_pad_gather_scatter_roundtrip_numpy_and_torch():
    rng = np.random.default_rng(0)
    x = rng.standard_normal((2, 3, 70, 4)).astype(np.float32)
    lay = BlockLayout(16, 70)  # 5 blocks, last one 6 valid rows
    xp = pad_to_blocks(x, lay)
    assert xp.shape == (2, 3, 80, 4) and not xp[:, :, 70:].any() and np.array_equal(xp[:, :, :70], x)
    idx = np.array([0, 2, 4])
    g = gather_blocks(xp, lay, idx)
    want = np.concatenate([xp[:, :, 0:16], xp[:, :, 32:48], xp[:, :, 64:80]], axis=2)
    assert np.array_equal(g, want)
    back = scatter_blocks(np.zeros_like(xp), idx, g)
    assert np.array_equal(back[:, :, 0:16], xp[:, :, 0:16]) and not back[:, :, 16:32].any()
    # torch path: identical values
    tx = torch.from_numpy(x)
    tp = pad_to_blocks(tx, lay)
    assert torch.equal(tp, torch.from_numpy(xp))
    tg = gather_blocks(tp, lay, torch.from_numpy(idx))
    assert torch.equal(tg, torch.from_numpy(g))
    assert torch.equal(scatter_blocks(torch.zeros_like(tp), idx, tg), torch.from_numpy(back))
    assert np.array_equal(concat_seq(x[:, :, :30], x[:, :, 30:]), x)
    assert torch.equal(concat_seq(tx[:, :, :30], tx[:, :, 30:]), tx)
    # per-(B,H) index lists and the empty gather
    per = np.stack([np.stack([np.array([h, 4]) for h in range(3)]) for _ in range(2)])
    gp = gather_blocks(xp, lay, per)
    assert np.array_equal(gp[1, 2, :16], xp[1, 2, 32:48])
    assert gather_blocks(xp, lay, np.zeros((2, 3, 0), np.int64)).shape == (2, 3, 0, 4)


def test_errors_match_reference_classes():
    x = np.zeros((1, 1, 32, 2), np.float32)
    lay = BlockLayout(16, 32)
    with pytest.raises(LayoutError):
        pad_to_blocks(x, BlockLayout(16, 40))
    with pytest.raises(BlockIndexError):
        gather_blocks(x, lay, np.array([0, 2]))
    with pytest.raises(ContractError):
        gather_blocks(x, lay, np.array([1, 0]))
    with pytest.raises(LayoutError):
        gather_blocks(x[:, :, :20], lay, np.array([0]))
    with pytest.raises(LayoutError):
        scatter_blocks(x, np.array([0]), np.zeros((1, 1, 15, 2)))
    with pytest.raises(LayoutError):
        concat_seq(x, np.zeros((1, 2, 4, 2)))
    with pytest.raises(InputError):
        ensure_tensor4(np.full((1, 1, 1, 1), np.nan))
    with pytest.raises(LayoutError):
        ensure_tensor4(np.zeros((1, 1, 1)))
    assert ensure_tensor4(np.ones((1, 1, 1, 1), np.int32)).dtype == np.float64
    assert ensure_tensor4(torch.ones(1, 1, 1, 1, dtype=torch.int32)).dtype == torch.float64
