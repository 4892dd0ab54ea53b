"""Standalone Taylor kernel (`taylor_sparse_forward`, reference taylor.py:45-194,
299-316) against the reference's own outputs (`tests/golden/taylor`, made by
`tests/golden/make_taylor_golden.py`) and the CPU oracle.

CPU: validation errors (same classes as taylor.py:60-103), FLOP tallies,
fixture inputs. GPU: outputs vs golden / oracle (max-abs 2e-2, cosine 0.999),
torch and strided inputs, the kc contract check, unsupported partial blocks.
"""

from __future__ import annotations

import os

import numpy as np
import pytest

from oracle import isa_oracle as O
from paper_2605_04569_b200.errors import ConfigError, ContractError, LayoutError
from paper_2605_04569_b200.taylor import TaylorKernelInput, flop_count, taylor_sparse_forward
from paper_2605_04569_b200.types import BlockMask

GOLD = os.path.join(os.path.dirname(__file__), "golden", "taylor")
CASES = sorted(f[:-4] for f in os.listdir(GOLD) if f.endswith(".npz"))


def make_inputs(B, H, t_q, t_k, D, k, seed):
    """Same draws as make_taylor_golden.make_inputs (pinned by the stored checksum)."""
    rng = np.random.default_rng(seed)
    b = 64
    q = O.round_bf16(rng.standard_normal((B, H, t_q * b, D)).astype(np.float32))
    kk = O.round_bf16(rng.standard_normal((B, H, t_k * b, D)).astype(np.float32))
    v = O.round_bf16(rng.standard_normal((B, H, t_k * b, D)).astype(np.float32))
    kc = kk.reshape(B, H, t_k, b, D).astype(np.float64).mean(axis=3).astype(np.float32)
    vc = v.reshape(B, H, t_k, b, D).astype(np.float64).mean(axis=3).astype(np.float32)
    idx = np.sort(np.stack([rng.permutation(t_k)[:k] for _ in range(B * H * t_q)]), axis=1)
    return q, kk, v, kc, vc, idx.reshape(B, H, t_q, k).astype(np.int64)


def _case(name):
    g = np.load(os.path.join(GOLD, f"{name}.npz"))
    B, H, t_q, t_k, D, k, seed = (int(x) for x in g["geom"])
    q, kk, v, kc, vc, idx = make_inputs(B, H, t_q, t_k, D, k, seed)
    assert np.isclose(q.sum() + kk.sum() + v.sum(), g["checksum"])
    np.testing.assert_array_equal(idx, g["mask"])
    inp = TaylorKernelInput(q=q, k_new=kk, v_new=v, kc=kc, vc=vc, mask=BlockMask(idx, t_k),
                            scale=float(g["scale"]), block_size=64)
    return inp, g


def _close(out, ref, max_abs=2e-2, min_cos=0.999):
    a = np.asarray(out, dtype=np.float64).ravel()
    r = np.asarray(ref, dtype=np.float64).ravel()
    err = float(np.max(np.abs(a - r)))
    cos = float(a @ r / (np.linalg.norm(a) * np.linalg.norm(r)))
    assert err <= max_abs and cos >= min_cos, f"max_abs={err:.3e} cos={cos:.6f}"


@pytest.mark.parametrize("name", CASES)
def test_flop_count_matches_reference(name):
    inp, g = _case(name)
    fc = flop_count(inp)
    assert [fc.exact_mas, fc.taylor_mas, fc.overhead_mas, fc.dense_equivalent_mas] == g["flops"].tolist()


def test_validation_errors():
    q, kk, v, kc, vc, idx = make_inputs(1, 1, 2, 3, 64, 2, 0)

    def inp(**kw):
        base = dict(q=q, k_new=kk, v_new=v, kc=kc, vc=vc, mask=BlockMask(idx, 3), scale=0.125, block_size=64)
        base.update(kw)
        return TaylorKernelInput(**base)

    cases = [
        (dict(q=q[:, :, :100]), LayoutError, "query length"),
        (dict(k_new=kk[:, :, :150]), LayoutError, "key length"),
        (dict(v_new=v[:, :, :128]), LayoutError, "mismatch"),
        (dict(kc=kc[:, :, :2]), LayoutError, "kc/vc"),
        (dict(mask=BlockMask(idx[:, :, :1], 3)), LayoutError, "mask indices shape"),
        (dict(mask=BlockMask(idx[..., :0], 3)), ContractError, "at least one"),
        (dict(mask=BlockMask(idx + 5, 3)), ContractError, "out of range"),
        (dict(mask=BlockMask(idx, 4)), ContractError, "out of range"),
        (dict(mask=BlockMask(idx[..., ::-1].copy(), 3)), ContractError, "sorted"),
        (dict(key_valid_rows=np.full((1, 1, 2), 64)), LayoutError, "key_valid_rows shape"),
        (dict(key_valid_rows=np.full((1, 1, 3), 65)), LayoutError, "lie in"),
        (dict(scale=0.0), LayoutError, "scale"),
        (dict(q=q[0]), LayoutError, "4 axes"),
    ]
    for kw, exc, msg in cases:
        with pytest.raises(exc, match=msg):
            inp(**kw).validated()


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_outputs_match_reference_golden(name):
    inp, g = _case(name)
    out = taylor_sparse_forward(inp)
    assert out.shape == g["out"].shape and out.dtype == np.float32
    _close(out, g["out"])


@pytest.mark.gpu
def test_larger_vs_oracle_torch_strided():
    """t_q != t_k at a few thousand tokens, torch bf16 inputs with (B,S,H,D)
    storage, mask on the device; against the oracle's taylor_head."""
    import torch

    B, H, t_q, t_k, D, k = 1, 3, 40, 72, 128, 6
    q, kk, v, kc, vc, idx = make_inputs(B, H, t_q, t_k, D, k, seed=77)
    dev = torch.device("cuda")

    def bshd(x):  # same values, (B,S,H,D) storage viewed as (B,H,S,D)
        return torch.from_numpy(x).to(dev, torch.bfloat16).permute(0, 2, 1, 3).contiguous().permute(0, 2, 1, 3)

    tq, tk, tv = bshd(q), bshd(kk), bshd(v)
    assert not tq.is_contiguous()
    out = taylor_sparse_forward(TaylorKernelInput(q=tq, k_new=tk, v_new=tv, kc=torch.from_numpy(kc).to(dev),
                                                  vc=torch.from_numpy(vc).to(dev),
                                                  mask=BlockMask(torch.from_numpy(idx).to(dev), t_k),
                                                  scale=1.0 / np.sqrt(D), block_size=64))
    assert out.dtype == torch.bfloat16 and out.is_cuda
    w = np.full(t_k, 64)
    for h in range(H):
        ref = O.taylor_head(q[0, h].astype(np.float64), kk[0, h].astype(np.float64), v[0, h].astype(np.float64),
                            kc[0, h].astype(np.float64), vc[0, h].astype(np.float64), idx[0, h], w,
                            1.0 / np.sqrt(D), 64)
        _close(out[0, h].float().cpu().numpy(), ref)


@pytest.mark.gpu
def test_contract_and_unsupported():
    q, kk, v, kc, vc, idx = make_inputs(1, 1, 2, 3, 64, 2, 1)
    base = dict(q=q, k_new=kk, v_new=v, kc=kc, vc=vc, mask=BlockMask(idx, 3), scale=0.125, block_size=64)
    with pytest.raises(ContractError, match="block mean"):
        taylor_sparse_forward(TaylorKernelInput(**dict(base, kc=kc + 0.1)))
    with pytest.raises(ConfigError, match="partial key blocks"):
        taylor_sparse_forward(TaylorKernelInput(**dict(base, key_valid_rows=np.array([[[64, 64, 60]]]),
                                                       kc=_partial_means(kk, [64, 64, 60]),
                                                       vc=_partial_means(v, [64, 64, 60]))))


def _partial_means(x, valid):
    out = np.zeros((1, 1, len(valid), x.shape[3]), np.float32)
    for t, n in enumerate(valid):
        out[0, 0, t] = x[0, 0, t * 64:t * 64 + n].astype(np.float64).mean(axis=0)
    return out


def _grad_close(got, ref, name):
    a = np.asarray(got, dtype=np.float64).ravel()
    r = np.asarray(ref, dtype=np.float64).ravel()
    cos = float(a @ r / (np.linalg.norm(a) * np.linalg.norm(r) + 1e-300))
    err = float(np.abs(a - r).max())
    assert cos >= 0.999 and err <= 3e-2 * float(np.abs(r).max()), (name, cos, err)


@pytest.mark.gpu
@pytest.mark.parametrize("name", [c for c in CASES if "dq" in np.load(os.path.join(GOLD, f"{c}.npz")).files])
def test_backward_matches_reference_golden(name):
    """taylor_sparse_backward (taylor.py:225-296) vs the reference's gradients."""
    from paper_2605_04569_b200.taylor import taylor_sparse_backward

    inp, g = _case(name)
    B, H, t_q, t_k, D, k, seed = (int(x) for x in g["geom"])
    do = O.round_bf16(np.random.default_rng(seed + 1000).standard_normal(g["out"].shape).astype(np.float32))
    grads = taylor_sparse_backward(inp, do)
    for key, got in (("dq", grads.dq), ("dk", grads.dk), ("dv", grads.dv)):
        _grad_close(got, g[key], key)
