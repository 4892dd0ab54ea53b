"""Exact attention drop-ins (`full_attention`, `online_softmax_attention`,
reference.py:79-170) on the sm_100a kernel, against the reference's own
`full_attention` outputs (`tests/golden/exact`, made by
`tests/golden/make_exact_golden.py`): S_q == S_k and S_q != S_k, ragged
lengths, head dims 64 / 128 / padded 96, the reference's errors."""

from __future__ import annotations

import os

import numpy as np
import pytest

from oracle import isa_oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden", "exact")
CASES = sorted(f[:-4] for f in os.listdir(GOLD) if f.endswith(".npz"))


def make_inputs(B, H, S_q, S_k, D, seed):
    """Same draws as make_exact_golden.make_inputs."""
    rng = np.random.default_rng(seed)
    q = O.round_bf16(rng.standard_normal((B, H, S_q, D)).astype(np.float32))
    k = O.round_bf16(rng.standard_normal((B, H, S_k, D)).astype(np.float32))
    v = O.round_bf16(rng.standard_normal((B, H, S_k, D)).astype(np.float32))
    return q, k, v


def _case(name):
    g = np.load(os.path.join(GOLD, f"{name}.npz"))
    B, H, S_q, S_k, D, seed = (int(x) for x in g["geom"])
    q, k, v = make_inputs(B, H, S_q, S_k, D, seed)
    assert np.isclose(q.sum() + k.sum() + v.sum(), g["checksum"])
    return (q, k, v), g


def test_errors_before_device():
    from paper_2605_04569_b200.errors import ConfigError, DegenerateRowError, LayoutError
    from paper_2605_04569_b200.exact import full_attention, online_softmax_attention
    from paper_2605_04569_b200.types import BlockLayout

    q, k, v = make_inputs(1, 2, 64, 128, 64, 0)
    with pytest.raises(LayoutError, match="batch/head/dim"):
        full_attention(q, k[:, :1], v)
    with pytest.raises(LayoutError, match="differ"):
        full_attention(q, k, v[:, :, :64])
    with pytest.raises(ConfigError, match="scale"):
        full_attention(q, k, v, scale=-1.0)
    with pytest.raises(LayoutError, match="key mask shape"):
        full_attention(q, k, v, mask=np.ones((1, 2, 5), bool))
    with pytest.raises(DegenerateRowError):
        full_attention(q, k, v, mask=np.zeros(128, bool))
    with pytest.raises(LayoutError, match="layout.seq_len"):
        online_softmax_attention(q, k, v, layout=BlockLayout(64, 100))
    with pytest.raises(LayoutError, match="4 axes"):
        full_attention(q[0], k, v)


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
def test_matches_reference_golden(name):
    import paper_2605_04569_b200 as P

    (q, k, v), g = _case(name)
    mask = g["mask"] if "mask" in g.files else np.ones(k.shape[2], bool)
    for fn in (P.full_attention, P.online_softmax_attention):
        out = fn(q, k, v, mask=mask)
        assert out.shape == g["out"].shape and out.dtype == np.float32
        a, r = out.astype(np.float64).ravel(), g["out"].astype(np.float64).ravel()
        err = float(np.abs(a - r).max())
        cos = float(a @ r / (np.linalg.norm(a) * np.linalg.norm(r)))
        assert err <= 2e-2 and cos >= 0.999, (name, err, cos)


@pytest.mark.gpu
def test_torch_strided_cross():
    import torch

    import paper_2605_04569_b200 as P

    q, k, v = make_inputs(2, 3, 700, 1500, 128, 5)
    dev = torch.device("cuda")
    tq, tk, tv = (torch.from_numpy(x).to(dev, torch.bfloat16).permute(0, 2, 1, 3).contiguous().permute(0, 2, 1, 3)
                  for x in (q, k, v))
    out = P.full_attention(tq, tk, tv)
    assert out.dtype == torch.bfloat16 and tuple(out.shape) == (2, 3, 700, 128)
    ref = torch.softmax((tq.float() @ tk.float().transpose(-1, -2)) / np.sqrt(128), -1) @ tv.float()
    assert (out.float() - ref).abs().max().item() < 2e-2


@pytest.mark.gpu
@pytest.mark.parametrize("name", [c for c in CASES if c.endswith("_bwd")])
def test_backward_matches_reference_golden(name):
    """full_attention_backward (reference.py:173-225) vs the reference's gradients."""
    import paper_2605_04569_b200 as P

    (q, k, v), g = _case(name)
    seed = int(g["geom"][5])
    do = O.round_bf16(np.random.default_rng(seed + 1000).standard_normal(g["out"].shape).astype(np.float32))
    grads = P.full_attention_backward(q, k, v, None, do)
    for key, got in (("dq", grads.dq), ("dk", grads.dk), ("dv", grads.dv)):
        a = np.asarray(got, dtype=np.float64).ravel()
        r = np.asarray(g[key], dtype=np.float64).ravel()
        cos = float(a @ r / (np.linalg.norm(a) * np.linalg.norm(r)))
        assert cos >= 0.999 and float(np.abs(a - r).max()) <= 3e-2 * float(np.abs(r).max()), (key, cos)


@pytest.mark.gpu
def test_online_state_matches_reference_contract():
    """OnlineState (reference.py:28-60): blockwise updates with weights equal
    the direct weighted softmax; an all-masked row raises DegenerateRowError."""
    import paper_2605_04569_b200 as P
    from paper_2605_04569_b200.errors import DegenerateRowError

    rng = np.random.default_rng(3)
    s = rng.standard_normal((5, 40)) * 3
    s[2, :7] = -np.inf
    vals = rng.standard_normal((40, 6))
    w = rng.integers(1, 65, 40).astype(np.float64)
    st = P.OnlineState(5, 6)
    for lo in range(0, 40, 16):
        st.update(s[:, lo:lo + 16], vals[lo:lo + 16], w[lo:lo + 16])
    out = st.finalize()
    p = np.where(np.isfinite(s), np.exp(s - s.max(axis=1, keepdims=True)), 0.0) * w
    np.testing.assert_allclose(out, (p @ vals) / p.sum(axis=1, keepdims=True), rtol=1e-12, atol=1e-12)
    st2 = P.OnlineState(2, 3)
    st2.update(np.full((2, 4), -np.inf), np.ones((4, 3)))
    with pytest.raises(DegenerateRowError):
        st2.finalize()


def test_backward_errors_before_device():
    from paper_2605_04569_b200.errors import ConfigError, LayoutError
    from paper_2605_04569_b200.exact import full_attention_backward

    q, k, v = make_inputs(1, 1, 64, 128, 64, 0)
    with pytest.raises(LayoutError, match="dO"):
        full_attention_backward(q, k, v, None, None)
    with pytest.raises(ConfigError, match="S_q == S_k"):
        full_attention_backward(q, k, v, None, np.zeros_like(q))


@pytest.mark.gpu
@pytest.mark.parametrize("S,D", [(4096, 128), (3000, 64), (700, 64)])
def test_backward_multi_tile_vs_torch_autograd(S, D):
    """full_attention_backward (reference.py:173-225) on the tcgen05 dK/dV and dQ
    kernels at sizes with many K/V tiles per CTA (both TMEM buffers and every
    ring slot cycle; 3000 / 700: ragged last block, odd block counts) vs torch
    fp32 autograd of softmax(QK^T/sqrt(D))V on the same bf16 inputs."""
    import torch

    import paper_2605_04569_b200 as P

    g = torch.Generator(device="cuda").manual_seed(S + D)
    q, k, v, do = (torch.randn((1, 2, S, D), generator=g, device="cuda").to(torch.bfloat16) for _ in range(4))
    got = P.full_attention_backward(q, k, v, None, do)
    qf, kf, vf = (x.float().requires_grad_(True) for x in (q, k, v))
    out = torch.softmax((qf @ kf.transpose(-1, -2)) / np.sqrt(D), -1) @ vf
    out.backward(do.float())
    for name, a, r in (("dq", got.dq, qf.grad), ("dk", got.dk, kf.grad), ("dv", got.dv, vf.grad)):
        a, r = a.float().flatten().double(), r.flatten().double()
        cos = float(a @ r / (a.norm() * r.norm()))
        err = float((a - r).abs().max())
        assert cos >= 0.999 and err <= 3e-2 * float(r.abs().max()), (name, cos, err)
