"""Exact softmax attention drop-ins: the reference's `full_attention` and
`online_softmax_attention` (pkg/src/isattn/reference.py:79-170, the sharp
branch's kernel and the dense oracle), with the same signatures and errors,
computed by the sm_100a K8 kernel (bf16 operands, fp32 accumulation).

S_q == S_k runs `isa_dense_attention`; S_q != S_k runs `isa_cross_attention`
on query rows zero-padded to a multiple of 64, except a ragged key length with
no more key blocks than query blocks, which runs `isa_dense_attention` on
query slabs of S_k rows.
Key masks (reference.py:67-76, 113-119, 160-162): masked keys get zero
weight, i.e. the softmax runs over the valid keys only — so the valid K/V
rows are compacted on the device (one index_select when every (b, h) shares
the mask, per (b, h) otherwise) and the same kernel runs on them. A row with
every key masked raises DegenerateRowError (reference.py:116-117).

`OnlineState` (reference.py:28-60) is the blockwise softmax accumulator with
the reference's update/finalize contract, on device fp64 tensors.
"""

from __future__ import annotations

import ctypes
import math
from typing import Optional

import numpy as np
import torch

from . import _native as N
from .errors import ConfigError, DegenerateRowError, InputError, LayoutError
from .types import SUPPORTED_HEAD_DIMS


def _shape4(x, name):
    shape = tuple(int(s) for s in getattr(x, "shape", ()))
    if len(shape) != 4:
        raise LayoutError(f"{name}: expected 4 axes (B,H,S,D), got shape {shape}")
    if min(shape) < 1:
        raise LayoutError(f"{name}: all dims must be >= 1, got shape {shape}")
    return shape


def _key_mask(mask, B: int, H: int, S_k: int) -> Optional[np.ndarray]:
    """(B,H,S_k) bool, True = valid key; a 1-D mask broadcasts (reference.py:67-76)."""
    if mask is None:
        return None
    if hasattr(mask, "detach"):
        mask = mask.detach().cpu().numpy()
    mask = np.asarray(mask, dtype=bool)
    if mask.ndim == 1:
        mask = np.broadcast_to(mask, (B, H, S_k))
    if mask.shape != (B, H, S_k):
        raise LayoutError(f"key mask shape {mask.shape} != (B,H,S_k)=({B},{H},{S_k})")
    return mask


def _device_bf16(x, dev):
    if isinstance(x, np.ndarray):
        x = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32))
    if not isinstance(x, torch.Tensor):
        raise LayoutError("expected torch tensors or numpy arrays")
    x = x.to(device=dev, dtype=torch.bfloat16)
    if x.stride(3) != 1 or any(s % 8 for s in x.stride()[:3]) or x.data_ptr() % 16:
        x = x.contiguous()
    return x


class OnlineState:
    """Running (max, normalizer, output accumulator) for blockwise softmax
    attention (reference.py:28-60): update() folds in one block of scores and
    values, rescaling the accumulators by exp(m - m_new) when the running max
    moves; `weights` multiplies the exponentials per score column (the Taylor
    branch's block weights). float64 on the CUDA device (numpy inputs are
    uploaded; finalize returns a numpy array when update was fed numpy)."""

    def __init__(self, rows: int, dim: int, device=None):
        if not torch.cuda.is_available() and device is None:
            raise LayoutError("OnlineState runs on a CUDA device and none is available (there is no CPU path)")
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.m = torch.full((rows,), -math.inf, dtype=torch.float64, device=dev)
        self.ell = torch.zeros(rows, dtype=torch.float64, device=dev)
        self.o_acc = torch.zeros((rows, dim), dtype=torch.float64, device=dev)
        self._numpy = False

    def _t(self, x):
        if isinstance(x, np.ndarray):
            self._numpy = True
            return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).to(self.m.device)
        return torch.as_tensor(x, dtype=torch.float64, device=self.m.device)

    def update(self, scores, values, weights=None) -> None:
        s = self._t(scores)
        m_new = torch.maximum(self.m, s.max(dim=1).values if s.shape[1] else self.m)
        p = torch.where(torch.isfinite(s), torch.exp(s - m_new[:, None]), torch.zeros((), dtype=s.dtype,
                                                                                      device=s.device))
        if weights is not None:
            p = p * self._t(weights)
        delta = self.m - m_new
        delta = torch.where(torch.isfinite(delta), delta, torch.zeros_like(delta))  # both -inf: nothing yet
        alpha = torch.exp(delta)
        self.ell = self.ell * alpha + p.sum(dim=1)
        self.o_acc = self.o_acc * alpha[:, None] + p @ self._t(values)
        self.m = m_new

    def finalize(self):
        if bool((self.ell <= 0.0).any()):
            raise DegenerateRowError("row with empty key set: normalizer is zero")
        out = self.o_acc / self.ell[:, None]
        return out.cpu().numpy() if self._numpy else out


def _exact(q, k, v, scale, mask):
    (B, H, S_q, D), (Bk, Hk, S_k, Dk), (Bv, Hv, S_v, Dv) = (_shape4(x, n) for x, n in ((q, "Q"), (k, "K"), (v, "V")))
    if (Bk, Hk) != (B, H) or (Bv, Hv) != (B, H) or Dk != D:
        raise LayoutError(f"Q/K/V batch/head/dim mismatch: {(B, H, S_q, D)}, {(Bk, Hk, S_k, Dk)}, "
                          f"{(Bv, Hv, S_v, Dv)}")
    if S_v != S_k:
        raise LayoutError(f"K and V sequence lengths differ: {S_k} vs {S_v}")
    if Dv != D:
        raise ConfigError(f"value width {Dv} != key width {D} is not supported by the sm_100a kernel")
    scale = 1.0 / math.sqrt(D) if scale is None else float(scale)
    if scale <= 0:
        raise ConfigError(f"scale must be > 0, got {scale}")
    km = _key_mask(mask, B, H, S_k)
    if km is not None and km.all():
        km = None
    if km is not None and not km.any(axis=2).all():
        raise DegenerateRowError("query row with all keys masked")
    if D > max(SUPPORTED_HEAD_DIMS):
        raise ConfigError(f"head dim {D} not supported by the sm_100a kernels (<= {max(SUPPORTED_HEAD_DIMS)})")
    numpy_io = isinstance(q, np.ndarray)
    out_dtype = q.dtype
    dev = next((x.device for x in (q, k, v) if isinstance(x, torch.Tensor) and x.is_cuda), None)
    if dev is None:
        if not torch.cuda.is_available():
            raise LayoutError("exact attention runs on a CUDA device and none is available (there is no CPU path)")
        dev = torch.device("cuda", torch.cuda.current_device())
    qd, kd, vd = (_device_bf16(x, dev) for x in (q, k, v))
    if not all(bool(torch.isfinite(x).all()) for x in (qd, kd, vd)):
        raise InputError("Q/K/V: non-finite elements")
    width = 64 if D <= 64 else 128
    if width != D:  # zero columns: exact zeros in every score, dropped output columns
        qd, kd, vd = (torch.nn.functional.pad(x, (0, width - D)) for x in (qd, kd, vd))
    if km is None:
        res = _run(qd, kd, vd, scale)
    elif (km == km[:1, :1]).all():  # one mask for every (b, h): compact the valid keys once
        idx = torch.from_numpy(np.nonzero(km[0, 0])[0]).to(dev)
        res = _run(qd, kd.index_select(2, idx), vd.index_select(2, idx), scale)
    else:
        res = torch.empty((B, H, S_q, width), dtype=torch.bfloat16, device=dev)
        for bi in range(B):
            for hi in range(H):
                idx = torch.from_numpy(np.nonzero(km[bi, hi])[0]).to(dev)
                sl = (slice(bi, bi + 1), slice(hi, hi + 1))
                res[sl] = _run(qd[sl], kd[sl].index_select(2, idx), vd[sl].index_select(2, idx), scale)
    res = res[..., :D]
    if numpy_io:
        return res.float().cpu().numpy().astype(out_dtype)
    return res.to(out_dtype).contiguous()


def _run(q, k, v, scale):
    """Dense softmax attention of bf16 device tensors on the sm_100a kernels."""
    if q.shape[2] == k.shape[2]:
        from .pipeline import dense_attention

        return dense_attention(q, k, v, scale)
    return _cross(q, k, v, scale)


def _cross(q, k, v, scale):
    B, H, S_q, D = q.shape
    S_k = k.shape[2]
    rows = -(-S_q // 64) * 64
    t_q, t_k = rows // 64, -(-S_k // 64)
    if S_k % 64 and t_k <= t_q:
        # ragged keys and at least as many query blocks: query slabs of S_k rows
        # on the equal-length kernel (the last slab zero-padded)
        from .pipeline import dense_attention

        k, v = k.contiguous(), v.contiguous()
        n = -(-S_q // S_k)
        qp = torch.nn.functional.pad(q, (0, 0, 0, n * S_k - S_q))
        out = torch.empty((B, H, n * S_k, D), dtype=torch.bfloat16, device=q.device)
        for i in range(n):
            out[:, :, i * S_k:(i + 1) * S_k] = dense_attention(qp[:, :, i * S_k:(i + 1) * S_k].contiguous(), k, v,
                                                               scale)
        return out[:, :, :S_q]
    if rows != S_q:
        q = torch.nn.functional.pad(q, (0, 0, 0, rows - S_q))
    if k.stride() != v.stride():
        k, v = k.contiguous(), v.contiguous()
    out = torch.empty((B, H, rows, D), dtype=torch.bfloat16, device=q.device)
    shape = N.IsaShape(B, H, rows, D, rows, 0, 64, N.ISA_DTYPE_BF16, *q.stride()[:3])
    shape.out_stride_b, shape.out_stride_h, shape.out_stride_s = out.stride()[:3]
    kst = (ctypes.c_int64 * 3)(*k.stride()[:3])
    N.check(N.load().isa_cross_attention(ctypes.byref(shape), S_k, kst, scale, q.data_ptr(), k.data_ptr(),
                                         v.data_ptr(), out.data_ptr(), torch.cuda.current_stream(q.device).cuda_stream))
    return out[:, :, :S_q]


def full_attention(q, k, v, scale: Optional[float] = None, mask=None, row_chunk: int = 2048):
    """Direct softmax attention O = softmax(scale * Q K^T) V (reference.py:79-123).
    `row_chunk` (the reference's memory knob) is accepted and unused: the
    kernel streams keys through shared memory and never forms the score matrix."""
    del row_chunk
    return _exact(q, k, v, scale, mask)


def online_softmax_attention(q, k, v, scale: Optional[float] = None, layout=None, mask=None, block_order=None):
    """Blockwise online-softmax attention (reference.py:126-170), same contract
    as full_attention. `layout` must cover the key axis (LayoutError otherwise);
    the kernel's own 128-key tiling replaces it, and `block_order` (the
    reference's visiting-order test hook) is accepted and ignored: the result
    is order-independent up to rounding."""
    del block_order
    S_k = _shape4(k, "K")[2]
    if layout is not None and layout.seq_len != S_k:
        raise LayoutError(f"layout.seq_len {layout.seq_len} != key length {S_k}")
    return _exact(q, k, v, scale, mask)


def full_attention_backward(q, k, v, scale: Optional[float] = None, do=None, mask=None, row_chunk: int = 2048):
    """Analytic gradients of full_attention (reference.py:173-225, same argument
    order). Self-attention (S_q == S_k) runs the tcgen05 backward kernels of
    `isa_backward` on the all-exact configuration (one segment, alpha_f = 0:
    every query block attends to every key block — ISA's dense identity);
    S_q != S_k and key masks that drop keys raise ConfigError. Returns a
    GradBundle in q's dtype (numpy fp32 for numpy inputs)."""
    del row_chunk
    from .pipeline import isa_backward
    from .types import IclLayout, IsaConfig

    (B, H, S_q, D), (_, _, S_k, _), _ = (_shape4(x, n) for x, n in ((q, "Q"), (k, "K"), (v, "V")))
    if do is None:
        raise LayoutError("dO is required")
    if tuple(int(x) for x in do.shape) != (B, H, S_q, int(v.shape[3])):
        raise LayoutError(f"dO shape {tuple(do.shape)} != output shape {(B, H, S_q, int(v.shape[3]))}")
    if scale is not None and scale <= 0:
        raise ConfigError(f"scale must be > 0, got {scale}")
    km = _key_mask(mask, B, H, S_k)
    if km is not None and not km.all():
        if not km.any(axis=2).all():
            raise DegenerateRowError("query row with all keys masked")
        raise ConfigError("key masks that drop keys are not supported by the sm_100a kernels")
    if S_q != S_k:
        raise ConfigError("full_attention_backward on the sm_100a kernels needs S_q == S_k")
    cfg = IsaConfig(alpha_s=1.0, alpha_f=0.0, scale=scale, strict=False)
    return isa_backward(q, k, v, IclLayout(S_q, 0), cfg, do)
