"""Standalone Taylor sparse attention kernel — drop-in for the reference's
`TaylorKernelInput` / `taylor_sparse_forward` / `flop_count`
(pkg/src/isattn/taylor.py:45-194, 299-316).

Every 64-row query block of `q` is a flat block: it attends exactly to the key
blocks its mask row lists (ascending) and to every other key block through the
block centroid `kc`/`vc` weighted by the block's row count (the 0th-order
Taylor surrogate, taylor.py:124-160). The computation is the pipeline's K7
kernel (`isa_taylor_forward` in the C ABI) on bf16 operands with fp32
accumulation; there is no CPU path.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Optional

import numpy as np

from .errors import ConfigError, ContractError, InputError, LayoutError
from .types import FlopCount, SUPPORTED_BLOCK, SUPPORTED_HEAD_DIMS


@dataclass
class TaylorKernelInput:
    """Everything the kernel consumes (taylor.py:45-58; same fields). kc/vc
    must be the valid-row block means of k_new/v_new."""

    q: object
    k_new: object
    v_new: object
    kc: object
    vc: object
    mask: object  # BlockMask (ours or the reference's): indices (B,H,t_q,k), num_key_blocks
    scale: float
    block_size: int
    key_valid_rows: Optional[np.ndarray] = None

    def validated(self) -> "TaylorKernelInput":
        """The reference checks, order and messages (taylor.py:60-103)."""
        q, k, v = (_shape4(x, n) for x, n in ((self.q, "Q"), (self.k_new, "K_new"), (self.v_new, "V_new")))
        b = self.block_size
        B, H, S_q, D = q
        if S_q % b:
            raise LayoutError(f"query length {S_q} not divisible by block size {b}")
        if k[2] % b:
            raise LayoutError(f"key length {k[2]} not divisible by block size {b}")
        if k[:2] != (B, H) or k[3] != D or v != k:
            raise LayoutError(f"Q/K_new/V_new mismatch: {q}, {k}, {v}")
        t_q, t_k = S_q // b, k[2] // b
        if tuple(self.kc.shape) != (B, H, t_k, D) or tuple(self.vc.shape) != (B, H, t_k, D):
            raise LayoutError(f"kc/vc must have shape (B,H,{t_k},{D})")
        idx = _np(self.mask.indices)
        if idx.ndim != 4 or idx.shape[:3] != (B, H, t_q):
            raise LayoutError(f"mask indices shape {idx.shape} != (B,H,{t_q},k)")
        if idx.shape[3] < 1:
            raise ContractError("every query block needs at least one exact key block")
        if self.mask.num_key_blocks != t_k or idx.max(initial=0) >= t_k or idx.min(initial=0) < 0:
            raise ContractError(f"mask indices out of range for {t_k} key blocks")
        if idx.shape[3] > 1 and np.any(np.diff(idx, axis=3) <= 0):
            raise ContractError("mask index lists must be sorted ascending without duplicates")
        if self.key_valid_rows is not None:
            w = np.asarray(self.key_valid_rows, dtype=np.int64)
            if w.shape != (B, H, t_k):
                raise LayoutError(f"key_valid_rows shape {w.shape} != (B,H,{t_k})")
            if w.min() < 1 or w.max() > b:
                raise LayoutError(f"key_valid_rows must lie in [1, {b}]")
        if self.scale <= 0:
            raise LayoutError(f"scale must be > 0, got {self.scale}")
        if __debug__:
            self._check_means()
        return self

    def _check_means(self):
        """kc must be the valid-row block mean of k_new (taylor.py:105-111, same tolerance)."""
        import torch

        dev = _device(self.q, self.k_new)
        k = _dev(self.k_new, dev, torch.float64)
        kc = _dev(self.kc, dev, torch.float64)
        B, H, t_k, D = kc.shape
        w = torch.as_tensor(self._weights(), device=dev)
        valid = torch.arange(self.block_size, device=dev) < w[..., None]
        means = (k.reshape(B, H, t_k, self.block_size, D) * valid[..., None]).sum(3) / w[..., None]
        if not torch.allclose(means, kc, rtol=1e-4, atol=1e-5):
            raise ContractError("kc is not the valid-row block mean of k_new")

    def _weights(self) -> np.ndarray:
        B, H, t_k = tuple(self.kc.shape)[:3]
        if self.key_valid_rows is None:
            return np.full((B, H, t_k), self.block_size, dtype=np.int64)
        return np.asarray(self.key_valid_rows, dtype=np.int64)


def _shape4(x, name):
    shape = tuple(int(s) for s in getattr(x, "shape", ()))
    if len(shape) != 4:
        raise LayoutError(f"{name}: expected 4 axes (B,H,S,D), got shape {shape}")
    if min(shape) < 1:
        raise LayoutError(f"{name}: all dims must be >= 1, got shape {shape}")
    return shape


def _np(x) -> np.ndarray:
    if hasattr(x, "detach"):
        return x.detach().cpu().numpy()
    return np.asarray(x)


def _device(*xs):
    import torch

    for x in xs:
        if isinstance(x, torch.Tensor) and x.is_cuda:
            return x.device
    if not torch.cuda.is_available():
        raise LayoutError("the Taylor kernel runs on a CUDA device and none is available (there is no CPU path)")
    return torch.device("cuda", torch.cuda.current_device())


def _dev(x, dev, dtype):
    import torch

    if isinstance(x, np.ndarray):
        x = torch.from_numpy(np.ascontiguousarray(x))
    return x.to(device=dev, dtype=dtype)


def taylor_sparse_forward(inp: TaylorKernelInput, visit_rng=None):
    """Forward pass, O = acc / ell per row (taylor.py:163-194). Returns an
    array like `q`: numpy in -> numpy of q's dtype out; torch -> torch of q's
    dtype on q's device. `visit_rng` (the reference's visiting-order test hook)
    is accepted and ignored: the kernel's order is fixed, and the reference
    requires results independent of it up to rounding."""
    import torch

    from . import _native as N

    del visit_rng
    inp = inp.validated()
    B, H, S_q, D = _shape4(inp.q, "Q")
    S_k = int(inp.k_new.shape[2])
    b = inp.block_size
    if b != SUPPORTED_BLOCK:
        raise ConfigError(f"block_size={b} is not supported by the sm_100a kernels (only {SUPPORTED_BLOCK})")
    if D not in SUPPORTED_HEAD_DIMS:
        raise ConfigError(f"head dim {D} not supported by the sm_100a kernels {SUPPORTED_HEAD_DIMS}")
    if inp.key_valid_rows is not None and np.any(np.asarray(inp.key_valid_rows) != b):
        raise ConfigError("partial key blocks (key_valid_rows < block_size) are not supported by the sm_100a "
                          "Taylor kernel")
    numpy_io = isinstance(inp.q, np.ndarray)
    out_dtype = inp.q.dtype
    dev = _device(inp.q, inp.k_new, inp.v_new)
    q, k, v = (_dev(x, dev, torch.bfloat16) for x in (inp.q, inp.k_new, inp.v_new))
    q = q if q.stride(3) == 1 and all(s % 8 == 0 for s in q.stride()[:3]) else q.contiguous()
    if k.stride() != v.stride() or k.stride(3) != 1 or any(s % 8 for s in k.stride()[:3]):
        k, v = k.contiguous(), v.contiguous()
    if not (bool(torch.isfinite(q).all()) and bool(torch.isfinite(k).all()) and bool(torch.isfinite(v).all())):
        raise InputError("Q/K_new/V_new: non-finite elements")
    kc, vc = (_dev(x, dev, torch.float32).contiguous() for x in (inp.kc, inp.vc))
    mask = _dev(_np(inp.mask.indices).astype(np.int64), dev, torch.int64).contiguous()
    kmask = int(mask.shape[3])
    out = torch.empty((B, H, S_q, D), dtype=torch.bfloat16, device=dev)
    shape = N.IsaShape(B, H, S_q, D, S_q, 0, b, N.ISA_DTYPE_BF16, q.stride(0), q.stride(1), q.stride(2))
    lib = N.load()
    nbytes = ctypes.c_size_t(0)
    N.check(lib.isa_taylor_workspace_bytes(ctypes.byref(shape), S_k, kmask, ctypes.byref(nbytes)))
    ws = torch.empty(max(int(nbytes.value), 1), dtype=torch.uint8, device=dev)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    kst = (ctypes.c_int64 * 3)(*k.stride()[:3])
    N.check(lib.isa_taylor_forward(ctypes.byref(shape), S_k, kst, kmask, float(inp.scale), q.data_ptr(),
                                   k.data_ptr(), v.data_ptr(), kc.data_ptr(), vc.data_ptr(), mask.data_ptr(),
                                   out.data_ptr(), ws.data_ptr(), nbytes.value, err.data_ptr(),
                                   torch.cuda.current_stream(dev).cuda_stream))
    if numpy_io:
        return out.float().cpu().numpy().astype(out_dtype)
    return out.to(out_dtype)


def flop_count(inp: TaylorKernelInput) -> FlopCount:
    """Tallies implied by the mask (taylor.py:299-316): per block pair, exact =
    2*b*b*D + 2*b*b*D, Taylor = 2*b*D + 2*b*D (FLOPs, 2 per multiply-add)."""
    B, H, S_q, D = _shape4(inp.q, "Q")
    b = inp.block_size
    t_q, t_k = S_q // b, int(inp.k_new.shape[2]) // b
    k = int(_np(inp.mask.indices).shape[3])
    exact_pair, taylor_pair = 4 * b * b * D, 4 * b * D
    return FlopCount(exact_mas=B * H * t_q * k * exact_pair, taylor_mas=B * H * t_q * (t_k - k) * taylor_pair,
                     overhead_mas=0, dense_equivalent_mas=B * H * t_q * t_k * exact_pair)


def taylor_sparse_backward(inp: TaylorKernelInput, do):
    """Gradients of taylor_sparse_forward (taylor.py:225-296): the Taylor
    branch's gradients to Q, and to K_new / V_new directly and through the
    block means. Self-attention geometry (S_q == S_k, full blocks) runs the
    tcgen05 backward of `isa_backward` with the caller's mask pinned as the
    routing (one segment, every query block flat); otherwise ConfigError."""
    import torch

    from .pipeline import isa_backward
    from .types import BlockMask, IclLayout, IsaConfig, IsaRouting, SelectionIndex, SharpnessSplit

    inp = inp.validated()
    B, H, S_q, D = _shape4(inp.q, "Q")
    S_k = int(inp.k_new.shape[2])
    b = inp.block_size
    if tuple(int(x) for x in do.shape) != (B, H, S_q, int(inp.v_new.shape[3])):
        raise LayoutError(f"dO shape {tuple(do.shape)} != output shape")
    if S_q != S_k:
        raise ConfigError("taylor_sparse_backward on the sm_100a kernels needs S_q == S_k")
    if inp.key_valid_rows is not None and np.any(np.asarray(inp.key_valid_rows) != b):
        raise ConfigError("partial key blocks (key_valid_rows < block_size) are not supported by the sm_100a "
                          "Taylor kernel")
    t = S_q // b
    idx = _np(inp.mask.indices).astype(np.int64)
    k = int(idx.shape[3])
    alpha_ns = min(1.0, (k + 0.5) / t)  # floor(alpha_ns * t) == k (coarse.py:169)
    cfg = IsaConfig(alpha_s=1.0, alpha_f=1.0, alpha_ns=alpha_ns, scale=inp.scale, block_size=b)
    flat = np.broadcast_to(np.arange(t, dtype=np.int64), (B, H, t)).copy()
    routing = IsaRouting(selection=SelectionIndex(np.zeros((B, H, 0), np.int64), 0),
                         split=SharpnessSplit(sharp=np.zeros((B, H, 0), np.int64), flat=flat,
                                              sharpness=np.zeros((B, H, t))),
                         mask=BlockMask(idx, t))
    return isa_backward(inp.q, inp.k_new, inp.v_new, IclLayout(S_q, 0), cfg, do, routing=routing)
