"""Function-level drop-ins for the reference's routing API (pkg/src/isattn/coarse.py:22-201):
`build_coarse`, `rank_context`, `build_block_mask`, `sharpness_split` and `CoarseSet`, on the
same sm_100a primitives the fused pipeline uses (C ABI `isa_pool_means`, `isa_topk_rows_f64`,
`isa_sharpness_rows_f64`, `isa_split_rows_f64`, `isa_coarse_scores`, `isa_ctx_saliency_f64`).
numpy callers get numpy arrays back (like the reference); torch callers get device tensors.
Block means, the fp64 coarse scores and the context saliency are bit-identical to the
reference's numpy arithmetic; every discrete decision matches it bit for bit.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import _native as N
from .errors import ConfigError, InputError, LayoutError
from .types import BlockLayout, BlockMask, IclLayout, SelectionIndex, SharpnessSplit, icl_from_any


@dataclass
class CoarseSet:
    """Pooled Q/K/V (one row per block) and the scaled fp64 block score matrix (coarse.py:22-49)."""

    qc: object  # (B, H, N_Q, D) fp32: device tensor, or numpy for numpy callers
    kc: object  # (B, H, N_K, D)
    vc: object
    s_coarse: object  # (B, H, N_Q, N_K) float64
    block_size: int
    scale_applied: bool = True

    @property
    def num_query_blocks(self) -> int:
        return int(self.qc.shape[2])

    @property
    def num_key_blocks(self) -> int:
        return int(self.kc.shape[2])

    def summary(self) -> dict:
        s = self.s_coarse
        return {"query_blocks": self.num_query_blocks, "key_blocks": self.num_key_blocks,
                "score_min": float(s.min()), "score_max": float(s.max()), "score_mean": float(s.mean())}


def _dev(x) -> torch.Tensor:
    """A CoarseSet field on the device (numpy fields are uploaded)."""
    if isinstance(x, np.ndarray):
        if not torch.cuda.is_available():
            raise LayoutError("the routing kernels run on a CUDA device and none is available (there is no CPU path)")
        return torch.from_numpy(np.ascontiguousarray(x)).cuda()
    return x


def _like(t: torch.Tensor, numpy_io: bool):
    return t.cpu().numpy() if numpy_io else t


def _device_tensor(x, name):
    if isinstance(x, np.ndarray):
        x = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32))
    if not isinstance(x, torch.Tensor) or x.dim() != 4:
        raise LayoutError(f"{name}: expected a 4-D (B,H,S,D) tensor or array")
    if not x.is_cuda:
        if not torch.cuda.is_available():
            raise LayoutError("the routing kernels run on a CUDA device and none is available (there is no CPU path)")
        x = x.cuda()
    if x.dtype not in (torch.bfloat16, torch.float32):
        x = x.float()
    return x.contiguous()


def _block_means(x: torch.Tensor, layout: BlockLayout) -> torch.Tensor:
    """block_mean (tensor.py:96-119): fp64 sums over each block's valid rows -> fp32, on the pool kernel."""
    B, H, S, D = x.shape
    if layout.seq_len != S:
        raise LayoutError(f"layout covers {layout.seq_len} rows, tensor has {S}")
    if layout.block_size != 64:
        raise ConfigError(f"block_size={layout.block_size} is not supported by the sm_100a kernels (only 64)")
    if D not in (64, 128):
        raise ConfigError(f"head dim {D} not supported by the pooling kernel (64 or 128)")
    T = layout.num_blocks
    means = torch.empty((3, B, H, T, D), dtype=torch.float32, device=x.device)
    err = torch.zeros(1, dtype=torch.int32, device=x.device)
    dt = N.ISA_DTYPE_BF16 if x.dtype == torch.bfloat16 else N.ISA_DTYPE_F32
    sh = N.IsaShape(B, H, S, D, S, 0, 64, dt, x.stride(0), x.stride(1), x.stride(2))
    N.check(N.load().isa_pool_means(ctypes.byref(sh), x.data_ptr(), x.data_ptr(), x.data_ptr(), means.data_ptr(),
                                    err.data_ptr(), torch.cuda.current_stream(x.device).cuda_stream))
    if int(err.item()) & N.ERRBIT_INPUT:  # ensure_tensor4's finiteness check (tensor.py:34-35)
        raise InputError("block_mean input: non-finite elements")
    return means[0]


def block_mean(x, layout: BlockLayout):
    """Per-block mean over each block's valid rows with fp64 accumulation
    (tensor.py:96-119) on the pooling kernel. `x` may hold layout.seq_len or
    layout.padded_len rows (padded rows never contribute). numpy in -> numpy
    float32 out; torch in -> fp32 device tensor."""
    numpy_io = isinstance(x, np.ndarray)
    t = _device_tensor(x, "block_mean input")
    if t.shape[2] not in (layout.seq_len, layout.padded_len):
        raise LayoutError(f"block_mean: seq length {t.shape[2]} matches neither layout.seq_len "
                          f"{layout.seq_len} nor padded_len {layout.padded_len}")
    if t.shape[2] != layout.seq_len:
        t = t[:, :, :layout.seq_len].contiguous()
    out = _block_means(t, layout)
    return out.cpu().numpy() if numpy_io else out


def build_coarse(q, k, v, q_layout: BlockLayout, k_layout: BlockLayout, scale: Optional[float] = None) -> CoarseSet:
    """Block means of Q (over q_layout) and K, V (over k_layout) and
    s_coarse = scale * qc . kc^T in float64 (coarse.py:110-127)."""
    if q_layout.block_size != k_layout.block_size:
        raise LayoutError("query and key layouts must share one block size")
    numpy_io = isinstance(q, np.ndarray)
    q, k, v = _device_tensor(q, "Q"), _device_tensor(k, "K"), _device_tensor(v, "V")
    if scale is None:
        scale = 1.0 / math.sqrt(q.shape[3])
    qc, kc, vc = _block_means(q, q_layout), _block_means(k, k_layout), _block_means(v, k_layout)
    B, H, t_q, D = qc.shape
    t_k = kc.shape[2]
    if kc.shape[:2] != (B, H):
        raise LayoutError(f"Q/K batch-head mismatch: {tuple(qc.shape)} vs {tuple(kc.shape)}")
    s = torch.empty((B, H, t_q, t_k), dtype=torch.float64, device=q.device)
    N.check(N.load().isa_coarse_scores(B * H, t_q, t_k, D, float(scale), qc.data_ptr(), kc.data_ptr(), s.data_ptr(),
                                       torch.cuda.current_stream(q.device).cuda_stream))
    return CoarseSet(qc=_like(qc, numpy_io), kc=_like(kc, numpy_io), vc=_like(vc, numpy_io),
                     s_coarse=_like(s, numpy_io), block_size=q_layout.block_size)


def _topk_rows(scores, k: int, method: int):
    """Top-k per row, ties to the lower index, ascending (coarse.py:130-136)."""
    numpy_io = isinstance(scores, np.ndarray)
    scores = _dev(scores)
    lead = tuple(scores.shape[:-1])
    n = int(scores.shape[-1])
    rows = int(np.prod(lead)) if lead else 1
    out = torch.empty(lead + (k,), dtype=torch.int64, device=scores.device)
    if k == 0 or rows == 0:
        return _like(out, numpy_io)
    s = scores.reshape(rows, n).contiguous().double()
    N.check(N.load().isa_topk_rows_f64(s.data_ptr(), rows, n, k, out.data_ptr(), method,
                                       torch.cuda.current_stream(s.device).cuda_stream))
    return _like(out, numpy_io)


def rank_context(cs: CoarseSet, icl: IclLayout, alpha_s: float) -> SelectionIndex:
    """Top floor(alpha_s * T_ctx) context blocks by their mean coarse score over
    the source query blocks (coarse.py:139-157)."""
    if not 0.0 <= alpha_s <= 1.0:
        raise ConfigError(f"alpha_s must be in [0, 1], got {alpha_s}")
    icl = icl_from_any(icl)
    b = cs.block_size
    n_src = -(-icl.l_src // b)
    n_ctx = -(-icl.l_ctx // b) if icl.l_ctx else 0
    if n_src + n_ctx != cs.num_key_blocks or n_src > cs.num_query_blocks:
        raise LayoutError(f"icl layout ({icl.l_src}, {icl.l_ctx}) inconsistent with coarse blocks "
                          f"({cs.num_query_blocks} x {cs.num_key_blocks}, b={b})")
    numpy_io = isinstance(cs.s_coarse, np.ndarray)
    B, H = cs.s_coarse.shape[:2]
    if n_ctx == 0:
        return SelectionIndex(np.zeros((B, H, 0), dtype=np.int64) if numpy_io else
                              torch.zeros((B, H, 0), dtype=torch.int64, device=cs.s_coarse.device), 0)
    s = _dev(cs.s_coarse).double().contiguous()
    t_q, t_k = s.shape[2], s.shape[3]
    ctx_scores = torch.empty((B, H, n_ctx), dtype=torch.float64, device=s.device)
    # the mean over source query blocks in numpy's summation order (ctx_mean_kernel)
    N.check(N.load().isa_ctx_saliency_f64(s.data_ptr(), B * H, t_q * t_k, t_k, n_src, n_ctx, ctx_scores.data_ptr(),
                                          torch.cuda.current_stream(s.device).cuda_stream))
    idx = _topk_rows(ctx_scores, int(math.floor(alpha_s * n_ctx)), 0)
    return SelectionIndex(_like(idx, numpy_io), n_ctx)


def build_block_mask(cs: CoarseSet, alpha_ns: float) -> BlockMask:
    """Top k = min(N_K, max(1, floor(alpha_ns * N_K))) key blocks per query block (coarse.py:160-170)."""
    if not 0.0 < alpha_ns <= 1.0:
        raise ConfigError(f"alpha_ns must be in (0, 1], got {alpha_ns}")
    n_k = cs.num_key_blocks
    k = min(n_k, max(1, int(math.floor(alpha_ns * n_k))))
    return BlockMask(_topk_rows(cs.s_coarse, k, 1), n_k)


def sharpness_split(cs: CoarseSet, icl: IclLayout, alpha_f: float, softmax_first: bool = True) -> SharpnessSplit:
    """Variance of the (softmaxed) coarse scores over the source key blocks per
    query block; the floor(alpha_f * T_q) least sharp go flat, ties keep the
    lower index sharp (coarse.py:173-201)."""
    if not 0.0 <= alpha_f <= 1.0:
        raise ConfigError(f"alpha_f must be in [0, 1], got {alpha_f}")
    icl = icl_from_any(icl)
    b = cs.block_size
    n_src = -(-icl.l_src // b)
    if n_src < 1 or n_src > cs.num_key_blocks:
        raise LayoutError(f"source block count {n_src} out of range for coarse set")
    numpy_io = isinstance(cs.s_coarse, np.ndarray)
    s_coarse = _dev(cs.s_coarse).double()
    B, H, T_q, _ = s_coarse.shape
    dev = s_coarse.device
    st = torch.cuda.current_stream(dev).cuda_stream
    lib = N.load()
    src = s_coarse[:, :, :, :n_src].reshape(B * H * T_q, n_src).contiguous()
    m = torch.empty((B, H, T_q), dtype=torch.float64, device=dev)
    N.check(lib.isa_sharpness_rows_f64(src.data_ptr(), B * H * T_q, n_src, int(bool(softmax_first)), m.data_ptr(), st))
    n_flat = int(math.floor(alpha_f * T_q))
    sharp = torch.empty((B, H, T_q - n_flat), dtype=torch.int64, device=dev)
    flat = torch.empty((B, H, n_flat), dtype=torch.int64, device=dev)
    N.check(lib.isa_split_rows_f64(m.data_ptr(), B * H, T_q, n_flat, sharp.data_ptr(), flat.data_ptr(), st))
    return SharpnessSplit(sharp=_like(sharp, numpy_io), flat=_like(flat, numpy_io), sharpness=_like(m, numpy_io))
