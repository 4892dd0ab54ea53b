"""DiT attention stack around the ISA operator (BASELINE.json configs[4],
SURVEY.md §8f rank 1: the 40-layer LIVEditor-14B-shaped attention stack).

Each layer is the attention half of a DiT block, x -> x + Attn(x):

    qkv = x @ W_qkv                       (B, S, 3E)   cuBLAS bf16 GEMM
    q, k = decoupled RoPE of the q/k heads (pipeline.py:469-490; positions
           restart at 0 for the context segment), written straight into
           (B, S, H, D) buffers
    o    = isa_forward(q, k, v)          (pipeline.py:307-316) on strided
           (B, H, S, D) views of those buffers, written straight into the
           (B, S, H*D) activation layout (no transposes)
    x    = x + o @ W_o                    cuBLAS bf16 GEMM

E = H * D (Wan / LIVEditor-14B: H = 40, D = 128, E = 5120). Source tokens come
first, then context tokens; ragged segments (e.g. 50,000 + 50,000) run with
cfg.strict = False. Norms and MLPs of the DiT block are outside the ISA path
and are not modelled. Weights are random-init (no checkpoints offline).
"""

from __future__ import annotations

import math
from typing import Optional

import torch

from . import pipeline as _P
from .types import IclLayout, IsaConfig, icl_from_any

__all__ = ["DiTAttentionLayer", "DiTAttentionStack"]


class DiTAttentionLayer:
    """One attention layer: QKV projection, decoupled RoPE, ISA (or dense)
    attention, output projection with residual add."""

    def __init__(self, heads: int = 40, head_dim: int = 128, device="cuda", dtype=torch.bfloat16,
                 generator: Optional[torch.Generator] = None, rope_base: float = 10000.0):
        self.H, self.D = heads, head_dim
        self.E = heads * head_dim
        self.rope_base = rope_base
        std = 1.0 / math.sqrt(self.E)
        self.w_qkv = (torch.randn(self.E, 3 * self.E, device=device, generator=generator) * std).to(dtype)
        self.w_o = (torch.randn(self.E, self.E, device=device, generator=generator) * std).to(dtype)

    def __call__(self, x: torch.Tensor, icl: IclLayout, cfg: IsaConfig, attention: str = "isa",
                 timings: Optional[dict] = None) -> torch.Tensor:
        icl = icl_from_any(icl)
        B, S, E = x.shape
        H, D = self.H, self.D
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)] if timings is not None else None
        rec = (lambda i: ev[i].record()) if ev else (lambda i: None)
        rec(0)
        qkv = (x.view(B * S, E) @ self.w_qkv).view(B, S, 3, H, D)
        rec(1)
        q_rot = torch.empty((B, S, H, D), dtype=x.dtype, device=x.device)
        k_rot = torch.empty_like(q_rot)
        for src, dst in ((qkv[:, :, 0], q_rot), (qkv[:, :, 1], k_rot)):
            _P.apply_decoupled_rope(src.permute(0, 2, 1, 3), icl, self.rope_base, out=dst.permute(0, 2, 1, 3))
        rec(2)
        q, k = q_rot.permute(0, 2, 1, 3), k_rot.permute(0, 2, 1, 3)
        v = qkv[:, :, 2].permute(0, 2, 1, 3)
        o = torch.empty((B, S, H, D), dtype=x.dtype, device=x.device)
        if attention == "isa":
            _P.isa_forward(q, k, v, icl, cfg, collect_trace=False, out=o.permute(0, 2, 1, 3), validate=False)
        elif attention == "dense":
            o.copy_(_P.dense_attention(q.contiguous(), k.contiguous(), v.contiguous()).permute(0, 2, 1, 3))
        else:
            raise ValueError(f"attention must be 'isa' or 'dense', got {attention!r}")
        rec(3)
        y = torch.addmm(x.view(B * S, E), o.view(B * S, E), self.w_o).view(B, S, E)
        rec(4)
        if ev:
            torch.cuda.synchronize()
            for name, a, b in (("qkv_gemm", 0, 1), ("rope", 1, 2), ("attention", 2, 3), ("out_gemm", 3, 4)):
                timings[name] = timings.get(name, 0.0) + ev[a].elapsed_time(ev[b])
        return y


class DiTAttentionStack:
    """`layers` DiTAttentionLayer applied in sequence (x_{l+1} = x_l + Attn_l(x_l))."""

    def __init__(self, layers: int = 40, heads: int = 40, head_dim: int = 128, device="cuda",
                 dtype=torch.bfloat16, seed: int = 0):
        g = torch.Generator(device=device).manual_seed(seed)
        self.layers = [DiTAttentionLayer(heads, head_dim, device, dtype, g) for _ in range(layers)]

    def __call__(self, x, icl, cfg, attention: str = "isa", timings: Optional[dict] = None):
        for layer in self.layers:
            x = layer(x, icl, cfg, attention, timings)
        return x
