"""DiT attention stack around the ISA operator (BASELINE.json configs[4],
SURVEY.md §8f rank 1: the 40-layer LIVEditor-14B-shaped attention stack).

Each layer is the attention half of a DiT block, x -> x + Attn(x):

    qkv = x @ W_qkv                       (B, S, 3E)   cuBLAS bf16 GEMM
    o   = isa_forward(q, k, v, rope_base)  decoupled RoPE of q/k (pipeline.py:
           469-490; positions restart at 0 for the context segment) fused into
           the ISA pooling pass, ISA attention (pipeline.py:307-316) on strided
           (B, H, S, D) views of the qkv buffer, written straight into the
           (B, S, H*D) activation layout (no transposes)
    x   = x + o @ W_o                     cuBLAS bf16 GEMM

E = H * D (Wan / LIVEditor-14B: H = 40, D = 128, E = 5120). Source tokens come
first, then context tokens; ragged segments (e.g. 50,000 + 50,000) run with
cfg.strict = False. Norms and MLPs of the DiT block are outside the ISA path
and are not modelled. Weights are random-init (no checkpoints offline).

Head-sharded across P GPUs (one process per GPU, `world`/`rank`): rank r owns
heads head_shard(H, r, P) (round-robin, parallel.py). The QKV projection is
column-parallel (each rank computes only its heads' q/k/v from the replicated
activations), the ISA layer runs on the local heads, and the output projection
is row-parallel: each rank multiplies its heads' outputs by their rows of W_o
and one all-reduce (sum) over NVLink forms x + o @ W_o on every rank. The
GEMM and the all-reduce run in sequence chunks so chunk c's all-reduce
overlaps chunk c+1's GEMM. Every stage of the ISA layer is per head
(reference.py:159-160, taylor.py:176-177), so the only exchange is that sum.
"""

from __future__ import annotations

import math
from typing import Callable, Optional

import torch

from . import pipeline as _P
from .parallel import head_shard
from .types import IclLayout, IsaConfig, icl_from_any

__all__ = ["DiTAttentionLayer", "DiTAttentionStack"]


class DiTAttentionLayer:
    """One attention layer: QKV projection, decoupled RoPE, ISA (or dense)
    attention, output projection with residual add. world > 1: this rank's
    head shard (column-parallel QKV, row-parallel O + all-reduce)."""

    def __init__(self, heads: int = 40, head_dim: int = 128, device="cuda", dtype=torch.bfloat16,
                 generator: Optional[torch.Generator] = None, rope_base: float = 10000.0, world: int = 1,
                 rank: int = 0, group=None, reduce_chunks: int = 4):
        self.H, self.D = heads, head_dim
        self.E = heads * head_dim
        self.rope_base = rope_base
        self.world, self.rank, self.group = world, rank, group
        self.reduce_chunks = max(1, reduce_chunks)
        std = 1.0 / math.sqrt(self.E)
        # full weights drawn identically on every rank (same generator seed), then sliced
        w_qkv = (torch.randn(self.E, 3 * self.E, device=device, generator=generator) * std).to(dtype)
        w_o = (torch.randn(self.E, self.E, device=device, generator=generator) * std).to(dtype)
        self.heads = head_shard(heads, rank, world)
        self.Hl = len(self.heads)
        if world == 1:
            self.w_qkv, self.w_o = w_qkv, w_o
        else:
            idx = torch.tensor(self.heads, device=device)
            cols = (torch.arange(3, device=device)[:, None, None] * self.E + idx[None, :, None] * head_dim
                    + torch.arange(head_dim, device=device)[None, None, :]).reshape(-1)
            self.w_qkv = w_qkv.index_select(1, cols).contiguous()          # (E, 3 * Hl * D)
            rows = (idx[:, None] * head_dim + torch.arange(head_dim, device=device)[None, :]).reshape(-1)
            self.w_o = w_o.index_select(0, rows).contiguous()              # (Hl * D, E)

    def attention_inputs(self, x: torch.Tensor):
        """qkv projection of this rank's heads: (B, S, 3, Hl, D)."""
        B, S, E = x.shape
        return (x.reshape(B * S, E) @ self.w_qkv).view(B, S, 3, self.Hl, self.D)

    def __call__(self, x: torch.Tensor, icl: IclLayout, cfg: IsaConfig, attention: str = "isa",
                 timings: Optional[dict] = None,
                 attend: Optional[Callable[[torch.Tensor, torch.Tensor, torch.Tensor, torch.Tensor], None]] = None
                 ) -> torch.Tensor:
        icl = icl_from_any(icl) if icl is not None else None
        B, S, E = x.shape
        H, D, Hl = self.H, self.D, self.Hl
        cuda = x.is_cuda
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)] if (timings is not None and cuda) else None
        rec = (lambda i: ev[i].record()) if ev else (lambda i: None)
        rec(0)
        qkv = self.attention_inputs(x)
        rec(1)
        q, k, v = (qkv[:, :, i].permute(0, 2, 1, 3) for i in range(3))  # strided (B, Hl, S, D) views
        o = torch.empty((B, S, Hl, D), dtype=x.dtype, device=x.device)
        if attend is not None:  # injected per-head attention (CPU tests of the sharding)
            attend(q, k, v, o.permute(0, 2, 1, 3))
        elif attention == "isa":
            _P.isa_forward(q, k, v, icl, cfg, collect_trace=False, out=o.permute(0, 2, 1, 3), validate=False,
                           rope_base=self.rope_base)
        elif attention == "dense":
            qr, kr = (_P.apply_decoupled_rope(t, icl, self.rope_base) for t in (q, k))
            o.copy_(_P.dense_attention(qr.contiguous(), kr.contiguous(), v.contiguous()).permute(0, 2, 1, 3))
        else:
            raise ValueError(f"attention must be 'isa' or 'dense', got {attention!r}")
        rec(2)
        y = self._project(x, o.view(B * S, Hl * D)).view(B, S, E)
        rec(3)
        if ev:
            torch.cuda.synchronize()
            for name, a, b in (("qkv_gemm", 0, 1), ("attention_with_rope", 1, 2), ("out_gemm_allreduce", 2, 3)):
                timings[name] = timings.get(name, 0.0) + ev[a].elapsed_time(ev[b])
        return y

    def _project(self, x: torch.Tensor, o: torch.Tensor) -> torch.Tensor:
        """x + o @ W_o: one fused addmm on one GPU; row-parallel partial sums +
        chunked all-reduce when sharded."""
        B, S, E = x.shape
        xf = x.reshape(B * S, E)
        if self.world == 1:
            return torch.addmm(xf, o, self.w_o)
        import torch.distributed as dist

        y = torch.empty_like(xf)
        n = B * S
        step = -(-n // self.reduce_chunks)
        works = []
        for lo in range(0, n, step):
            hi = min(lo + step, n)
            torch.mm(o[lo:hi], self.w_o, out=y[lo:hi])  # this rank's heads' share of the projection
            works.append(dist.all_reduce(y[lo:hi], group=self.group, async_op=True))  # under the next chunk's GEMM
        for w in works:
            w.wait()
        return y.add_(xf)


class DiTAttentionStack:
    """`layers` DiTAttentionLayer applied in sequence (x_{l+1} = x_l + Attn_l(x_l))."""

    def __init__(self, layers: int = 40, heads: int = 40, head_dim: int = 128, device="cuda",
                 dtype=torch.bfloat16, seed: int = 0, world: int = 1, rank: int = 0, group=None):
        g = torch.Generator(device=device).manual_seed(seed)
        self.layers = [DiTAttentionLayer(heads, head_dim, device, dtype, g, world=world, rank=rank, group=group)
                       for _ in range(layers)]

    def __call__(self, x, icl, cfg, attention: str = "isa", timings: Optional[dict] = None, attend=None):
        for layer in self.layers:
            x = layer(x, icl, cfg, attention, timings, attend)
        return x
