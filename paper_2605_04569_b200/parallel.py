"""Head-parallel ISA across the GPUs of one node.

Every ISA stage is per (batch, head) — coarse scores, selection, split, mask
and both attention branches (coarse.py:5-6; every reference loop
is `for bi: for hi:`, e.g. reference.py:159-160, taylor.py:176-177) — so heads
shard with no exchange during compute. Heads are assigned round-robin (rank r
owns heads r, r+P, r+2P, ...), so the c-th chunked all-gather (head c*P + r
from every rank r) lands as one contiguous [c*P, (c+1)*P) head slab of the
final (1, H, S, D) output: no permute copy. The only collective is the NCCL
all-gather over NVLink that reassembles the output; chunk c's all-gather runs
on a side stream while chunk c+1 computes.
"""

from __future__ import annotations

from typing import List, Optional

import torch
import torch.distributed as dist


def head_shard(num_heads: int, rank: int, world: int) -> List[int]:
    """Round-robin head ownership: rank r owns r, r+P, r+2P, ..."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} / world {world}")
    return list(range(rank, num_heads, world))


def local_heads(x: torch.Tensor, rank: int, world: int) -> torch.Tensor:
    """This rank's heads of a full (B, H, S, D) tensor (a strided view)."""
    return x[:, rank::world]


def gather_heads(out_local: torch.Tensor, out_full: torch.Tensor, world: int, group=None,
                 chunks: Optional[List[int]] = None) -> None:
    """All-gather head shards into out_full (B, H, S, D) (round-robin layout).

    B == 1 with H % P == 0: one all_gather_into_tensor per local head chunk c
    straight into the contiguous slab out_full[0, c*P:(c+1)*P] (viewed as the
    concatenation (P*S, D), which NCCL and gloo both accept, so the CPU gloo
    tests run this exact path). Otherwise a generic all_gather of shards
    padded to ceil(H/P) heads and a strided scatter (uneven head counts, B > 1)."""
    B, Hl, S, D = out_local.shape
    H = out_full.shape[1]
    if B == 1 and out_full.is_contiguous() and H % world == 0:
        for c in (chunks if chunks is not None else range(Hl)):
            dist.all_gather_into_tensor(out_full[0, c * world:(c + 1) * world].view(world * S, D),
                                        out_local[0, c].contiguous(), group=group)
        return
    h_max = -(-H // world)
    send = out_local
    if Hl < h_max:
        send = torch.cat([out_local, out_local.new_zeros(B, h_max - Hl, S, D)], dim=1)
    parts = [torch.empty_like(send) for _ in range(world)]
    dist.all_gather(parts, send.contiguous(), group=group)
    for r in range(world):
        n_r = len(range(r, H, world))
        out_full[:, r::world] = parts[r][:, :n_r]


def isa_forward_sharded(prepared, out_full: torch.Tensor, my_heads: List[int], world: int, group=None,
                        comm_stream: Optional[torch.cuda.Stream] = None) -> torch.Tensor:
    """One ISA layer over this rank's heads (a `pipeline.prepare()`d call on the
    local (1, H/P, S, D) inputs), then the head all-gather into `out_full`.

    The gather is issued on `comm_stream` (created on demand) after an event on
    the compute stream, so NCCL traffic overlaps whatever the caller enqueues
    next; the function returns after enqueuing and makes the compute stream
    wait for the gather."""
    out_local = prepared()
    if world == 1:
        out_full.copy_(out_local)
        return out_full
    compute = torch.cuda.current_stream()
    comm = comm_stream or _comm_stream(out_local.device)
    ev = torch.cuda.Event()
    ev.record(compute)
    comm.wait_event(ev)
    with torch.cuda.stream(comm):
        gather_heads(out_local, out_full, world, group)
    compute.wait_stream(comm)
    return out_full


_COMM = {}


def _comm_stream(device) -> torch.cuda.Stream:
    key = str(device)
    if key not in _COMM:
        _COMM[key] = torch.cuda.Stream(device=device)
    return _COMM[key]
