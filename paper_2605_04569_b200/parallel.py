"""Head-parallel ISA across the GPUs of one node.

Every ISA stage is per (batch, head) — coarse scores, selection, split, mask
and both attention branches (coarse.py:5-6; every reference loop
is `for bi: for hi:`, e.g. reference.py:159-160, taylor.py:176-177) — so heads
shard with no exchange during compute. Heads are assigned round-robin (rank r
owns heads r, r+P, r+2P, ...), so the all-gather of local head c (head c*P + r
from every rank r) lands as one contiguous [c*P, (c+1)*P) head slab of the
final (1, H, S, D) output: no permute copy. The only collective is that NCCL
all-gather over NVLink, which reassembles the output.

`ShardedIsa` overlaps it with compute in one of two schedules:

* "signal" (default on CUDA): ONE fused call computes all local heads (no
  loss of grid efficiency) and publishes per-head completion counters from
  inside the attention grid (`isa_forward_signal`: every CTA adds 1 to its
  head's counter after its output rows are final). The communication stream
  waits on each head's counter (`cuStreamWaitValue32`, GEQ on a monotonically
  growing target) and all-gathers that head's slab while later heads still
  compute: compute-to-collective overlap at head granularity.
* "chunks": the local heads are cut into chunks, each a separate prepared
  call on one of two alternating compute streams, chunk c's all-gathers
  running on the comm stream while chunk c+1 computes (measured on one B200:
  per-head chunks cost 16% of compute at 5 heads per rank, hence "signal").

The same schedule code drives the CPU (gloo) tests through a stream adapter
whose "streams" execute inline.
"""

from __future__ import annotations

from typing import Callable, List, Optional

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


def chunk_ranges(n_local: int, chunk_heads: int) -> List[range]:
    """Local head index ranges of the compute/gather chunks."""
    if chunk_heads < 1:
        raise ValueError("chunk_heads must be >= 1")
    return [range(c, min(c + chunk_heads, n_local)) for c in range(0, n_local, chunk_heads)]


def gather_slab(out_chunk: torch.Tensor, first_local: int, out_full: torch.Tensor, world: int, group=None) -> None:
    """All-gather the local heads of one chunk (out_chunk (1, m, S, D), local
    heads first_local .. first_local + m - 1) into out_full: local head c of
    every rank is the contiguous slab out_full[0, c*P:(c+1)*P], viewed as
    (P*S, D) — NCCL and gloo both take it, so the CPU tests run this path."""
    S, D = out_chunk.shape[2], out_chunk.shape[3]
    for j in range(out_chunk.shape[1]):
        c = first_local + j
        dist.all_gather_into_tensor(out_full[0, c * world:(c + 1) * world].view(world * S, D),
                                    out_chunk[0, j].contiguous().view(S, D), group=group)


def gather_heads(out_local: torch.Tensor, out_full: torch.Tensor, world: int, group=None,
                 chunks: Optional[List[int]] = None) -> None:
    """All-gather head shards into out_full (B, H, S, D) (round-robin layout).

    B == 1 with H % P == 0 and a contiguous out_full: per-local-head slabs
    (gather_slab). Otherwise a generic all_gather of shards padded to
    ceil(H/P) heads and a strided scatter (uneven head counts, B > 1)."""
    B, Hl, S, D = out_local.shape
    H = out_full.shape[1]
    if B == 1 and out_full.is_contiguous() and H % world == 0:
        for c in (chunks if chunks is not None else range(Hl)):
            gather_slab(out_local[:, c:c + 1], c, out_full, world, group)
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


# ---------------------------------------------------------------- stream adapters
class CudaStreams:
    """Two compute streams (alternating per chunk) and one comm stream, joined
    with the caller's current stream at the start and end of a step."""

    def __init__(self, device):
        self.device = torch.device(device)
        self.compute = [torch.cuda.Stream(self.device), torch.cuda.Stream(self.device)]
        self.comm = torch.cuda.Stream(self.device)

    def begin(self):
        self.main = torch.cuda.current_stream(self.device)
        ev = torch.cuda.Event()
        ev.record(self.main)
        for s in (*self.compute, self.comm):
            s.wait_event(ev)

    def run(self, i: int, fn: Callable[[], None]):
        s = self.compute[i % 2]
        with torch.cuda.stream(s):
            fn()
        ev = torch.cuda.Event()
        ev.record(s)
        return ev

    def after(self, ev, fn: Callable[[], None]) -> None:
        self.comm.wait_event(ev)
        with torch.cuda.stream(self.comm):
            fn()

    def after_head(self, prep, bh: int, fn: Callable[[], None]) -> None:
        """Comm-stream work once head bh of the signalling call is final."""
        prep.wait_head(self.comm, bh)
        with torch.cuda.stream(self.comm):
            fn()

    def end(self):
        for s in (*self.compute, self.comm):
            self.main.wait_stream(s)


class InlineStreams:
    """CPU stand-in: every 'stream' executes inline, in issue order (gloo tests)."""

    def begin(self):
        pass

    def run(self, i: int, fn):
        fn()
        return None

    def after(self, ev, fn):
        fn()

    def after_head(self, prep, bh, fn):
        fn()

    def end(self):
        pass


# ---------------------------------------------------------------- the sharded layer
class ShardedIsa:
    """One ISA layer over this rank's heads with the output all-gather
    overlapped with compute ("signal" or "chunks" schedule, module docstring).

    q/k/v: this rank's (1, H/P, S, D) inputs (heads head_shard(H, rank, P)).
    `compute(lo, hi)` (optional) replaces the prepared ISA call for local
    heads [lo, hi) and returns their (1, hi-lo, S, D) output — the CPU tests
    use it; on CUDA each call is a `pipeline.prepare()`d call.
    """

    def __init__(self, q, k, v, icl, cfg, world: int, group=None, chunk_heads: int = 1,
                 compute: Optional[Callable[[int, int], torch.Tensor]] = None, streams=None,
                 mode: str = "signal"):
        if mode not in ("signal", "chunks"):
            raise ValueError("mode must be 'signal' or 'chunks'")
        self.world, self.group, self.mode = world, group, mode
        self.shape = tuple(q.shape)
        if self.shape[0] != 1:
            raise ValueError("ShardedIsa takes B = 1 (the head-sharded north-star layout)")
        n_local = self.shape[1]
        self.chunks = [range(0, n_local)] if mode == "signal" else chunk_ranges(n_local, chunk_heads)
        self._preps = [None] * len(self.chunks)
        if compute is None:
            from .pipeline import prepare

            self._preps = [prepare(q[:, r.start:r.stop], k[:, r.start:r.stop], v[:, r.start:r.stop], icl, cfg,
                                   signal=(mode == "signal")) for r in self.chunks]
            self._calls = [p.__call__ for p in self._preps]
            self._outs = [p.out for p in self._preps]
        else:
            self._outs = [None] * len(self.chunks)

            def host_call(i, r):
                def call():
                    self._outs[i] = compute(r.start, r.stop)
                return call

            self._calls = [host_call(i, r) for i, r in enumerate(self.chunks)]
        self.streams = streams or (CudaStreams(q.device) if q.is_cuda else InlineStreams())

    def _move(self, i: int, r: range, j: Optional[int], out_full: torch.Tensor):
        """Comm-stream work for chunk i (all its heads, or only local head j of it)."""
        lo, hi = (r.start, r.stop) if j is None else (j, j + 1)
        src = self._outs[i][:, lo - r.start:hi - r.start]
        if self.world > 1:
            gather_slab(src, lo, out_full, self.world, self.group)
        else:
            out_full[:, lo:hi].copy_(src)

    def __call__(self, out_full: torch.Tensor, gather: bool = True) -> torch.Tensor:
        """Compute every local head and (gather=True) all-gather the outputs
        into out_full (1, H, S, D), overlapped with the remaining compute.
        gather=False runs the compute alone (scaling without the collective).
        Returns out_full; the caller's stream is ordered after all of it."""
        n_local = self.shape[1]
        if tuple(out_full.shape[2:]) != self.shape[2:] or out_full.shape[1] != n_local * self.world:
            raise ValueError(f"out_full {tuple(out_full.shape)} must be (1, {n_local * self.world}, S, D): "
                             "the slab gather needs H divisible by the world size")
        st = self.streams
        st.begin()
        for i, r in enumerate(self.chunks):
            ev = st.run(i, self._calls[i])
            if not gather:
                continue
            if self.mode == "signal":
                for j in r:  # head j's slab as soon as head j is final
                    st.after_head(self._preps[i], j, lambda i=i, r=r, j=j: self._move(i, r, j, out_full))
            else:
                st.after(ev, lambda i=i, r=r: self._move(i, r, None, out_full))
        st.end()
        return out_full

    def local_output(self) -> List[torch.Tensor]:
        """This rank's local head outputs, one (1, 1, S, D) tensor per local head."""
        return [o[:, j:j + 1] for o in self._outs for j in range(o.shape[1])]


def isa_forward_sharded(q, k, v, icl, cfg, out_full: torch.Tensor, world: int, group=None,
                        mode: str = "signal", chunk_heads: int = 1) -> torch.Tensor:
    """One-shot convenience: ShardedIsa over this rank's (1, H/P, S, D) heads."""
    return ShardedIsa(q, k, v, icl, cfg, world, group, chunk_heads, mode=mode)(out_full)
