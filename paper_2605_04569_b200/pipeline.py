"""The ISA forward operator on B200 — drop-in for the reference pipeline API.

Public functions keep the reference signatures (pkg/src/isattn/pipeline.py):

    isa_forward(q, k, v, icl, cfg, collect_trace=True) -> (out, IsaTrace | None)   :307-316
    isa_routing(q, k, v, icl, cfg) -> IsaRouting                                   :302-304
    isa_forward_with_routing(q, k, v, icl, cfg, routing) -> out                    :319-328

plus `dense_attention` (the full_attention oracle / dense baseline,
reference.py:79-123) on the same sm_100a kernel.

Inputs may be torch CUDA tensors (bf16 or fp32; any B/H/S strides with a
contiguous D axis), or HOST data: numpy arrays (cast to float32 like the
reference, result returned as a numpy float32 array) or CPU torch tensors
(bf16/fp32; result returned as a CPU tensor of the input dtype). Host data is
streamed through the GPU head-chunk by head-chunk by the native
`isa_forward_host` (H2D of chunk c+1 and D2H of chunk c-1 overlap the device
pipeline of chunk c; pass page-locked tensors for the overlap). All compute
runs in libisa_b200.so; there is no CPU path.
"""

from __future__ import annotations

import ctypes
import dataclasses
import math
from typing import Optional

import numpy as np
import torch

from . import _native as N
from .errors import BlockIndexError, ConfigError, ContractError, DegenerateRowError, InputError, LayoutError
from .types import (
    BlockMask,
    GradBundle,
    IclLayout,
    IsaConfig,
    IsaDims,
    IsaRouting,
    IsaTrace,
    SelectionIndex,
    SharpnessSplit,
    SUPPORTED_HEAD_DIMS,
    _LazyStageTimes,
    cfg_from_any,
    icl_from_any,
)

__all__ = ["isa_forward", "isa_routing", "isa_forward_with_routing", "isa_backward", "dense_attention", "prepare",
           "apply_decoupled_rope"]


def _ptr(t: Optional[torch.Tensor]) -> Optional[int]:
    return None if t is None else t.data_ptr()


class _Inputs:
    """Validated device views of q/k/v plus the ABI descriptors (pipeline.py:136-154)."""

    def __init__(self, q, k, v, icl, cfg):
        self.cfg = cfg_from_any(cfg).validate_b200()
        self.icl = icl_from_any(icl)
        self.numpy_io = isinstance(q, np.ndarray)
        self.host = all(isinstance(x, np.ndarray) or (isinstance(x, torch.Tensor) and not x.is_cuda)
                        for x in (q, k, v))
        if self.host:
            if not torch.cuda.is_available():
                raise LayoutError("host Q/K/V are streamed through a CUDA device and none is available "
                                  "(there is no CPU path)")
            q, k, v = (self._to_host(x, n) for x, n in ((q, "Q"), (k, "K"), (v, "V")))
            if q.dtype != k.dtype or q.dtype != v.dtype:
                q, k, v = q.float(), k.float(), v.float()
        else:
            q, k, v = (self._to_device(x, n) for x, n in ((q, "Q"), (k, "K"), (v, "V")))
        if not (q.shape == k.shape == v.shape):
            raise LayoutError(f"Q/K/V must share one shape, got {tuple(q.shape)}, {tuple(k.shape)}, {tuple(v.shape)}")
        if q.stride() != k.stride() or q.stride() != v.stride() or q.dtype != k.dtype or q.dtype != v.dtype:
            k, v = (x.contiguous() if x.stride() != q.stride() else x for x in (k, v))
            q = q.contiguous()
            k, v = k.contiguous().to(q.dtype), v.contiguous().to(q.dtype)
        if q.shape[2] != self.icl.total:
            raise LayoutError(f"sequence length {q.shape[2]} != icl total {self.icl.total}")
        b = self.cfg.block_size
        if self.cfg.strict and (self.icl.l_src % b or self.icl.l_ctx % b):
            raise ConfigError(
                f"strict mode requires L_src and L_ctx divisible by b={b}, got ({self.icl.l_src}, {self.icl.l_ctx})")
        if q.shape[3] not in SUPPORTED_HEAD_DIMS:
            raise ConfigError(f"head dim {q.shape[3]} not supported by the sm_100a kernels {SUPPORTED_HEAD_DIMS}")
        self.q, self.k, self.v = q, k, v
        self.dims = IsaDims.derive(q.shape, self.icl, self.cfg)
        d = self.dims
        self.shape = N.IsaShape(d.B, d.H, d.S, d.D, self.icl.l_src, self.icl.l_ctx, b,
                                N.ISA_DTYPE_BF16 if q.dtype == torch.bfloat16 else N.ISA_DTYPE_F32,
                                q.stride(0), q.stride(1), q.stride(2))
        self.knobs = N.IsaKnobs(d.scale, d.k_ctx, d.n_flat, max(d.k, 1), int(bool(self.cfg.softmax_first)), 0,
                                float(self.cfg.gamma), int(bool(self.cfg.residual_softmax)))

    @staticmethod
    def _to_host(x, name):
        """Host operand for the streamed path: contiguous (B,H,S,D), bf16 or fp32."""
        if isinstance(x, np.ndarray):
            x = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32))
        if x.dim() != 4:
            raise LayoutError(f"{name}: expected 4 axes (B,H,S,D), got shape {tuple(x.shape)}")
        if min(x.shape) < 1:
            raise LayoutError(f"{name}: all dims must be >= 1, got shape {tuple(x.shape)}")
        if x.dtype not in (torch.bfloat16, torch.float32):
            if not x.is_floating_point():
                raise InputError(f"{name}: floating-point input required")
            x = x.float()
        return x.contiguous()

    @staticmethod
    def _to_device(x, name):
        if isinstance(x, np.ndarray):
            if x.ndim != 4:
                raise LayoutError(f"{name}: expected 4 axes (B,H,S,D), got shape {x.shape}")
            x = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda()
        if not isinstance(x, torch.Tensor):
            raise LayoutError(f"{name}: expected a torch tensor or numpy array")
        if x.dim() != 4:
            raise LayoutError(f"{name}: expected 4 axes (B,H,S,D), got shape {tuple(x.shape)}")
        if min(x.shape) < 1:
            raise LayoutError(f"{name}: all dims must be >= 1, got shape {tuple(x.shape)}")
        if not x.is_cuda:
            raise LayoutError(f"{name}: Q, K and V must all be CUDA tensors or all host data (no CPU path)")
        if x.dtype not in (torch.bfloat16, torch.float32):
            if not x.is_floating_point():
                raise InputError(f"{name}: floating-point input required")
            x = x.float()
        if x.stride(3) != 1:
            x = x.contiguous()
        elem = x.element_size()
        if any((s * elem) % 16 for s in x.stride()[:3]) or x.data_ptr() % 16:
            x = x.contiguous()
        return x

    @property
    def device(self):
        return torch.device("cuda", torch.cuda.current_device()) if self.host else self.q.device

    def workspace(self):
        nbytes = ctypes.c_size_t(0)
        N.check(N.load().isa_workspace_bytes(ctypes.byref(self.shape), ctypes.byref(self.knobs), ctypes.byref(nbytes)))
        return torch.empty(int(nbytes.value), dtype=torch.uint8, device=self.q.device), int(nbytes.value)


def _routing_buffers(d: IsaDims, device):
    B, H = d.B, d.H
    i64 = dict(dtype=torch.int64, device=device)
    return {
        "selection": torch.empty((B, H, d.k_ctx), **i64),
        "sharp": torch.empty((B, H, d.n_sharp), **i64),
        "flat": torch.empty((B, H, d.n_flat), **i64),
        "mask": torch.empty((B, H, d.n_flat, d.k), **i64),
        "sharpness": torch.empty((B, H, d.T), dtype=torch.float64, device=device),
        "ctx_scores": torch.empty((B, H, d.t_ctx), dtype=torch.float64, device=device),
        "taylor_kernel": torch.empty((B, H), dtype=torch.int32, device=device),
    }


def _routing_struct(bufs) -> N.IsaRoutingOut:
    return N.IsaRoutingOut(*(_ptr(bufs[n]) if bufs[n].numel() else None
                             for n in ("selection", "sharp", "flat", "mask", "sharpness", "ctx_scores",
                                       "taylor_kernel")))


def _make_routing(d: IsaDims, bufs, numpy_io: bool = False) -> IsaRouting:
    """Routing value types over the exported buffers: device tensors, or numpy
    arrays for numpy callers (the reference's types hold numpy, coarse.py:52-107)."""
    cv = (lambda t: t.cpu().numpy()) if numpy_io else (lambda t: t)
    sel = SelectionIndex(cv(bufs["selection"]), d.t_ctx)
    split = SharpnessSplit(cv(bufs["sharp"]), cv(bufs["flat"]), cv(bufs["sharpness"]))
    mask = BlockMask(cv(bufs["mask"]), d.t_new) if d.n_flat else None
    return IsaRouting(selection=sel, split=split, mask=mask)


def _raise_flags(err: torch.Tensor):
    """Device error word (ISA_ERRBIT_*) -> the reference's exceptions. Pinned
    routing is checked in the reference's order: the selection gather
    (pipeline.py:189-192 via tensor.py:120-133), then the sharp/flat gathers,
    then the Taylor mask (taylor.py:80-84)."""
    flags = int(err.item())
    if flags & N.ERRBIT_INPUT:
        raise InputError("Q/K/V: non-finite elements")
    if flags & N.ERRBIT_SEL_RANGE:
        raise BlockIndexError("gather_blocks: pinned selection block index out of range [0, T_ctx)")
    if flags & N.ERRBIT_SEL_ORDER:
        raise ContractError("gather_blocks: pinned selection lists must be sorted ascending without duplicates")
    if flags & N.ERRBIT_SPLIT_RANGE:
        raise BlockIndexError("gather_blocks: pinned sharp/flat block index out of range [0, T)")
    if flags & N.ERRBIT_SPLIT_ORDER:
        raise ContractError("pinned sharp/flat lists must be sorted ascending without duplicates "
                            "and partition the query blocks")
    if flags & N.ERRBIT_MASK:
        raise ContractError("pinned mask indices out of range for the K_new blocks or not sorted ascending "
                            "without duplicates")
    if flags & N.ERRBIT_DEGENERATE:
        raise DegenerateRowError("row with empty key set: normalizer is zero")


class _LazySummary(dict):
    """coarse_summary of the reference trace (coarse.py:41-49), computed on access
    from the pooled means (torch fp64 on device; diagnostics only)."""

    def __init__(self, qc, kc, scale):
        super().__init__()
        self._args = (qc, kc, scale)

    def _resolve(self):
        if self._args is not None:
            qc, kc, scale = self._args
            self._args = None
            s = scale * torch.einsum("bhid,bhjd->bhij", qc.double(), kc.double())
            dict.update(self, {"query_blocks": int(qc.shape[2]), "key_blocks": int(kc.shape[2]),
                               "score_min": float(s.min()), "score_max": float(s.max()),
                               "score_mean": float(s.mean())})

    def items(self):
        self._resolve()
        return dict.items(self)

    def __getitem__(self, key):
        self._resolve()
        return dict.__getitem__(self, key)

    def __repr__(self):
        self._resolve()
        return dict.__repr__(self)


def _pinned_struct(routing, d: IsaDims, device):
    """IsaRouting (ours or the reference's numpy one) -> device int64 buffers."""
    def dev(x, shape):
        if x is None:
            return None
        t = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.asarray(x, dtype=np.int64))
        t = t.to(device=device, dtype=torch.int64).contiguous()
        if tuple(t.shape) != tuple(shape):
            raise LayoutError(f"pinned routing shape {tuple(t.shape)} != {tuple(shape)}")
        return t
    sel = dev(routing.selection.indices, (d.B, d.H, d.k_ctx))
    sharp = dev(routing.split.sharp, (d.B, d.H, d.n_sharp))
    flat = dev(routing.split.flat, (d.B, d.H, d.n_flat))
    mask = dev(routing.mask.indices, (d.B, d.H, d.n_flat, d.k)) if routing.mask is not None else None
    keep = (sel, sharp, flat, mask)
    return N.IsaRoutingIn(*(_ptr(t) if t is not None and t.numel() else None for t in keep)), keep


_SIDE_STREAMS: dict = {}


def _side_streams(dev):
    """Two long-lived copy streams per device for the host-streamed path."""
    key = dev.index
    if key not in _SIDE_STREAMS:
        _SIDE_STREAMS[key] = (torch.cuda.Stream(dev), torch.cuda.Stream(dev))
    return _SIDE_STREAMS[key]


def _run_host(inp: _Inputs, collect_trace: bool, pinned=None, out=None, validate=True, heads_per_chunk=0):
    """Host data in, host data out: native head-chunk streaming (isa_forward_host)."""
    lib = N.load()
    d = inp.dims
    dev = inp.device
    st_b, ws_b = ctypes.c_size_t(0), ctypes.c_size_t(0)
    N.check(lib.isa_forward_host_bytes(ctypes.byref(inp.shape), ctypes.byref(inp.knobs), int(heads_per_chunk),
                                       ctypes.byref(st_b), ctypes.byref(ws_b)))
    stage = torch.empty(int(st_b.value), dtype=torch.uint8, device=dev)
    ws = torch.empty(int(ws_b.value), dtype=torch.uint8, device=dev)
    pin = inp.q.is_pinned()
    if out is None:
        out = torch.empty((d.B, d.H, d.S, d.D), dtype=inp.q.dtype, pin_memory=pin)
    elif not (isinstance(out, torch.Tensor) and not out.is_cuda and out.is_contiguous()
              and tuple(out.shape) == (d.B, d.H, d.S, d.D) and out.dtype == inp.q.dtype):
        raise LayoutError("out must be a contiguous host (B,H,S,D) tensor of the input dtype")
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    bufs = _routing_buffers(d, dev) if collect_trace else None
    rout = _routing_struct(bufs) if bufs is not None else None
    pin_struct, keep = (None, None)
    if pinned is not None:
        pin_struct, keep = _pinned_struct(pinned, d, dev)
    main = torch.cuda.current_stream(dev)
    s_in, s_out = _side_streams(dev)
    streams = (ctypes.c_void_p * 3)(main.cuda_stream, s_in.cuda_stream, s_out.cuda_stream)
    e0 = e1 = None
    if collect_trace:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(main)
    N.check(lib.isa_forward_host(ctypes.byref(inp.shape), ctypes.byref(inp.knobs), _ptr(inp.q), _ptr(inp.k),
                                 _ptr(inp.v), _ptr(out), int(heads_per_chunk), _ptr(stage), st_b.value, _ptr(ws),
                                 ws_b.value, ctypes.byref(pin_struct) if pin_struct else None,
                                 ctypes.byref(rout) if rout else None, _ptr(err), streams))
    if collect_trace:
        e1.record(main)
    # host results must be complete on return (CPU tensors carry no stream order)
    if validate:
        _raise_flags(err)
    else:
        main.synchronize()
    # stage/ws return to the caching allocator on the main stream, which has
    # joined both copy streams: later reuse is ordered after their last use
    trace = None
    if collect_trace:
        times = _LazyStageTimes({"kernel": (e0, e1)})
        for name in ("coarse", "select", "split", "reconstruct"):
            dict.__setitem__(times, name, 0.0)  # not separable: stages of all chunks interleave
        routing = _make_routing(d, bufs, inp.numpy_io)
        trace = IsaTrace(coarse_summary={"host_streamed": True}, selection=routing.selection,
                         split=routing.split, mask=routing.mask, flops=d.flops(), stage_times_us=times,
                         ctx_scores=bufs["ctx_scores"], taylor_kernel=bufs["taylor_kernel"])
    del keep
    if inp.numpy_io:
        out = out.float().numpy()
    return out, trace, bufs


def _set_out_strides(shape: N.IsaShape, out, d: IsaDims, dtype):
    """Caller-provided output: any (B,H,S,D) view with a contiguous D axis and
    16-byte aligned strides (e.g. a permuted (B,S,H*D) activation buffer)."""
    if not (isinstance(out, torch.Tensor) and out.is_cuda and tuple(out.shape) == (d.B, d.H, d.S, d.D)
            and out.dtype == dtype and out.stride(3) == 1):
        raise LayoutError("out must be a CUDA (B,H,S,D) tensor of the input dtype with a contiguous D axis")
    e = out.element_size()
    if out.data_ptr() % 16 or any((st * e) % 16 for st in out.stride()[:3]):
        raise LayoutError("out strides must be multiples of 16 bytes")
    shape.out_stride_b, shape.out_stride_h, shape.out_stride_s = out.stride()[:3]


def _run(inp: _Inputs, collect_trace: bool, pinned=None, out: Optional[torch.Tensor] = None, validate=True,
         heads_per_chunk: int = 0):
    if inp.host:
        return _run_host(inp, collect_trace, pinned=pinned, out=out, validate=validate,
                         heads_per_chunk=heads_per_chunk)
    lib = N.load()
    d = inp.dims
    dev = inp.q.device
    ws, nbytes = inp.workspace()
    if out is None:
        out = torch.empty((d.B, d.H, d.S, d.D), dtype=inp.q.dtype, device=dev)
    else:
        _set_out_strides(inp.shape, out, d, inp.q.dtype)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    bufs = _routing_buffers(d, dev) if collect_trace else None
    rout = _routing_struct(bufs) if bufs is not None else None
    pin_struct, keep = (None, None)
    if pinned is not None:
        pin_struct, keep = _pinned_struct(pinned, d, dev)
    events = None
    evs = None
    if collect_trace:
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
        events = N.IsaEvents()
        for i, e in enumerate(evs):
            e.record()  # materialise the cudaEvent_t handle
            events.ev[i] = e.cuda_event
    stream = torch.cuda.current_stream(dev).cuda_stream
    N.check(lib.isa_forward(ctypes.byref(inp.shape), ctypes.byref(inp.knobs), _ptr(inp.q), _ptr(inp.k), _ptr(inp.v),
                            _ptr(out), _ptr(ws), nbytes, ctypes.byref(pin_struct) if pin_struct else None,
                            ctypes.byref(rout) if rout else None, _ptr(err),
                            ctypes.byref(events) if events else None, stream))
    if validate:
        _raise_flags(err)
    trace = None
    if collect_trace:
        T, D = d.T, d.D
        means = ws[256: 256 + 3 * d.B * d.H * T * D * 4].view(torch.float32).view(3, d.B, d.H, T, D)
        qc, kc = means[0].clone(), means[1].clone()
        times = _LazyStageTimes({"coarse": (evs[0], evs[1]), "select": (evs[1], evs[2]),
                                 "split": (evs[2], evs[3]), "kernel": (evs[3], evs[5])})
        dict.__setitem__(times, "reconstruct", 0.0)
        routing = _make_routing(d, bufs, inp.numpy_io)
        trace = IsaTrace(coarse_summary=_LazySummary(qc, kc, d.scale), selection=routing.selection,
                         split=routing.split, mask=routing.mask, flops=d.flops(), stage_times_us=times,
                         ctx_scores=bufs["ctx_scores"], taylor_kernel=bufs["taylor_kernel"])
    del keep
    if inp.numpy_io:
        out = out.float().cpu().numpy()
    return out, trace, bufs


def _kernel_width(D: int) -> int:
    return 64 if D <= 64 else 128


def _pad_head_dim(cfg, *xs):
    """Head dims the kernels are not instantiated for (D < 128, not 64): the D
    axis is zero-padded to the next kernel width (64 or 128). Zero columns add
    exact zeros to every dot product (the fp64 block-mean scores included, so
    routing is unchanged) and V's zero columns only produce output columns that
    are dropped; the scale stays 1/sqrt(D) of the real width. Returns None when
    no padding applies, else (cfg with the scale fixed, padded arrays...)."""
    shape = getattr(xs[0], "shape", None)
    if shape is None or len(shape) != 4:
        return None
    D = int(shape[-1])
    if D in SUPPORTED_HEAD_DIMS or D > max(SUPPORTED_HEAD_DIMS) or D < 1:
        return None
    cfg = cfg_from_any(cfg)
    cfg = dataclasses.replace(cfg, scale=cfg.scale if cfg.scale is not None else 1.0 / math.sqrt(D))
    w = _kernel_width(D) - D
    padded = []
    for x in xs:
        if isinstance(x, np.ndarray):
            padded.append(np.pad(np.asarray(x, dtype=np.float32), ((0, 0),) * 3 + ((0, w),)))
        elif isinstance(x, torch.Tensor):
            padded.append(torch.nn.functional.pad(x, (0, w)))
        else:
            raise LayoutError("expected torch tensors or numpy arrays")
    return (cfg, *padded)


def _unpad(x, D: int):
    if isinstance(x, np.ndarray):
        return np.ascontiguousarray(x[..., :D])
    return x[..., :D].contiguous()


_TAYLOR_FLAGS = {None: 0, "auto": 0, "k7": 2, "k7t": 4}


def isa_forward(q, k, v, icl: IclLayout, cfg: IsaConfig, collect_trace: bool = True, *, out=None, validate=True,
                heads_per_chunk: int = 0, taylor_kernel: Optional[str] = None, rope_base: Optional[float] = None):
    """Run the full pipeline; returns (output, IsaTrace or None) (pipeline.py:307-316).

    The output has the input dtype (bf16 in -> bf16 out; fp32 in -> fp32 out,
    computed with bf16 tensor cores and fp32 accumulation). Routing decisions
    are exact float64 restatements of the reference and match it bit-for-bit.
    Host inputs (numpy / CPU tensors) are streamed through the GPU in chunks of
    `heads_per_chunk` heads (0 = about 150 MB of inputs); the result is complete on return.
    Head dims other than 64/128 (up to 128) run zero-padded (`_pad_head_dim`).
    `taylor_kernel` ("k7" | "k7t" | None = per-head automatic choice) forces
    the D = 128 Taylor-branch kernel (test / A-B hook; same operator).
    `rope_base` (bf16 inputs) applies the decoupled RoPE of
    `apply_decoupled_rope(., icl, rope_base)` (pipeline.py:469-490) to Q and K
    inside the pooling pass: the result equals RoPE followed by isa_forward
    bit for bit, without the separate read + write of Q and K.
    """
    if taylor_kernel not in _TAYLOR_FLAGS:
        raise ConfigError(f"taylor_kernel must be one of {sorted(k for k in _TAYLOR_FLAGS if k)} or None")
    padded = _pad_head_dim(cfg, q, k, v)
    if padded is not None:
        D = int(q.shape[-1])
        pcfg, pq, pk, pv = padded
        if rope_base is not None:
            raise ConfigError("fused RoPE needs a kernel head dim (64 or 128)")
        res, trace = isa_forward(pq, pk, pv, icl, pcfg, collect_trace, validate=validate,
                                 heads_per_chunk=heads_per_chunk, taylor_kernel=taylor_kernel)
        res = _unpad(res, D)
        if trace is not None:  # FLOP tallies of the real head dim
            trace.flops = IsaDims.derive(q.shape, icl_from_any(icl), pcfg).flops()
        if out is not None:
            out[...] = res
            res = out
        return res, trace
    inp = _Inputs(q, k, v, icl, cfg)
    inp.knobs.flags |= _TAYLOR_FLAGS[taylor_kernel]
    if rope_base is not None:
        if not rope_base > 0:
            raise ConfigError(f"rope base must be > 0, got {rope_base}")
        inp.knobs.rope_base = float(rope_base)
    res, trace, _ = _run(inp, collect_trace, out=out, validate=validate, heads_per_chunk=heads_per_chunk)
    return res, trace


def isa_routing(q, k, v, icl: IclLayout, cfg: IsaConfig) -> IsaRouting:
    """Stages 1-3 only (pipeline.py:302-304). Index tensors stay on the GPU for
    torch callers; numpy callers get numpy arrays, like the reference."""
    padded = _pad_head_dim(cfg, q, k, v)
    if padded is not None:
        return isa_routing(*padded[1:], icl, padded[0])
    numpy_io = isinstance(q, np.ndarray)
    inp = _Inputs(q, k, v, icl, cfg)
    if inp.host:  # routing reads all of Q/K/V once: one plain upload
        inp = _Inputs(*(t.cuda() for t in (inp.q, inp.k, inp.v)), icl, cfg)
    lib = N.load()
    d = inp.dims
    ws, nbytes = inp.workspace()
    err = torch.zeros(1, dtype=torch.int32, device=inp.q.device)
    bufs = _routing_buffers(d, inp.q.device)
    rout = _routing_struct(bufs)
    stream = torch.cuda.current_stream(inp.q.device).cuda_stream
    N.check(lib.isa_routing(ctypes.byref(inp.shape), ctypes.byref(inp.knobs), _ptr(inp.q), _ptr(inp.k), _ptr(inp.v),
                            _ptr(ws), nbytes, ctypes.byref(rout), _ptr(err), stream))
    _raise_flags(err)
    return _make_routing(d, bufs, numpy_io)


def isa_forward_with_routing(q, k, v, icl: IclLayout, cfg: IsaConfig, routing) -> object:
    """Forward pass with pinned routing (pipeline.py:319-328). Accepts our
    IsaRouting or the reference's (numpy index arrays)."""
    padded = _pad_head_dim(cfg, q, k, v)
    if padded is not None:
        return _unpad(isa_forward_with_routing(*padded[1:], icl, padded[0], routing), int(q.shape[-1]))
    res, _, _ = _run(_Inputs(q, k, v, icl, cfg), False, pinned=routing)
    return res


def isa_backward(q, k, v, icl: IclLayout, cfg: IsaConfig, do, *, routing=None) -> GradBundle:
    """Gradients of isa_forward with routing frozen at this forward's decisions
    (pipeline.py:373-466, same signature, incl. the gamma residual). `routing` optionally pins
    the decisions (ours or the reference's IsaRouting). Computes in bf16 tensor
    arithmetic with fp32 accumulation; returns tensors in q's dtype (numpy fp32
    for numpy inputs)."""
    padded = _pad_head_dim(cfg, q, k, v, do)
    if padded is not None:
        D = int(q.shape[-1])
        g = isa_backward(*padded[1:4], icl, padded[0], padded[4], routing=routing)
        return GradBundle(_unpad(g.dq, D), _unpad(g.dk, D), _unpad(g.dv, D))
    numpy_io = isinstance(q, np.ndarray)
    inp = _Inputs(q, k, v, icl, cfg)
    if inp.host:
        inp = _Inputs(*(t.cuda() for t in (inp.q, inp.k, inp.v)), icl, cfg)
    out_dtype = inp.q.dtype
    if inp.q.dtype != torch.bfloat16:  # the backward kernels take bf16 operands
        inp = _Inputs(*(t.to(torch.bfloat16) for t in (inp.q, inp.k, inp.v)), icl, cfg)
    d = inp.dims
    if isinstance(do, np.ndarray):
        do = torch.from_numpy(np.ascontiguousarray(do, dtype=np.float32))
    if not isinstance(do, torch.Tensor) or tuple(do.shape) != (d.B, d.H, d.S, d.D):
        raise LayoutError(f"dO shape {tuple(getattr(do, 'shape', ()))} != output shape {(d.B, d.H, d.S, d.D)}")
    do = do.to(device=inp.q.device, dtype=torch.bfloat16)
    if do.stride() != inp.q.stride():
        do = torch.empty_strided(inp.q.shape, inp.q.stride(), dtype=torch.bfloat16, device=inp.q.device).copy_(do)
    lib = N.load()
    nbytes = ctypes.c_size_t(0)
    N.check(lib.isa_backward_workspace_bytes(ctypes.byref(inp.shape), ctypes.byref(inp.knobs), ctypes.byref(nbytes)))
    ws = torch.empty(int(nbytes.value), dtype=torch.uint8, device=inp.q.device)
    grads = [torch.empty((d.B, d.H, d.S, d.D), dtype=torch.float32, device=inp.q.device) for _ in range(3)]
    err = torch.zeros(1, dtype=torch.int32, device=inp.q.device)
    pin_struct, keep = (None, None)
    if routing is not None:
        pin_struct, keep = _pinned_struct(routing, d, inp.q.device)
    N.check(lib.isa_backward(ctypes.byref(inp.shape), ctypes.byref(inp.knobs), _ptr(inp.q), _ptr(inp.k),
                             _ptr(inp.v), _ptr(do), *(_ptr(g) for g in grads), _ptr(ws), nbytes.value,
                             ctypes.byref(pin_struct) if pin_struct else None, _ptr(err),
                             torch.cuda.current_stream(inp.q.device).cuda_stream))
    _raise_flags(err)
    del keep
    if numpy_io:
        return GradBundle(*(g.cpu().numpy() for g in grads))
    return GradBundle(*(g.to(out_dtype) for g in grads))


def dense_attention(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, scale: Optional[float] = None,
                    out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """Dense non-causal softmax attention (reference.py:79-123) on the sm_100a
    kernel with identity block tables: the ISA speed-up denominator (K8)."""
    if q.dtype != torch.bfloat16:
        raise ConfigError("dense_attention takes bf16 tensors")
    B, H, S, D = q.shape
    if D not in SUPPORTED_HEAD_DIMS and D < max(SUPPORTED_HEAD_DIMS):  # zero-padded head dim
        scale = scale if scale is not None else 1.0 / math.sqrt(D)
        w = _kernel_width(D) - D
        res = dense_attention(*(torch.nn.functional.pad(x, (0, w)) for x in (q, k, v)), scale)[..., :D]
        if out is None:
            return res.contiguous()
        out.copy_(res)
        return out
    if D not in SUPPORTED_HEAD_DIMS:
        raise ConfigError(f"head dim {D} not supported")
    scale = scale if scale is not None else 1.0 / math.sqrt(D)
    q, k, v = (x if x.stride(3) == 1 else x.contiguous() for x in (q, k, v))
    if q.stride() != k.stride() or q.stride() != v.stride():
        q, k, v = q.contiguous(), k.contiguous(), v.contiguous()
    if out is None:
        out = torch.empty((B, H, S, D), dtype=q.dtype, device=q.device)
    shape = N.IsaShape(B, H, S, D, S, 0, 64, N.ISA_DTYPE_BF16, q.stride(0), q.stride(1), q.stride(2))
    N.check(N.load().isa_dense_attention(ctypes.byref(shape), scale, _ptr(q), _ptr(k), _ptr(v), _ptr(out),
                                         torch.cuda.current_stream(q.device).cuda_stream))
    return out


def apply_decoupled_rope(x, icl: IclLayout, base: float = 10000.0, *, out: Optional[torch.Tensor] = None):
    """Rotary rotation with positions restarting at zero for the context
    segment (pipeline.py:469-490, same signature). Pairs (2i, 2i+1) rotate by
    pos * base^(-2i/D). Angles in fp64, rotation in fp32 on the GPU; returns a
    new tensor of x's dtype (numpy in -> numpy out, like the reference), or
    writes `out` (any (B,H,S,D) view with a contiguous D axis)."""
    icl = icl_from_any(icl)
    numpy_io = isinstance(x, np.ndarray)
    if numpy_io:
        if x.ndim != 4:
            raise LayoutError(f"rope input: expected 4 axes (B,H,S,D), got shape {x.shape}")
        x = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda()
    if not (isinstance(x, torch.Tensor) and x.is_cuda and x.dim() == 4):
        raise LayoutError("rope input must be a CUDA (B,H,S,D) tensor or a numpy array")
    B, H, S, D = x.shape
    if D % 2:
        raise ConfigError(f"decoupled rope needs an even head dim, got D={D}")
    if S != icl.total:
        raise LayoutError(f"sequence length {S} != icl total {icl.total}")
    if x.dtype not in (torch.bfloat16, torch.float32):
        x = x.float()
    if x.stride(3) != 1 or any((st * x.element_size()) % 16 for st in x.stride()[:3]) or x.data_ptr() % 16:
        x = x.contiguous()
    if out is None:
        out = torch.empty((B, H, S, D), dtype=x.dtype, device=x.device)
    shape = N.IsaShape(B, H, S, D, icl.l_src, icl.l_ctx, 64,
                       N.ISA_DTYPE_BF16 if x.dtype == torch.bfloat16 else N.ISA_DTYPE_F32,
                       x.stride(0), x.stride(1), x.stride(2))
    if not (isinstance(out, torch.Tensor) and out.is_cuda and tuple(out.shape) == (B, H, S, D)
            and out.dtype == x.dtype and out.stride(3) == 1):
        raise LayoutError("out must be a CUDA (B,H,S,D) tensor of x's dtype with a contiguous D axis")
    shape.out_stride_b, shape.out_stride_h, shape.out_stride_s = out.stride()[:3]
    N.check(N.load().isa_decoupled_rope(ctypes.byref(shape), float(base), _ptr(x), _ptr(out),
                                        torch.cuda.current_stream(x.device).cuda_stream))
    if numpy_io:
        return out.cpu().numpy()
    return out


def prepare(q, k, v, icl, cfg, separate_branches: bool = False, signal: bool = False,
            rope_base: Optional[float] = None):
    """Validated inputs + a reusable workspace for repeated calls (bench/CUDA graphs).

    separate_branches launches the exact and Taylor attention branches as two
    kernels (per-branch profiling) instead of the default fused grid;
    signal publishes per-head completion counters (see _Prepared)."""
    inp = _Inputs(q, k, v, icl, cfg)
    if separate_branches:
        inp.knobs.flags |= N.FLAG_SEPARATE_BRANCHES
    if rope_base is not None:
        inp.knobs.rope_base = float(rope_base)
    ws, nbytes = inp.workspace()
    return _Prepared(inp, ws, nbytes, signal=signal)


class _Prepared:
    """Pre-validated call: no per-call allocation; graph-capturable.

    signal=True publishes per-head completion (isa_forward_signal): after
    the n-th call, head_done[b*H + h] reaches n * done_inc once head h's output
    rows are final; `wait_head(stream, h)` makes another stream wait for that
    (the multi-GPU overlap in parallel.py)."""

    def __init__(self, inp: _Inputs, ws, nbytes, signal: bool = False):
        self.inp, self.ws, self.nbytes = inp, ws, nbytes
        d = inp.dims
        self.out = torch.empty((d.B, d.H, d.S, d.D), dtype=inp.q.dtype, device=inp.q.device)
        self.err = torch.zeros(1, dtype=torch.int32, device=inp.q.device)
        self.head_done = torch.zeros(d.B * d.H, dtype=torch.int32, device=inp.q.device) if signal else None
        self.done_inc = ctypes.c_int32(0)
        self.calls = 0

    def __call__(self, stream=None):
        inp = self.inp
        st = stream if stream is not None else torch.cuda.current_stream(inp.q.device).cuda_stream
        if self.head_done is not None:
            N.check(N.load().isa_forward_signal(ctypes.byref(inp.shape), ctypes.byref(inp.knobs), _ptr(inp.q),
                                                _ptr(inp.k), _ptr(inp.v), _ptr(self.out), _ptr(self.ws), self.nbytes,
                                                _ptr(self.err), _ptr(self.head_done), ctypes.byref(self.done_inc),
                                                st))
            self.calls += 1
            return self.out
        N.check(N.load().isa_forward(ctypes.byref(inp.shape), ctypes.byref(inp.knobs), _ptr(inp.q), _ptr(inp.k),
                                     _ptr(inp.v), _ptr(self.out), _ptr(self.ws), self.nbytes, None, None,
                                     _ptr(self.err), None, st))
        return self.out

    def wait_head(self, stream, bh: int) -> None:
        """Enqueue on `stream` a wait until head bh of the latest call is final."""
        target = self.calls * self.done_inc.value
        if target >= 2 ** 31:
            raise OverflowError("head_done counter range exhausted; re-prepare")
        N.check(N.load().isa_stream_wait_geq(stream.cuda_stream, self.head_done.data_ptr() + 4 * bh, target))
