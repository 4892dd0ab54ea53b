"""ISA4 tensor containers (reference `tensor.py:192-219`, `workload.py:147-175`).

Byte format (kept identical so files move between the reference CLI and this
one): the 4-byte magic ``ISA4``, four little-endian u32 dims (B, H, S, D), then
the B*H*S*D elements, little-endian, float32 ("single") or float64 ("double").
A ``<prefix>.meta`` sidecar holds three lines: L_src, L_ctx, precision.

B200 side: `load_tensor4(..., pinned=True)` reads the payload straight into a
page-locked torch buffer (`readinto`), so the host->HBM copy that follows is a
single DMA with no staging copy.
"""

from __future__ import annotations

import os
import struct
from typing import Tuple

import numpy as np

from .errors import FormatError, InputError, LayoutError
from .types import IclLayout

PRECISIONS = {"single": np.float32, "double": np.float64}
MAGIC = b"ISA4"
_DIMS = struct.Struct("<4I")
_HDR = len(MAGIC) + _DIMS.size


def _dtype(precision: str) -> np.dtype:
    if precision not in PRECISIONS:
        raise FormatError(f"unknown precision {precision!r}")
    return np.dtype(PRECISIONS[precision]).newbyteorder("<")


def _check4(x: np.ndarray, name: str) -> np.ndarray:
    # the (B,H,S,D) contract of ensure_tensor4 (tensor.py:25-36)
    if x.ndim != 4:
        raise LayoutError(f"{name}: expected 4 axes (B,H,S,D), got shape {x.shape}")
    if min(x.shape) < 1:
        raise LayoutError(f"{name}: all dims must be >= 1, got shape {x.shape}")
    if not np.all(np.isfinite(x)):
        raise InputError(f"{name}: non-finite elements")
    return x


def save_tensor4(path, x, precision: str = "single") -> None:
    """Write one container (tensor.py:192-199). Accepts numpy arrays or torch tensors."""
    if hasattr(x, "detach"):  # torch (any float dtype, any device)
        x = x.detach().double().cpu().numpy()
    x = np.asarray(x)
    if not np.issubdtype(x.dtype, np.floating):
        x = x.astype(np.float64)
    payload = np.ascontiguousarray(_check4(x, "save_tensor4 input"), dtype=_dtype(precision))
    with open(path, "wb") as f:
        f.write(MAGIC + _DIMS.pack(*payload.shape))
        f.write(memoryview(payload).cast("B"))


def _read_header(f, path) -> Tuple[int, int, int, int]:
    head = f.read(_HDR)
    if head[:4] != MAGIC:
        raise FormatError(f"{path}: bad magic {head[:4]!r} at byte 0 (want {MAGIC!r})")
    if len(head) < _HDR:
        raise FormatError(f"{path}: truncated header at byte {len(head)}")
    dims = _DIMS.unpack_from(head, 4)
    if min(dims) < 1:
        raise FormatError(f"{path}: zero dim in header {dims}")
    return dims


def load_tensor4(path, precision: str = "single", pinned: bool = False):
    """Read one container (tensor.py:202-219): the same FormatError cases with
    byte offsets (bad magic, short header, zero dim, size mismatch) and the
    finiteness check. Returns a numpy array, or with `pinned=True` a
    page-locked torch tensor of the stored dtype."""
    dt = _dtype(precision)
    size = os.path.getsize(path)
    with open(path, "rb") as f:
        dims = _read_header(f, path)
        need = _HDR + int(np.prod(dims, dtype=np.int64)) * dt.itemsize
        if size != need:
            raise FormatError(f"{path}: expected {need} bytes, file ends at byte {size}")
        if pinned:
            import torch

            t = torch.empty(dims, dtype=torch.float32 if precision == "single" else torch.float64).pin_memory()
            f.readinto(memoryview(t.numpy()).cast("B"))
            _check4(t.numpy(), f"load_tensor4({path})")
            return t
        arr = np.empty(dims, dtype=dt)
        f.readinto(memoryview(arr).cast("B"))
    return _check4(arr.astype(PRECISIONS[precision], copy=False), f"load_tensor4({path})")


def dump(prefix: str, q, k, v, icl: IclLayout, precision: str = "single") -> None:
    """<prefix>.{q,k,v}.isa4 plus the three-line <prefix>.meta sidecar (workload.py:147-153)."""
    for name, x in (("q", q), ("k", k), ("v", v)):
        save_tensor4(f"{prefix}.{name}.isa4", x, precision)
    with open(f"{prefix}.meta", "w") as f:
        f.write(f"{icl.l_src}\n{icl.l_ctx}\n{precision}\n")


def load(prefix: str, pinned: bool = False):
    """Inverse of dump() (workload.py:156-175): parses the sidecar, loads the
    three containers and checks they agree with each other and with L_src + L_ctx."""
    try:
        with open(f"{prefix}.meta") as f:
            fields = [line.strip() for line in f]
        l_src, l_ctx, precision = int(fields[0]), int(fields[1]), fields[2]
    except (OSError, ValueError, IndexError) as exc:
        raise FormatError(f"{prefix}.meta: cannot parse sidecar header: {exc}") from exc
    if precision not in PRECISIONS:
        raise FormatError(f"{prefix}.meta: unknown precision {precision!r}")
    q, k, v = (load_tensor4(f"{prefix}.{n}.isa4", precision, pinned) for n in ("q", "k", "v"))
    if tuple(q.shape) != tuple(k.shape) or tuple(q.shape) != tuple(v.shape):
        raise FormatError(f"{prefix}: Q/K/V container dims disagree: {tuple(q.shape)}, {tuple(k.shape)}, "
                          f"{tuple(v.shape)}")
    if l_src + l_ctx != q.shape[2]:
        raise LayoutError(f"{prefix}.meta: L_src + L_ctx = {l_src + l_ctx} != stored sequence length {q.shape[2]}")
    return q, k, v, IclLayout(l_src, l_ctx)
