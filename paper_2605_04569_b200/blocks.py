"""Block-layout utilities of the reference (tensor.py:25-36, 67-75, 122-190):
`ensure_tensor4`, `pad_to_blocks`, `gather_blocks`, `scatter_blocks`,
`concat_seq`, with the same checks and error classes.

These are pure data movement (bit-exact copies). The fused pipeline never
materialises them — TMA reads blocks in place through the block table and the
attention epilogues write rows at their original positions — so here they are
plain tensor indexing on whatever device the input lives on (numpy in -> numpy
out, torch in -> torch out).
"""

from __future__ import annotations

import numpy as np

from .errors import BlockIndexError, ContractError, InputError, LayoutError
from .types import BlockLayout


def _is_torch(x) -> bool:
    return hasattr(x, "detach")


def ensure_tensor4(x, name: str = "tensor"):
    """4 axes, every dim >= 1, floating point (ints cast to float64), finite (tensor.py:25-36)."""
    if _is_torch(x):
        import torch

        if x.dim() != 4:
            raise LayoutError(f"{name}: expected 4 axes (B,H,S,D), got shape {tuple(x.shape)}")
        if min(x.shape) < 1:
            raise LayoutError(f"{name}: all dims must be >= 1, got shape {tuple(x.shape)}")
        if not x.is_floating_point():
            x = x.to(torch.float64)
        if not bool(torch.isfinite(x).all()):
            raise InputError(f"{name}: non-finite elements")
        return x
    x = np.asarray(x)
    if x.ndim != 4:
        raise LayoutError(f"{name}: expected 4 axes (B,H,S,D), got shape {x.shape}")
    if min(x.shape) < 1:
        raise LayoutError(f"{name}: all dims must be >= 1, got shape {x.shape}")
    if not np.issubdtype(x.dtype, np.floating):
        x = x.astype(np.float64)
    if not np.all(np.isfinite(x)):
        raise InputError(f"{name}: non-finite elements")
    return x


def pad_to_blocks(x, layout: BlockLayout):
    """Zero rows from layout.seq_len up to layout.padded_len (tensor.py:67-75)."""
    if x.shape[2] != layout.seq_len:
        raise LayoutError(f"seq length {x.shape[2]} != layout.seq_len {layout.seq_len}")
    pad = layout.padded_len - layout.seq_len
    if pad == 0:
        return x
    if _is_torch(x):
        import torch

        return torch.nn.functional.pad(x, (0, 0, 0, pad))
    B, H, _, D = x.shape
    return np.concatenate([x, np.zeros((B, H, pad, D), dtype=x.dtype)], axis=2)


def _block_index(idx, B: int, H: int, num_blocks: int, name: str) -> np.ndarray:
    """Per-(B,H) sorted block lists as int64 (B,H,k), validated (tensor.py:122-135)."""
    if _is_torch(idx):
        idx = idx.detach().cpu().numpy()
    idx = np.asarray(idx, dtype=np.int64)
    if idx.ndim == 1:
        idx = np.broadcast_to(idx, (B, H, idx.shape[0])).copy()
    if idx.ndim != 3 or idx.shape[:2] != (B, H):
        raise LayoutError(f"{name}: index array must have shape (B,H,k), got {idx.shape}")
    if idx.size:
        if idx.min() < 0 or idx.max() >= num_blocks:
            raise BlockIndexError(f"{name}: block index out of range [0, {num_blocks})")
        if np.any(np.diff(idx, axis=2) <= 0):
            raise ContractError(f"{name}: block-index lists must be sorted ascending without duplicates")
    return idx


def gather_blocks(x, layout: BlockLayout, idx):
    """Whole blocks by per-(B,H) sorted index lists, copied bit-exactly (tensor.py:138-154)."""
    if len(x.shape) != 4:
        raise LayoutError(f"gather_blocks: expected 4 axes, got shape {tuple(x.shape)}")
    if x.shape[2] != layout.padded_len:
        raise LayoutError(f"gather_blocks: seq length {x.shape[2]} != layout.padded_len {layout.padded_len}")
    B, H, _, D = (int(s) for s in x.shape)
    T, b = layout.num_blocks, layout.block_size
    idx = _block_index(idx, B, H, T, "gather_blocks")
    k = idx.shape[2]
    if _is_torch(x):
        import torch

        if k == 0:
            return x.new_zeros((B, H, 0, D))
        it = torch.from_numpy(idx).to(x.device)[:, :, :, None, None].expand(B, H, k, b, D)
        return torch.gather(x.reshape(B, H, T, b, D), 2, it).reshape(B, H, k * b, D)
    x = np.asarray(x)
    if k == 0:
        return np.zeros((B, H, 0, D), dtype=x.dtype)
    out = np.take_along_axis(x.reshape(B, H, T, b, D), idx[:, :, :, None, None], axis=2)
    return out.reshape(B, H, k * b, D)


def scatter_blocks(dst, idx, src):
    """A copy of dst with the indexed blocks replaced by src's blocks, in list order (tensor.py:157-179)."""
    if len(dst.shape) != 4 or len(src.shape) != 4:
        raise LayoutError("scatter_blocks: dst and src must have 4 axes")
    B, H, S, D = (int(s) for s in dst.shape)
    if src.shape[0] != B or src.shape[1] != H or src.shape[3] != D:
        raise LayoutError(f"scatter_blocks: src shape {tuple(src.shape)} incompatible with dst {tuple(dst.shape)}")
    torch_io = _is_torch(dst)
    if src.shape[2] == 0:
        return dst.clone() if torch_io else np.asarray(dst).copy()
    k = (idx.shape[-1]) if hasattr(idx, "shape") else np.asarray(idx).shape[-1]
    if src.shape[2] % k:
        raise LayoutError(f"scatter_blocks: src seq length {src.shape[2]} not divisible by |idx|={k}")
    b = int(src.shape[2]) // k
    if S % b:
        raise LayoutError(f"scatter_blocks: dst seq length {S} not divisible by block size {b}")
    T = S // b
    idx = _block_index(idx, B, H, T, "scatter_blocks")
    if torch_io:
        import torch

        out = dst.reshape(B, H, T, b, D).clone()
        it = torch.from_numpy(idx).to(dst.device)[:, :, :, None, None].expand(B, H, k, b, D)
        out.scatter_(2, it, src.reshape(B, H, k, b, D).to(dst.dtype))
        return out.reshape(B, H, S, D)
    out = np.asarray(dst).reshape(B, H, T, b, D).copy()
    np.put_along_axis(out, idx[:, :, :, None, None], np.asarray(src).reshape(B, H, k, b, D).astype(out.dtype),
                      axis=2)
    return out.reshape(B, H, S, D)


def concat_seq(a, b):
    """Concatenate along the sequence axis, a's rows first (tensor.py:182-189)."""
    if len(a.shape) != 4 or len(b.shape) != 4:
        raise LayoutError("concat_seq: operands must have 4 axes")
    if a.shape[0] != b.shape[0] or a.shape[1] != b.shape[1] or a.shape[3] != b.shape[3]:
        raise LayoutError(f"concat_seq: (B,H,D) mismatch: {tuple(a.shape)} vs {tuple(b.shape)}")
    if _is_torch(a):
        import torch

        return torch.cat([a, b], dim=2)
    return np.concatenate([np.asarray(a), np.asarray(b)], axis=2)
