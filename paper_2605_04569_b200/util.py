"""Error metrics of the reference (util.py:8-29), same definitions, for numpy
arrays or torch tensors (device tensors are reduced on the GPU in float64)."""

from __future__ import annotations

import numpy as np


def _pair(a, b):
    if hasattr(a, "detach") or hasattr(b, "detach"):
        import torch

        dev = a.device if hasattr(a, "device") else b.device
        a = torch.as_tensor(a, device=dev).double()
        b = torch.as_tensor(b, device=dev).double()
        return a, b, torch
    return np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64), np


def max_relative_error(a, ref) -> float:
    """max |a - ref| normalised by the largest reference magnitude (util.py:8-13)."""
    a, r, lib = _pair(a, ref)
    if a.size == 0 if lib is np else a.numel() == 0:
        return 0.0
    scale = max(float(lib.abs(r).max()), np.finfo(np.float64).tiny)
    return float(lib.abs(a - r).max()) / scale


def mean_relative_error(a, ref) -> float:
    """mean |a - ref| normalised by the mean reference magnitude (util.py:16-21)."""
    a, r, lib = _pair(a, ref)
    if a.size == 0 if lib is np else a.numel() == 0:
        return 0.0
    scale = max(float(lib.abs(r).mean()), np.finfo(np.float64).tiny)
    return float(lib.abs(a - r).mean()) / scale


def elementwise_relative_error(a, b, floor: float = 1e-12) -> float:
    """max_i |a_i - b_i| / (max(|a_i|, |b_i|) + floor) (util.py:24-29)."""
    a, b, lib = _pair(a, b)
    if a.size == 0 if lib is np else a.numel() == 0:
        return 0.0
    denom = lib.maximum(lib.abs(a), lib.abs(b)) + floor
    return float((lib.abs(a - b) / denom).max())
