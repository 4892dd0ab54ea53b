"""Deterministic inputs with duplicated and near-tied context blocks at the
top-k boundary of the context selection, shared by the golden generator
(make_coarse_golden.py, run with the reference) and the tests (no reference
needed). Pure numpy; test infrastructure.

The context saliency of block c is the mean over source query blocks of
scale * <qc_i, kc_c> (coarse.py:155). Column 0 of Q alternates +a / -a
between consecutive source blocks, so sum_i qc_i[0] = 0. Per head, with the
k_ctx-th ranked context block c_k and the next two c_n, c_m:

* block c_n becomes an exact copy of c_k: a tie in any arithmetic, straddling
  the top-k boundary (the stable rule keeps the lower index);
* block c_m becomes c_k with column 0 of every row raised by one bf16 step:
  in exact arithmetic it ties with c_k too (its extra term is scaled by
  sum_i qc_i[0] = 0), so only the fp64 rounding of the per-(i, c) scores and
  of the sequential mean decides where it lands (a "near tie").
"""

from __future__ import annotations

import math

import numpy as np


def _bf16(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even fp32 -> bf16 -> fp32 (same as oracle.round_bf16)."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(np.float32).reshape(x.shape)


def _bf16_up(x: np.ndarray) -> np.ndarray:
    """The next bf16 value above each (finite, non-max) bf16 value x."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.int64)
    u = np.where(x > 0, u + 0x10000, np.where(x < 0, u - 0x10000, 0x10000))
    return u.astype(np.uint32).view(np.float32).reshape(x.shape)


def tie_inputs(B: int, H: int, l_src: int, l_ctx: int, D: int, seed: int, alpha_s: float = 0.25, b: int = 64):
    rng = np.random.default_rng(seed)
    S = l_src + l_ctx
    q, k, v = (_bf16(rng.standard_normal((B, H, S, D)).astype(np.float32)) for _ in range(3))
    t_src, t_ctx = l_src // b, l_ctx // b
    for i in range(t_src):
        q[:, :, i * b:(i + 1) * b, 0] = np.float32(0.75) if i % 2 == 0 else np.float32(-0.75)
    k_ctx = int(math.floor(alpha_s * t_ctx))
    assert 1 <= k_ctx <= t_ctx - 3
    qm = q[:, :, :l_src].reshape(B, H, t_src, b, D).astype(np.float64).mean(axis=(2, 3))
    kc = k[:, :, l_src:].reshape(B, H, t_ctx, b, D).astype(np.float64).mean(axis=3)
    score = np.einsum("bhd,bhcd->bhc", qm, kc)
    for bi in range(B):
        for hi in range(H):
            order = np.argsort(-score[bi, hi], kind="stable")
            c_k, c_n, c_m = (l_src + int(order[j]) * b for j in (k_ctx - 1, k_ctx, k_ctx + 1))
            src = k[bi, hi, c_k:c_k + b].copy()
            k[bi, hi, c_n:c_n + b] = src
            bumped = src.copy()
            bumped[:, 0] = _bf16_up(src[:, 0])
            k[bi, hi, c_m:c_m + b] = bumped
    return q, k, v
