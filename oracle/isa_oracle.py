"""CPU oracle for the ISA forward path — TEST INFRASTRUCTURE ONLY.

This module is a numpy (float64) restatement of the reference algorithm in
`/root/reference/pkg/src/isattn` (the `isattn` package, pure numpy; there is
no native code to compile). It is the checker for the CUDA path: only
`tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline/reference
leg may import it. The product package `paper_2605_04569_b200` never imports
it and has no CPU fallback.

Parity pinning: every function below is validated against golden vectors
produced by the reference itself (`tests/golden/make_golden.py` imports
`isattn` from /root/reference in the build container and commits the
outputs to `tests/golden/*.npz`); see tests/test_oracle_golden.py.

Each function cites the reference file:line it restates. Paths are relative
to /root/reference/pkg/src/isattn/.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Optional

import numpy as np

# ----------------------------------------------------------------------------
# Layout helpers (tensor.py)
# ----------------------------------------------------------------------------


def block_layout(b: int, s: int):
    """BlockLayout (tensor.py:39-64): (num_blocks, padded_len, valid_rows)."""
    t = -(-s // b)
    valid = np.full(t, b, dtype=np.int64)
    if s % b:
        valid[-1] = s % b
    return t, t * b, valid


def pad_to_blocks(x: np.ndarray, b: int) -> np.ndarray:
    """Zero-pad the sequence axis to a multiple of b (tensor.py:67-75)."""
    s = x.shape[2]
    t, padded, _ = block_layout(b, s)
    if padded == s:
        return x
    B, H, _, D = x.shape
    return np.concatenate([x, np.zeros((B, H, padded - s, D), dtype=x.dtype)], axis=2)


def block_mean(x: np.ndarray, b: int) -> np.ndarray:
    """Valid-row block means, fp64 sum then cast to storage dtype (tensor.py:96-119)."""
    s = x.shape[2]
    t, padded, valid = block_layout(b, s)
    xp = pad_to_blocks(x, b)
    B, H, _, D = xp.shape
    sums = xp.reshape(B, H, t, b, D).sum(axis=3, dtype=np.float64)  # padded rows are zero
    return (sums / valid[None, None, :, None]).astype(x.dtype)


def icl_means(x: np.ndarray, l_src: int, l_ctx: int, b: int) -> np.ndarray:
    """Per-segment block means concatenated source-first (pipeline.py:238-243)."""
    parts = [block_mean(x[:, :, :l_src], b)]
    if l_ctx:
        parts.append(block_mean(x[:, :, l_src:], b))
    return np.concatenate(parts, axis=2)


def icl_pad(x: np.ndarray, l_src: int, l_ctx: int, b: int) -> np.ndarray:
    """Pad each segment independently (pipeline.py:230-236)."""
    src = pad_to_blocks(x[:, :, :l_src], b)
    if not l_ctx:
        return src
    return np.concatenate([src, pad_to_blocks(x[:, :, l_src:], b)], axis=2)


# ----------------------------------------------------------------------------
# Routing (coarse.py, util.py)
# ----------------------------------------------------------------------------


def softmax_rows(s: np.ndarray) -> np.ndarray:
    """Max-subtracted fp64 softmax along the last axis (util.py:32-40)."""
    s = np.asarray(s, dtype=np.float64)
    m = np.max(s, axis=-1, keepdims=True)
    m = np.where(np.isfinite(m), m, 0.0)
    with np.errstate(invalid="ignore"):
        e = np.exp(s - m)
    e = np.where(np.isfinite(s), e, 0.0)
    return e / e.sum(axis=-1, keepdims=True)


def topk_rows(scores: np.ndarray, k: int) -> np.ndarray:
    """k largest along the last axis, ties to the lowest index, sorted ascending
    (coarse.py:130-136)."""
    if k == 0:
        return np.zeros(scores.shape[:-1] + (0,), dtype=np.int64)
    order = np.argsort(-scores, axis=-1, kind="stable")
    return np.sort(order[..., :k], axis=-1).astype(np.int64)


def rank_context(s_coarse: np.ndarray, t_src: int, t_ctx: int, alpha_s: float) -> np.ndarray:
    """Context-block saliency = mean over source query rows; keep floor(alpha_s*T_ctx)
    (coarse.py:139-157)."""
    B, H = s_coarse.shape[:2]
    if t_ctx == 0:
        return np.zeros((B, H, 0), dtype=np.int64)
    ctx_scores = s_coarse[:, :, :t_src, t_src:].mean(axis=2)
    k_ctx = int(math.floor(alpha_s * t_ctx))
    return topk_rows(ctx_scores, k_ctx)


def sharpness_split(s_coarse: np.ndarray, t_src: int, alpha_f: float, softmax_first: bool = True):
    """Variance of (softmaxed) source-column scores; floor(alpha_f*T) least sharp go
    flat; stable ties keep the lower index sharp (coarse.py:173-201)."""
    src = s_coarse[:, :, :, :t_src]
    rows = softmax_rows(src) if softmax_first else src
    m = rows.var(axis=-1)
    T = m.shape[2]
    n_flat = int(math.floor(alpha_f * T))
    order = np.argsort(-m, axis=-1, kind="stable")
    sharp = np.sort(order[..., : T - n_flat], axis=-1).astype(np.int64)
    flat = np.sort(order[..., T - n_flat :], axis=-1).astype(np.int64)
    return sharp, flat, m


def block_mask(s_flat: np.ndarray, alpha_ns: float) -> np.ndarray:
    """Top-k key blocks per flat query block, k = min(N_K, max(1, floor(alpha_ns*N_K)))
    (coarse.py:160-170)."""
    n_k = s_flat.shape[-1]
    k = min(n_k, max(1, int(math.floor(alpha_ns * n_k))))
    return topk_rows(s_flat, k)


# ----------------------------------------------------------------------------
# Attention branches (reference.py, taylor.py)
# ----------------------------------------------------------------------------


def masked_softmax_attention(qf, kf, vf, scale, key_valid, row_chunk=2048):
    """Exact softmax attention of fp64 rows over keys with a validity mask.

    Same map as online_softmax_attention (reference.py:126-170, OnlineState
    reference.py:42-60): the online recurrence equals the direct max-subtracted
    softmax up to fp64 reordering; full_attention (reference.py:79-123) is the
    direct form used here.
    """
    out = np.empty((qf.shape[0], vf.shape[1]))
    for lo in range(0, qf.shape[0], row_chunk):
        s = scale * (qf[lo : lo + row_chunk] @ kf.T)
        s[:, ~key_valid] = -np.inf
        m = s.max(axis=1)
        p = np.exp(s - m[:, None])
        p[:, ~key_valid] = 0.0
        out[lo : lo + row_chunk] = (p @ vf) / p.sum(axis=1)[:, None]
    return out


def taylor_head(qf, kf, vf, kc, vc, idx, w, scale, b):
    """One (batch, head) of the Taylor kernel (taylor.py:124-160), finalized O/ell
    (taylor.py:193). Exact blocks then one batched centroid update."""
    t_q, t_k = qf.shape[0] // b, kf.shape[0] // b
    d = qf.shape[1]
    qb = qf.reshape(t_q, b, d)
    kb = kf.reshape(t_k, b, d)
    vb = vf.reshape(t_k, b, d)
    col_valid = np.arange(b) < w[:, None]
    member = np.zeros((t_q, t_k), dtype=bool)
    np.put_along_axis(member, idx, True, axis=1)
    m = np.full((t_q, b), -np.inf)
    ell = np.zeros((t_q, b))
    acc = np.zeros((t_q, b, d))
    for slot in range(idx.shape[1]):
        j = idx[:, slot]
        s = scale * np.matmul(qb, kb[j].transpose(0, 2, 1))
        s = np.where(col_valid[j][:, None, :], s, -np.inf)
        m_new = np.maximum(m, s.max(axis=2))
        with np.errstate(invalid="ignore"):
            p = np.exp(s - m_new[..., None])
        p = np.where(np.isfinite(s), p, 0.0)
        delta = m - m_new
        delta[~np.isfinite(delta)] = 0.0
        alpha = np.exp(delta)
        ell = ell * alpha + p.sum(axis=2)
        acc = acc * alpha[..., None] + np.matmul(p, vb[j])
        m = m_new
    s_c = scale * (qb @ kc.T)
    s_c = np.where(member[:, None, :], -np.inf, s_c)
    m_new = np.maximum(m, s_c.max(axis=2, initial=-np.inf))
    with np.errstate(invalid="ignore"):
        pe = np.exp(s_c - m_new[..., None])
    pe = np.where(np.isfinite(s_c), pe, 0.0) * w
    delta = m - m_new
    delta[~np.isfinite(delta)] = 0.0
    alpha = np.exp(delta)
    ell = ell * alpha + pe.sum(axis=2)
    acc = acc * alpha[..., None] + pe @ vc
    return (acc / ell[..., None]).reshape(t_q * b, d)


# ----------------------------------------------------------------------------
# Pipeline (pipeline.py)
# ----------------------------------------------------------------------------


@dataclass
class OracleRouting:
    selection: np.ndarray  # (B,H,k_ctx) int64
    sharp: np.ndarray  # (B,H,n_sharp)
    flat: np.ndarray  # (B,H,n_flat)
    sharpness: np.ndarray  # (B,H,T) fp64
    mask: Optional[np.ndarray]  # (B,H,n_flat,k) or None
    ctx_scores: Optional[np.ndarray] = None  # (B,H,T_ctx) fp64 (diagnostics)
    s_flat: Optional[np.ndarray] = None  # (B,H,n_flat,t_new) fp64 (diagnostics)


class OracleAssembly:
    """Stages 1-3 of _Assembly (pipeline.py:133-228), storage dtype fp32."""

    def __init__(self, q, k, v, l_src, l_ctx, *, alpha_s=0.125, alpha_ns=0.0625, alpha_f=0.5,
                 block_size=64, scale=None, softmax_first=True, gamma=0.0, residual_softmax=True,
                 routing: Optional[OracleRouting] = None):
        b = block_size
        self.gamma, self.residual_softmax = gamma, residual_softmax
        self.q, self.k, self.v = (np.asarray(x, dtype=np.float32) for x in (q, k, v))  # pipeline.py:150-151
        B, H, S, D = self.q.shape
        self.b, self.l_src, self.l_ctx = b, l_src, l_ctx
        self.scale = scale if scale is not None else 1.0 / math.sqrt(D)  # pipeline.py:154
        self.t_src = -(-l_src // b)
        self.t_ctx = -(-l_ctx // b) if l_ctx else 0
        self.T = self.t_src + self.t_ctx
        self.qp, self.kp, self.vp = (icl_pad(x, l_src, l_ctx, b) for x in (self.q, self.k, self.v))
        self.orig_rows = np.concatenate([np.arange(l_src), self.t_src * b + np.arange(l_ctx)]).astype(np.int64)
        _, _, src_valid = block_layout(b, l_src)
        ctx_valid = block_layout(b, l_ctx)[2] if l_ctx else np.zeros(0, np.int64)
        # stage 1 (pipeline.py:176-183)
        self.qc, self.kc, self.vc = (icl_means(x, l_src, l_ctx, b) for x in (self.q, self.k, self.v))
        self.s_coarse = self.scale * np.einsum("bhid,bhjd->bhij", self.qc.astype(np.float64), self.kc.astype(np.float64))
        # stage 2 (pipeline.py:186-211)
        if routing is not None:
            sel = routing.selection
        else:
            sel = rank_context(self.s_coarse, self.t_src, self.t_ctx, alpha_s)
        self.sel = sel
        k_ctx = sel.shape[2]
        self.t_new = self.t_src + k_ctx
        ts = self.t_src * b
        if self.t_ctx and k_ctx:
            kb_ctx = self.kp[:, :, ts:].reshape(B, H, self.t_ctx, b, D)
            vb_ctx = self.vp[:, :, ts:].reshape(B, H, self.t_ctx, b, D)
            k_sel = np.take_along_axis(kb_ctx, sel[..., None, None], axis=2).reshape(B, H, k_ctx * b, D)
            v_sel = np.take_along_axis(vb_ctx, sel[..., None, None], axis=2).reshape(B, H, k_ctx * b, D)
            self.k_new = np.concatenate([self.kp[:, :, :ts], k_sel], axis=2)
            self.v_new = np.concatenate([self.vp[:, :, :ts], v_sel], axis=2)
            self.valid_new = np.concatenate(
                [np.broadcast_to(src_valid, (B, H, self.t_src)), ctx_valid[sel]], axis=2)
        else:
            self.k_new = self.kp[:, :, :ts]
            self.v_new = self.vp[:, :, :ts]
            self.valid_new = np.broadcast_to(src_valid, (B, H, self.t_src)).copy()
        self.key_mask_new = (np.arange(b)[None, None, None, :] < self.valid_new[..., None]).reshape(B, H, self.t_new * b)
        self.kc_new = _masked_block_means(self.k_new, self.valid_new, b)
        self.vc_new = _masked_block_means(self.v_new, self.valid_new, b)
        # stage 3 (pipeline.py:214-228)
        if routing is not None:
            self.sharp, self.flat = routing.sharp, routing.flat
            self.sharpness = routing.sharpness
        else:
            self.sharp, self.flat, self.sharpness = sharpness_split(self.s_coarse, self.t_src, alpha_f, softmax_first)
        self.n_flat = self.flat.shape[2]
        self.n_sharp = self.sharp.shape[2]
        self.s_flat = None
        if self.n_flat:
            qc_flat = np.take_along_axis(self.qc, self.flat[..., None], axis=2)
            self.s_flat = self.scale * np.einsum("bhid,bhjd->bhij", qc_flat.astype(np.float64), self.kc_new.astype(np.float64))
            self.mask = routing.mask if routing is not None else block_mask(self.s_flat, alpha_ns)
        else:
            self.mask = None

    def routing(self) -> OracleRouting:
        ctx_scores = None
        if self.t_ctx:
            ctx_scores = self.s_coarse[:, :, : self.t_src, self.t_src:].mean(axis=2)
        return OracleRouting(self.sel, self.sharp, self.flat, self.sharpness, self.mask, ctx_scores, self.s_flat)

    def coarse_residual(self) -> np.ndarray:
        """O_coarse, one row per query block, float64 (pipeline.py:261-267)."""
        if self.residual_softmax:
            p = softmax_rows(self.s_coarse)
        else:
            p = self.s_coarse / self.scale  # raw, unscaled scores
        return p @ self.vc.astype(np.float64)

    def forward(self, block_fraction: float = 1.0) -> np.ndarray:
        """Stages 4-5 of _forward (pipeline.py:331-358), incl. the gamma
        coarse residual (pipeline.py:354-356).

        block_fraction < 1 computes only the first ceil(f*n) sharp and flat
        query blocks of each head (bench.py's bounded CPU sample; rows are
        independent so time scales linearly); the rest of the output is 0."""
        B, H, Sp, D = self.qp.shape
        b = self.b
        out_pad = np.zeros((B, H, Sp, D), dtype=np.float64)
        qb = self.qp.reshape(B, H, self.T, b, D)
        ob = out_pad.reshape(B, H, self.T, b, D)
        for bi in range(B):
            for hi in range(H):
                kf = self.k_new[bi, hi].astype(np.float64)
                vf = self.v_new[bi, hi].astype(np.float64)
                ns = int(math.ceil(block_fraction * self.n_sharp))
                nf = int(math.ceil(block_fraction * self.n_flat))
                if ns:  # pipeline.py:338-343
                    sel = self.sharp[bi, hi, :ns]
                    rows = qb[bi, hi, sel].reshape(-1, D).astype(np.float64)
                    o = masked_softmax_attention(rows, kf, vf, self.scale, self.key_mask_new[bi, hi])
                    ob[bi, hi, sel] = o.reshape(-1, b, D)
                if nf:  # pipeline.py:344-347, taylor.py:163-194
                    sel = self.flat[bi, hi, :nf]
                    rows = qb[bi, hi, sel].reshape(-1, D).astype(np.float64)
                    o = taylor_head(rows, kf, vf, self.kc_new[bi, hi].astype(np.float64),
                                    self.vc_new[bi, hi].astype(np.float64), self.mask[bi, hi, :nf],
                                    self.valid_new[bi, hi], self.scale, b)
                    ob[bi, hi, sel] = o.reshape(-1, b, D)
        out_pad = out_pad.astype(np.float32)  # scatter into the storage-dtype buffer (pipeline.py:350-353)
        if self.gamma:  # pipeline.py:354-356
            residual = np.repeat(self.coarse_residual(), b, axis=2)
            out_pad = (out_pad.astype(np.float64) + self.gamma * residual).astype(np.float32)
        out = out_pad[:, :, self.orig_rows]  # pipeline.py:357 (storage dtype fp32)
        return out


def _masked_block_means(x, valid, b):
    """pipeline.py:292-299."""
    B, H, S, D = x.shape
    t = S // b
    blocks = x.reshape(B, H, t, b, D).astype(np.float64)
    keep = np.arange(b)[None, None, None, :] < valid[..., None]
    means = (blocks * keep[..., None]).sum(axis=3) / valid[..., None]
    return means.astype(x.dtype)


def isa_routing(q, k, v, l_src, l_ctx, **cfg) -> OracleRouting:
    """pipeline.py:302-304."""
    return OracleAssembly(q, k, v, l_src, l_ctx, **cfg).routing()


def isa_forward(q, k, v, l_src, l_ctx, **cfg):
    """pipeline.py:307-316 (output, routing)."""
    asm = OracleAssembly(q, k, v, l_src, l_ctx, **cfg)
    return asm.forward(), asm.routing()


def full_attention(q, k, v, scale=None):
    """Dense softmax attention in fp64, output fp32 (reference.py:79-123)."""
    q = np.asarray(q)
    B, H, S, D = q.shape
    scale = scale if scale is not None else 1.0 / math.sqrt(D)
    out = np.empty(q.shape, dtype=np.float32)
    valid = np.ones(k.shape[2], dtype=bool)
    for bi in range(B):
        for hi in range(H):
            out[bi, hi] = masked_softmax_attention(q[bi, hi].astype(np.float64), k[bi, hi].astype(np.float64),
                                                   v[bi, hi].astype(np.float64), scale, valid)
    return out


# ----------------------------------------------------------------------------
# Synthetic inputs (workload.py) — restated so golden inputs regenerate on the
# GPU box, where /root/reference does not exist.
# ----------------------------------------------------------------------------


def workload_head(kind: str, seq_len: int, dim: int, seed: int, bi: int, hi: int, n_clusters=None,
                  cluster_noise=0.25, rank=8, lowrank_noise=0.1):
    """workload.py:77-106: one (batch, head) of Q/K/V from its Philox stream."""
    rng = np.random.Generator(np.random.Philox(key=seed * 2**16 + bi * 256 + hi))
    s, d = seq_len, dim
    if kind == "iid-gaussian":
        return rng.standard_normal((3, s, d))
    if kind == "clustered":
        n = min(n_clusters if n_clusters is not None else max(1, s // 256), s)
        run = -(-s // n)
        member = np.minimum(np.arange(s) // run, n - 1)
        k_centers = rng.standard_normal((n, d))
        v_centers = rng.standard_normal((n, d))
        kk = k_centers[member] + cluster_noise * rng.standard_normal((s, d))
        vv = v_centers[member] + cluster_noise * rng.standard_normal((s, d))
        target = rng.integers(0, n, size=n)
        tau = rng.uniform(0.25, 2.5, size=n)
        qq = tau[member, None] * k_centers[target[member]] + 0.5 * rng.standard_normal((s, d))
        return np.stack([qq, kk, vv])
    if kind == "lowrank":
        r = min(rank, d)
        qq = rng.standard_normal((s, r)) @ rng.standard_normal((r, d)) / math.sqrt(r)
        kk = rng.standard_normal((s, r)) @ rng.standard_normal((r, d)) / math.sqrt(r)
        qq = qq + lowrank_noise * rng.standard_normal((s, d))
        kk = kk + lowrank_noise * rng.standard_normal((s, d))
        vv = rng.standard_normal((s, d))
        return np.stack([qq, kk, vv])
    raise ValueError(kind)


def workload(kind: str, batch: int, heads: int, seq_len: int, dim: int, seed: int):
    """workload.py:127-144 with context_attenuation = 1 (fp32 storage)."""
    q = np.empty((batch, heads, seq_len, dim), dtype=np.float32)
    k = np.empty_like(q)
    v = np.empty_like(q)
    for bi in range(batch):
        for hi in range(heads):
            qh, kh, vh = workload_head(kind, seq_len, dim, seed, bi, hi)
            q[bi, hi], k[bi, hi], v[bi, hi] = qh, kh, vh
    return q, k, v


def round_bf16(x: np.ndarray) -> np.ndarray:
    """Round fp32 to the nearest bf16 value (ties to even), returned as fp32."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def apply_decoupled_rope(x: np.ndarray, l_src: int, l_ctx: int, base: float = 10000.0) -> np.ndarray:
    """Rotary rotation, positions restarting at 0 for the context segment;
    fp64 math, result in x's dtype (pipeline.py:469-490)."""
    B, H, S, D = x.shape
    pos = np.concatenate([np.arange(l_src), np.arange(l_ctx)]).astype(np.float64)
    inv_freq = base ** (-np.arange(0, D, 2, dtype=np.float64) / D)
    theta = pos[:, None] * inv_freq[None, :]
    cos, sin = np.cos(theta), np.sin(theta)
    xf = x.astype(np.float64).reshape(B, H, S, D // 2, 2)
    even, odd = xf[..., 0], xf[..., 1]
    out = np.empty_like(xf)
    out[..., 0] = even * cos - odd * sin
    out[..., 1] = even * sin + odd * cos
    return out.reshape(B, H, S, D).astype(x.dtype)
