"""Seeded synthetic Q/K/V workloads (reference `workload.py:23-144`).

The bench CLI (`cli.py`) needs the reference's exact inputs so its CSV rows can
be compared row for row with `isa-bench` runs: each (batch, head) pair draws
from its own numpy Philox stream keyed ``seed * 2**16 + b * 256 + h``
(`workload.py:77-78`), with the draws in the reference's order, so the arrays
are bit-identical (pinned by `tests/golden/workload`). Generation is host work
(numpy); the arrays are then staged once into HBM by the caller.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, replace
from typing import Optional

import numpy as np

from .errors import ConfigError
from .tensorio import PRECISIONS, load
from .types import IclLayout

KINDS = ("iid-gaussian", "clustered", "lowrank", "loaded")


@dataclass
class WorkloadSpec:
    """Shape, structure and seed of one workload (workload.py:23-74); same fields and defaults."""

    batch: int = 1
    heads: int = 4
    seq_len: int = 4096
    dim: int = 64
    l_src: Optional[int] = None  # None -> seq_len // 2
    l_ctx: Optional[int] = None  # None -> seq_len - l_src
    kind: str = "clustered"
    n_clusters: Optional[int] = None  # None -> max(1, seq_len // 256)
    cluster_noise: float = 0.25
    rank: int = 8
    lowrank_noise: float = 0.1
    context_attenuation: float = 1.0
    seed: int = 0
    precision: str = "single"
    path: Optional[str] = None  # kind == "loaded"

    def resolved(self) -> "WorkloadSpec":
        """Defaults filled in and every field range-checked (ConfigError), as workload.py:49-74."""
        l_src = self.seq_len // 2 if self.l_src is None else self.l_src
        l_ctx = self.seq_len - l_src if self.l_ctx is None else self.l_ctx
        n_clusters = max(1, self.seq_len // 256) if self.n_clusters is None else self.n_clusters
        spec = replace(self, l_src=l_src, l_ctx=l_ctx, n_clusters=n_clusters)
        if spec.kind not in KINDS:
            raise ConfigError(f"unknown workload kind {spec.kind!r}")
        if min(spec.batch, spec.heads, spec.seq_len, spec.dim) < 1:
            raise ConfigError("batch/heads/seq_len/dim must all be >= 1")
        if l_src + l_ctx != spec.seq_len or l_src < 1 or l_ctx < 0:
            raise ConfigError(f"l_src + l_ctx must equal seq_len with l_src >= 1, "
                              f"got {l_src}+{l_ctx} != {spec.seq_len}")
        if spec.cluster_noise < 0 or spec.lowrank_noise < 0:
            raise ConfigError("noise levels must be >= 0")
        if not 0.0 <= spec.context_attenuation <= 1.0:
            raise ConfigError(f"context_attenuation must be in [0, 1], got {spec.context_attenuation}")
        if n_clusters < 1 or spec.rank < 1:
            raise ConfigError("n_clusters and rank must be >= 1")
        if spec.precision not in PRECISIONS:
            raise ConfigError(f"precision must be one of {sorted(PRECISIONS)}")
        if spec.kind == "loaded" and not spec.path:
            raise ConfigError("kind='loaded' needs a path")
        return spec


def head_stream(seed: int, b: int, h: int) -> np.random.Generator:
    """The per-(batch, head) Philox stream (workload.py:77-78)."""
    return np.random.Generator(np.random.Philox(key=seed * 2**16 + b * 256 + h))


def _clustered(spec: WorkloadSpec, g: np.random.Generator):
    # workload.py:85-97. Draw order: key centres, value centres, key noise,
    # value noise, per-run target cluster, per-run temperature, query noise.
    S, D = spec.seq_len, spec.dim
    n = min(spec.n_clusters, S)
    run_len = -(-S // n)
    run_of = np.minimum(np.arange(S) // run_len, n - 1)
    kcen = g.standard_normal((n, D))
    vcen = g.standard_normal((n, D))
    k = kcen[run_of] + spec.cluster_noise * g.standard_normal((S, D))
    v = vcen[run_of] + spec.cluster_noise * g.standard_normal((S, D))
    aim = g.integers(0, n, size=n)
    tau = g.uniform(0.25, 2.5, size=n)
    q = tau[run_of, None] * kcen[aim[run_of]] + 0.5 * g.standard_normal((S, D))
    return q, k, v


def _lowrank(spec: WorkloadSpec, g: np.random.Generator):
    # workload.py:98-105. Draw order: Q factors, K factors, Q noise, K noise, V.
    S, D = spec.seq_len, spec.dim
    r = min(spec.rank, D)
    norm = math.sqrt(r)
    qa = g.standard_normal((S, r))
    q = qa @ g.standard_normal((r, D)) / norm
    ka = g.standard_normal((S, r))
    k = ka @ g.standard_normal((r, D)) / norm
    q = q + spec.lowrank_noise * g.standard_normal((S, D))
    k = k + spec.lowrank_noise * g.standard_normal((S, D))
    v = g.standard_normal((S, D))
    return q, k, v


def _head(spec: WorkloadSpec, g: np.random.Generator):
    if spec.kind == "iid-gaussian":  # workload.py:83-84: one (3, S, D) draw
        q, k, v = g.standard_normal((3, spec.seq_len, spec.dim))
        return q, k, v
    if spec.kind == "clustered":
        return _clustered(spec, g)
    if spec.kind == "lowrank":
        return _lowrank(spec, g)
    raise ConfigError(f"kind {spec.kind!r} has no generator")


def _attenuate(q: np.ndarray, k: np.ndarray, spec: WorkloadSpec) -> np.ndarray:
    """Shrink the part of every context key inside the source-query row space
    by `context_attenuation` (workload.py:109-124): numerical rank from the SVD
    at 1e-10 of the top singular value, projection onto that basis."""
    a = spec.context_attenuation
    if a == 1.0 or spec.l_ctx == 0:
        return k
    _, sv, vt = np.linalg.svd(q[: spec.l_src], full_matrices=False)
    rank = int(np.count_nonzero(sv > sv[0] * 1e-10)) if sv.size else 0
    if rank == 0:
        return k
    basis = vt[:rank]
    ctx = k[spec.l_src:]
    inside = (ctx @ basis.T) @ basis
    k = k.copy()
    k[spec.l_src:] = a * inside + (ctx - inside)
    return k


def generate(spec: WorkloadSpec):
    """(Q, K, V, IclLayout) for the spec (workload.py:127-144): numpy arrays of
    the spec's precision, bit-identical to the reference generator's."""
    spec = spec.resolved()
    if spec.kind == "loaded":
        return load(spec.path)
    dt = PRECISIONS[spec.precision]
    shape = (spec.batch, spec.heads, spec.seq_len, spec.dim)
    q, k, v = (np.empty(shape, dtype=dt) for _ in range(3))
    for b in range(spec.batch):
        for h in range(spec.heads):
            qh, kh, vh = _head(spec, head_stream(spec.seed, b, h))
            q[b, h], k[b, h], v[b, h] = qh, _attenuate(qh, kh, spec), vh
    return q, k, v, IclLayout(spec.l_src, spec.l_ctx)
