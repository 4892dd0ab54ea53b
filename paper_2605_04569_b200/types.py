"""Host-side value types of the ISA operator, mirroring the reference interface.

Every class here keeps the reference's field names, defaults and validation
messages so `isattn` callers can switch without edits:

- `IsaConfig`           <- pkg/src/isattn/pipeline.py:51-88
- `IsaRouting`          <- pipeline.py:91-97
- `IsaTrace`            <- pipeline.py:100-130
- `IclLayout`           <- pkg/src/isattn/tensor.py:78-93
- `BlockLayout`         <- tensor.py:39-64
- `SelectionIndex`      <- pkg/src/isattn/coarse.py:52-69
- `BlockMask`           <- coarse.py:72-88
- `SharpnessSplit`      <- coarse.py:91-107
- `FlopCount`           <- pkg/src/isattn/taylor.py:24-42

Index tensors are torch int64 tensors that live on the GPU (routing never
leaves the device unless the caller asks); `.numpy()` helpers copy to host.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Union, Optional

import numpy as np

from .errors import ConfigError, LayoutError

# Precisions the reference accepts (tensor.py:19). The B200 path computes in
# bf16 tensor-core arithmetic with fp32 accumulation; "single" is the only
# accepted value (ConfigError otherwise, see IsaConfig.validate_b200).
PRECISIONS = ("double", "single")

SUPPORTED_BLOCK = 64
SUPPORTED_HEAD_DIMS = (64, 128)



# tensor.py:17-19: the reference's tensor alias and storage dtypes. The B200
# operator takes numpy arrays or torch tensors; "double" is accepted by
# IsaConfig.validate (pipeline.py:73-88) and rejected by the sm_100a kernels
# (validate_b200), which compute in bf16 with fp32 accumulation.
Tensor4 = Union[np.ndarray, "torch.Tensor"]
DTYPES = {"single": np.float32, "double": np.float64}

@dataclass
class GradBundle:
    """Gradients w.r.t. the attention primals; dims match Q/K/V (reference.py:20-25)."""

    dq: object
    dk: object
    dv: object


@dataclass
class IsaConfig:
    """Sparsity knobs and behavioral flags (pipeline.py:51-71, same defaults)."""

    alpha_s: float = 0.125
    alpha_ns: float = 0.0625
    alpha_f: float = 0.5
    gamma: float = 0.0
    block_size: int = 64
    scale: Optional[float] = None
    softmax_first: bool = True
    residual_softmax: bool = True
    deterministic: bool = True
    precision: str = "single"
    strict: bool = True

    def validate(self) -> "IsaConfig":
        """Same checks, order and messages as pipeline.py:73-88."""
        if not 0.0 <= self.alpha_s <= 1.0:
            raise ConfigError(f"alpha_s must be in [0, 1], got {self.alpha_s}")
        if not 0.0 < self.alpha_ns <= 1.0:
            raise ConfigError(f"alpha_ns must be in (0, 1], got {self.alpha_ns}")
        if not 0.0 <= self.alpha_f <= 1.0:
            raise ConfigError(f"alpha_f must be in [0, 1], got {self.alpha_f}")
        if self.gamma < 0.0:
            raise ConfigError(f"gamma must be >= 0, got {self.gamma}")
        if self.block_size < 1:
            raise ConfigError(f"block_size must be >= 1, got {self.block_size}")
        if self.scale is not None and self.scale <= 0.0:
            raise ConfigError(f"scale must be > 0, got {self.scale}")
        if self.precision not in PRECISIONS:
            raise ConfigError(f"precision must be one of {sorted(PRECISIONS)}, got {self.precision!r}")
        return self

    def validate_b200(self) -> "IsaConfig":
        """Reference validation plus the limits of this tier's kernels.

        Values the reference accepts but the sm_100a path does not implement
        raise ConfigError instead of silently degrading.
        """
        self.validate()
        if self.block_size != SUPPORTED_BLOCK:
            raise ConfigError(
                f"block_size={self.block_size} is not supported by the sm_100a kernels (only {SUPPORTED_BLOCK})"
            )
        if self.precision != "single":
            raise ConfigError("precision='double' is not available on the bf16 tensor-core path")
        return self


def cfg_from_any(cfg) -> IsaConfig:
    """Accept our IsaConfig or a duck-typed reference `isattn.IsaConfig`."""
    if isinstance(cfg, IsaConfig):
        return cfg
    names = IsaConfig.__dataclass_fields__.keys()
    return IsaConfig(**{n: getattr(cfg, n) for n in names if hasattr(cfg, n)})


@dataclass(frozen=True)
class IclLayout:
    """Source/context split: source tokens first, context after (tensor.py:78-93)."""

    l_src: int
    l_ctx: int

    def __post_init__(self):
        if self.l_src < 1:
            raise LayoutError(f"l_src must be >= 1, got {self.l_src}")
        if self.l_ctx < 0:
            raise LayoutError(f"l_ctx must be >= 0, got {self.l_ctx}")

    @property
    def total(self) -> int:
        return self.l_src + self.l_ctx


def icl_from_any(icl) -> IclLayout:
    if isinstance(icl, IclLayout):
        return icl
    return IclLayout(int(icl.l_src), int(icl.l_ctx))


@dataclass
class BlockLayout:
    """Partition of a length-S sequence into blocks (tensor.py:39-64)."""

    block_size: int
    seq_len: int
    padded_len: int = field(init=False)
    num_blocks: int = field(init=False)
    valid_rows: np.ndarray = field(init=False, repr=False)

    def __post_init__(self):
        if self.block_size < 1:
            raise LayoutError(f"block_size must be >= 1, got {self.block_size}")
        if self.seq_len < 1:
            raise LayoutError(f"seq_len must be >= 1, got {self.seq_len}")
        b, s = self.block_size, self.seq_len
        self.num_blocks = -(-s // b)
        self.padded_len = self.num_blocks * b
        valid = np.full(self.num_blocks, b, dtype=np.int64)
        if s % b:
            valid[-1] = s % b
        self.valid_rows = valid


def _to_np(x) -> np.ndarray:
    if hasattr(x, "detach"):
        return x.detach().cpu().numpy()
    return np.asarray(x)


@dataclass
class SelectionIndex:
    """Retained context block indices, ascending per (batch, head) (coarse.py:52-69)."""

    indices: object  # torch int64 (B, H, k_ctx), device
    num_context_blocks: int

    @property
    def k_ctx(self) -> int:
        return int(self.indices.shape[2])

    def numpy(self) -> np.ndarray:
        return _to_np(self.indices)

    def to_text(self) -> str:
        idx = self.numpy()
        B, H, _ = idx.shape
        return "\n".join(f"b={bi} h={hi}: {idx[bi, hi].tolist()}" for bi in range(B) for hi in range(H))


@dataclass
class BlockMask:
    """Per flat query block, the K_new blocks computed exactly (coarse.py:72-88)."""

    indices: object  # torch int64 (B, H, n_flat, k), device
    num_key_blocks: int

    @property
    def k(self) -> int:
        return int(self.indices.shape[3])

    def numpy(self) -> np.ndarray:
        return _to_np(self.indices)

    def member_mask(self) -> np.ndarray:
        idx = self.numpy()
        B, H, NQ, _ = idx.shape
        m = np.zeros((B, H, NQ, self.num_key_blocks), dtype=bool)
        np.put_along_axis(m, idx, True, axis=3)
        return m


@dataclass
class SharpnessSplit:
    """Sharp/flat partition of query blocks (coarse.py:91-107)."""

    sharp: object  # torch int64 (B, H, n_sharp)
    flat: object  # torch int64 (B, H, n_flat)
    sharpness: object  # torch float64 (B, H, T)

    def to_text(self) -> str:
        sharp, flat = _to_np(self.sharp), _to_np(self.flat)
        B, H, _ = sharp.shape
        return "\n".join(
            f"b={bi} h={hi}: sharp={sharp[bi, hi].tolist()} flat={flat[bi, hi].tolist()}"
            for bi in range(B)
            for hi in range(H)
        )


@dataclass
class FlopCount:
    """FLOP tallies by branch (taylor.py:24-42; the "mas" fields count 2 per multiply-add)."""

    exact_mas: int = 0
    taylor_mas: int = 0
    overhead_mas: int = 0
    dense_equivalent_mas: int = 0

    def total(self) -> int:
        return self.exact_mas + self.taylor_mas + self.overhead_mas

    def to_text(self) -> str:
        return (
            f"exact_mas={self.exact_mas}\n"
            f"taylor_mas={self.taylor_mas}\n"
            f"overhead_mas={self.overhead_mas}\n"
            f"dense_equivalent_mas={self.dense_equivalent_mas}\n"
        )


@dataclass
class IsaRouting:
    """The discrete decisions of one forward run (pipeline.py:91-97)."""

    selection: SelectionIndex
    split: SharpnessSplit
    mask: Optional[BlockMask]


class _LazyStageTimes(dict):
    """Stage times from CUDA events; resolved (one sync) on first access."""

    def __init__(self, events):
        super().__init__()
        self._events = events
        self._resolved = False

    def _resolve(self):
        if not self._resolved:
            self._resolved = True
            for name, (a, b) in self._events.items():
                b.synchronize()
                dict.__setitem__(self, name, a.elapsed_time(b) * 1e3)

    def __getitem__(self, key):
        self._resolve()
        return dict.__getitem__(self, key)

    def items(self):
        self._resolve()
        return dict.items(self)

    def keys(self):
        self._resolve()
        return dict.keys(self)

    def values(self):
        self._resolve()
        return dict.values(self)

    def __iter__(self):
        self._resolve()
        return dict.__iter__(self)

    def __len__(self):
        self._resolve()
        return dict.__len__(self)

    def __repr__(self):
        self._resolve()
        return dict.__repr__(self)


@dataclass
class IsaTrace:
    """Per-call trace (pipeline.py:100-130). stage_times_us come from CUDA events."""

    coarse_summary: dict
    selection: SelectionIndex
    split: SharpnessSplit
    mask: Optional[BlockMask]
    flops: FlopCount
    stage_times_us: dict = field(default_factory=dict)
    # B200 extensions (not in the reference trace): the context saliency
    # scores (B,H,T_ctx) fp64, bit-identical to coarse.py:155, and the
    # Taylor-branch kernel run per head (B,H) int32: 0 = K7 union tiles, 1 = K7T
    ctx_scores: object = None
    taylor_kernel: object = None

    def to_text(self) -> str:
        lines = ["isa_trace:", "  coarse:"]
        for key, val in self.coarse_summary.items():
            lines.append(f"    {key}: {val}")
        lines.append("  selection:")
        lines.append(f"    k_ctx: {self.selection.k_ctx}")
        for row in self.selection.to_text().splitlines():
            lines.append(f"    {row}")
        lines.append("  split:")
        for row in self.split.to_text().splitlines():
            lines.append(f"    {row}")
        lines.append("  mask:")
        lines.append(f"    k: {0 if self.mask is None else self.mask.k}")
        lines.append("  flops:")
        for row in self.flops.to_text().strip().splitlines():
            key, val = row.split("=", 1)
            lines.append(f"    {key}: {val}")
        lines.append("  stage_times_us:")
        for key, val in self.stage_times_us.items():
            lines.append(f"    {key}: {val:.1f}")
        return "\n".join(lines) + "\n"


@dataclass(frozen=True)
class IsaDims:
    """Every integer the pipeline derives from (shape, icl, cfg).

    The counts use the reference's exact float expressions so that the
    representation-sensitive floors agree: k_ctx (coarse.py:156), n_flat
    (coarse.py:197), k (coarse.py:169). Block counts follow
    pipeline.py:158-162 (per-segment ceil).
    """

    B: int
    H: int
    S: int
    D: int
    b: int
    l_src: int
    l_ctx: int
    t_src: int
    t_ctx: int
    T: int
    k_ctx: int
    t_new: int
    n_flat: int
    n_sharp: int
    k: int  # exact blocks per flat query block (0 when n_flat == 0)
    scale: float
    gamma: float = 0.0  # coarse residual weight (pipeline.py:354-356)

    @staticmethod
    def derive(shape, icl: IclLayout, cfg: IsaConfig) -> "IsaDims":
        B, H, S, D = (int(x) for x in shape)
        b = cfg.block_size
        t_src = -(-icl.l_src // b)
        t_ctx = -(-icl.l_ctx // b) if icl.l_ctx else 0
        T = t_src + t_ctx
        k_ctx = int(math.floor(cfg.alpha_s * t_ctx)) if t_ctx else 0
        t_new = t_src + k_ctx
        n_flat = int(math.floor(cfg.alpha_f * T))
        n_sharp = T - n_flat
        k = min(t_new, max(1, int(math.floor(cfg.alpha_ns * t_new)))) if n_flat else 0
        scale = cfg.scale if cfg.scale is not None else 1.0 / math.sqrt(D)
        return IsaDims(B, H, S, D, b, icl.l_src, icl.l_ctx, t_src, t_ctx, T, k_ctx, t_new, n_flat, n_sharp, k, scale,
                       float(cfg.gamma))

    def flops(self) -> FlopCount:
        """Reference accounting (pipeline.py:269-289 with taylor.py:299-316)."""
        B, H, D, b = self.B, self.H, self.D, self.b
        per_exact_pair = 4 * b * b * D
        per_taylor_pair = 4 * b * D
        exact = B * H * self.n_sharp * self.t_new * per_exact_pair
        taylor = 0
        if self.n_flat:
            exact += B * H * self.n_flat * self.k * per_exact_pair
            taylor = B * H * self.n_flat * (self.t_new - self.k) * per_taylor_pair
        overhead = 2 * B * H * self.T * self.T * D
        if self.n_flat:
            overhead += 2 * B * H * self.n_flat * self.t_new * D
        if self.gamma:
            overhead += 2 * B * H * self.T * self.T * D  # residual P V^c (pipeline.py:284-285)
        return FlopCount(
            exact_mas=exact,
            taylor_mas=taylor,
            overhead_mas=overhead,
            dense_equivalent_mas=B * H * self.T * self.T * per_exact_pair,
        )
