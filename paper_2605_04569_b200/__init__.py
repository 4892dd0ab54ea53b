"""B200-native (sm_100a) In-context Sparse Attention forward — drop-in for the
reference `isattn` operator path (pkg/src/isattn/pipeline.py:302-328).

    from paper_2605_04569_b200 import isa_forward, IsaConfig, IclLayout
    out, trace = isa_forward(q, k, v, IclLayout(L_src, L_ctx), IsaConfig())

The compute lives in libisa_b200.so (hand-written tcgen05/TMA kernels, C ABI in
include/isa_b200.h); this package is the host-side mirror of the reference
interface. There is no CPU fallback.
"""

from .errors import (
    BlockIndexError,
    ConfigError,
    ContractError,
    DegenerateRowError,
    FormatError,
    InputError,
    IsaError,
    LayoutError,
    NativeError,
    NumericError,
)
from .types import (
    DTYPES,
    BlockLayout,
    BlockMask,
    FlopCount,
    GradBundle,
    IclLayout,
    IsaConfig,
    IsaDims,
    IsaRouting,
    IsaTrace,
    SelectionIndex,
    SharpnessSplit,
    Tensor4,
)

from .blocks import concat_seq, ensure_tensor4, gather_blocks, pad_to_blocks, scatter_blocks
from .tensorio import dump, load, load_tensor4, save_tensor4
from .util import elementwise_relative_error, max_relative_error, mean_relative_error
from .workload import WorkloadSpec, generate
from .taylor import TaylorKernelInput, flop_count, taylor_sparse_backward, taylor_sparse_forward

__version__ = "0.1.0"


def __getattr__(name):
    # The operator entry points import torch; keep `import paper_2605_04569_b200`
    # light for host-only consumers (types, errors, build).
    if name in ("isa_forward", "isa_routing", "isa_forward_with_routing", "isa_backward", "dense_attention",
                "prepare", "apply_decoupled_rope"):
        from . import pipeline

        return getattr(pipeline, name)
    if name in ("CoarseSet", "build_coarse", "rank_context", "build_block_mask", "sharpness_split", "block_mean"):
        from . import coarse

        return getattr(coarse, name)
    if name in ("full_attention", "online_softmax_attention", "full_attention_backward", "OnlineState"):
        from . import exact

        return getattr(exact, name)
    if name in ("isa_forward_sharded", "head_shard"):
        from . import parallel

        return getattr(parallel, name)
    if name in ("DiTAttentionLayer", "DiTAttentionStack"):
        from . import stack

        return getattr(stack, name)
    raise AttributeError(name)
