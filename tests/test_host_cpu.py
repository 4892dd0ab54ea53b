"""Host-side logic of the B200 operator (no GPU needed): the reference-mirroring
types, the integer derivations, the C ABI surface and its error codes."""

import ctypes
import math
import os
import re
import sys

import numpy as np
import pytest

from paper_2605_04569_b200 import errors as E
from paper_2605_04569_b200.types import BlockLayout, IclLayout, IsaConfig, IsaDims

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
REF_SRC = "/root/reference/pkg/src"


def _reference():
    if not os.path.isdir(REF_SRC):
        pytest.skip("reference package not present (GPU box)")
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import isattn

    return isattn


# ------------------------------------------------------------------ config / layout parity with the reference
@pytest.mark.parametrize("kw", [
    dict(alpha_s=-0.1), dict(alpha_s=1.5), dict(alpha_ns=0.0), dict(alpha_ns=1.1), dict(alpha_f=-1e-9),
    dict(alpha_f=2.0), dict(gamma=-1.0), dict(block_size=0), dict(scale=0.0), dict(scale=-2.0),
    dict(precision="half"),
])
def test_config_validation_matches_reference(kw):
    ref = _reference()
    with pytest.raises(ref.ConfigError) as r:
        ref.IsaConfig(**kw).validate()
    with pytest.raises(E.ConfigError) as o:
        IsaConfig(**kw).validate()
    assert str(r.value) == str(o.value)


def test_config_defaults_match_reference():
    ref = _reference()
    a, b = ref.IsaConfig(), IsaConfig()
    for name in IsaConfig.__dataclass_fields__:
        assert getattr(a, name) == getattr(b, name), name


def test_b200_limits_raise_config_error():
    for kw in (dict(block_size=32), dict(precision="double")):
        with pytest.raises(E.ConfigError):
            IsaConfig(**kw).validate_b200()
    IsaConfig().validate_b200()
    IsaConfig(gamma=0.5, residual_softmax=False).validate_b200()  # coarse residual is implemented
    with pytest.raises(E.ConfigError):
        IsaConfig(gamma=-1.0).validate_b200()


def test_layouts_match_reference():
    ref = _reference()
    for b, s in [(64, 1), (64, 64), (64, 65), (64, 50000), (4, 13)]:
        r, o = ref.BlockLayout(b, s), BlockLayout(b, s)
        assert (r.num_blocks, r.padded_len) == (o.num_blocks, o.padded_len)
        np.testing.assert_array_equal(r.valid_rows, o.valid_rows)
    with pytest.raises(E.LayoutError):
        IclLayout(0, 5)
    with pytest.raises(E.LayoutError):
        IclLayout(5, -1)
    assert IclLayout(3, 4).total == 7


def test_derived_counts_use_reference_float_expressions():
    """k_ctx (coarse.py:156), n_flat (coarse.py:197), k (coarse.py:169) on a
    sweep that includes representation-sensitive products like 0.3*10."""
    rng = np.random.default_rng(0)
    alphas = [0.0, 0.0625, 0.1, 0.125, 0.25, 0.3, 0.5, 0.7, 0.75, 0.9, 1.0] + list(rng.random(20))
    for a_s in alphas:
        for a_f in alphas[:12]:
            for a_ns in [0.0625, 0.1, 0.3, 1.0]:
                for l_src, l_ctx in [(1024, 1024), (640, 1920), (50000, 50000), (64, 0)]:
                    cfg = IsaConfig(alpha_s=a_s, alpha_f=a_f, alpha_ns=a_ns)
                    d = IsaDims.derive((1, 1, l_src + l_ctx, 128), IclLayout(l_src, l_ctx), cfg)
                    t_src, t_ctx = -(-l_src // 64), (-(-l_ctx // 64) if l_ctx else 0)
                    T = t_src + t_ctx
                    k_ctx = int(math.floor(a_s * t_ctx)) if t_ctx else 0
                    t_new = t_src + k_ctx
                    n_flat = int(math.floor(a_f * T))
                    assert (d.T, d.k_ctx, d.t_new, d.n_flat, d.n_sharp) == (T, k_ctx, t_new, n_flat, T - n_flat)
                    if n_flat:
                        assert d.k == min(t_new, max(1, int(math.floor(a_ns * t_new))))


def test_flops_match_reference_pipeline_flops():
    ref = _reference()
    rng = np.random.default_rng(1)
    q, k, v = (rng.standard_normal((1, 2, 512, 8)) for _ in range(3))
    for over in (dict(), dict(alpha_f=0.0, alpha_s=1.0), dict(alpha_f=1.0, alpha_ns=1.0), dict(alpha_s=0.5)):
        cfg = dict(block_size=64, **over)
        _, tr = ref.isa_forward(q, k, v, ref.IclLayout(256, 256), ref.IsaConfig(**cfg))
        ours = IsaDims.derive(q.shape, IclLayout(256, 256), IsaConfig(**cfg)).flops()
        assert (tr.flops.exact_mas, tr.flops.taylor_mas, tr.flops.overhead_mas, tr.flops.dense_equivalent_mas) == \
            (ours.exact_mas, ours.taylor_mas, ours.overhead_mas, ours.dense_equivalent_mas)


def test_error_taxonomy_mirrors_reference():
    ref = _reference()
    for name in ("IsaError", "LayoutError", "InputError", "BlockIndexError", "ContractError", "ConfigError",
                 "FormatError", "DegenerateRowError", "NumericError"):
        ours, theirs = getattr(E, name), getattr(ref, name)
        assert [c.__name__ for c in ours.__mro__[:-2]] == [c.__name__ for c in theirs.__mro__[:-2]]


# ------------------------------------------------------------------ the C ABI (.so) without a GPU
def _header_functions():
    text = open(os.path.join(ROOT, "include", "isa_b200.h")).read()
    return sorted(set(re.findall(r"^int\s+(isa_\w+)\s*\(|^const char\*\s+(isa_\w+)\s*\(", text, re.M)))


def test_library_exports_every_header_symbol():
    from paper_2605_04569_b200 import _native as N

    lib = N.load()
    names = {a or b for a, b in _header_functions()}
    assert names == set(N.EXPORTED_SYMBOLS), names ^ set(N.EXPORTED_SYMBOLS)
    for name in names:
        assert hasattr(lib, name)
    assert lib.isa_abi_version() == N.ISA_ABI_VERSION


def _shape(N, B=1, H=40, S=65536, D=128, l_src=32768, l_ctx=32768, block=64, dtype=0):
    return N.IsaShape(B, H, S, D, l_src, l_ctx, block, dtype, H * S * D, S * D, D)


def test_workspace_query_and_status_codes_on_cpu():
    """isa_workspace_bytes is pure host arithmetic: callable without a GPU,
    and its validation maps onto the reference exception classes."""
    from paper_2605_04569_b200 import _native as N

    lib = N.load()
    nb = ctypes.c_size_t(0)
    kn = N.IsaKnobs(1 / math.sqrt(128), 64, 512, 36, 1, 0)
    assert lib.isa_workspace_bytes(ctypes.byref(_shape(N)), ctypes.byref(kn), ctypes.byref(nb)) == 0
    assert 100e6 < nb.value < 1e9
    cases = [
        (_shape(N, block=32), kn, E.ConfigError),
        (_shape(N, D=96), kn, E.ConfigError),
        (_shape(N, l_src=1000), kn, E.LayoutError),
        (_shape(N), N.IsaKnobs(0.0, 64, 512, 36, 1, 0), E.ConfigError),
        (_shape(N), N.IsaKnobs(0.1, 513, 512, 36, 1, 0), E.ConfigError),
        (_shape(N), N.IsaKnobs(0.1, 64, 512, 0, 1, 0), E.ConfigError),
    ]
    for sh, k, err in cases:
        rc = lib.isa_workspace_bytes(ctypes.byref(sh), ctypes.byref(k), ctypes.byref(nb))
        assert E.STATUS_TO_ERROR[rc] is err
        with pytest.raises(err):
            N.check(rc)


def test_native_missing_library_fails_loudly(tmp_path):
    from paper_2605_04569_b200 import _native as N

    with pytest.raises(E.NativeError):
        N._lib_saved = N._lib
        try:
            N._lib = None
            N.load(str(tmp_path / "nope.so"))
        finally:
            N._lib = N._lib_saved


def test_cpu_tensors_are_rejected_no_fallback():
    """Host data is only ever streamed through the GPU: without one the call
    fails loudly instead of computing on the CPU."""
    torch = pytest.importorskip("torch")
    import paper_2605_04569_b200 as P

    if torch.cuda.is_available():
        pytest.skip("a GPU is present: host data takes the streamed path")
    x = torch.zeros(1, 1, 128, 64)
    with pytest.raises(E.LayoutError):
        P.isa_forward(x, x, x, P.IclLayout(64, 64), P.IsaConfig())
    with pytest.raises(E.LayoutError):
        P.isa_forward(x.numpy(), x.numpy(), x.numpy(), P.IclLayout(64, 64), P.IsaConfig())


def test_host_stream_plan_on_cpu():
    """isa_forward_host_bytes: staging = 2 slots x (3 inputs + 1 output) chunks;
    the chunk workspace equals isa_workspace_bytes of a (1, hc, S, D) problem."""
    from paper_2605_04569_b200 import _native as N

    lib = N.load()
    kn = N.IsaKnobs(1 / math.sqrt(128), 64, 512, 36, 1, 0)
    st, ws = ctypes.c_size_t(0), ctypes.c_size_t(0)
    assert lib.isa_forward_host_bytes(ctypes.byref(_shape(N)), ctypes.byref(kn), 5, ctypes.byref(st),
                                      ctypes.byref(ws)) == 0
    assert st.value == 2 * 4 * 5 * 65536 * 128 * 2
    one = ctypes.c_size_t(0)
    assert lib.isa_workspace_bytes(ctypes.byref(_shape(N, H=5)), ctypes.byref(kn), ctypes.byref(one)) == 0
    assert ws.value == one.value
    # default chunking: about 150 MB of inputs (3 heads of 3 x 65536 x 128 bf16)
    assert lib.isa_forward_host_bytes(ctypes.byref(_shape(N)), ctypes.byref(kn), 0, ctypes.byref(st),
                                      ctypes.byref(ws)) == 0
    assert st.value == 2 * 4 * 3 * 65536 * 128 * 2
    # non-contiguous host layouts are rejected (LayoutError)
    sh = _shape(N)
    sh.stride_s = 256
    rc = lib.isa_forward_host_bytes(ctypes.byref(sh), ctypes.byref(kn), 5, ctypes.byref(st), ctypes.byref(ws))
    assert E.STATUS_TO_ERROR[rc] is E.LayoutError


def test_head_dim_padding_plan():
    """Head dims other than 64/128 (up to 128) are zero-padded to the next
    kernel width with the scale pinned to 1/sqrt(D) of the real width."""
    import math

    import torch

    from paper_2605_04569_b200 import IsaConfig
    from paper_2605_04569_b200.pipeline import _pad_head_dim, _unpad

    for D, width in ((1, 64), (32, 64), (63, 64), (65, 128), (96, 128), (127, 128)):
        x = torch.randn(1, 2, 3, D)
        cfg, px, pn = _pad_head_dim(IsaConfig(), x, x.numpy())
        assert px.shape[-1] == width and pn.shape[-1] == width
        assert cfg.scale == 1.0 / math.sqrt(D)
        assert torch.equal(px[..., :D], x) and not px[..., D:].any()
        assert torch.equal(_unpad(px, D), x)
    assert _pad_head_dim(IsaConfig(scale=0.5), torch.ones(1, 1, 1, 40))[0].scale == 0.5
    for D in (64, 128, 129, 256):
        assert _pad_head_dim(IsaConfig(), torch.ones(1, 1, 1, D)) is None


def test_error_metrics_match_reference_definitions():
    """util.py:8-29 restated: numpy and (CPU) torch inputs give the same numbers."""
    import numpy as np
    import torch

    from paper_2605_04569_b200 import elementwise_relative_error, max_relative_error, mean_relative_error

    rng = np.random.default_rng(3)
    a, r = rng.standard_normal((2, 3, 5, 4)), rng.standard_normal((2, 3, 5, 4))
    assert max_relative_error(a, r) == float(np.max(np.abs(a - r))) / float(np.max(np.abs(r)))
    assert abs(mean_relative_error(a, r) - float(np.mean(np.abs(a - r))) / float(np.mean(np.abs(r)))) < 1e-15
    want = float(np.max(np.abs(a - r) / (np.maximum(np.abs(a), np.abs(r)) + 1e-12)))
    assert abs(elementwise_relative_error(a, r) - want) < 1e-15
    assert abs(max_relative_error(torch.from_numpy(a), torch.from_numpy(r)) - max_relative_error(a, r)) < 1e-15
    assert max_relative_error(np.zeros(0), np.zeros(0)) == 0.0
