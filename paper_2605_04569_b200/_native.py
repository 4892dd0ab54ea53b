"""ctypes binding of libisa_b200.so (C ABI declared in include/isa_b200.h).

The library is required: importing the operator API on a machine without the
built .so raises `NativeError` at call time instead of falling back to any CPU
path. Every call passes raw device pointers and the current CUDA stream.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import ISA_OK, STATUS_TO_ERROR, NativeError

HERE = os.path.dirname(os.path.abspath(__file__))
# ISA_B200_LIB points at an alternative build of the same C ABI (A/B kernel measurements)
LIB_PATH = os.environ.get("ISA_B200_LIB") or os.path.join(HERE, "libisa_b200.so")

ISA_ABI_VERSION = 4
ISA_DTYPE_BF16 = 0
ISA_DTYPE_F32 = 1

EXPORTED_SYMBOLS = (
    "isa_abi_version",
    "isa_last_error",
    "isa_last_launch_count",
    "isa_workspace_bytes",
    "isa_forward",
    "isa_routing",
    "isa_dense_attention",
    "isa_pool_means",
    "isa_topk_rows_f64",
    "isa_sharpness_rows_f64",
    "isa_split_rows_f64",
    "isa_forward_host_bytes",
    "isa_forward_host",
    "isa_decoupled_rope",
    "isa_backward_workspace_bytes",
    "isa_backward",
    "isa_taylor_workspace_bytes",
    "isa_taylor_forward",
    "isa_cross_attention",
    "isa_coarse_scores",
    "isa_ctx_saliency_f64",
    "isa_forward_signal",
    "isa_stream_wait_geq",
)

# IsaKnobs.flags
FLAG_SEPARATE_BRANCHES = 1
FLAG_TAYLOR_K7 = 2
FLAG_TAYLOR_K7T = 4
FLAG_FUSED_GRID = 8
FLAG_SINGLE_CTA = 16

# err_word bits (include/isa_b200.h ISA_ERRBIT_*)
ERRBIT_INPUT = 1
ERRBIT_DEGENERATE = 2
ERRBIT_SEL_RANGE = 4
ERRBIT_SEL_ORDER = 8
ERRBIT_SPLIT_RANGE = 16
ERRBIT_SPLIT_ORDER = 32
ERRBIT_MASK = 64


class IsaShape(ctypes.Structure):
    _fields_ = [
        ("batch", ctypes.c_int32),
        ("heads", ctypes.c_int32),
        ("seq_len", ctypes.c_int32),
        ("head_dim", ctypes.c_int32),
        ("l_src", ctypes.c_int32),
        ("l_ctx", ctypes.c_int32),
        ("block", ctypes.c_int32),
        ("dtype", ctypes.c_int32),
        ("stride_b", ctypes.c_int64),
        ("stride_h", ctypes.c_int64),
        ("stride_s", ctypes.c_int64),
        ("out_stride_b", ctypes.c_int64),
        ("out_stride_h", ctypes.c_int64),
        ("out_stride_s", ctypes.c_int64),
    ]


class IsaKnobs(ctypes.Structure):
    _fields_ = [
        ("scale", ctypes.c_double),
        ("k_ctx", ctypes.c_int32),
        ("n_flat", ctypes.c_int32),
        ("k_mask", ctypes.c_int32),
        ("softmax_first", ctypes.c_int32),
        ("flags", ctypes.c_int32),
        ("gamma", ctypes.c_double),
        ("residual_softmax", ctypes.c_int32),
        ("_pad", ctypes.c_int32),
        ("rope_base", ctypes.c_double),
    ]


class IsaRoutingOut(ctypes.Structure):
    _fields_ = [
        ("selection", ctypes.c_void_p),
        ("sharp", ctypes.c_void_p),
        ("flat", ctypes.c_void_p),
        ("mask", ctypes.c_void_p),
        ("sharpness", ctypes.c_void_p),
        ("ctx_scores", ctypes.c_void_p),
        ("taylor_kernel", ctypes.c_void_p),
    ]


class IsaRoutingIn(ctypes.Structure):
    _fields_ = [
        ("selection", ctypes.c_void_p),
        ("sharp", ctypes.c_void_p),
        ("flat", ctypes.c_void_p),
        ("mask", ctypes.c_void_p),
    ]


class IsaEvents(ctypes.Structure):
    _fields_ = [("ev", ctypes.c_void_p * 6)]


_lib = None
_lock = threading.Lock()

_P = ctypes.c_void_p
_I = ctypes.c_int32
_SIGS = {
    "isa_abi_version": (ctypes.c_int, []),
    "isa_last_error": (ctypes.c_char_p, []),
    "isa_last_launch_count": (ctypes.c_int, []),
    "isa_workspace_bytes": (ctypes.c_int, [ctypes.POINTER(IsaShape), ctypes.POINTER(IsaKnobs),
                                           ctypes.POINTER(ctypes.c_size_t)]),
    "isa_forward": (ctypes.c_int, [ctypes.POINTER(IsaShape), ctypes.POINTER(IsaKnobs), _P, _P, _P, _P, _P,
                                   ctypes.c_size_t, ctypes.POINTER(IsaRoutingIn), ctypes.POINTER(IsaRoutingOut),
                                   _P, ctypes.POINTER(IsaEvents), _P]),
    "isa_routing": (ctypes.c_int, [ctypes.POINTER(IsaShape), ctypes.POINTER(IsaKnobs), _P, _P, _P, _P,
                                   ctypes.c_size_t, ctypes.POINTER(IsaRoutingOut), _P, _P]),
    "isa_dense_attention": (ctypes.c_int, [ctypes.POINTER(IsaShape), ctypes.c_double, _P, _P, _P, _P, _P]),
    "isa_pool_means": (ctypes.c_int, [ctypes.POINTER(IsaShape), _P, _P, _P, _P, _P, _P]),
    "isa_topk_rows_f64": (ctypes.c_int, [_P, _I, _I, _I, _P, _I, _P]),
    "isa_sharpness_rows_f64": (ctypes.c_int, [_P, _I, _I, _I, _P, _P]),
    "isa_split_rows_f64": (ctypes.c_int, [_P, _I, _I, _I, _P, _P, _P]),
    "isa_forward_signal": (ctypes.c_int, [ctypes.POINTER(IsaShape), ctypes.POINTER(IsaKnobs), _P, _P, _P, _P, _P,
                                          ctypes.c_size_t, _P, _P, ctypes.POINTER(ctypes.c_int32), _P]),
    "isa_stream_wait_geq": (ctypes.c_int, [_P, _P, _I]),
    "isa_coarse_scores": (ctypes.c_int, [_I, _I, _I, _I, ctypes.c_double, _P, _P, _P, _P]),
    "isa_ctx_saliency_f64": (ctypes.c_int, [_P, _I, ctypes.c_int64, ctypes.c_int64, _I, _I, _P, _P]),
    "isa_backward_workspace_bytes": (ctypes.c_int, [ctypes.POINTER(IsaShape), ctypes.POINTER(IsaKnobs),
                                                    ctypes.POINTER(ctypes.c_size_t)]),
    "isa_backward": (ctypes.c_int, [ctypes.POINTER(IsaShape), ctypes.POINTER(IsaKnobs), _P, _P, _P, _P, _P, _P, _P,
                                    _P, ctypes.c_size_t, ctypes.POINTER(IsaRoutingIn), _P, _P]),
    "isa_decoupled_rope": (ctypes.c_int, [ctypes.POINTER(IsaShape), ctypes.c_double, _P, _P, _P]),
    "isa_cross_attention": (ctypes.c_int, [ctypes.POINTER(IsaShape), _I, ctypes.POINTER(ctypes.c_int64),
                                           ctypes.c_double, _P, _P, _P, _P, _P]),
    "isa_taylor_workspace_bytes": (ctypes.c_int, [ctypes.POINTER(IsaShape), _I, _I,
                                                  ctypes.POINTER(ctypes.c_size_t)]),
    "isa_taylor_forward": (ctypes.c_int, [ctypes.POINTER(IsaShape), _I, ctypes.POINTER(ctypes.c_int64), _I,
                                          ctypes.c_double, _P, _P, _P, _P, _P, _P, _P, _P, ctypes.c_size_t, _P,
                                          _P]),
    "isa_forward_host_bytes": (ctypes.c_int, [ctypes.POINTER(IsaShape), ctypes.POINTER(IsaKnobs), _I,
                                              ctypes.POINTER(ctypes.c_size_t), ctypes.POINTER(ctypes.c_size_t)]),
    "isa_forward_host": (ctypes.c_int, [ctypes.POINTER(IsaShape), ctypes.POINTER(IsaKnobs), _P, _P, _P, _P, _I, _P,
                                        ctypes.c_size_t, _P, ctypes.c_size_t, ctypes.POINTER(IsaRoutingIn),
                                        ctypes.POINTER(IsaRoutingOut), _P, ctypes.POINTER(_P)]),
}


def load(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load (once) and type the C ABI. Raises NativeError when the .so is absent."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise NativeError(
                f"{path} not built; run `python -m paper_2605_04569_b200.build` (there is no CPU fallback)")
        lib = ctypes.CDLL(path)
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.isa_abi_version() != ISA_ABI_VERSION:
            raise NativeError(f"ABI mismatch: library {lib.isa_abi_version()} != {ISA_ABI_VERSION}")
        _lib = lib
        return lib


def check(status: int) -> None:
    """Map an IsaStatus onto the reference exception classes (errors.py)."""
    if status == ISA_OK:
        return
    lib = load()
    msg = lib.isa_last_error().decode(errors="replace")
    raise STATUS_TO_ERROR.get(status, NativeError)(msg)
