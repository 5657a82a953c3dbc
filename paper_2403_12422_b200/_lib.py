"""ctypes binding of libjetfire.so (the C ABI declared in include/jetfire.h).

The product path has no CPU fallback: if the shared library or a CUDA
device is missing, every op raises ``JetfireUnavailable``.
"""

from __future__ import annotations

import ctypes
import os
import threading

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# JF_LIBJETFIRE: an alternative in-tree build (diagnostics / A-B of kernel variants)
LIB_PATH = os.environ.get("JF_LIBJETFIRE") or os.path.join(_HERE, "libjetfire.so")

JF_EFLAG_NONFINITE = 1
JF_EFLAG_OVERFLOW = 2
MODE_EXACT = 0
MODE_FAST = 1
OUT_INT8 = 0
OUT_F32 = 1
OUT_INT8_DEQ = 2


class JetfireUnavailable(RuntimeError):
    """libjetfire.so or a CUDA device is missing (there is no CPU fallback)."""


_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int32
_F32 = ctypes.c_float
_SZ = ctypes.c_size_t

# name -> (restype, argtypes); mirrors include/jetfire.h exactly
SIGNATURES = {
    "jf_version": (ctypes.c_int, []),
    "jf_last_error": (ctypes.c_char_p, []),
    "jf_sm_count": (ctypes.c_int, []),
    "jf_quantize_f32": (ctypes.c_int, [_P, _I64, _I64, _I64, _P, _P, _P, _P]),
    "jf_quantize_bf16": (ctypes.c_int, [_P, _I64, _I64, _I64, _P, _P, _P, _P]),
    "jf_dequantize_f32": (ctypes.c_int, [_P, _P, _I64, _I64, _P, _P]),
    "jf_dequantize_bf16": (ctypes.c_int, [_P, _P, _I64, _I64, _P, _P]),
    "jf_transpose": (ctypes.c_int, [_P, _P, _I64, _I64, _P, _P, _P]),
    "jf_gemm_fwd": (ctypes.c_int, [_P, _P, _P, _P, _P, _I64, _I64, _I64, _I32, _I32, _P, _P, _P, _P, _P]),
    "jf_gemm_dgrad": (ctypes.c_int, [_P, _P, _P, _P, _P, _P, _I64, _I64, _I64, _I32, _I32, _P, _P, _P,
                                     _P, _P, _P]),
    "jf_gemm_wgrad": (ctypes.c_int, [_P, _P, _P, _P, _P, _P, _P, _P, _I64, _I64, _I64, _I32, _I32, _P, _P, _P,
                                     _P, _P, _P]),
    "jf_gemm_scratch_bytes": (_SZ, [_I32, _I64, _I64, _I64]),
    "jf_widen_codes": (ctypes.c_int, [_P, _I64, _I64, _P, _I32, _P]),
    "jf_gemm_f16": (ctypes.c_int, [_P, _P, _I64, _I64, _P, _P, _I64, _I64, _P, _I64, _I64, _I64, _I32, _I32,
                                   _P, _P, _P, _P, _P]),
    "jf_gemm_partials": (ctypes.c_int, [_P, _P, _I64, _I64, _I64, _I64, _P, _P]),
    "jf_add_stats": (ctypes.c_int, [_P, _P, _P, _P, _I64, _I64, _I64, _P, _P, _P, _P, _P, _P]),
    "jf_ln_fwd": (ctypes.c_int, [_P, _P, _P, _P, _I64, _I64, _I64, _P, _P, _F32, _P, _P, _P, _P, _P, _P]),
    "jf_ln_bwd": (ctypes.c_int, [_P, _P, _P, _P, _P, _P, _P, _I64, _I64, _P, _P, _P, _P, _P, _P, _P]),
    "jf_ln_bwd_workspace_bytes": (_SZ, [_I64, _I64]),
    "jf_gelu_tables_bytes": (_SZ, []),
    "jf_gelu_build_tables": (ctypes.c_int, [_P, _P]),
    "jf_gelu_fwd": (ctypes.c_int, [_P, _P, _I64, _I64, _P, _P, _P, _P, _P]),
    "jf_gelu_bwd": (ctypes.c_int, [_P, _P, _P, _P, _I64, _I64, _P, _P, _P, _P, _P]),
    "jf_colsum": (ctypes.c_int, [_P, _P, _I64, _I64, _P, _P, _P]),
    "jf_colsum_workspace_bytes": (_SZ, [_I64, _I64]),
    "jf_philox_keep": (ctypes.c_int, [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_double, _I64, _P, _P]),
    "jf_dropout": (ctypes.c_int, [_P, _P, _P, _F32, _I64, _I64, _P, _P, _P, _P]),
    "jf_gemm_set_option": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_int]),
    "jf_adamw": (ctypes.c_int, [_P, _P, _P, _P, _I64, _F32, ctypes.c_double, ctypes.c_double, _F32, _F32, _F32,
                                _F32, _P]),
    "jf_adamw_multi": (ctypes.c_int, [_P, _P, _P, _I32, _I64, _F32, ctypes.c_double, ctypes.c_double, _F32, _F32,
                                      _F32, _P]),
    "jf_adamw_quantize": (ctypes.c_int, [_P, _P, _P, _P, _I64, _I64, _F32, ctypes.c_double, ctypes.c_double, _F32,
                                         _F32, _F32, _F32, _P, _P, _P, _P]),
    "jf_adamw_quantize_multi": (ctypes.c_int, [_P, _I32, _I64, _F32, ctypes.c_double, ctypes.c_double, _F32, _F32,
                                               _F32, _P, _P]),
    "jf_cross_entropy_bf16": (ctypes.c_int, [_P, _I64, _I64, _I64, _P, _P, _P, _P, _P, _P]),
    "jf_dequantize_qkv_heads": (ctypes.c_int, [_P, _P, _I64, _I64, _I64, _I64, _P, _P, _P, _P]),
    "jf_quantize_heads_bf16": (ctypes.c_int, [_P, _I64, _I64, _I64, _I64, _I64, _I64, _I64, _P, _I64, _P, _I64,
                                              _P, _P]),
    "jf_attn_supported": (ctypes.c_int, [_I64, _I64]),
    "jf_attn_set_mn_desc": (ctypes.c_int, [ctypes.c_uint32, ctypes.c_uint32]),
    "jf_attn_set_trace": (ctypes.c_int, [_P]),
    "jf_attn_fwd_q": (ctypes.c_int, [_P, _P, _I64, _I64, _I64, _I64, _P, _P, _P, _P, _P, _P]),
    "jf_attn_bwd_q": (ctypes.c_int, [_P, _P, _P, _P, _P, _P, _P, _I64, _I64, _I64, _I64, _P, _P, _P, _P]),
}

_lib = None
_lock = threading.Lock()


def load_library(path: str = LIB_PATH):
    """Load and type the shared library (no CUDA device needed)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise JetfireUnavailable(
                f"{path} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            )
        lib = ctypes.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        extra = getattr(lib, "jf_set_gemm_magic", None)
        if extra is not None:
            extra.restype = None
            extra.argtypes = [ctypes.c_int]
        _lib = lib
        return lib


def lib():
    """The library, after checking a CUDA device exists (fails loudly otherwise)."""
    if not torch.cuda.is_available():
        raise JetfireUnavailable("no CUDA device: the Jetfire B200 path has no CPU fallback")
    return load_library()


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)
_get_device = getattr(torch._C, "_cuda_getDevice", None)


def stream_handle() -> int:
    """The current CUDA stream of the current device (C-level lookups: this runs once per
    kernel launch, and torch.cuda.current_stream() costs ~10 us of Python)."""
    if _raw_stream is not None and _get_device is not None:
        return _raw_stream(_get_device())
    return torch.cuda.current_stream().cuda_stream


# kernels each C entry point enqueues (for bench.py's gpu_launches tally)
KERNELS_PER_CALL = {
    "quantize": 1, "dequantize": 1, "transpose": 1, "gemm_fwd": 1, "gemm_dgrad": 1, "gemm_wgrad": 1,
    "gemm_partials": 1, "add_stats": 1, "ln_fwd": 2, "ln_bwd": 3, "gelu_fwd": 1, "gelu_bwd": 1,
    "colsum": 2, "dropout": 1, "philox_keep": 1, "gelu_tables": 1, "dequant_qkv_heads": 1, "quantize_heads": 1,
    "cross_entropy": 1, "attn_fwd": 1, "attn_bwd": 2, "adamw": 1, "adamw_quantize": 1, "adamw_multi": 1, "adamw_quantize_multi": 1, "widen_codes": 1, "gemm_f16": 1,
}
launch_count = [0]


def check(rc: int, what: str) -> None:
    launch_count[0] += KERNELS_PER_CALL.get(what, 1)
    if rc != 0:
        msg = _lib.jf_last_error().decode(errors="replace") if _lib is not None else ""
        raise RuntimeError(f"libjetfire {what} failed (status {rc}): {msg}")
