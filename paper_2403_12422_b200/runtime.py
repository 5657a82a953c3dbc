"""Runtime knobs and the asynchronous error word.

Kernels that can hit a data-dependent error (non-finite input, binary16
scale overflow — qtensor.py:189,210) OR a flag into one device int32; the
host turns it into the reference's ``ValueError`` text.  In ``eager`` mode
(the default, exactly the reference's behaviour) every op that can fail
synchronizes and checks; in ``deferred`` mode the check happens at
``check_errors()`` (once per training step), so steps stay sync-free.
"""

from __future__ import annotations

import functools
import os
import threading

import torch

from . import _lib

_MSG_NONFINITE = "input contains non-finite values"
_MSG_OVERFLOW = "scale overflows the binary16 range; input magnitude too large"

_state = threading.local()
_config = {"error_check": "eager", "promotion": "exact", "operands": "int8", "attention": "sdpa"}
_gemm_options = {"tma_scales": 1}


def set_error_check(mode: str) -> None:
    """'eager' (raise from the failing call, reference semantics) or 'deferred'."""
    if mode not in ("eager", "deferred"):
        raise ValueError(f"error_check must be 'eager' or 'deferred', got {mode!r}")
    _config["error_check"] = mode


def get_error_check() -> str:
    return _config["error_check"]


def set_promotion(mode: str) -> None:
    """GEMM promotion: 'exact' (bit-exact with qgemm.py) or 'fast' (one rounding less)."""
    if mode not in ("exact", "fast"):
        raise ValueError(f"promotion must be 'exact' or 'fast', got {mode!r}")
    _config["promotion"] = mode


def set_gemm_option(key: str, value: int) -> None:
    """Diagnostics / A-B: libjetfire GEMM launch option (jf_gemm_set_option).  Results are
    bit-identical for every option; ``tma_scales=0`` also brings back the transposed
    operand copies the generic kernel needs."""
    rc = _lib.lib().jf_gemm_set_option(key.encode(), int(value))
    if rc != 0:
        raise ValueError(f"unknown GEMM option {key!r}")
    _gemm_options[key] = int(value)


def gemm_option(key: str) -> int | None:
    return _gemm_options.get(key)


def get_promotion() -> str:
    return _config["promotion"]


def set_gemm_operands(kind: str) -> None:
    """GEMM operand path for shapes that are multiples of 128: 'int8' (default: tcgen05
    kind::i8 on the codes as stored, int32 TMEM partials -- the north-star design), 'f16'
    (opt-in experiment: the codes widened to f16 -- exact -- and multiplied with
    kind::f16, whose f32 partials need no int->float conversion in the promotion; the
    widened copies are GEMM operand staging in HBM), or 'auto' (f16 for GEMMs of at least
    F16_MIN_FLOP, int8 below).  All are bit-identical; DESIGN.md section 3 has the numbers."""
    if kind not in ("int8", "f16", "auto"):
        raise ValueError(f"operands must be 'int8', 'f16' or 'auto', got {kind!r}")
    _config["operands"] = kind


def set_attention(kind: str) -> None:
    """Attention island of the INT8 block (qlayers.py:187-236, boundary :350-351/:406-408):
    'sdpa' (default: codes dequantized to bf16 head tensors, cuDNN SDPA, outputs
    requantized by boundary kernels) or 'fused' (libjetfire's tcgen05 attention kernels
    read the INT8 QKV / dO codes and write INT8 O / dQ|dK|dV directly: no bf16 head
    tensor in HBM).  Both compute in bf16 with FP32 accumulation; 'fused' needs
    seq % 256 == 0 and head_dim in {64, 128} (other shapes use 'sdpa')."""
    if kind not in ("sdpa", "fused"):
        raise ValueError(f"attention must be 'sdpa' or 'fused', got {kind!r}")
    _config["attention"] = kind


def attention() -> str:
    return _config["attention"]


# 'auto' threshold: measured on B200 -- 4096x12288x4096 and larger gain 7% with f16
# operands, 4096^3 breaks even, the 8192x1024-wide GPT-2 GEMMs lose to the widening launches.
F16_MIN_FLOP = 2 ** 38


def gemm_operands() -> str:
    return _config["operands"]


# ── weight-gradient overlap ───────────────────────────────────────────────
# dW = dY^T X does not feed the rest of backward, so TransformerBlock.backward
# issues it on a side stream (QuantLinear.backward(defer_wgrad=True)): its tiles
# fill the SMs the dgrad GEMM and the elementwise kernels leave idle (few-tile
# GEMMs of 1024-wide models), and joins before publishing the gradients.
# Bit-identical either way; on by default.
_overlap = {"wgrad": True}
_side_streams: dict = {}
_pending: list = []


def set_overlap_wgrad(flag: bool) -> None:
    _overlap["wgrad"] = bool(flag)


def overlap_wgrad() -> bool:
    return _overlap["wgrad"]


def side_stream(device) -> "torch.cuda.Stream":
    import torch

    key = torch.device(device).index
    if key not in _side_streams:
        _side_streams[key] = torch.cuda.Stream(device=device)
    return _side_streams[key]


def defer_join(event, outputs, keepalive=()) -> None:
    """Record side-stream work the current stream must wait for.  ``keepalive``: inputs
    the side stream reads -- referenced until the join, so the caching allocator cannot
    hand their memory to new work before the side stream is done with it.  Outputs need
    no bookkeeping: the side stream waits on the current stream before every new batch
    of work, so a block the current stream freed is never still in use there."""
    _pending.append((event, outputs, keepalive))


def join_side_streams() -> None:
    """Make the current stream wait for all deferred side-stream work."""
    if not _pending:
        return
    import torch

    main = torch.cuda.current_stream()
    for ev, _, _ in _pending:
        main.wait_event(ev)
    _pending.clear()


def promotion_code(mode: str | None) -> int:
    m = mode or _config["promotion"]
    if m not in ("exact", "fast"):
        raise ValueError(f"promotion must be 'exact' or 'fast', got {m!r}")
    return _lib.MODE_EXACT if m == "exact" else _lib.MODE_FAST


def _word(device=None) -> torch.Tensor:
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    words = getattr(_state, "words", None)
    if words is None:
        words = _state.words = {}
    w = words.get(dev.index)
    if w is None:
        w = words[dev.index] = torch.zeros(1, dtype=torch.int32, device=dev)
    return w


_cur_dev = getattr(torch._C, "_cuda_getDevice", None) or torch.cuda.current_device


def err_ptr() -> int:
    """Device address of this thread's error word on the current device (cached: this runs
    once per kernel launch)."""
    dev = _cur_dev()
    ptrs = getattr(_state, "ptrs", None)
    if ptrs is None:
        ptrs = _state.ptrs = {}
    p = ptrs.get(dev)
    if p is None:
        p = ptrs[dev] = _word(dev).data_ptr()
    return p


def check_errors() -> None:
    """Synchronize on the error word; raise the reference's ValueError if set."""
    w = _word()
    flags = int(w.item())
    if flags:
        w.zero_()
        if flags & _lib.JF_EFLAG_NONFINITE:
            raise ValueError(_MSG_NONFINITE)
        raise ValueError(_MSG_OVERFLOW)


def maybe_check() -> None:
    # (no host sync while a CUDA graph is being captured: the error word is read after replay)
    if _config["error_check"] == "eager" and not torch.cuda.is_current_stream_capturing():
        check_errors()


# ── NVTX ranges (SURVEY.md §5 tracing) ──────────────────────────────────────
# Off by default (one dict lookup per op).  ``set_nvtx(True)`` or JF_NVTX=1 wraps every
# public op (quantizer, the three GEMMs, Add+stats, LayerNorm, GELU, dropout, the
# attention island, QuantLinear / TransformerBlock fwd+bwd, the model step and AdamW) in
# a named range, so an nsys timeline or ``ncu --nvtx`` attributes kernels to operators.
_nvtx = {"on": os.environ.get("JF_NVTX", "0") == "1"}


def set_nvtx(flag: bool) -> None:
    _nvtx["on"] = bool(flag)


def nvtx_enabled() -> bool:
    return _nvtx["on"]


def traced(name: str):
    """Decorator: run ``fn`` inside NVTX range ``name`` when NVTX is on."""
    def deco(fn):
        @functools.wraps(fn)
        def wrapper(*args, **kwargs):
            if not _nvtx["on"]:
                return fn(*args, **kwargs)
            torch.cuda.nvtx.range_push(name)
            try:
                return fn(*args, **kwargs)
            finally:
                torch.cuda.nvtx.range_pop()
        return wrapper
    return deco
