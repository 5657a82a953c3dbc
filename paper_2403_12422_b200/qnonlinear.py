"""Fused INT8-in/INT8-out operators on the GPU (drop-in for int8flow.qnonlinear).

Mirrors ``int8flow/qnonlinear.py``: RowStats :103-131, add_forward
:246-267, NormParams :273-287, LayerNormContext :290-297, layernorm_forward
:300-330, layernorm_backward :333-355, gelu_forward/backward :150-175,
DropoutState / dropout_forward / dropout_backward :181-240,
count_elementwise :76-97.  Each op is one libjetfire launch (K6-K10) that
dequantizes, computes in the reference's float32 order, and requantizes per
32x32 block before anything reaches HBM.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from . import runtime as _rt
from .qgemm import AccessCounters, ExecMode
from .qtensor import BlockQuantTensor, empty_like_shape, snap_to_f16


def count_elementwise(counters, mode, in_elems, out_elems, dequant_elems=0, quant_elems=0) -> None:
    """Analytic traffic tally (qnonlinear.py:76-97)."""
    if counters is None:
        return
    if mode is ExecMode.INT8_DATA_FLOW:
        counters.int8_load_store += in_elems + out_elems
        counters.dequant_ops += dequant_elems
        counters.quant_ops += quant_elems
    else:
        counters.fp16_load_store += in_elems + out_elems


@dataclass
class RowStats:
    """Per-row, per-column-block mean and sum of squares (CUDA float32 [N, C/width])."""

    mean: torch.Tensor
    sumsq: torch.Tensor
    width: int

    def __post_init__(self):
        if tuple(self.mean.shape) != tuple(self.sumsq.shape):
            raise ValueError("mean and sumsq shapes differ")

    @property
    def cols(self) -> int:
        return self.mean.shape[1] * self.width


@dataclass
class NormParams:
    gamma: torch.Tensor
    beta: torch.Tensor
    eps: float = 1e-5

    def __post_init__(self):
        if self.eps <= 0:
            raise ValueError(f"eps must be positive, got {self.eps}")
        self.gamma = _vec(self.gamma)
        self.beta = _vec(self.beta)
        if self.gamma.shape != self.beta.shape or self.gamma.dim() != 1:
            raise ValueError("gamma and beta must be equal-length vectors")


def _vec(v) -> torch.Tensor:
    if isinstance(v, np.ndarray):
        v = torch.from_numpy(np.ascontiguousarray(v, dtype=np.float32))
    v = torch.as_tensor(v, dtype=torch.float32)
    if not v.is_cuda and torch.cuda.is_available():
        v = v.cuda()
    return v.contiguous()


@dataclass
class LayerNormContext:
    """Saved for backward: the INT8 input plus per-row moments (x-hat is recomputed)."""

    xq: BlockQuantTensor
    mu: torch.Tensor
    inv_std: torch.Tensor


# ── GELU ────────────────────────────────────────────────────────────────

_GELU_TABLES: dict[int, torch.Tensor] = {}


def gelu_tables(device=None) -> torch.Tensor:
    """Per-device lookup tables f(code * s) for all binary16 scales (built once, 64 MB)."""
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    tab = _GELU_TABLES.get(dev.index)
    if tab is None:
        L = _lib.lib()
        tab = torch.empty(int(L.jf_gelu_tables_bytes()) // 4, dtype=torch.float32, device=dev)
        _lib.check(L.jf_gelu_build_tables(tab.data_ptr(), _lib.stream_handle()), "gelu_tables")
        _GELU_TABLES[dev.index] = tab
    return tab



@_rt.traced("jf.gelu_fwd")
def gelu_forward(xq: BlockQuantTensor, counters: AccessCounters | None = None) -> BlockQuantTensor:
    """y = x * CDF(x), requantized per block — kernel K9 (qnonlinear.py:150-158)."""
    nc = xq.rows * xq.cols
    count_elementwise(counters, ExecMode.INT8_DATA_FLOW, nc, nc, dequant_elems=nc, quant_elems=nc)
    L = _lib.lib()
    y = empty_like_shape(xq.rows, xq.cols, xq.device)
    _lib.check(L.jf_gelu_fwd(xq.values.data_ptr(), xq.scales.data_ptr(), xq.rows, xq.cols,
                             y.values.data_ptr(), y.scales.data_ptr(), gelu_tables(xq.device.index).data_ptr(),
                             _rt.err_ptr(), _lib.stream_handle()), "gelu_fwd")
    _rt.maybe_check()
    return y


@_rt.traced("jf.gelu_bwd")
def gelu_backward(xq: BlockQuantTensor, dyq: BlockQuantTensor,
                  counters: AccessCounters | None = None) -> BlockQuantTensor:
    """dX = dY * (x pdf(x) + CDF(x)) — kernel K10 (qnonlinear.py:161-175)."""
    if xq.shape != dyq.shape:
        raise ValueError(f"shape mismatch: x {xq.shape}, dY {dyq.shape}")
    nc = xq.rows * xq.cols
    count_elementwise(counters, ExecMode.INT8_DATA_FLOW, 2 * nc, nc, dequant_elems=2 * nc,
                      quant_elems=nc)
    L = _lib.lib()
    y = empty_like_shape(xq.rows, xq.cols, xq.device)
    _lib.check(L.jf_gelu_bwd(xq.values.data_ptr(), xq.scales.data_ptr(), dyq.values.data_ptr(),
                             dyq.scales.data_ptr(), xq.rows, xq.cols, y.values.data_ptr(),
                             y.scales.data_ptr(), gelu_tables(xq.device.index).data_ptr(), _rt.err_ptr(),
                             _lib.stream_handle()), "gelu_bwd")
    _rt.maybe_check()
    return y


# ── Dropout (scale folding) ─────────────────────────────────────────────


@dataclass
class DropoutState:
    """Drop probability, seed and the materialized keep mask (qnonlinear.py:181-204).

    The mask is drawn on the device (``jf_philox_keep``): numpy's Philox4x64-10
    stream keyed by ``seed`` and its 53-bit ``random()`` doubles, restated in CUDA,
    so masks are bit-identical to the reference's without a host draw or upload.
    The key words come from numpy's own seed conversion (``Philox(key=seed)``).
    """

    p: float
    seed: object
    mask: torch.Tensor | None

    @classmethod
    def generate(cls, p, seed, shape) -> "DropoutState":
        if not 0.0 <= p < 1.0:
            raise ValueError(f"drop probability must be in [0, 1), got {p}")
        if p == 0.0:
            return cls(p, seed, None)  # identity: every element kept
        k0, k1 = (int(w) for w in np.random.Philox(key=seed).state["state"]["key"])
        rows, cols = shape
        mask = torch.empty((rows, cols), dtype=torch.bool, device="cuda")
        _lib.check(_lib.lib().jf_philox_keep(k0, k1, float(p), rows * cols, mask.data_ptr(),
                                             _lib.stream_handle()), "philox_keep")
        return cls(p, seed, mask)

    @property
    def keep_factor(self) -> np.float32:
        return np.float32(1.0 / (1.0 - self.p))


def _apply_dropout(tq: BlockQuantTensor, state: DropoutState) -> BlockQuantTensor:
    if state.mask is not None and tuple(state.mask.shape) != tq.shape:
        raise ValueError(f"mask shape {tuple(state.mask.shape)} does not match tensor {tq.shape}")
    if state.mask is None:
        # p = 0: values untouched and snap_to_f16(s * 1.0) == s (qnonlinear.py:216-217)
        return tq
    L = _lib.lib()
    y = empty_like_shape(tq.rows, tq.cols, tq.device)
    keep = state.mask.to(device=tq.device, dtype=torch.uint8).contiguous()
    _lib.check(L.jf_dropout(tq.values.data_ptr(), tq.scales.data_ptr(), keep.data_ptr(),
                            float(state.keep_factor), tq.rows, tq.cols, y.values.data_ptr(),
                            y.scales.data_ptr(), _rt.err_ptr(), _lib.stream_handle()), "dropout")
    try:
        _rt.maybe_check()
    except ValueError:
        raise ValueError("dropout scale correction overflows binary16") from None
    return y


@_rt.traced("jf.dropout_fwd")
def dropout_forward(xq, state: DropoutState, counters: AccessCounters | None = None):
    nc = xq.rows * xq.cols
    count_elementwise(counters, ExecMode.INT8_DATA_FLOW, nc, nc)
    return _apply_dropout(xq, state)


@_rt.traced("jf.dropout_bwd")
def dropout_backward(dyq, state: DropoutState, counters: AccessCounters | None = None):
    nc = dyq.rows * dyq.cols
    count_elementwise(counters, ExecMode.INT8_DATA_FLOW, nc, nc)
    return _apply_dropout(dyq, state)


# ── Add with statistics ─────────────────────────────────────────────────


@_rt.traced("jf.add_stats")
def add_forward(x1q: BlockQuantTensor, x2q: BlockQuantTensor | None, stats_width: int = 64,
                counters: AccessCounters | None = None) -> tuple[BlockQuantTensor, RowStats]:
    """y = x1 + x2 in FP32, requantized, plus stats of the FP32 y — kernel K6.

    ``x2q`` may be ``None`` (or an all-zero ``zeros_like`` tensor) for the
    block-entry Add(x, 0) (qlayers.py:347): the kernel then skips the read.
    """
    if x2q is not None and (x1q.shape != x2q.shape or x1q.block != x2q.block):
        raise ValueError(
            f"operands differ: {x1q.shape}/b{x1q.block} vs {x2q.shape}/b{x2q.block}")
    n, c = x1q.shape
    if c % stats_width:
        raise ValueError(f"stats width {stats_width} does not divide {c} columns")
    nc = n * c
    count_elementwise(counters, ExecMode.INT8_DATA_FLOW, 2 * nc, nc, dequant_elems=2 * nc,
                      quant_elems=nc)
    L = _lib.lib()
    y = empty_like_shape(n, c, x1q.device)
    mean = torch.empty((n, c // stats_width), dtype=torch.float32, device=x1q.device)
    sumsq = torch.empty_like(mean)
    rc = L.jf_add_stats(x1q.values.data_ptr(), x1q.scales.data_ptr(),
                        _lib.ptr(x2q and x2q.values), _lib.ptr(x2q and x2q.scales), n, c,
                        stats_width, y.values.data_ptr(), y.scales.data_ptr(), mean.data_ptr(),
                        sumsq.data_ptr(), _rt.err_ptr(), _lib.stream_handle())
    if rc == 3:
        raise ValueError(f"stats width {stats_width} is not supported by the GPU kernel "
                         f"(lcm(32, width) must be <= 256)")
    _lib.check(rc, "add_stats")
    _rt.maybe_check()
    return y, RowStats(mean, sumsq, stats_width)


# ── LayerNorm ───────────────────────────────────────────────────────────


@_rt.traced("jf.ln_fwd")
def layernorm_forward(xq: BlockQuantTensor, stats: RowStats, params: NormParams,
                      counters: AccessCounters | None = None):
    """Normalize rows using the Add-provided statistics — kernel K7 (qnonlinear.py:300-330)."""
    if stats.mean.shape[0] != xq.rows or stats.cols != xq.cols:
        raise ValueError(
            f"stats for {stats.mean.shape[0]}x{stats.cols} do not match tensor {xq.shape}")
    if params.gamma.shape[0] != xq.cols:
        raise ValueError("parameter length does not match channel count")
    nc = xq.rows * xq.cols
    count_elementwise(counters, ExecMode.INT8_DATA_FLOW, nc, nc, dequant_elems=nc, quant_elems=nc)
    L = _lib.lib()
    n, c = xq.shape
    y = empty_like_shape(n, c, xq.device)
    mu = torch.empty(n, dtype=torch.float32, device=xq.device)
    inv_std = torch.empty_like(mu)
    g = params.gamma.to(xq.device)
    b = params.beta.to(xq.device)
    _lib.check(L.jf_ln_fwd(xq.values.data_ptr(), xq.scales.data_ptr(), stats.mean.data_ptr(),
                           stats.sumsq.data_ptr(), n, c, stats.width, g.data_ptr(), b.data_ptr(),
                           float(np.float32(params.eps)), y.values.data_ptr(), y.scales.data_ptr(),
                           mu.data_ptr(), inv_std.data_ptr(), _rt.err_ptr(), _lib.stream_handle()),
               "ln_fwd")
    _rt.maybe_check()
    return y, LayerNormContext(xq, mu, inv_std)


@_rt.traced("jf.ln_bwd")
def layernorm_backward(ctx: LayerNormContext, dyq: BlockQuantTensor, params: NormParams,
                       counters: AccessCounters | None = None):
    """Three-term LayerNorm gradient — kernel K8 (qnonlinear.py:333-355).

    Returns (dX quantized, dgamma FP32, dbeta FP32).
    """
    if dyq.shape != ctx.xq.shape:
        raise ValueError(f"dY {dyq.shape} does not match saved input {ctx.xq.shape}")
    nc = dyq.rows * dyq.cols
    count_elementwise(counters, ExecMode.INT8_DATA_FLOW, 2 * nc, nc, dequant_elems=2 * nc,
                      quant_elems=nc)
    L = _lib.lib()
    n, c = dyq.shape
    dx = empty_like_shape(n, c, dyq.device)
    dgamma = torch.empty(c, dtype=torch.float32, device=dyq.device)
    dbeta = torch.empty_like(dgamma)
    ws = torch.empty(int(L.jf_ln_bwd_workspace_bytes(n, c)), dtype=torch.uint8, device=dyq.device)
    g = params.gamma.to(dyq.device)
    _lib.check(L.jf_ln_bwd(ctx.xq.values.data_ptr(), ctx.xq.scales.data_ptr(), ctx.mu.data_ptr(),
                           ctx.inv_std.data_ptr(), dyq.values.data_ptr(), dyq.scales.data_ptr(),
                           g.data_ptr(), n, c, dx.values.data_ptr(), dx.scales.data_ptr(),
                           dgamma.data_ptr(), dbeta.data_ptr(), ws.data_ptr(), _rt.err_ptr(),
                           _lib.stream_handle()), "ln_bwd")
    _rt.maybe_check()
    return dx, dgamma, dbeta


def column_sum(xq: BlockQuantTensor) -> torch.Tensor:
    """dequantize(x).sum(axis=0) in FP32 (QuantLinear dbias, qlayers.py:180) — kernel K11."""
    L = _lib.lib()
    out = torch.empty(xq.cols, dtype=torch.float32, device=xq.device)
    ws = torch.empty(int(L.jf_colsum_workspace_bytes(xq.rows, xq.cols)), dtype=torch.uint8,
                     device=xq.device)
    _lib.check(L.jf_colsum(xq.values.data_ptr(), xq.scales.data_ptr(), xq.rows, xq.cols,
                           out.data_ptr(), ws.data_ptr(), _lib.stream_handle()), "colsum")
    return out


__all__ = [
    "DropoutState", "LayerNormContext", "NormParams", "RowStats", "add_forward", "column_sum",
    "count_elementwise", "dropout_backward", "dropout_forward", "gelu_backward", "gelu_forward",
    "layernorm_backward", "layernorm_forward", "snap_to_f16",
]
