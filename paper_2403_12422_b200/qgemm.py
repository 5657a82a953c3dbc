"""Per-block INT8 GEMMs on tcgen05 (drop-in for int8flow.qgemm).

Mirrors ``int8flow/qgemm.py``: ExecMode :28-32, AccessCounters :35-66,
TileConfig :69-108, DenseResult :111-120, _count_call :130-162,
micro_mm_16 :168-180, block_mm_forward :282-309, block_mm_grad_input
:312-333, block_mm_grad_weight :336-357, CounterLog :360-415.

The three products run in libjetfire's tcgen05 kind::i8 kernel (K3-K5).
``cfg`` and ``threads`` are accepted for API compatibility: on the GPU the
tile shape is fixed by the hardware design and the result is independent
of both, exactly like the reference's bit-transparency guarantee
(SPEC.md:154).  Access counters stay the reference's analytic closed forms.
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum

import numpy as np
import torch

from . import _lib
from . import runtime as _rt
from .qtensor import BLOCK, BlockQuantTensor, empty_like_shape


class ExecMode(Enum):
    INT8_DATA_FLOW = "int8"
    QCD_EMULATION = "qcd"


@dataclass
class AccessCounters:
    int8_load_store: int = 0
    fp16_load_store: int = 0
    int_mac: int = 0
    dequant_ops: int = 0
    quant_ops: int = 0

    def reset(self) -> None:
        self.int8_load_store = self.fp16_load_store = self.int_mac = 0
        self.dequant_ops = self.quant_ops = 0

    def merge(self, other: "AccessCounters") -> None:
        self.int8_load_store += other.int8_load_store
        self.fp16_load_store += other.fp16_load_store
        self.int_mac += other.int_mac
        self.dequant_ops += other.dequant_ops
        self.quant_ops += other.quant_ops

    def as_tuple(self) -> tuple[int, int, int, int, int]:
        return (self.int8_load_store, self.fp16_load_store, self.int_mac, self.dequant_ops,
                self.quant_ops)


@dataclass(frozen=True)
class TileConfig:
    """Analytic tile sizes B_N x B_C x B_D (validated like qgemm.py:83-96)."""

    b_n: int = 128
    b_c: int = 32
    b_d: int = 128
    block: int = 32

    def __post_init__(self):
        if self.block <= 0 or self.block % 16:
            raise ValueError(f"block size must be a positive multiple of 16, got {self.block}")
        if self.b_c != self.block:
            raise ValueError(f"inner tile width {self.b_c} must equal the block size {self.block}")
        for name, v in (("b_n", self.b_n), ("b_d", self.b_d)):
            if v <= 0 or v % self.block:
                raise ValueError(f"{name}={v} must be a positive multiple of block {self.block}")

    @classmethod
    def default_for(cls, block: int = 32) -> "TileConfig":
        outer = block * max(1, 128 // block)
        return cls(outer, block, outer, block)

    def clamped(self, n: int, d: int) -> "TileConfig":
        return TileConfig(min(self.b_n, n), self.b_c, min(self.b_d, d), self.block)


@dataclass
class DenseResult:
    """Full-precision output of the QCD emulation mode: values + trivial scale."""

    values: torch.Tensor
    scale: float = 1.0

    @property
    def shape(self):
        return tuple(self.values.shape)


def _spans(total: int, step: int):
    return [(t0, min(t0 + step, total)) for t0 in range(0, total, step)]


def _count_call(counters, n, c, d, cfg, mode, quantize_output) -> None:
    """Analytic cost model, identical closed forms to qgemm.py:130-162."""
    t_c = c // cfg.b_c
    nspans = _spans(n, cfg.b_n)
    dspans = _spans(d, cfg.b_d)
    for n0, n1 in nspans:
        bn = n1 - n0
        for d0, d1 in dspans:
            bd = d1 - d0
            counters.int_mac += bn * bd * c
            traffic = (bn + bd) * c + bn * bd
            if mode is ExecMode.INT8_DATA_FLOW:
                counters.int8_load_store += traffic
                counters.dequant_ops += bn * bd * t_c
                if quantize_output:
                    counters.quant_ops += bn * bd
            else:
                counters.fp16_load_store += traffic
    if mode is ExecMode.QCD_EMULATION:
        counters.dequant_ops += n * d


def _resolve_cfg(cfg, block):
    if cfg is None:
        return TileConfig.default_for(block)
    if cfg.block != block:
        raise ValueError(f"tile config block {cfg.block} does not match tensor block {block}")
    return cfg


def micro_mm_16(a, bt):
    """Exact 16x16x16 int8 product with int32 accumulation (qgemm.py:168-180).

    The GPU's unit is one tcgen05 kind::i8 MMA (K=32); this host helper keeps
    the reference's API for tests and documentation.
    """
    a = np.asarray(a.cpu() if isinstance(a, torch.Tensor) else a)
    bt = np.asarray(bt.cpu() if isinstance(bt, torch.Tensor) else bt)
    if a.shape != (16, 16) or bt.shape != (16, 16):
        raise ValueError(f"expected 16x16 operands, got {a.shape} and {bt.shape}")
    if a.dtype != np.int8 or bt.dtype != np.int8:
        raise TypeError("micro kernel operates on int8 inputs")
    return a.astype(np.int32) @ bt.astype(np.int32)


_OUT_KIND = {"int8": _lib.OUT_INT8, "f32": _lib.OUT_F32, "int8+deq": _lib.OUT_INT8_DEQ}


class GemmTimer:
    """Records CUDA events around every GEMM kernel launch on the current stream.

    Used by bench.py to measure the dominant kernel live inside the timed
    region: ``ops`` is the algorithmic work 2*M*N*K per launch.
    """

    def __init__(self):
        self.records: list[tuple[str, int, torch.cuda.Event, torch.cuda.Event]] = []

    def __enter__(self):
        global _TIMER
        _TIMER = self
        return self

    def __exit__(self, *exc):
        global _TIMER
        _TIMER = None

    def summary(self) -> dict:
        torch.cuda.synchronize()
        ms = sum(a.elapsed_time(b) for _, _, a, b in self.records)
        ops = sum(o for _, o, _, _ in self.records)
        return {"launches": len(self.records), "ms": ms, "ops": ops}


_TIMER: GemmTimer | None = None


def _timed(kind: str, ops: int, call):
    if _TIMER is None:
        return call()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    rc = call()
    b.record()
    _TIMER.records.append((kind, ops, a, b))
    return rc


def _outputs(m: int, n: int, device, out: str):
    yq = ys = yf = None
    if out in ("int8", "int8+deq"):
        t = empty_like_shape(m, n, device)
        yq, ys = t, t
    if out in ("f32", "int8+deq"):
        yf = torch.empty((m, n), dtype=torch.float32, device=device)
    return yq, yf


def _finish(yq, yf, mode, out):
    _rt.maybe_check()
    if mode is ExecMode.QCD_EMULATION:
        return DenseResult(yf)
    if out == "f32":
        return yf
    if out == "int8+deq":
        return yq, yf
    return yq


def _prep(mode, quantize, out):
    if out is None:
        out = "f32" if (not quantize or mode is ExecMode.QCD_EMULATION) else "int8"
    if out not in _OUT_KIND:
        raise ValueError(f"unknown output kind {out!r}")
    return out


@_rt.traced("jf.gemm_fwd")
def block_mm_forward(xq: BlockQuantTensor, wq: BlockQuantTensor, cfg: TileConfig | None = None,
                     mode: ExecMode = ExecMode.INT8_DATA_FLOW, counters: AccessCounters | None = None,
                     *, bias=None, threads: int = 1, quantize: bool = True,
                     promotion: str | None = None, out: str | None = None,
                     w16: torch.Tensor | None = None):
    """Y = X W^T (+bias) for X [N x C], W [D x C] — kernel K3 (qgemm.py:282-309).

    ``w16`` (optional): W's f16-widened codes, cached by QuantLinear for the f16 operand path.
    """
    if xq.cols != wq.cols:
        raise ValueError(f"inner dims differ: X is {xq.shape}, W is {wq.shape}")
    if xq.block != wq.block:
        raise ValueError(f"mixed block sizes {xq.block} and {wq.block}")
    cfg = _resolve_cfg(cfg, xq.block)
    out = _prep(mode, quantize, out)
    if counters is not None:
        _count_call(counters, xq.rows, xq.cols, wq.rows, cfg, mode, quantize)
    L = _lib.lib()
    if bias is not None:
        bias = bias if isinstance(bias, torch.Tensor) else torch.as_tensor(np.asarray(bias))
        bias = bias.to(device=xq.device, dtype=torch.float32).contiguous()
    yq, yf = _outputs(xq.rows, wq.rows, xq.device, out)
    n, c, d = xq.rows, xq.cols, wq.rows
    if f16_ok(n, c, d):
        b16 = w16 if w16 is not None else widen_codes(wq.values)
        _lib.check(_gemm_f16("fwd", widen_codes(xq.values), xq.scales, (c // 32, 1), b16, wq.scales, (c // 32, 1),
                             bias, n, d, c, promotion, out, yq, yf), "gemm_f16")
        return _finish(yq, yf, mode, out)
    _lib.check(_timed("fwd", 2 * xq.rows * xq.cols * wq.rows, lambda: L.jf_gemm_fwd(
        xq.values.data_ptr(), xq.scales.data_ptr(), wq.values.data_ptr(), wq.scales.data_ptr(),
        _lib.ptr(bias), xq.rows, xq.cols, wq.rows, _rt.promotion_code(promotion), _OUT_KIND[out],
        _lib.ptr(yq and yq.values), _lib.ptr(yq and yq.scales), _lib.ptr(yf), _rt.err_ptr(),
        _lib.stream_handle())), "gemm_fwd")
    return _finish(yq, yf, mode, out)


def f16_ok(m: int, n: int, k: int) -> bool:
    """True when the f16-widened operand path applies to an m x n x k GEMM
    (runtime.set_gemm_operands: 'f16', or 'auto' and 2mnk >= runtime.F16_MIN_FLOP; every
    dim a multiple of 128)."""
    kind = _rt.gemm_operands()
    if kind == "int8" or m % 128 or n % 128 or k % 128:
        return False
    return kind == "f16" or 2 * m * n * k >= _rt.F16_MIN_FLOP


def widen_codes(values: torch.Tensor, transpose: bool = False) -> torch.Tensor:
    """f16 copy of int8 codes (exact), optionally transposed (libjetfire jf_widen_codes)."""
    L = _lib.lib()
    rows, cols = values.shape
    out = torch.empty((cols, rows) if transpose else (rows, cols), dtype=torch.float16, device=values.device)
    _lib.check(L.jf_widen_codes(values.data_ptr(), rows, cols, out.data_ptr(), int(transpose),
                                _lib.stream_handle()), "widen_codes")
    return out


def _gemm_f16(kind, a16, sa, sa_st, b16, sb, sb_st, bias, m, n, k, promotion, out, yq, yf):
    L = _lib.lib()
    return _timed(kind, 2 * m * n * k, lambda: L.jf_gemm_f16(
        a16.data_ptr(), sa.data_ptr(), sa_st[0], sa_st[1], b16.data_ptr(), sb.data_ptr(), sb_st[0], sb_st[1],
        _lib.ptr(bias), m, n, k, _rt.promotion_code(promotion), _OUT_KIND[out], _lib.ptr(yq and yq.values),
        _lib.ptr(yq and yq.scales), _lib.ptr(yf), _rt.err_ptr(), _lib.stream_handle()))


def mn_major_ok(*dims: int) -> bool:
    """True when the GEMM reads MN-major operands as stored (every dim a multiple of 128):
    dgrad then needs no W^T and wgrad no transposed dY / X (libjetfire gemm_tc_kernel)."""
    return _rt.gemm_option("tma_scales") != 0 and all(d % 128 == 0 for d in dims)


@_rt.traced("jf.gemm_dgrad")
def block_mm_grad_input(dyq: BlockQuantTensor, wq: BlockQuantTensor, cfg: TileConfig | None = None,
                        mode: ExecMode = ExecMode.INT8_DATA_FLOW,
                        counters: AccessCounters | None = None, *, threads: int = 1,
                        quantize: bool = True, promotion: str | None = None,
                        out: str | None = None, wt: BlockQuantTensor | None = None,
                        w16t: torch.Tensor | None = None):
    """dX = dY W for dY [N x D], W [D x C] — kernel K4 (qgemm.py:312-333).

    ``wt`` (optional) is W's transposed codes, cached by QuantLinear so the
    kernel never re-transposes a weight between updates; ``w16t`` the same
    for the f16 operand path (W^T widened to f16).
    """
    if dyq.cols != wq.rows:
        raise ValueError(f"inner dims differ: dY is {dyq.shape}, W is {wq.shape}")
    if dyq.block != wq.block:
        raise ValueError(f"mixed block sizes {dyq.block} and {wq.block}")
    cfg = _resolve_cfg(cfg, dyq.block)
    out = _prep(mode, quantize, out)
    if counters is not None:
        _count_call(counters, dyq.rows, dyq.cols, wq.cols, cfg, mode, quantize)
    L = _lib.lib()
    n, d, c = dyq.rows, dyq.cols, wq.cols
    yq, yf = _outputs(n, c, dyq.device, out)
    if f16_ok(n, d, c):
        # A = dY [n x d] (K = d); B = W^T [c x d], grid element (J, ci) = W.scales[ci, J]
        b16 = w16t if w16t is not None else widen_codes(wq.values, transpose=True)
        _lib.check(_gemm_f16("dgrad", widen_codes(dyq.values), dyq.scales, (d // 32, 1), b16, wq.scales,
                             (1, c // 32), None, n, c, d, promotion, out, yq, yf), "gemm_f16")
        return _finish(yq, yf, mode, out)
    if wt is None and not mn_major_ok(n, d, c):
        wt = wq.transposed()
    _lib.check(_timed("dgrad", 2 * n * d * c, lambda: L.jf_gemm_dgrad(
        dyq.values.data_ptr(), dyq.scales.data_ptr(), wq.values.data_ptr(), wq.scales.data_ptr(),
        _lib.ptr(wt and wt.values), _lib.ptr(wt and wt.scales), n, d, c,
        _rt.promotion_code(promotion), _OUT_KIND[out], _lib.ptr(yq and yq.values),
        _lib.ptr(yq and yq.scales), _lib.ptr(yf), None, _rt.err_ptr(),
        _lib.stream_handle())), "gemm_dgrad")
    return _finish(yq, yf, mode, out)


@_rt.traced("jf.gemm_wgrad")
def block_mm_grad_weight(dyq: BlockQuantTensor, xq: BlockQuantTensor, cfg: TileConfig | None = None,
                         mode: ExecMode = ExecMode.INT8_DATA_FLOW,
                         counters: AccessCounters | None = None, *, threads: int = 1,
                         quantize: bool = True, promotion: str | None = None,
                         out: str | None = None):
    """dW = dY^T X for dY [N x D], X [N x C] -> [D x C] — kernel K5 (qgemm.py:336-357)."""
    if dyq.rows != xq.rows:
        raise ValueError(f"batch dims differ: dY is {dyq.shape}, X is {xq.shape}")
    if dyq.block != xq.block:
        raise ValueError(f"mixed block sizes {dyq.block} and {xq.block}")
    cfg = _resolve_cfg(cfg, dyq.block)
    out = _prep(mode, quantize, out)
    if counters is not None:
        _count_call(counters, dyq.cols, dyq.rows, xq.cols, cfg, mode, quantize)
    L = _lib.lib()
    n, d, c = dyq.rows, dyq.cols, xq.cols
    if f16_ok(n, d, c):
        # A = dY^T [d x n] (K = n), grid (I, ci) = dY.scales[ci, I]; B = X^T [c x n] likewise
        yq, yf = _outputs(d, c, dyq.device, out)
        _lib.check(_gemm_f16("wgrad", widen_codes(dyq.values, transpose=True), dyq.scales, (1, d // 32),
                             widen_codes(xq.values, transpose=True), xq.scales, (1, c // 32), None, d, c, n,
                             promotion, out, yq, yf), "gemm_f16")
        return _finish(yq, yf, mode, out)
    dyt = xt = None
    if not mn_major_ok(n, d, c):  # generic shapes: K(=tokens)-major transposed copies
        dyt = dyq.transposed()   # dY^T [d x n] (codes + grid)
        xt = xq.transposed()     # X^T [c x n]
    yq, yf = _outputs(d, c, dyq.device, out)
    _lib.check(_timed("wgrad", 2 * n * d * c, lambda: L.jf_gemm_wgrad(
        dyq.values.data_ptr(), dyq.scales.data_ptr(), xq.values.data_ptr(), xq.scales.data_ptr(),
        _lib.ptr(dyt and dyt.values), _lib.ptr(dyt and dyt.scales), _lib.ptr(xt and xt.values),
        _lib.ptr(xt and xt.scales), n, d, c,
        _rt.promotion_code(promotion), _OUT_KIND[out],
        _lib.ptr(yq and yq.values), _lib.ptr(yq and yq.scales), _lib.ptr(yf), None, _rt.err_ptr(),
        _lib.stream_handle())), "gemm_wgrad")
    return _finish(yq, yf, mode, out)


def transpose_codes(values: torch.Tensor) -> torch.Tensor:
    """Transposed int8 codes (libjetfire transpose kernel; scales are read transposed in place)."""
    L = _lib.lib()
    n, c = values.shape
    out = torch.empty((c, n), dtype=torch.int8, device=values.device)
    _lib.check(L.jf_transpose(values.data_ptr(), None, n, c, out.data_ptr(), None,
                              _lib.stream_handle()), "transpose")
    return out


def block_partials(a: torch.Tensor, bt: torch.Tensor, kblk: int) -> torch.Tensor:
    """Debug: exact int32 P = A[:, 32k:32k+32] . Bt[:, 32k:32k+32]^T from the tcgen05 MMA."""
    L = _lib.lib()
    m, k = a.shape
    n = bt.shape[0]
    p = torch.empty((m, n), dtype=torch.int32, device=a.device)
    _lib.check(L.jf_gemm_partials(a.data_ptr(), bt.data_ptr(), m, n, k, kblk, p.data_ptr(),
                                  _lib.stream_handle()), "gemm_partials")
    return p


# ── counter logging (qgemm.py:360-415) ──────────────────────────────────

COUNTER_CSV_HEADER = "op_name,N,C,D,B,mode,int8_ls,fp16_ls,int_mac,dequant,quant"


@dataclass
class CounterRecord:
    op_name: str
    n: int
    c: int
    d: int
    block: int
    mode: str
    counters: AccessCounters

    def csv_row(self) -> str:
        k = self.counters
        return (f"{self.op_name},{self.n},{self.c},{self.d},{self.block},{self.mode},"
                f"{k.int8_load_store},{k.fp16_load_store},{k.int_mac},{k.dequant_ops},{k.quant_ops}")


class CounterLog:
    def __init__(self) -> None:
        self.records: list[CounterRecord] = []

    def add(self, op_name, n, c, d, block, mode: ExecMode, counters: AccessCounters) -> None:
        self.records.append(CounterRecord(op_name, n, c, d, block, mode.value, counters))

    def total(self) -> AccessCounters:
        out = AccessCounters()
        for rec in self.records:
            out.merge(rec.counters)
        return out

    def to_csv(self) -> str:
        return "\n".join([COUNTER_CSV_HEADER] + [r.csv_row() for r in self.records]) + "\n"


__all__ = [
    "BLOCK", "AccessCounters", "CounterLog", "CounterRecord", "COUNTER_CSV_HEADER", "DenseResult",
    "ExecMode", "TileConfig", "block_mm_forward", "block_mm_grad_input", "block_mm_grad_weight",
    "block_partials", "micro_mm_16",
]
