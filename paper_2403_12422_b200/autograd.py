"""torch.autograd form of the INT8 data flow.

The reference drives backward by hand (``qlayers.py:385-427``).  Here the
same operators are ``torch.autograd.Function``s so a block can sit in an
ordinary autograd graph, while every tensor handed between them stays a
``BlockQuantTensor`` in HBM: ``QTensor`` is a float32-typed tensor subclass
with NO float storage that carries the INT8 codes + scale grid (and, after
an Add, the FP32 row statistics the next LayerNorm consumes,
``qnonlinear.py:103-144``).  Autograd sees an ``[N, C]`` float tensor; the
kernels see INT8.

Gradient accumulation for a tensor used twice (the residual stream) is
autograd's own ``add`` of two ``QTensor`` gradients, dispatched to the
Jetfire Add kernel K6 — the same ``add_forward(dh_branch, dy)`` the
reference runs by hand (``qlayers.py:402,411``).  Any other torch op applied
to a ``QTensor`` sees its dequantized FP32 value (an explicit boundary).
"""

from __future__ import annotations

import torch
import torch.nn as nn
from torch.utils._pytree import tree_map

from .qgemm import block_mm_forward, block_mm_grad_input, block_mm_grad_weight, mn_major_ok
from .qlayers import AttentionCore, BlockConfig, QuantLinear
from .qnonlinear import (
    NormParams,
    add_forward,
    column_sum,
    gelu_backward,
    gelu_forward,
    layernorm_backward,
    layernorm_forward,
)
from .qtensor import BlockQuantTensor, dequantize, quantize_per_block

aten = torch.ops.aten


class QTensor(torch.Tensor):
    """A BlockQuantTensor that autograd treats as an [N, C] float32 tensor."""

    @staticmethod
    def __new__(cls, bq: BlockQuantTensor, stats=None, requires_grad: bool = False):
        t = torch.Tensor._make_wrapper_subclass(cls, bq.shape, dtype=torch.float32,
                                                device=bq.values.device, requires_grad=requires_grad)
        t.bq = bq
        t.stats = stats
        return t

    def __init__(self, bq, stats=None, requires_grad=False):  # state set in __new__
        pass

    def __repr__(self):
        return f"QTensor({self.bq!r}, stats={'yes' if self.stats is not None else 'no'})"

    __torch_function__ = torch._C._disabled_torch_function_impl

    @classmethod
    def __torch_dispatch__(cls, func, types, args=(), kwargs=None):
        kwargs = kwargs or {}
        if func in (aten.detach.default, aten.alias.default):
            x = args[0]
            return QTensor(x.bq, x.stats)
        if func in (aten.add.Tensor, aten.add_.Tensor) and len(args) == 2 and \
                all(isinstance(a, QTensor) for a in args) and kwargs.get("alpha", 1) == 1:
            y, stats = add_forward(args[0].bq, args[1].bq, _width(args[0].bq.cols))
            if func is aten.add_.Tensor:
                args[0].bq, args[0].stats = y, stats
                return args[0]
            return QTensor(y, stats)

        def unwrap(x):
            return dequantize(x.bq) if isinstance(x, QTensor) else x
        return func(*tree_map(unwrap, args), **tree_map(unwrap, kwargs))


def _width(c: int) -> int:
    return 64 if c % 64 == 0 else 32


def as_block_quant(g) -> BlockQuantTensor:
    """A gradient reaching a backward: QTensor payload, or quantize a float one."""
    if isinstance(g, QTensor):
        return g.bq
    return quantize_per_block(g.contiguous())


# ── Functions ───────────────────────────────────────────────────────────


class Quantize(torch.autograd.Function):
    """FP -> INT8 entry (qtensor.py:219-246); backward hands back deq(dY)."""

    @staticmethod
    def forward(ctx, x):
        return QTensor(quantize_per_block(x.detach().contiguous()))

    @staticmethod
    def backward(ctx, g):
        return dequantize(as_block_quant(g))


class Dequantize(torch.autograd.Function):
    """INT8 -> FP exit (qtensor.py:249-255); backward quantizes the incoming gradient."""

    @staticmethod
    def forward(ctx, xq, dtype=torch.float32):
        return dequantize(xq.bq, dtype)

    @staticmethod
    def backward(ctx, g):
        return QTensor(quantize_per_block(g.contiguous())), None


class Linear(torch.autograd.Function):
    """QuantLinear (qlayers.py:149-181): Y = X W^T + b; dX, dW = deq(requant(dY^T X)), db."""

    @staticmethod
    def forward(ctx, xq, weight, bias, layer: QuantLinear):
        ctx.layer, ctx.xq = layer, xq.bq
        ctx.has_bias = bias is not None
        return QTensor(block_mm_forward(xq.bq, layer.weight_q, bias=layer.bias, w16=layer.weight_f16(xq.bq.rows)))

    @staticmethod
    def backward(ctx, g):
        dyq = as_block_quant(g)
        lay = ctx.layer
        d, c = lay.master_weight.shape
        dxq = block_mm_grad_input(dyq, lay.weight_q, wt=None if mn_major_ok(dyq.rows, d, c) else lay.weight_qt,
                                  w16t=lay.weight_f16(dyq.rows, transpose=True))
        _, dw = block_mm_grad_weight(dyq, ctx.xq, out="int8+deq")
        db = column_sum(dyq) if ctx.has_bias else None
        return QTensor(dxq), dw, db, None


class Add(torch.autograd.Function):
    """Residual Add + RowStats (qnonlinear.py:246-267); x2 may be None (Add(x, 0))."""

    @staticmethod
    def forward(ctx, x1, x2, width):
        y, stats = add_forward(x1.bq, None if x2 is None else x2.bq, width)
        ctx.has_x2 = x2 is not None
        return QTensor(y, stats)

    @staticmethod
    def backward(ctx, g):
        return g, (g if ctx.has_x2 else None), None


class LayerNorm(torch.autograd.Function):
    """LayerNorm on Add-provided statistics (qnonlinear.py:300-355)."""

    @staticmethod
    def forward(ctx, xq, gamma, beta, eps):
        if xq.stats is None:
            raise ValueError("layernorm input must come from an Add (no row statistics)")
        params = NormParams(gamma.detach(), beta.detach(), eps)
        y, lctx = layernorm_forward(xq.bq, xq.stats, params)
        ctx.lctx, ctx.params = lctx, params
        return QTensor(y)

    @staticmethod
    def backward(ctx, g):
        dx, dgamma, dbeta = layernorm_backward(ctx.lctx, as_block_quant(g), ctx.params)
        return QTensor(dx), dgamma, dbeta, None


class Gelu(torch.autograd.Function):
    """Exact-erf GELU (qnonlinear.py:150-175)."""

    @staticmethod
    def forward(ctx, xq):
        ctx.xq = xq.bq
        return QTensor(gelu_forward(xq.bq))

    @staticmethod
    def backward(ctx, g):
        return QTensor(gelu_backward(ctx.xq, as_block_quant(g)))


class Attention(torch.autograd.Function):
    """The FP island (qlayers.py:350-351, 406-408): deq(QKV) -> SDPA -> quantize."""

    @staticmethod
    def forward(ctx, qkv, batch, seq, heads, dtype):
        core = AttentionCore(heads, qkv.shape[1] // 3 // heads, dtype=dtype)
        ctx.core, ctx.batch, ctx.seq = core, batch, seq
        if core.supports_q():
            return QTensor(core.forward_q(qkv.bq, batch, seq))
        out = core.forward(dequantize(qkv.bq, dtype), batch, seq)
        return QTensor(quantize_per_block(out))

    @staticmethod
    def backward(ctx, g):
        core = ctx.core
        if core.supports_q():
            return QTensor(core.backward_q(as_block_quant(g), ctx.batch, ctx.seq)), None, None, None, None
        d = core.backward(dequantize(as_block_quant(g), core.dtype), ctx.batch, ctx.seq)
        return QTensor(quantize_per_block(d)), None, None, None, None


# ── Modules ─────────────────────────────────────────────────────────────


class JetfireLinear(nn.Module):
    """nn.Linear-shaped module on the INT8 data flow (FP32 master weight + bias)."""

    def __init__(self, in_features: int, out_features: int, bias: bool = True, device="cuda"):
        super().__init__()
        self.weight = nn.Parameter(torch.empty(out_features, in_features, device=device))
        self.bias = nn.Parameter(torch.zeros(out_features, device=device)) if bias else None
        nn.init.normal_(self.weight, std=in_features ** -0.5)
        self._q = None

    def quant(self) -> QuantLinear:
        if self._q is None:  # shares storage with the Parameters (no copies)
            self._q = QuantLinear(self.weight.detach(), None if self.bias is None else self.bias.detach())
        return self._q

    def mark_updated(self) -> None:
        """Call after the optimizer step: the INT8 weight copy is re-derived lazily."""
        if self._q is not None:
            self._q.mark_updated()

    def forward(self, xq: QTensor) -> QTensor:
        return Linear.apply(xq, self.weight, self.bias, self.quant())


class JetfireTransformerBlock(nn.Module):
    """Pre-norm block, INT8 between every operator (qlayers.py:329-383), autograd-driven."""

    def __init__(self, config: BlockConfig, device="cuda", attn_dtype=torch.bfloat16):
        super().__init__()
        if config.dropout_p != 0.0:
            raise ValueError("the autograd block implements dropout p = 0 (every BASELINE config)")
        c, h = config.c_model, config.hidden
        self.config, self.attn_dtype = config, attn_dtype
        self.qkv = JetfireLinear(c, 3 * c, device=device)
        self.proj = JetfireLinear(c, c, device=device)
        self.mlp1 = JetfireLinear(c, h, device=device)
        self.mlp2 = JetfireLinear(h, c, device=device)
        self.ln1_gamma = nn.Parameter(torch.ones(c, device=device))
        self.ln1_beta = nn.Parameter(torch.zeros(c, device=device))
        self.ln2_gamma = nn.Parameter(torch.ones(c, device=device))
        self.ln2_beta = nn.Parameter(torch.zeros(c, device=device))

    def mark_updated(self) -> None:
        for m in (self.qkv, self.proj, self.mlp1, self.mlp2):
            m.mark_updated()

    def forward(self, x: QTensor, batch: int, seq: int) -> QTensor:
        cfg = self.config
        w = cfg.stats_width
        a1 = Add.apply(x, None, w)
        qkv = self.qkv(LayerNorm.apply(a1, self.ln1_gamma, self.ln1_beta, cfg.eps))
        att = Attention.apply(qkv, batch, seq, cfg.heads, self.attn_dtype)
        h = Add.apply(a1, self.proj(att), w)
        m = self.mlp2(Gelu.apply(self.mlp1(LayerNorm.apply(h, self.ln2_gamma, self.ln2_beta, cfg.eps))))
        return Add.apply(h, m, w)


def quantize(x: torch.Tensor) -> QTensor:
    return Quantize.apply(x)


def dequantize_q(xq: QTensor, dtype=torch.float32) -> torch.Tensor:
    return Dequantize.apply(xq, dtype)


__all__ = ["Add", "Attention", "Dequantize", "Gelu", "JetfireLinear", "JetfireTransformerBlock",
           "LayerNorm", "Linear", "QTensor", "Quantize", "as_block_quant", "dequantize_q", "quantize"]
