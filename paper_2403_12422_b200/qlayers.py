"""Quantized Linear and the pre-norm transformer block on the GPU.

Drop-in for ``int8flow/qlayers.py``: BlockConfig :59-85, QuantLinear
:91-181, AttentionCore :187-236 (the FP32 island, here torch SDPA),
TransformerBlock :256-444.  Every tensor handed between operators inside
the block is a BlockQuantTensor (INT8 codes + scales in HBM); the hot ops
are libjetfire kernels.  Parameters and parameter gradients are FP32 CUDA
tensors; the INT8 weight copy (and its transpose, for the input-gradient
GEMM) is refreshed lazily after ``mark_updated()``.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch
import torch.nn.functional as F

from .qgemm import (
    AccessCounters,
    TileConfig,
    block_mm_forward,
    block_mm_grad_input,
    block_mm_grad_weight,
    f16_ok,
    mn_major_ok,
    widen_codes,
)
from .qnonlinear import (
    DropoutState,
    NormParams,
    add_forward,
    column_sum,
    dropout_backward,
    dropout_forward,
    gelu_backward,
    gelu_forward,
    layernorm_backward,
    layernorm_forward,
)
from . import _lib
from . import runtime as _rt
from .qtensor import BlockQuantTensor, dequantize, empty_like_shape, quantize_per_block


@dataclass(frozen=True)
class BlockConfig:
    c_model: int = 64
    heads: int = 4
    hidden: int = 256
    block: int = 32
    dropout_p: float = 0.0
    eps: float = 1e-5

    def __post_init__(self):
        if self.c_model % self.block or self.hidden % self.block:
            raise ValueError("model and hidden widths must be block multiples")
        if self.c_model % self.heads:
            raise ValueError("head count must divide the model width")
        if not 0.0 <= self.dropout_p < 1.0:
            raise ValueError("dropout probability must be in [0, 1)")

    @property
    def head_dim(self) -> int:
        return self.c_model // self.heads

    @property
    def stats_width(self) -> int:
        return 64 if self.c_model % 64 == 0 else self.block


def _f32_cuda(a) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        return a.detach().to(device="cuda", dtype=torch.float32).contiguous()
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


class QuantLinear:
    """FP32 master weight [D x C] + lazily refreshed INT8 copy (qlayers.py:91-181)."""

    def __init__(self, master_weight, bias=None, block: int = 32, cfg: TileConfig | None = None):
        if isinstance(master_weight, np.ndarray) and master_weight.ndim != 2:
            raise ValueError("weight must be a D x C matrix")
        if isinstance(master_weight, torch.Tensor) and master_weight.dim() != 2:
            raise ValueError("weight must be a D x C matrix")
        self.master_weight = _f32_cuda(master_weight)
        self.bias = None if bias is None else _f32_cuda(bias)
        if self.bias is not None and tuple(self.bias.shape) != (self.master_weight.shape[0],):
            raise ValueError("bias length must match the output width")
        self.block = block
        self.cfg = cfg
        self._weight_q: BlockQuantTensor | None = None
        self._weight_qt: BlockQuantTensor | None = None
        self._weight_f16: list = [None, None]  # f16-widened W, W^T (f16 operand path)
        self.saved_input: BlockQuantTensor | None = None

    @classmethod
    def initialize(cls, rng: np.random.Generator, d: int, c: int, *, bias: bool = True,
                   block: int = 32, gain: float = 1.0) -> "QuantLinear":
        w = (rng.standard_normal((d, c)) * gain / np.sqrt(c)).astype(np.float32)
        b = np.zeros(d, dtype=np.float32) if bias else None
        return cls(w, b, block)

    @property
    def out_features(self) -> int:
        return self.master_weight.shape[0]

    @property
    def in_features(self) -> int:
        return self.master_weight.shape[1]

    @property
    def weight_q(self) -> BlockQuantTensor:
        if self._weight_q is None:
            self._weight_q = quantize_per_block(self.master_weight, self.block)
        return self._weight_q

    @property
    def weight_qt(self) -> BlockQuantTensor:
        """W^T codes + scales, cached with weight_q (dgrad operand for shapes that are not
        multiples of 128; otherwise the GEMM reads W MN-major as stored)."""
        if self._weight_qt is None:
            self._weight_qt = self.weight_q.transposed()
        return self._weight_qt

    def weight_f16(self, n_tokens: int, transpose: bool = False):
        """W (or W^T) widened to f16 for the f16 operand path, cached with weight_q; None
        when that path does not apply to this shape."""
        d, c = self.master_weight.shape
        if not f16_ok(n_tokens, d, c):
            return None
        if self._weight_f16[transpose] is None:
            self._weight_f16[transpose] = widen_codes(self.weight_q.values, transpose=transpose)
        return self._weight_f16[transpose]

    def set_weight_q(self, wq: BlockQuantTensor) -> None:
        """Install freshly requantized codes (optimizer step; may be the same buffers,
        rewritten in place); drops the derived copies."""
        self.drop_derived()
        self._weight_q = wq

    def drop_derived(self) -> None:
        """Forget the copies derived from weight_q (W^T codes, f16-widened W / W^T)."""
        self._weight_qt = None
        self._weight_f16 = [None, None]

    def mark_updated(self) -> None:
        """The master weight changed (qlayers.py:145-147).  An existing INT8 copy is
        requantized IN PLACE (same buffers), so a captured CUDA graph that reads it keeps
        reading live weights; derived copies are dropped."""
        if self._weight_q is not None:
            quantize_per_block(self.master_weight, self.block, out=self._weight_q)
        self.drop_derived()

    @_rt.traced("jf.QuantLinear.forward")
    def forward(self, xq: BlockQuantTensor, counters: AccessCounters | None = None,
                threads: int = 1) -> BlockQuantTensor:
        self.saved_input = xq
        return block_mm_forward(xq, self.weight_q, cfg=self.cfg, counters=counters, bias=self.bias,
                                threads=threads, w16=self.weight_f16(xq.rows))

    @_rt.traced("jf.QuantLinear.backward")
    def backward(self, dyq: BlockQuantTensor, counters: AccessCounters | None = None,
                 threads: int = 1, defer_wgrad: bool = False):
        """(dX quantized, dW FP32 = deq(requant(dY^T X)), dbias FP32).

        ``defer_wgrad``: issue dW / dbias on the runtime side stream; the caller must
        ``runtime.join_side_streams()`` before reading them (TransformerBlock does)."""
        if self.saved_input is None:
            raise RuntimeError("backward called before forward")
        d, c = self.master_weight.shape
        wt = None if mn_major_ok(dyq.rows, d, c) else self.weight_qt  # W^T only for generic shapes
        dxq = block_mm_grad_input(dyq, self.weight_q, cfg=self.cfg, counters=counters,
                                  threads=threads, wt=wt, w16t=self.weight_f16(dyq.rows, transpose=True))
        x = self.saved_input
        if defer_wgrad and counters is None:
            # dW (+ dbias) on the side stream, joined by the caller (runtime.join_side_streams)
            main = torch.cuda.current_stream()
            side = _rt.side_stream(dyq.device)
            side.wait_stream(main)
            with torch.cuda.stream(side):
                _, dw = block_mm_grad_weight(dyq, x, cfg=self.cfg, threads=threads, out="int8+deq")
                dbias = None if self.bias is None else column_sum(dyq)
                ev = torch.cuda.Event()
                ev.record(side)
            # dY and X stay referenced until the join (no record_stream: the caching
            # allocator's per-free event bookkeeping stalled the host)
            _rt.defer_join(ev, [dw, dbias], keepalive=(dyq, x))
            return dxq, dw, dbias
        _, dw = block_mm_grad_weight(dyq, x, cfg=self.cfg, counters=counters,
                                     threads=threads, out="int8+deq")
        dbias = None if self.bias is None else column_sum(dyq)
        return dxq, dw, dbias


class AttentionCore:
    """Causal multi-head attention: the FP32 island (qlayers.py:187-236).

    Runs torch SDPA (flash / cuDNN kernels) in ``dtype`` — float32 matches
    the reference's island, bfloat16 is the fast path.  Input/output are
    dense [batch*seq, 3C] / [batch*seq, C] tensors, as in the reference.
    """

    def __init__(self, heads: int, head_dim: int, causal: bool = True, dtype=torch.float32):
        self.heads = heads
        self.head_dim = head_dim
        self.causal = causal
        self.dtype = dtype
        self._saved = None

    def _split(self, t, batch, seq):
        return t.view(batch, seq, self.heads, self.head_dim).transpose(1, 2)

    def forward(self, qkv: torch.Tensor, batch: int, seq: int) -> torch.Tensor:
        c = self.heads * self.head_dim
        if tuple(qkv.shape) != (batch * seq, 3 * c):
            raise ValueError(f"expected ({batch * seq}, {3 * c}), got {tuple(qkv.shape)}")
        qkv = qkv.detach().to(self.dtype).requires_grad_(True)
        with torch.enable_grad():
            q = self._split(qkv[:, :c], batch, seq)
            k = self._split(qkv[:, c:2 * c], batch, seq)
            v = self._split(qkv[:, 2 * c:], batch, seq)
            o = F.scaled_dot_product_attention(q, k, v, is_causal=self.causal)
            out = o.transpose(1, 2).reshape(batch * seq, c)
        self._saved = (qkv, out)
        return out.detach()

    def backward(self, dout: torch.Tensor, batch: int, seq: int) -> torch.Tensor:
        if self._saved is None:
            raise RuntimeError("backward called before forward")
        qkv, out = self._saved
        (g,) = torch.autograd.grad(out, qkv, dout.to(out.dtype))
        self._saved = None
        return g

    # ── INT8 boundary without dense intermediates (BF16 island) ──
    def supports_q(self) -> bool:
        return self.dtype == torch.bfloat16 and self.head_dim % 16 == 0

    def fused(self, seq: int) -> bool:
        """runtime.set_attention('fused') and a shape the fused kernels take."""
        return (_rt.attention() == "fused" and self.dtype == torch.bfloat16
                and bool(_lib.lib().jf_attn_supported(seq, self.head_dim)))

    def _forward_fused(self, qkv_q: BlockQuantTensor, batch: int, seq: int) -> BlockQuantTensor:
        """One kernel: INT8 QKV codes -> causal attention (tcgen05, bf16 operands, FP32
        accumulation) -> INT8 O codes + block scales.  Saves O (bf16) and the per-row
        log-sum-exp for the backward."""
        L = _lib.lib()
        c = self.heads * self.head_dim
        dev = qkv_q.device
        out = empty_like_shape(batch * seq, c, dev)
        o_bf = torch.empty(batch * seq, c, dtype=torch.bfloat16, device=dev)
        lse = torch.empty(batch, self.heads, seq, dtype=torch.float32, device=dev)
        _lib.check(L.jf_attn_fwd_q(qkv_q.values.data_ptr(), qkv_q.scales.data_ptr(), batch, seq, self.heads,
                                   self.head_dim, out.values.data_ptr(), out.scales.data_ptr(), o_bf.data_ptr(),
                                   lse.data_ptr(), _rt.err_ptr(), _lib.stream_handle()), "attn_fwd")
        _rt.maybe_check()
        self._saved = ("fused", qkv_q, o_bf, lse)
        return out

    def _backward_fused(self, dattn_q: BlockQuantTensor, batch: int, seq: int) -> BlockQuantTensor:
        """Two kernels (dQ, then dK/dV): INT8 dO codes in, INT8 dQ|dK|dV out."""
        _, qkv_q, o_bf, lse = self._saved
        self._saved = None
        L = _lib.lib()
        c = self.heads * self.head_dim
        dev = dattn_q.device
        dqkv = empty_like_shape(batch * seq, 3 * c, dev)
        dsum = torch.empty(batch, self.heads, seq, dtype=torch.float32, device=dev)
        _lib.check(L.jf_attn_bwd_q(qkv_q.values.data_ptr(), qkv_q.scales.data_ptr(), dattn_q.values.data_ptr(),
                                   dattn_q.scales.data_ptr(), o_bf.data_ptr(), lse.data_ptr(), dsum.data_ptr(),
                                   batch, seq, self.heads, self.head_dim, dqkv.values.data_ptr(),
                                   dqkv.scales.data_ptr(), _rt.err_ptr(), _lib.stream_handle()), "attn_bwd")
        _rt.maybe_check()
        return dqkv

    @_rt.traced("jf.attention.forward")
    def forward_q(self, qkv_q: BlockQuantTensor, batch: int, seq: int) -> BlockQuantTensor:
        """deq(QKV) -> SDPA -> quantize (qlayers.py:350-351), per-head layouts end to end:
        the codes are dequantized straight into contiguous [b, h, s, d] q/k/v and the
        attention output is quantized from whatever strides SDPA returns."""
        c = self.heads * self.head_dim
        if qkv_q.shape != (batch * seq, 3 * c):
            raise ValueError(f"expected ({batch * seq}, {3 * c}), got {qkv_q.shape}")
        if self.fused(seq):
            return self._forward_fused(qkv_q, batch, seq)
        L = _lib.lib()
        shape = (batch, self.heads, seq, self.head_dim)
        q, k, v = (torch.empty(shape, dtype=torch.bfloat16, device=qkv_q.device) for _ in range(3))
        _lib.check(L.jf_dequantize_qkv_heads(qkv_q.values.data_ptr(), qkv_q.scales.data_ptr(), batch, seq,
                                             self.heads, self.head_dim, q.data_ptr(), k.data_ptr(), v.data_ptr(),
                                             _lib.stream_handle()), "dequant_qkv_heads")
        q.requires_grad_(True)
        k.requires_grad_(True)
        v.requires_grad_(True)
        with torch.enable_grad():
            o = F.scaled_dot_product_attention(q, k, v, is_causal=self.causal)
        self._saved = (q, k, v, o)
        out = empty_like_shape(batch * seq, c, qkv_q.device)
        _quantize_heads(o.detach(), out, 0)
        return out

    @_rt.traced("jf.attention.backward")
    def backward_q(self, dattn_q: BlockQuantTensor, batch: int, seq: int) -> BlockQuantTensor:
        """deq(dO) -> SDPA backward -> quantize dQ|dK|dV into one [N, 3C] tensor (qlayers.py:406-408)."""
        if self._saved is None:
            raise RuntimeError("backward called before forward")
        if self._saved[0] == "fused":
            return self._backward_fused(dattn_q, batch, seq)
        q, k, v, o = self._saved
        self._saved = None
        c = self.heads * self.head_dim
        dout = dequantize(dattn_q, torch.bfloat16).view(batch, seq, self.heads, self.head_dim).transpose(1, 2)
        dq, dk, dv = torch.autograd.grad(o, (q, k, v), dout)
        dqkv = empty_like_shape(batch * seq, 3 * c, dattn_q.device)
        for i, g in enumerate((dq, dk, dv)):
            _quantize_heads(g, dqkv, i * c)
        return dqkv


def _quantize_heads(t: torch.Tensor, out: BlockQuantTensor, col0: int) -> None:
    """bf16 t [b, h, s, d] (any strides with a contiguous d) -> columns [col0, col0 + h*d) of out."""
    b, h, s, d = t.shape
    sb, sh, ss, sd = t.stride()
    if sd != 1:
        t = t.contiguous()
        sb, sh, ss, sd = t.stride()
    L = _lib.lib()
    n, ctot = out.shape
    _lib.check(L.jf_quantize_heads_bf16(t.data_ptr(), b, s, h, d, sb, ss, sh, out.values.data_ptr() + col0,
                                        ctot, out.scales.data_ptr() + 4 * (col0 // 32), ctot // 32,
                                        _rt.err_ptr(), _lib.stream_handle()), "quantize_heads")
    _rt.maybe_check()


@dataclass
class _SavedForward:
    batch: int
    seq: int
    ctx1: object
    ctx2: object
    m1: BlockQuantTensor
    drop1: DropoutState
    drop2: DropoutState
    quant_saves: list = field(default_factory=list)


class TransformerBlock:
    """Pre-norm transformer block with INT8 tensors between all operators.

    Wiring (qlayers.py:329-383): Add(x,0)+stats -> LN -> QKV -> attention ->
    proj -> dropout -> Add+stats -> LN -> MLP1 -> GELU -> MLP2 -> dropout -> Add.
    """

    def __init__(self, config: BlockConfig, qkv: QuantLinear, proj: QuantLinear, mlp1: QuantLinear,
                 mlp2: QuantLinear, ln1: NormParams, ln2: NormParams, attn_dtype=torch.float32):
        self.config = config
        self.qkv, self.proj, self.mlp1, self.mlp2 = qkv, proj, mlp1, mlp2
        self.ln1, self.ln2 = ln1, ln2
        self.attn = AttentionCore(config.heads, config.head_dim, dtype=attn_dtype)
        self._saved: _SavedForward | None = None

    @classmethod
    def initialize(cls, rng: np.random.Generator, config: BlockConfig, *, residual_gain: float = 1.0,
                   attn_dtype=torch.float32) -> "TransformerBlock":
        c, h, b = config.c_model, config.hidden, config.block
        return cls(
            config,
            qkv=QuantLinear.initialize(rng, 3 * c, c, block=b),
            proj=QuantLinear.initialize(rng, c, c, block=b, gain=residual_gain),
            mlp1=QuantLinear.initialize(rng, h, c, block=b),
            mlp2=QuantLinear.initialize(rng, c, h, block=b, gain=residual_gain),
            ln1=NormParams(np.ones(c, np.float32), np.zeros(c, np.float32), config.eps),
            ln2=NormParams(np.ones(c, np.float32), np.zeros(c, np.float32), config.eps),
            attn_dtype=attn_dtype,
        )

    @classmethod
    def from_parameters(cls, config: BlockConfig, params: dict, attn_dtype=torch.float32):
        p = params
        return cls(config, QuantLinear(p["qkv.w"], p["qkv.b"]), QuantLinear(p["proj.w"], p["proj.b"]),
                   QuantLinear(p["mlp1.w"], p["mlp1.b"]), QuantLinear(p["mlp2.w"], p["mlp2.b"]),
                   NormParams(p["ln1.gamma"], p["ln1.beta"], config.eps),
                   NormParams(p["ln2.gamma"], p["ln2.beta"], config.eps), attn_dtype=attn_dtype)

    def parameters(self) -> dict[str, torch.Tensor]:
        return {
            "qkv.w": self.qkv.master_weight, "qkv.b": self.qkv.bias,
            "proj.w": self.proj.master_weight, "proj.b": self.proj.bias,
            "mlp1.w": self.mlp1.master_weight, "mlp1.b": self.mlp1.bias,
            "mlp2.w": self.mlp2.master_weight, "mlp2.b": self.mlp2.bias,
            "ln1.gamma": self.ln1.gamma, "ln1.beta": self.ln1.beta,
            "ln2.gamma": self.ln2.gamma, "ln2.beta": self.ln2.beta,
        }

    def mark_updated(self) -> None:
        for lin in (self.qkv, self.proj, self.mlp1, self.mlp2):
            lin.mark_updated()

    @_rt.traced("jf.TransformerBlock.forward")
    def forward(self, xq: BlockQuantTensor, batch: int, seq: int, *, dropout_seed: int = 0,
                train: bool = True, counters: AccessCounters | None = None,
                threads: int = 1) -> BlockQuantTensor:
        cfg = self.config
        p = cfg.dropout_p if train else 0.0
        n = batch * seq
        if xq.shape != (n, cfg.c_model):
            raise ValueError(f"expected ({n}, {cfg.c_model}), got {xq.shape}")
        width = cfg.stats_width

        a1, stats1 = add_forward(xq, None, width, counters)           # Add(x, zeros_like(x))
        ln1_out, ctx1 = layernorm_forward(a1, stats1, self.ln1, counters)
        qkv_q = self.qkv.forward(ln1_out, counters, threads)
        if self.attn.supports_q():
            attn_q = self.attn.forward_q(qkv_q, batch, seq)
        else:
            attn = self.attn.forward(dequantize(qkv_q, self.attn.dtype), batch, seq)
            attn_q = quantize_per_block(attn, cfg.block)
        proj_q = self.proj.forward(attn_q, counters, threads)
        drop1 = DropoutState.generate(p, (dropout_seed, 1), proj_q.shape)
        branch1 = dropout_forward(proj_q, drop1, counters)
        h, stats2 = add_forward(a1, branch1, width, counters)

        ln2_out, ctx2 = layernorm_forward(h, stats2, self.ln2, counters)
        m1 = self.mlp1.forward(ln2_out, counters, threads)
        g = gelu_forward(m1, counters)
        m2 = self.mlp2.forward(g, counters, threads)
        drop2 = DropoutState.generate(p, (dropout_seed, 2), m2.shape)
        branch2 = dropout_forward(m2, drop2, counters)
        out, _ = add_forward(h, branch2, width, counters)

        self._saved = _SavedForward(batch, seq, ctx1, ctx2, m1, drop1, drop2, quant_saves=[
            ctx1.xq, self.qkv.saved_input, self.proj.saved_input, ctx2.xq,
            self.mlp1.saved_input, m1, self.mlp2.saved_input])
        return out

    @_rt.traced("jf.TransformerBlock.backward")
    def backward(self, dyq: BlockQuantTensor, counters: AccessCounters | None = None,
                 threads: int = 1, grad_hook=None):
        """(dX, grads) as qlayers.py:385-427.  ``grad_hook(grads, names)`` (optional) is called
        as soon as the named FP32 parameter gradients are final, in backward order, so a
        data-parallel caller can overlap their all-reduce with the rest of backward."""
        if self._saved is None:
            raise RuntimeError("backward called before forward")
        s = self._saved
        width = self.config.stats_width

        dm2 = dropout_backward(dyq, s.drop2, counters)
        ov = _rt.overlap_wgrad()
        dg, dw_mlp2, db_mlp2 = self.mlp2.backward(dm2, counters, threads, defer_wgrad=ov)
        dm1 = gelu_backward(s.m1, dg, counters)
        dln2, dw_mlp1, db_mlp1 = self.mlp1.backward(dm1, counters, threads, defer_wgrad=ov)
        dh_branch, dgamma2, dbeta2 = layernorm_backward(s.ctx2, dln2, self.ln2, counters)
        if grad_hook is not None:
            _rt.join_side_streams()
            grad_hook({"mlp2.w": dw_mlp2, "mlp2.b": db_mlp2, "mlp1.w": dw_mlp1, "mlp1.b": db_mlp1,
                       "ln2.gamma": dgamma2, "ln2.beta": dbeta2},
                      ["mlp2.w", "mlp2.b", "mlp1.w", "mlp1.b", "ln2.gamma", "ln2.beta"])
        dh, _ = add_forward(dh_branch, dyq, width, counters)

        dproj = dropout_backward(dh, s.drop1, counters)
        dattn_q, dw_proj, db_proj = self.proj.backward(dproj, counters, threads, defer_wgrad=ov)
        if self.attn.supports_q():
            dqkv_q = self.attn.backward_q(dattn_q, s.batch, s.seq)
        else:
            dqkv = self.attn.backward(dequantize(dattn_q, self.attn.dtype), s.batch, s.seq)
            dqkv_q = quantize_per_block(dqkv, self.config.block)
        dln1, dw_qkv, db_qkv = self.qkv.backward(dqkv_q, counters, threads, defer_wgrad=ov)
        da1_branch, dgamma1, dbeta1 = layernorm_backward(s.ctx1, dln1, self.ln1, counters)
        dx, _ = add_forward(da1_branch, dh, width, counters)
        _rt.join_side_streams()

        if grad_hook is not None:
            grad_hook({"proj.w": dw_proj, "proj.b": db_proj, "qkv.w": dw_qkv, "qkv.b": db_qkv,
                       "ln1.gamma": dgamma1, "ln1.beta": dbeta1},
                      ["proj.w", "proj.b", "qkv.w", "qkv.b", "ln1.gamma", "ln1.beta"])
        grads = {
            "qkv.w": dw_qkv, "qkv.b": db_qkv, "proj.w": dw_proj, "proj.b": db_proj,
            "mlp1.w": dw_mlp1, "mlp1.b": db_mlp1, "mlp2.w": dw_mlp2, "mlp2.b": db_mlp2,
            "ln1.gamma": dgamma1, "ln1.beta": dbeta1, "ln2.gamma": dgamma2, "ln2.beta": dbeta2,
        }
        return dx, grads

    def drop_derived_weights(self) -> None:
        for lin in (self.qkv, self.proj, self.mlp1, self.mlp2):
            lin.drop_derived()

    def saved_activation_bytes(self) -> int:
        if self._saved is None:
            raise RuntimeError("no forward pass recorded")
        return sum(t.nbytes_saved() for t in self._saved.quant_saves)

    def fp16_baseline_bytes(self) -> int:
        if self._saved is None:
            raise RuntimeError("no forward pass recorded")
        return sum(2 * t.values.numel() for t in self._saved.quant_saves)


__all__ = ["AttentionCore", "BlockConfig", "QuantLinear", "TransformerBlock"]
