"""numpy-facing ``int8flow.qlayers``: QuantLinear and TransformerBlock are the GPU
module's (every operator on the GPU); the FP32 ``AttentionCore``, the FP32/fake-quant
twin ``ReferenceBlock`` and the checkpoint I/O are the reference's own."""

from __future__ import annotations

from types import SimpleNamespace

import numpy as np
import torch

from paper_2403_12422_b200 import qlayers as _g
from paper_2403_12422_b200 import qnonlinear as _gn

from ._ref import qlayers as _r
from .qnonlinear import NormParams
from .qtensor import gpu, host, wrap

BlockConfig = _g.BlockConfig
AttentionCore = _r.AttentionCore
ReferenceBlock = _r.ReferenceBlock
save_params = _r.save_params
load_params = _r.load_params


def _cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


class QuantLinear:
    """Reference attribute semantics (mutable numpy ``master_weight``/``bias``, lazily
    cached ``weight_q`` refreshed by ``mark_updated``) over a GPU QuantLinear."""

    def __init__(self, master_weight, bias=None, block: int = 32, cfg=None):
        self._inner = _g.QuantLinear(master_weight, bias, block, cfg)  # reference checks
        self.master_weight = np.ascontiguousarray(master_weight, dtype=np.float32)
        self.bias = None if bias is None else np.asarray(bias, dtype=np.float32)
        self.block = block
        self.cfg = cfg
        self._weight_q = None

    @classmethod
    def initialize(cls, rng, d: int, c: int, *, bias: bool = True, block: int = 32, gain: float = 1.0):
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
    def weight_q(self):
        if self._weight_q is None:
            inner = self._inner
            inner.master_weight.copy_(_cuda(self.master_weight))
            inner._weight_q = None          # a NEW tensor (the reference re-creates it)
            inner.drop_derived()
            self._weight_q = wrap(inner.weight_q)
        return self._weight_q

    def mark_updated(self) -> None:
        self._weight_q = None

    def _sync(self) -> None:
        self.weight_q  # noqa: B018  (refresh from the numpy master if invalidated)
        if self.bias is not None:
            self._inner.bias.copy_(_cuda(self.bias))  # read at every call, as the reference

    @property
    def saved_input(self):
        return wrap(self._inner.saved_input)

    def forward(self, xq, counters=None, threads: int = 1):
        self._sync()
        return wrap(self._inner.forward(gpu(xq), counters, threads))

    def backward(self, dyq, counters=None, threads: int = 1):
        dxq, dw, db = self._inner.backward(gpu(dyq), counters, threads)
        return wrap(dxq), host(dw), host(db)


def _drop_host(st):
    """GPU DropoutState (mask None = keep all at p = 0) -> the reference's numpy form."""
    from .qnonlinear import DropoutState

    mask = None if st.mask is None else st.mask.cpu().numpy().astype(bool)
    return DropoutState(st.p, st.seed, mask)


def _norm_gpu(p) -> _gn.NormParams:
    return _gn.NormParams(np.asarray(p.gamma, np.float32), np.asarray(p.beta, np.float32), p.eps)


class TransformerBlock:
    """The GPU TransformerBlock (qlayers.py:256-444 wiring, INT8 between all operators),
    with the reference's numpy-facing attributes."""

    def __init__(self, config, qkv, proj, mlp1, mlp2, ln1, ln2):
        self.config = config
        self.qkv, self.proj, self.mlp1, self.mlp2 = qkv, proj, mlp1, mlp2
        self.ln1, self.ln2 = ln1, ln2
        self._inner = None
        self._saved = None

    @classmethod
    def initialize(cls, rng, config, *, residual_gain: float = 1.0) -> "TransformerBlock":
        c, h, b = config.c_model, config.hidden, config.block
        return cls(
            config,
            qkv=QuantLinear.initialize(rng, 3 * c, c, block=b),
            proj=QuantLinear.initialize(rng, c, c, block=b, gain=residual_gain),
            mlp1=QuantLinear.initialize(rng, h, c, block=b),
            mlp2=QuantLinear.initialize(rng, c, h, block=b, gain=residual_gain),
            ln1=NormParams(np.ones(c, np.float32), np.zeros(c, np.float32), config.eps),
            ln2=NormParams(np.ones(c, np.float32), np.zeros(c, np.float32), config.eps),
        )

    def parameters(self) -> dict:
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

    def forward(self, xq, batch: int, seq: int, *, dropout_seed: int = 0, train: bool = True,
                counters=None, threads: int = 1):
        lins = (self.qkv, self.proj, self.mlp1, self.mlp2)
        for lin in lins:
            lin._sync()
        self._inner = _g.TransformerBlock(self.config, *(lin._inner for lin in lins), _norm_gpu(self.ln1),
                                          _norm_gpu(self.ln2), attn_dtype=torch.float32)
        out = self._inner.forward(gpu(xq), batch, seq, dropout_seed=dropout_seed, train=train,
                                  counters=counters, threads=threads)
        sv = self._inner._saved
        self._saved = SimpleNamespace(quant_saves=[wrap(t) for t in sv.quant_saves],
                                      drop1=_drop_host(sv.drop1), drop2=_drop_host(sv.drop2))
        return wrap(out)

    def backward(self, dyq, counters=None, threads: int = 1):
        if self._inner is None:
            raise RuntimeError("backward called before forward")
        dx, grads = self._inner.backward(gpu(dyq), counters, threads)
        return wrap(dx), {k: host(v) for k, v in grads.items()}

    def saved_activation_bytes(self) -> int:
        if self._inner is None:
            raise RuntimeError("no forward pass recorded")
        return self._inner.saved_activation_bytes()

    def fp16_baseline_bytes(self) -> int:
        if self._inner is None:
            raise RuntimeError("no forward pass recorded")
        return self._inner.fp16_baseline_bytes()
