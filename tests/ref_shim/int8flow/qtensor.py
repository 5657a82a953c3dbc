"""numpy-facing ``int8flow.qtensor`` over the GPU module (hot path on the GPU)."""

from __future__ import annotations

import numpy as np
import torch

from paper_2403_12422_b200 import qtensor as _g

from ._ref import qtensor as _r

INT8_MAX = _r.INT8_MAX
snap_to_f16 = _r.snap_to_f16  # host helper (qtensor.py:26-28), not a kernel
# ablation-only quantization schemes (qtensor.py:31-70, 267-310; out of scope)
PER_TENSOR, PER_TOKEN, PER_CHANNEL = _r.PER_TENSOR, _r.PER_TOKEN, _r.PER_CHANNEL
QuantScheme, SchemeKind = _r.QuantScheme, _r.SchemeKind
quantize_with_scheme, quantization_error = _r.quantize_with_scheme, _r.quantization_error


def _frozen(a: np.ndarray) -> np.ndarray:
    a = np.array(a, copy=True)
    a.flags.writeable = False
    return a


class BlockQuantTensor:
    """The reference container (frozen numpy ``values``/``scales``) mirrored by a CUDA
    BlockQuantTensor that every op runs on."""

    def __init__(self, values, scales, block: int):
        # the GPU module's constructor applies the reference's Type/ValueError checks
        self._gpu = _g.BlockQuantTensor(np.asarray(values), np.asarray(scales), block)
        self.values = _frozen(values)
        self.scales = _frozen(scales)
        self.block = block

    @classmethod
    def from_gpu(cls, t: _g.BlockQuantTensor) -> "BlockQuantTensor":
        obj = cls.__new__(cls)
        obj._gpu = t
        obj.values = _frozen(t.values.cpu().numpy())
        obj.scales = _frozen(t.scales.cpu().numpy())
        obj.block = t.block
        return obj

    @property
    def gpu(self) -> _g.BlockQuantTensor:
        return self._gpu

    @property
    def rows(self) -> int:
        return self.values.shape[0]

    @property
    def cols(self) -> int:
        return self.values.shape[1]

    @property
    def block_rows(self) -> int:
        return self.scales.shape[0]

    @property
    def block_cols(self) -> int:
        return self.scales.shape[1]

    @property
    def shape(self) -> tuple[int, int]:
        return self.values.shape

    def dequantize(self) -> np.ndarray:
        return _g.dequantize(self._gpu).cpu().numpy()

    def transposed(self) -> "BlockQuantTensor":
        return BlockQuantTensor.from_gpu(self._gpu.transposed())

    def validate(self) -> None:
        self._gpu.validate()

    def to_bytes(self) -> bytes:
        return self._gpu.to_bytes()

    @classmethod
    def from_bytes(cls, raw: bytes) -> "BlockQuantTensor":
        return cls.from_gpu(_g.BlockQuantTensor.from_bytes(raw))


def gpu(t: BlockQuantTensor | None):
    return None if t is None else t.gpu


def wrap(t):
    return None if t is None else BlockQuantTensor.from_gpu(t)


def quantize_per_block(x, block: int) -> BlockQuantTensor:
    return BlockQuantTensor.from_gpu(_g.quantize_per_block(np.asarray(x), block))


def dequantize(xq: BlockQuantTensor) -> np.ndarray:
    return xq.dequantize()


def zeros_like(xq: BlockQuantTensor) -> BlockQuantTensor:
    return BlockQuantTensor.from_gpu(_g.zeros_like(xq.gpu))


def host(t):
    """CUDA tensor -> numpy (FP32 outputs of the GPU ops)."""
    if isinstance(t, torch.Tensor):
        return t.detach().cpu().numpy()
    return t
