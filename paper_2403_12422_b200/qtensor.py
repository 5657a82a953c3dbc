"""Block-quantized INT8 tensors on the GPU (drop-in for int8flow.qtensor).

Mirrors ``int8flow/qtensor.py`` (BlockQuantTensor :73-181,
quantize_per_block :219-246, dequantize :249-255, zeros_like :258-264,
snap_to_f16 :26-28) with CUDA tensors: ``values`` is an int8 [N, C] CUDA
tensor, ``scales`` a float32 [N/32, C/32] CUDA tensor of binary16-grid
values.  All compute runs in libjetfire (sm_100a); the block size is fixed
at 32 (any other block raises ValueError: there is no CPU fallback).
"""

from __future__ import annotations

import struct

import numpy as np
import torch

from . import _lib
from . import runtime as _rt

INT8_MAX = 127
BLOCK = 32
_MAGIC = b"JQT1"


def _as_cuda(x, dtype=None) -> torch.Tensor:
    if isinstance(x, np.ndarray):
        x = torch.from_numpy(np.ascontiguousarray(x))
    if not isinstance(x, torch.Tensor):
        x = torch.as_tensor(x)
    if dtype is not None and x.dtype != dtype:
        x = x.to(dtype)
    if not x.is_cuda:
        _lib.lib()  # raises JetfireUnavailable without a device
        x = x.cuda()
    return x


def snap_to_f16(x):
    """Round to the nearest binary16 value, kept as float32 (qtensor.py:26-28)."""
    if isinstance(x, torch.Tensor):
        return x.to(torch.float16).to(torch.float32)
    return np.asarray(x, dtype=np.float16).astype(np.float32)


class BlockQuantTensor:
    """INT8 codes [N, C] + one binary16-grid FP32 scale per 32 x 32 block."""

    __slots__ = ("values", "scales", "block")

    def __init__(self, values, scales, block: int = BLOCK):
        if isinstance(values, np.ndarray):
            if values.dtype != np.int8:
                raise TypeError(f"values must be int8, got {values.dtype}")
            values = torch.from_numpy(np.ascontiguousarray(values))
        if isinstance(scales, np.ndarray):
            if scales.dtype != np.float32:
                raise TypeError(f"scales must be float32, got {scales.dtype}")
            scales = torch.from_numpy(np.ascontiguousarray(scales))
        if values.dtype != torch.int8:
            raise TypeError(f"values must be int8, got {values.dtype}")
        if scales.dtype != torch.float32:
            raise TypeError(f"scales must be float32, got {scales.dtype}")
        if values.dim() != 2:
            raise ValueError(f"expected a 2-D matrix, got shape {tuple(values.shape)}")
        n, c = values.shape
        if n % block or c % block:
            raise ValueError(f"shape {n}x{c} is not a multiple of block size {block}")
        if tuple(scales.shape) != (n // block, c // block):
            raise ValueError(
                f"scale grid {tuple(scales.shape)} does not match {n}x{c} blocked by {block}"
            )
        if block != BLOCK:
            raise ValueError(f"the B200 path supports block size {BLOCK} only, got {block}")
        self.values = _as_cuda(values).contiguous()
        self.scales = _as_cuda(scales).contiguous()
        self.block = block

    # -- shape ------------------------------------------------------------
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
        return (self.rows, self.cols)

    @property
    def device(self):
        return self.values.device

    def nbytes_saved(self) -> int:
        """Reference accounting: 1 B per code + 2 B (binary16) per scale (qlayers.py:431-438)."""
        return self.values.numel() + 2 * self.scales.numel()

    # -- ops ---------------------------------------------------------------
    def dequantize(self, dtype=torch.float32) -> torch.Tensor:
        return dequantize(self, dtype)

    def transposed(self) -> "BlockQuantTensor":
        """Transposed matrix; square blocks, so the scale grid transposes too."""
        L = _lib.lib()
        qt = torch.empty((self.cols, self.rows), dtype=torch.int8, device=self.device)
        st = torch.empty((self.block_cols, self.block_rows), dtype=torch.float32, device=self.device)
        _lib.check(L.jf_transpose(self.values.data_ptr(), self.scales.data_ptr(), self.rows, self.cols,
                                  qt.data_ptr(), st.data_ptr(), _lib.stream_handle()), "transpose")
        return BlockQuantTensor(qt, st, self.block)

    def numpy(self) -> tuple[np.ndarray, np.ndarray]:
        return self.values.cpu().numpy(), self.scales.cpu().numpy()

    def validate(self) -> None:
        """Format invariants (qtensor.py:138-150); raises AssertionError."""
        v = self.values
        assert int(v.min()) >= -INT8_MAX if v.numel() else True, "value below -127"
        assert int(v.max()) <= INT8_MAX if v.numel() else True, "value above 127"
        s = self.scales
        assert bool(torch.isfinite(s).all()), "non-finite scale"
        assert bool((s >= 0).all()), "negative scale"
        assert torch.equal(s, snap_to_f16(s)), "scale off the binary16 grid"
        blk = v.view(self.block_rows, 32, self.block_cols, 32).abs().amax(dim=(1, 3)) > 0
        assert not bool((blk & (s == 0)).any()), "zero scale on nonzero block"

    # -- JQT1 fixture format (qtensor.py:152-181) ----------------------------
    def to_bytes(self) -> bytes:
        q, s = self.numpy()
        header = _MAGIC + struct.pack("<III", self.rows, self.cols, self.block)
        return header + q.tobytes() + s.astype(np.float16).view(np.uint16).astype("<u2").tobytes()

    @classmethod
    def from_bytes(cls, raw: bytes) -> "BlockQuantTensor":
        if raw[:4] != _MAGIC:
            raise ValueError(f"bad magic {raw[:4]!r}, expected {_MAGIC!r}")
        rows, cols, block = struct.unpack_from("<III", raw, 4)
        vals = np.frombuffer(raw, np.int8, rows * cols, 16).reshape(rows, cols).copy()
        nb = (rows // block) * (cols // block)
        bits = np.frombuffer(raw, "<u2", nb, 16 + rows * cols)
        scales = bits.view(np.float16).astype(np.float32).reshape(rows // block, cols // block)
        return cls(vals, scales, block)

    def save(self, path) -> None:
        with open(path, "wb") as fh:
            fh.write(self.to_bytes())

    @classmethod
    def load(cls, path) -> "BlockQuantTensor":
        with open(path, "rb") as fh:
            return cls.from_bytes(fh.read())

    def __repr__(self) -> str:
        return f"BlockQuantTensor(shape={self.shape}, block={self.block}, device={self.device})"


def empty_like_shape(n: int, c: int, device) -> BlockQuantTensor:
    """Uninitialized codes + scales (internal: outputs written by a kernel)."""
    t = BlockQuantTensor.__new__(BlockQuantTensor)
    t.values = torch.empty((n, c), dtype=torch.int8, device=device)
    t.scales = torch.empty((n // BLOCK, c // BLOCK), dtype=torch.float32, device=device)
    t.block = BLOCK
    return t


def _check_block(block: int) -> None:
    if block <= 0:
        raise ValueError(f"block size must be positive, got {block}")
    if block != BLOCK:
        raise ValueError(f"the B200 path supports block size {BLOCK} only, got {block}")


def quantize_per_block(x, block: int = BLOCK, *, out: BlockQuantTensor | None = None) -> BlockQuantTensor:
    """Per-block absmax INT8 quantizer (qtensor.py:219-246) — kernel K1.

    ``x``: float32 or bfloat16 2-D tensor (CUDA; numpy arrays are uploaded).
    Raises the reference's ValueErrors (2-D, block, multiple, non-finite,
    binary16 overflow).  ``out`` (extension): write the codes and scales into
    an existing tensor of the same shape (stable addresses for captured graphs).
    """
    if not isinstance(x, torch.Tensor):
        x = np.asarray(x)
        if x.ndim != 2:
            raise ValueError(f"expected a 2-D matrix, got shape {x.shape}")
        x = _as_cuda(np.ascontiguousarray(x, dtype=np.float32))
    if x.dim() != 2:
        raise ValueError(f"expected a 2-D matrix, got shape {tuple(x.shape)}")
    n, c = x.shape
    if block <= 0:
        raise ValueError(f"block size must be positive, got {block}")
    if n % block or c % block:
        raise ValueError(f"shape {n}x{c} is not a multiple of block size {block}")
    _check_block(block)
    L = _lib.lib()
    x = _as_cuda(x)
    if x.dtype not in (torch.float32, torch.bfloat16):
        x = x.to(torch.float32)
    if x.stride(1) != 1 or x.stride(0) < c or (x.data_ptr() % 16):
        x = x.contiguous()
    if out is None:
        out = empty_like_shape(n, c, x.device)
    elif out.shape != (n, c) or out.device != x.device:
        raise ValueError(f"out has shape {out.shape}, expected {(n, c)}")
    fn = L.jf_quantize_f32 if x.dtype == torch.float32 else L.jf_quantize_bf16
    if x.dtype == torch.bfloat16 and x.stride(0) % 8:
        x = x.contiguous()
    _lib.check(fn(x.data_ptr(), n, c, x.stride(0), out.values.data_ptr(), out.scales.data_ptr(),
                  _rt.err_ptr(), _lib.stream_handle()), "quantize")
    _rt.maybe_check()
    return out


def dequantize(xq: BlockQuantTensor, dtype=torch.float32) -> torch.Tensor:
    """codes * block scale (qtensor.py:249-255) — kernel K2; exact in float32."""
    L = _lib.lib()
    y = torch.empty(xq.shape, dtype=dtype, device=xq.device)
    if dtype == torch.float32:
        rc = L.jf_dequantize_f32(xq.values.data_ptr(), xq.scales.data_ptr(), xq.rows, xq.cols,
                                 y.data_ptr(), _lib.stream_handle())
    elif dtype == torch.bfloat16:
        rc = L.jf_dequantize_bf16(xq.values.data_ptr(), xq.scales.data_ptr(), xq.rows, xq.cols,
                                  y.data_ptr(), _lib.stream_handle())
    else:
        raise TypeError(f"dequantize supports float32/bfloat16 outputs, got {dtype}")
    _lib.check(rc, "dequantize")
    return y


def zeros_like(xq: BlockQuantTensor) -> BlockQuantTensor:
    """All-zero codes with scale 1 per block (qtensor.py:258-264)."""
    return BlockQuantTensor(torch.zeros_like(xq.values), torch.ones_like(xq.scales), xq.block)
