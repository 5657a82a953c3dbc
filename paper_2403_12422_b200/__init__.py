"""Jetfire INT8 data flow on B200 (sm_100a): a drop-in for the hot path of
the reference ``int8flow`` package (arXiv 2403.12422).

Same names and signatures as ``int8flow`` for the hot path — per-block
quantizer, block INT8 GEMMs, fused INT8 GELU / Add+stats / LayerNorm /
Dropout, QuantLinear and TransformerBlock — with every kernel in
``libjetfire.so`` (hand-written tcgen05/TMA CUDA, C ABI in
``include/jetfire.h``).  There is no CPU fallback.
"""

from . import autograd, dist, runtime
from ._lib import JetfireUnavailable, load_library
from .qgemm import (
    COUNTER_CSV_HEADER,
    AccessCounters,
    CounterLog,
    DenseResult,
    ExecMode,
    TileConfig,
    block_mm_forward,
    block_mm_grad_input,
    block_mm_grad_weight,
    block_partials,
    micro_mm_16,
)
from .qlayers import AttentionCore, BlockConfig, QuantLinear, TransformerBlock
from .qnonlinear import (
    DropoutState,
    LayerNormContext,
    NormParams,
    RowStats,
    add_forward,
    column_sum,
    count_elementwise,
    dropout_backward,
    dropout_forward,
    gelu_backward,
    gelu_forward,
    layernorm_backward,
    layernorm_forward,
)
from .qtensor import INT8_MAX, BlockQuantTensor, dequantize, quantize_per_block, snap_to_f16, zeros_like
from .runtime import check_errors, set_error_check, set_promotion


def require_cuda():
    """Load libjetfire and check for a CUDA device; raises JetfireUnavailable."""
    from . import _lib

    return _lib.lib()


__all__ = [
    "COUNTER_CSV_HEADER", "INT8_MAX", "AccessCounters", "AttentionCore", "BlockConfig",
    "BlockQuantTensor", "CounterLog", "DenseResult", "DropoutState", "ExecMode", "JetfireUnavailable",
    "LayerNormContext", "NormParams", "QuantLinear", "RowStats", "TileConfig", "TransformerBlock",
    "add_forward", "block_mm_forward", "block_mm_grad_input", "block_mm_grad_weight", "block_partials",
    "check_errors", "column_sum", "count_elementwise", "dequantize", "dropout_backward",
    "dropout_forward", "gelu_backward", "gelu_forward", "layernorm_backward", "layernorm_forward",
    "autograd", "dist", "load_library", "micro_mm_16", "quantize_per_block", "require_cuda", "runtime", "set_error_check",
    "set_promotion", "snap_to_f16", "zeros_like",
]

__version__ = "0.1.0"
