"""numpy-facing ``int8flow.qgemm``: the three block GEMMs run on the GPU (tcgen05)."""

from __future__ import annotations

import numpy as np

from paper_2403_12422_b200 import qgemm as _g

from .qtensor import gpu, host, wrap

COUNTER_CSV_HEADER = _g.COUNTER_CSV_HEADER
AccessCounters = _g.AccessCounters
CounterLog = _g.CounterLog
ExecMode = _g.ExecMode
TileConfig = _g.TileConfig


DenseResult = _g.DenseResult


def _out(r):
    from paper_2403_12422_b200.qtensor import BlockQuantTensor as GB

    if isinstance(r, _g.DenseResult):
        return _g.DenseResult(host(r.values), r.scale)
    if isinstance(r, GB):
        return wrap(r)
    return host(r)


def _bias(b):
    return None if b is None else np.asarray(b, dtype=np.float32)


def block_mm_forward(xq, wq, cfg=None, mode=ExecMode.INT8_DATA_FLOW, counters=None, *, bias=None,
                     threads: int = 1, quantize: bool = True):
    return _out(_g.block_mm_forward(gpu(xq), gpu(wq), cfg, mode, counters, bias=_bias(bias),
                                    threads=threads, quantize=quantize))


def block_mm_grad_input(dyq, wq, cfg=None, mode=ExecMode.INT8_DATA_FLOW, counters=None, *,
                        threads: int = 1, quantize: bool = True):
    return _out(_g.block_mm_grad_input(gpu(dyq), gpu(wq), cfg, mode, counters, threads=threads,
                                       quantize=quantize))


def block_mm_grad_weight(dyq, xq, cfg=None, mode=ExecMode.INT8_DATA_FLOW, counters=None, *,
                         threads: int = 1, quantize: bool = True):
    return _out(_g.block_mm_grad_weight(gpu(dyq), gpu(xq), cfg, mode, counters, threads=threads,
                                        quantize=quantize))


def micro_mm_16(a, bt):
    return host(_g.micro_mm_16(a, bt))
