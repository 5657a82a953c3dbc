"""numpy-facing ``int8flow.qnonlinear``: GELU, Add+stats, LayerNorm and dropout run on
the GPU; the FP32 helper functions the suites use as oracles come from the reference."""

from __future__ import annotations

import numpy as np
import torch

from paper_2403_12422_b200 import qnonlinear as _g

from ._ref import qnonlinear as _r
from .qtensor import gpu, host, wrap

# FP32 helpers / oracles (not kernels): the reference's own
norm_cdf = _r.norm_cdf
gelu_f32 = _r.gelu_f32
gelu_grad_f32 = _r.gelu_grad_f32
layernorm_f32 = _r.layernorm_f32
layernorm_grad_f32 = _r.layernorm_grad_f32
compute_row_stats = _r.compute_row_stats
count_elementwise = _g.count_elementwise
NormParams = _r.NormParams            # numpy dataclass; converted per call
RowStats = _r.RowStats
LayerNormContext = _r.LayerNormContext
DropoutState = _r.DropoutState        # numpy Philox mask, as the reference draws it


def _stats_gpu(s) -> _g.RowStats:
    return _g.RowStats(torch.from_numpy(np.ascontiguousarray(s.mean)).cuda(),
                       torch.from_numpy(np.ascontiguousarray(s.sumsq)).cuda(), s.width)


def _params_gpu(p) -> _g.NormParams:
    return _g.NormParams(np.asarray(p.gamma, np.float32), np.asarray(p.beta, np.float32), p.eps)


def _drop_gpu(state) -> _g.DropoutState:
    mask = np.asarray(state.mask)
    if state.p == 0.0 and mask.all():
        return _g.DropoutState(state.p, state.seed, None)
    return _g.DropoutState(state.p, state.seed, torch.from_numpy(np.ascontiguousarray(mask)).cuda())


def gelu_forward(xq, counters=None):
    return wrap(_g.gelu_forward(gpu(xq), counters))


def gelu_backward(xq, dyq, counters=None):
    return wrap(_g.gelu_backward(gpu(xq), gpu(dyq), counters))


def dropout_forward(xq, state, counters=None):
    return wrap(_g.dropout_forward(gpu(xq), _drop_gpu(state), counters))


def dropout_backward(dyq, state, counters=None):
    return wrap(_g.dropout_backward(gpu(dyq), _drop_gpu(state), counters))


def add_forward(x1q, x2q, stats_width: int = 64, counters=None):
    y, st = _g.add_forward(gpu(x1q), gpu(x2q), stats_width, counters)
    return wrap(y), RowStats(host(st.mean), host(st.sumsq), st.width)


def layernorm_forward(xq, stats, params, counters=None):
    if stats.mean.shape[0] != xq.rows or stats.cols != xq.cols:
        raise ValueError(f"stats for {stats.mean.shape[0]}x{stats.cols} do not match tensor {xq.shape}")
    y, ctx = _g.layernorm_forward(gpu(xq), _stats_gpu(stats), _params_gpu(params), counters)
    return wrap(y), LayerNormContext(xq, host(ctx.mu), host(ctx.inv_std))


def layernorm_backward(ctx, dyq, params, counters=None):
    gctx = _g.LayerNormContext(gpu(ctx.xq), torch.from_numpy(np.ascontiguousarray(ctx.mu)).cuda(),
                               torch.from_numpy(np.ascontiguousarray(ctx.inv_std)).cuda())
    dx, dg, db = _g.layernorm_backward(gctx, gpu(dyq), _params_gpu(params), counters)
    return wrap(dx), host(dg), host(db)


