"""Small-shape driver for compute-sanitizer (memcheck / racecheck / synccheck):
one launch of each hand-written pipeline -- the tcgen05 GEMM kernels (TMA-staged
scales, MN-major operands, a second tile per CTA, generic-shape kernel with partial tiles, int32
partials, f16-widened operands), Add+stats, LayerNorm fwd/bwd, GELU fwd/bwd,
the quantizer, the column sum, the fused INT8-boundary attention (forward and
both backward kernels, head_dim 64 and 128) and the device Philox dropout mask.  Usage:
  compute-sanitizer --tool racecheck python tools/sanitize_driver.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_12422_b200 as jf  # noqa: E402
from paper_2403_12422_b200 import runtime  # noqa: E402


def q(shape, scale=1.0, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return jf.quantize_per_block(torch.randn(shape, generator=g, device="cuda") * scale)


def main():
    jf.require_cuda()
    x, w, dy = q((256, 384), seed=1), q((256, 384), 0.05, seed=2), q((256, 256), 0.1, seed=3)
    for prom in ("exact", "fast"):
        runtime.set_promotion(prom)
        jf.block_mm_forward(x, w, bias=torch.zeros(256, device="cuda"))   # i8s, K-major
        jf.block_mm_grad_input(dy, w)                                      # i8s, MN-major B
        jf.block_mm_grad_weight(dy, x, quantize=False)                     # i8s, MN-major A and B
    runtime.set_promotion("exact")
    # more output tiles (256) than SMs: CTAs run a tile's epilogue and then a second tile
    xb, wb = q((2048, 128), seed=10), q((2048, 128), 0.1, seed=11)
    jf.block_mm_forward(xb, wb, bias=torch.zeros(2048, device="cuda"))
    xg, wg = q((160, 96), seed=4), q((224, 96), seed=5)                    # generic kernel, partial tiles
    jf.block_mm_forward(xg, wg)
    jf.block_partials(xg.values, wg.values, 1)                            # int32 partials
    runtime.set_gemm_operands("f16")
    jf.block_mm_forward(x, w)                                              # f16-widened operands
    runtime.set_gemm_operands("int8")
    a, st = jf.add_forward(x, q((256, 384), seed=6), 64)
    ln = jf.NormParams(torch.ones(384, device="cuda"), torch.zeros(384, device="cuda"))
    y, ctx = jf.layernorm_forward(a, st, ln)
    jf.layernorm_backward(ctx, q((256, 384), 0.1, seed=7), ln)
    g = jf.gelu_forward(x)
    jf.gelu_backward(x, g)
    jf.column_sum(dy)
    runtime.set_attention("fused")
    for h, d in ((2, 64), (1, 128)):
        core = jf.AttentionCore(h, d, dtype=torch.bfloat16)
        qkv = q((256, 3 * h * d), seed=8)
        assert core.fused(256)
        core.forward_q(qkv, 1, 256)
        core.backward_q(q((256, h * d), 0.1, seed=9), 1, 256)
    runtime.set_attention("sdpa")
    st_ = jf.DropoutState.generate(0.2, (5, 1), (256, 384))
    jf.dropout_forward(x, st_)
    torch.cuda.synchronize()
    jf.check_errors()
    print("sanitize driver ok")


if __name__ == "__main__":
    main()
