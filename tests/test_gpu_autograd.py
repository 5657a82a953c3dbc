"""autograd form of the block (paper_2403_12422_b200.autograd) vs the
hand-driven TransformerBlock: same kernels, same order -> same bits."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _pair(jf, attn_dtype):
    from paper_2403_12422_b200 import autograd as A

    torch.manual_seed(0)
    cfg = jf.BlockConfig(c_model=128, heads=4, hidden=512, block=32, dropout_p=0.0)
    mod = A.JetfireTransformerBlock(cfg, attn_dtype=attn_dtype)
    with torch.no_grad():
        for m in (mod.qkv, mod.proj, mod.mlp1, mod.mlp2):
            m.bias.normal_(std=0.1)
        mod.ln1_gamma.uniform_(0.5, 1.5)
        mod.ln2_beta.normal_(std=0.1)
    p = {"qkv.w": mod.qkv.weight, "qkv.b": mod.qkv.bias, "proj.w": mod.proj.weight, "proj.b": mod.proj.bias,
         "mlp1.w": mod.mlp1.weight, "mlp1.b": mod.mlp1.bias, "mlp2.w": mod.mlp2.weight, "mlp2.b": mod.mlp2.bias,
         "ln1.gamma": mod.ln1_gamma, "ln1.beta": mod.ln1_beta, "ln2.gamma": mod.ln2_gamma,
         "ln2.beta": mod.ln2_beta}
    blk = jf.TransformerBlock.from_parameters(cfg, {k: v.detach().clone() for k, v in p.items()},
                                              attn_dtype=attn_dtype)
    return A, cfg, mod, blk, p


@pytest.mark.parametrize("attn_dtype", [torch.float32, torch.bfloat16])
def test_autograd_block_matches_explicit(jf, attn_dtype):
    A, cfg, mod, blk, p = _pair(jf, attn_dtype)
    batch, seq = 2, 64
    n = batch * seq
    x = torch.randn(n, cfg.c_model, device="cuda")
    dy = 0.1 * torch.randn(n, cfg.c_model, device="cuda")
    xq = jf.quantize_per_block(x)
    dyq = jf.quantize_per_block(dy)

    ref_out = blk.forward(xq, batch, seq)
    ref_dx, ref_g = blk.backward(dyq)

    xin = A.QTensor(xq, requires_grad=True)
    out = mod(xin, batch, seq)
    assert isinstance(out, A.QTensor)
    assert torch.equal(out.bq.values, ref_out.values) and torch.equal(out.bq.scales, ref_out.scales)
    out.backward(A.QTensor(dyq))
    assert isinstance(xin.grad, A.QTensor)
    assert torch.equal(xin.grad.bq.values, ref_dx.values)
    assert torch.equal(xin.grad.bq.scales, ref_dx.scales)
    for k, t in p.items():
        assert torch.equal(t.grad, ref_g[k]), k


def test_autograd_quantize_boundary(jf):
    from paper_2403_12422_b200 import autograd as A

    lin = A.JetfireLinear(64, 96)
    x = torch.randn(32, 64, device="cuda", requires_grad=True)
    y = A.dequantize_q(lin(A.quantize(x)))
    ref = jf.block_mm_forward(jf.quantize_per_block(x.detach()), lin.quant().weight_q, bias=lin.bias.detach())
    assert torch.equal(y, ref.dequantize())
    g = torch.randn_like(y)
    y.backward(g)
    gq = jf.quantize_per_block(g)
    want = jf.block_mm_grad_input(gq, lin.quant().weight_q).dequantize()
    assert torch.equal(x.grad, want)
    assert torch.equal(lin.bias.grad, jf.column_sum(gq))
    # optimizer step -> the INT8 copy is re-derived
    with torch.no_grad():
        lin.weight.add_(1.0)
    lin.mark_updated()
    assert torch.equal(lin.quant().weight_q.values, jf.quantize_per_block(lin.weight.detach()).values)


def test_layernorm_needs_stats(jf):
    from paper_2403_12422_b200 import autograd as A

    xq = A.quantize(torch.randn(32, 64, device="cuda"))
    with pytest.raises(ValueError, match="statistics"):
        A.LayerNorm.apply(xq, torch.ones(64, device="cuda"), torch.zeros(64, device="cuda"), 1e-5)
