"""Fused INT8-boundary attention (csrc/attn.cu) vs the oracle.

The reference's island (qlayers.py:187-236) is FP32 attention between a dequantize of
the QKV codes (qlayers.py:350-351) and a quantize of its output; backward dequantizes
dO and quantizes dQ|dK|dV (qlayers.py:406-408).  The fused kernels do the crossings
inside the attention kernels and compute with bf16 operands and FP32 accumulation, so
parity is the tolerance class: FP outputs relative to the tensor's
max-abs, output codes within +-1 of the oracle's quantization of its FP32 result.
"""
import numpy as np
import pytest
import torch

from oracle import int8flow_oracle as O

pytestmark = pytest.mark.gpu

# max-abs-relative tolerances (bf16 operands: 2^-9 relative rounding of Q/K/V/P/dS)
TOL_O, TOL_G = 1.0e-2, 1.5e-2


def cu(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def npy(t):
    return t.detach().cpu().numpy()


def rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


@pytest.fixture
def fused(jf):
    jf.runtime.set_attention("fused")
    yield
    jf.runtime.set_attention("sdpa")


def _inputs(jf, rng, b, s, h, d):
    c = h * d
    qkv = jf.quantize_per_block(cu(rng.standard_normal((b * s, 3 * c)).astype(np.float32)))
    dattn = jf.quantize_per_block(cu((0.1 * rng.standard_normal((b * s, c))).astype(np.float32)))
    return qkv, dattn


@pytest.mark.parametrize("b,s,h,d", [(1, 256, 2, 64), (2, 512, 2, 128), (1, 1024, 16, 64)])
def test_fused_attention_vs_oracle(jf, fused, b, s, h, d):
    rng = np.random.default_rng(7 + s + d)
    c = h * d
    qkv, dattn = _inputs(jf, rng, b, s, h, d)
    core = jf.AttentionCore(h, d, dtype=torch.bfloat16)
    assert core.fused(s)
    out = core.forward_q(qkv, b, s)
    ro, saved = O.attention_f32(O.dequantize(npy(qkv.values), npy(qkv.scales)), b, s, h)
    assert rel(npy(out.dequantize()), ro) <= TOL_O
    # codes vs the oracle's quantization of its own FP32 output: the bf16 operands move
    # O by ~4e-3 of its max, about half a quantization step (1/127 of the block max), so
    # codes flip at rounding boundaries (measured ~10%, never by more than 2)
    oq, os_ = O.quantize(ro)
    dcode = np.abs(npy(out.values).astype(np.int32) - oq.astype(np.int32))
    assert dcode.max() <= 2 and (dcode > 0).mean() <= 0.2, ((dcode > 0).mean(), dcode.max())
    assert np.abs(npy(out.scales) / os_ - 1).max() <= 0.02
    dqkv = core.backward_q(dattn, b, s)
    rg = O.attention_f32_backward(O.dequantize(npy(dattn.values), npy(dattn.scales)), saved, b, s, h)
    got = npy(dqkv.dequantize())
    for i in range(3):
        sl = slice(i * c, (i + 1) * c)
        assert rel(got[:, sl], rg[:, sl]) <= TOL_G, ("qkv"[i], rel(got[:, sl], rg[:, sl]))


def test_fused_attention_deterministic(jf, fused):
    """No atomics: dQ and dK/dV come from separate kernels, so two runs are bit-identical."""
    rng = np.random.default_rng(3)
    b, s, h, d = 1, 512, 4, 128
    qkv, dattn = _inputs(jf, rng, b, s, h, d)
    outs = []
    for _ in range(2):
        core = jf.AttentionCore(h, d, dtype=torch.bfloat16)
        o = core.forward_q(qkv, b, s)
        g = core.backward_q(dattn, b, s)
        outs.append((o.values.clone(), o.scales.clone(), g.values.clone(), g.scales.clone()))
    for x, y in zip(*outs):
        assert torch.equal(x, y)


@pytest.mark.parametrize("b,s,h,d", [(2, 2048, 32, 128), (8, 1024, 16, 64)])
def test_fused_attention_config4_vs_torch_fp32(jf, fused, b, s, h, d):
    """BASELINE config 4's attention shape (batch 2, seq 2048, 32 heads x 128) and the
    GPT-2-medium shape (batch 8, seq 1024, 16 heads x 64) against a torch FP32 SDPA of the
    same dequantized inputs (the numpy oracle's seq^2 x heads probability tensor does not
    fit a test's budget)."""
    rng = np.random.default_rng(4 + d)
    c = h * d
    qkv, dattn = _inputs(jf, rng, b, s, h, d)
    core = jf.AttentionCore(h, d, dtype=torch.bfloat16)
    out = core.forward_q(qkv, b, s)
    dqkv = core.backward_q(dattn, b, s)
    dense = qkv.dequantize().view(b, s, 3, h, d)
    q, k, v = (dense[:, :, i].transpose(1, 2).contiguous().requires_grad_(True) for i in range(3))
    o = torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True)
    do = dattn.dequantize().view(b, s, h, d).transpose(1, 2)
    gq, gk, gv = torch.autograd.grad(o, (q, k, v), do)
    ro = o.detach().transpose(1, 2).reshape(b * s, c)
    assert ((out.dequantize() - ro).abs().max() / ro.abs().max()).item() <= TOL_O
    got = dqkv.dequantize()
    for i, g in enumerate((gq, gk, gv)):
        r = g.transpose(1, 2).reshape(b * s, c)
        e = ((got[:, i * c:(i + 1) * c] - r).abs().max() / r.abs().max()).item()
        assert e <= TOL_G, ("qkv"[i], e)
    jf.check_errors()


def test_fused_matches_sdpa_path(jf):
    """The fused kernels and the SDPA island (both bf16) agree on the same codes."""
    rng = np.random.default_rng(5)
    b, s, h, d = 1, 512, 4, 64
    qkv, dattn = _inputs(jf, rng, b, s, h, d)
    res = {}
    for mode in ("sdpa", "fused"):
        jf.runtime.set_attention(mode)
        try:
            core = jf.AttentionCore(h, d, dtype=torch.bfloat16)
            o = core.forward_q(qkv, b, s).dequantize()
            g = core.backward_q(dattn, b, s).dequantize()
        finally:
            jf.runtime.set_attention("sdpa")
        res[mode] = (o, g)
    for a, r in zip(res["fused"], res["sdpa"]):
        assert ((a - r).abs().max() / r.abs().max()).item() <= 2e-2


def test_fused_unsupported_shape_uses_sdpa(jf, fused):
    """seq % 256 != 0 (or head_dim not in {64, 128}): the island falls back to the SDPA
    kernels, still on the GPU."""
    rng = np.random.default_rng(6)
    b, s, h, d = 2, 64, 4, 32
    qkv, dattn = _inputs(jf, rng, b, s, h, d)
    core = jf.AttentionCore(h, d, dtype=torch.bfloat16)
    assert not core.fused(s)
    out = core.forward_q(qkv, b, s)
    ro, _ = O.attention_f32(O.dequantize(npy(qkv.values), npy(qkv.scales)), b, s, h)
    assert rel(npy(out.dequantize()), ro) <= 2e-2
