"""Full-size checks at the BASELINE config-4 shapes (hidden 4096, MLP 16384,
4096 tokens), through properties that do not need a full-size oracle run
(the oracle comparisons live in test_gpu_kernels.py):

* the quantizer against the vectorised oracle on one full activation;
* GEMM cross-identities: fwd(X, W) is dgrad(X, Wᵀ) (K-major vs MN-major B
  operand) and wgrad(dY, X) is fwd(dYᵀ, Xᵀ) -- the same chunk products in the
  same K order, so the bits must agree; the int8 and f16-widened operand
  paths agree;
* the whole block fwd+bwd raises no error flag and repeats bit for bit up to
  the attention backward (cuDNN's dQ accumulation is not deterministic).
"""

import numpy as np
import pytest
import torch

from oracle import int8flow_oracle as O

pytestmark = pytest.mark.gpu

N, C, H = 4096, 4096, 16384


def _q(jf, shape, scale=1.0, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return jf.quantize_per_block(torch.randn(shape, generator=g, device="cuda") * scale)


def _eq(a, b):
    return torch.equal(a.values, b.values) and torch.equal(a.scales, b.scales)


def test_quantize_full_activation_vs_oracle(jf):
    rng = np.random.default_rng(0)
    x = rng.standard_normal((N, H), dtype=np.float32)
    x[:, rng.choice(H, H // 100, replace=False)] *= 30.0  # SURVEY §8d outlier variant
    t = jf.quantize_per_block(torch.from_numpy(x).cuda())
    q, s = O.quantize(x)
    assert np.array_equal(t.values.cpu().numpy(), q)
    assert np.array_equal(t.scales.cpu().numpy(), s)


def test_gemm_fwd_equals_dgrad_on_transposed_weight(jf):
    x = _q(jf, (N, C), seed=1)
    w = _q(jf, (H, C), C ** -0.5, seed=2)           # mlp1 weight [H x C]
    y = jf.block_mm_forward(x, w)                   # X W^T, W read K-major
    y2 = jf.block_mm_grad_input(x, w.transposed())  # X (W^T), W^T read MN-major
    assert _eq(y, y2)


def test_gemm_wgrad_equals_fwd_on_transposes(jf):
    dy = _q(jf, (N, C), 0.1, seed=3)
    x = _q(jf, (N, H), seed=4)
    dw = jf.block_mm_grad_weight(dy, x)             # dY^T X, both read MN-major
    dw2 = jf.block_mm_forward(dy.transposed(), x.transposed())  # (dY^T)(X^T)^T, K-major
    assert _eq(dw, dw2)


def test_gemm_operand_paths_agree_full_size(jf):
    from paper_2403_12422_b200 import runtime

    x = _q(jf, (N, C), seed=5)
    w = _q(jf, (3 * C, C), C ** -0.5, seed=6)        # qkv weight
    prev = runtime.gemm_operands()
    try:
        runtime.set_gemm_operands("int8")
        a = jf.block_mm_forward(x, w)
        runtime.set_gemm_operands("f16")
        b = jf.block_mm_forward(x, w)
    finally:
        runtime.set_gemm_operands(prev)
    assert _eq(a, b)


def test_block_full_size_deterministic(jf):
    from paper_2403_12422_b200.qlayers import BlockConfig, QuantLinear, TransformerBlock

    rng = np.random.default_rng(7)
    cfg = BlockConfig(c_model=C, heads=32, hidden=H)
    lin = [QuantLinear.initialize(rng, d, c) for d, c in ((3 * C, C), (C, C), (H, C), (C, H))]
    blk = TransformerBlock(cfg, *lin, jf.NormParams(torch.ones(C, device="cuda"), torch.zeros(C, device="cuda")),
                           jf.NormParams(torch.ones(C, device="cuda"), torch.zeros(C, device="cuda")),
                           attn_dtype=torch.bfloat16)
    x = _q(jf, (N, C), seed=8)
    dy = _q(jf, (N, C), 0.1, seed=9)
    runs = []
    for _ in range(2):
        out = blk.forward(x, 2, 2048)
        dx, grads = blk.backward(dy)
        runs.append((out, dx, {k: v.clone() for k, v in grads.items() if v is not None}))
    jf.check_errors()
    (o1, d1, g1), (o2, d2, g2) = runs
    assert _eq(o1, o2)
    # everything upstream of the attention backward (cuDNN's dQ accumulation is not
    # bit-deterministic) must repeat bit for bit
    for k in ("mlp2.w", "mlp2.b", "mlp1.w", "mlp1.b", "ln2.gamma", "ln2.beta"):
        assert torch.equal(g1[k], g2[k]), k
    for k in g1:
        assert bool(torch.isfinite(g1[k]).all()), k
    assert bool(torch.isfinite(d1.dequantize()).all())
