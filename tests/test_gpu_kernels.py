"""GPU parity: every libjetfire kernel vs the CPU oracle and the reference's
golden fixtures (tests/golden, produced by the unmodified reference).

Contract: codes, scales, int32 partials, exact-mode FP32
accumulators, Add statistics, LayerNorm and GELU-forward outputs are
bit-exact; GELU backward (numpy SIMD exp) and the axis-0 parameter-gradient
sums are compared under stated tolerances.
"""

import numpy as np
import pytest
import torch

from oracle import int8flow_oracle as O

pytestmark = pytest.mark.gpu


def cu(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def npy(t):
    return t.detach().cpu().numpy()


def bqt(jf, q, s):
    return jf.BlockQuantTensor(cu(q), cu(s))


def same(t, ref):
    a = npy(t) if isinstance(t, torch.Tensor) else t
    return a.shape == ref.shape and a.tobytes() == np.ascontiguousarray(ref, dtype=a.dtype).tobytes()


# ── K1 / K2 ─────────────────────────────────────────────────────────────


def test_quantize_golden(jf, golden):
    g = golden("quant")
    for name in g["names"]:
        t = jf.quantize_per_block(cu(g[f"{name}_x"]))
        assert same(t.values, g[f"{name}_q"]), name
        assert same(t.scales, g[f"{name}_s"]), name
        assert same(t.dequantize(), g[f"{name}_deq"]), name


def test_quantize_bf16_input(jf, golden):
    g = golden("quant")
    x = cu(g["bf16_x"]).to(torch.bfloat16)
    t = jf.quantize_per_block(x)
    assert same(t.values, g["bf16_q"]) and same(t.scales, g["bf16_s"])


@pytest.mark.parametrize("shape", [(32, 32), (96, 160), (256, 4096), (2048, 1056)])
@pytest.mark.parametrize("scale", [1e-6, 1.0, 3e3])
def test_quantize_random_vs_oracle(jf, shape, scale):
    rng = np.random.default_rng(shape[0] * 7 + shape[1])
    x = (rng.standard_normal(shape) * scale).astype(np.float32)
    x[rng.random(shape) < 0.01] *= 30.0
    q, s = O.quantize(x)
    t = jf.quantize_per_block(cu(x))
    assert same(t.values, q) and same(t.scales, s)


def test_quantize_strided_input(jf):
    rng = np.random.default_rng(3)
    big = rng.standard_normal((64, 256)).astype(np.float32)
    view = cu(big)[:, 64:192]
    q, s = O.quantize(big[:, 64:192])
    t = jf.quantize_per_block(view)
    assert same(t.values, q) and same(t.scales, s)


def test_quantize_errors(jf, golden):
    g = golden("quant")
    with pytest.raises(ValueError, match="finite"):
        jf.quantize_per_block(cu(g["err_nan_x"]))
    with pytest.raises(ValueError, match="overflow"):
        jf.quantize_per_block(cu(g["err_overflow_x"]))
    x = torch.ones((32, 32), device="cuda")
    x[5, 5] = float("inf")
    with pytest.raises(ValueError, match="finite"):
        jf.quantize_per_block(x)
    with pytest.raises(ValueError, match="multiple"):
        jf.quantize_per_block(torch.ones((30, 32), device="cuda"))
    with pytest.raises(ValueError, match="2-D"):
        jf.quantize_per_block(torch.ones(32, device="cuda"))
    # the error word is cleared after raising: a clean call succeeds
    jf.quantize_per_block(torch.ones((32, 32), device="cuda"))


def test_deferred_error_check(jf):
    jf.set_error_check("deferred")
    try:
        x = torch.full((32, 32), float("nan"), device="cuda")
        jf.quantize_per_block(x)  # does not raise yet
        with pytest.raises(ValueError, match="finite"):
            jf.check_errors()
        jf.check_errors()  # cleared
    finally:
        jf.set_error_check("eager")


def test_f16_snap_sweep(jf):
    # scale = snap(absmax/127) over a dense sweep of magnitudes incl. subnormal f16
    mags = np.geomspace(1e-40, 8.3e6, 20000).astype(np.float32)
    x = np.zeros((32, 32 * len(mags) // 1), np.float32)[:, :0]
    blocks = []
    for m in mags[:4096]:
        b = np.zeros((32, 32), np.float32)
        b[0, 0] = m
        b[1, 1] = -m / 3
        blocks.append(b)
    x = np.concatenate(blocks, axis=1)
    q, s = O.quantize(x)
    t = jf.quantize_per_block(cu(x))
    assert same(t.scales, s) and same(t.values, q)


def test_transpose(jf):
    rng = np.random.default_rng(5)
    q, s = O.quantize(rng.standard_normal((96, 160)).astype(np.float32))
    t = bqt(jf, q, s).transposed()
    assert same(t.values, q.T.copy()) and same(t.scales, s.T.copy())


def test_zeros_like_and_validate(jf):
    q, s = O.quantize(np.random.default_rng(1).standard_normal((64, 64)).astype(np.float32))
    t = bqt(jf, q, s)
    t.validate()
    z = jf.zeros_like(t)
    z.validate()
    assert int(z.values.abs().max()) == 0 and bool((z.scales == 1).all())


# ── K3-K5 GEMMs ─────────────────────────────────────────────────────────


def test_partials_bit_exact(jf, golden):
    g = golden("gemm")
    for i in range(int(g["nshapes"])):
        p = f"s{i}_"
        x, w = cu(g[p + "x_q"]), cu(g[p + "w_q"])
        got = jf.block_partials(x, w, 0)
        assert same(got, g[p + "part0"]), i
    rng = np.random.default_rng(9)
    a = rng.integers(-127, 128, (256, 512), dtype=np.int8)
    b = rng.integers(-127, 128, (384, 512), dtype=np.int8)
    a[:, 64:96] = 127
    b[:, 64:96] = -127  # extreme chunk: -32*127^2
    for k in (0, 2, 15):
        ref = (a[:, 32 * k:32 * k + 32].astype(np.int64) @ b[:, 32 * k:32 * k + 32].T.astype(np.int64))
        assert same(jf.block_partials(cu(a), cu(b), k), ref.astype(np.int32)), k


def test_gemm_golden_exact(jf, golden):
    if True:
        g = golden("gemm")
        for i in range(int(g["nshapes"])):
            p = f"s{i}_"
            x, w, dy = (bqt(jf, g[p + k + "_q"], g[p + k + "_s"]) for k in ("x", "w", "dy"))
            bias = cu(g[p + "bias"])
            assert same(jf.block_mm_forward(x, w, quantize=False), g[p + "fwd_acc"]), i
            y = jf.block_mm_forward(x, w, bias=bias)
            assert same(y.values, g[p + "fwd_q"]) and same(y.scales, g[p + "fwd_s"]), i
            y = jf.block_mm_forward(x, w)
            assert same(y.values, g[p + "fwdnb_q"]) and same(y.scales, g[p + "fwdnb_s"]), i
            assert same(jf.block_mm_grad_input(dy, w, quantize=False), g[p + "dgrad_acc"]), i
            y = jf.block_mm_grad_input(dy, w)
            assert same(y.values, g[p + "dgrad_q"]) and same(y.scales, g[p + "dgrad_s"]), i
            assert same(jf.block_mm_grad_weight(dy, x, quantize=False), g[p + "wgrad_acc"]), i
            y = jf.block_mm_grad_weight(dy, x)
            assert same(y.values, g[p + "wgrad_q"]) and same(y.scales, g[p + "wgrad_s"]), i


def _rand_q(rng, shape, scale=1.0):
    return O.quantize((rng.standard_normal(shape) * scale).astype(np.float32))


@pytest.mark.parametrize("n,c,d", [(128, 128, 128), (384, 640, 256), (1024, 1024, 4096), (160, 4096, 96)])
def test_gemm_random_exact_vs_oracle(jf, n, c, d):
    rng = np.random.default_rng(n + c + d)
    xq, xs = _rand_q(rng, (n, c))
    wq, ws = _rand_q(rng, (d, c), 1 / np.sqrt(c))
    dq, ds = _rand_q(rng, (n, d), 0.1)
    bias = (0.1 * rng.standard_normal(d)).astype(np.float32)
    X, W, DY = bqt(jf, xq, xs), bqt(jf, wq, ws), bqt(jf, dq, ds)
    rq, rs = O.mm_forward(xq, xs, wq, ws, bias)
    y = jf.block_mm_forward(X, W, bias=cu(bias))
    assert same(y.values, rq) and same(y.scales, rs)
    rq, rs = O.mm_grad_input(dq, ds, wq, ws)
    y = jf.block_mm_grad_input(DY, W)
    assert same(y.values, rq) and same(y.scales, rs)
    acc = O.mm_grad_weight(dq, ds, xq, xs, quantize_out=False)
    assert same(jf.block_mm_grad_weight(DY, X, quantize=False), acc)


@pytest.mark.parametrize("promotion", ["exact", "fast"])
@pytest.mark.parametrize("shape", [(256, 384, 512), (2048, 256, 2304)])
def test_gemm_paths_bit_identical(jf, promotion, shape):
    """Staged-scales kernel with MN-major operands (dgrad reads W, wgrad reads dY and X as
    stored) vs the generic kernel on transposed copies: same bits, every output kind.  The
    second shape has more tiles than SMs (persistent loop)."""
    from paper_2403_12422_b200 import runtime

    rng = np.random.default_rng(5)
    n, c, d = shape
    X = bqt(jf, *_rand_q(rng, (n, c)))
    W = bqt(jf, *_rand_q(rng, (d, c), 1 / np.sqrt(c)))
    DY = bqt(jf, *_rand_q(rng, (n, d), 0.1))
    bias = cu((0.1 * rng.standard_normal(d)).astype(np.float32))
    def run():
        return (jf.block_mm_forward(X, W, bias=bias, promotion=promotion),
                jf.block_mm_grad_input(DY, W, promotion=promotion, wt=W.transposed()),
                jf.block_mm_grad_weight(DY, X, promotion=promotion, out="int8+deq"),
                jf.block_mm_grad_weight(DY, X, promotion=promotion, quantize=False))
    prev = runtime.gemm_operands()
    try:
        runtime.set_gemm_operands("int8")
        staged = run()
        runtime.set_gemm_option("tma_scales", 0)
        generic = run()
    finally:
        runtime.set_gemm_option("tma_scales", 1)
        runtime.set_gemm_operands(prev)
    for other in (generic,):
        for a, b in ((staged[0], other[0]), (staged[1], other[1])):
            assert torch.equal(a.values, b.values) and torch.equal(a.scales, b.scales)
        assert torch.equal(staged[2][0].values, other[2][0].values)
        assert torch.equal(staged[2][1], other[2][1])
        assert torch.equal(staged[3], other[3])


def test_widen_codes(jf):
    from paper_2403_12422_b200.qgemm import widen_codes

    rng = np.random.default_rng(3)
    q = torch.from_numpy(rng.integers(-127, 128, size=(192, 320), dtype=np.int8)).cuda()
    assert torch.equal(widen_codes(q), q.to(torch.float16))
    assert torch.equal(widen_codes(q, transpose=True), q.t().contiguous().to(torch.float16))


@pytest.mark.parametrize("promotion", ["exact", "fast"])
@pytest.mark.parametrize("shape", [(256, 384, 512), (2048, 256, 2304)])
def test_gemm_f16_operands_bit_identical(jf, promotion, shape):
    """The f16-widened operand path (kind::f16 MMA, f32 partials) vs the int8 kernels: same
    bits for fwd (+bias), dgrad and wgrad, every output kind."""
    from paper_2403_12422_b200 import runtime

    rng = np.random.default_rng(11)
    n, c, d = shape
    X = bqt(jf, *_rand_q(rng, (n, c)))
    W = bqt(jf, *_rand_q(rng, (d, c), 1 / np.sqrt(c)))
    DY = bqt(jf, *_rand_q(rng, (n, d), 0.1))
    bias = cu((0.1 * rng.standard_normal(d)).astype(np.float32))

    def run():
        return (jf.block_mm_forward(X, W, bias=bias, promotion=promotion),
                jf.block_mm_forward(X, W, promotion=promotion, quantize=False),
                jf.block_mm_grad_input(DY, W, promotion=promotion),
                jf.block_mm_grad_weight(DY, X, promotion=promotion, out="int8+deq"),
                jf.block_mm_grad_weight(DY, X, promotion=promotion, quantize=False))
    prev = runtime.gemm_operands()
    try:
        runtime.set_gemm_operands("int8")
        ref = run()
        runtime.set_gemm_operands("f16")
        got = run()
    finally:
        runtime.set_gemm_operands(prev)
    for a, b in ((ref[0], got[0]), (ref[2], got[2])):
        assert torch.equal(a.values, b.values) and torch.equal(a.scales, b.scales)
    assert torch.equal(ref[1], got[1])
    assert torch.equal(ref[3][0].values, got[3][0].values) and torch.equal(ref[3][1], got[3][1])
    assert torch.equal(ref[4], got[4])


def test_quantlinear_f16_weight_cache(jf):
    """QuantLinear caches the widened W / W^T and drops them on mark_updated / set_weight_q."""
    from paper_2403_12422_b200 import runtime
    from paper_2403_12422_b200.qlayers import QuantLinear

    rng = np.random.default_rng(12)
    lin = QuantLinear.initialize(rng, 256, 384)
    x = jf.quantize_per_block(torch.from_numpy(rng.standard_normal((128, 384)).astype(np.float32)).cuda())
    prev = runtime.gemm_operands()
    try:
        runtime.set_gemm_operands("int8")
        ref = lin.forward(x)
        runtime.set_gemm_operands("f16")
        got = lin.forward(x)
        assert lin._weight_f16[0] is not None
        lin.master_weight.mul_(2.0)
        lin.mark_updated()
        assert lin._weight_f16 == [None, None]
        got2 = lin.forward(x)
        runtime.set_gemm_operands("int8")
        ref2 = lin.forward(x)
    finally:
        runtime.set_gemm_operands(prev)
    assert torch.equal(ref.values, got.values) and torch.equal(ref.scales, got.scales)
    assert torch.equal(ref2.values, got2.values) and torch.equal(ref2.scales, got2.scales)


def test_gemm_fast_mode_tolerance(jf):
    if True:
        rng = np.random.default_rng(77)
        n, c, d = 512, 2048, 768
        xq, xs = _rand_q(rng, (n, c))
        wq, ws = _rand_q(rng, (d, c), 1 / np.sqrt(c))
        X, W = bqt(jf, xq, xs), bqt(jf, wq, ws)
        acc = O.mm_forward(xq, xs, wq, ws, quantize_out=False)
        got = npy(jf.block_mm_forward(X, W, quantize=False, promotion="fast"))
        rel = np.abs(got - acc).max() / np.abs(acc).max()
        assert rel <= 1e-3, rel          # north-star tolerance
        assert rel <= 1e-6, rel          # what the fast promotion actually achieves
        rq, rs = O.quantize(acc)
        y = jf.block_mm_forward(X, W, promotion="fast")
        diff = np.abs(npy(y.values).astype(int) - rq.astype(int))
        assert diff.max() <= 1 and (diff > 0).mean() <= 1e-4


def test_gemm_shape_errors(jf):
    rng = np.random.default_rng(2)
    a = bqt(jf, *_rand_q(rng, (64, 64)))
    b = bqt(jf, *_rand_q(rng, (64, 96)))
    with pytest.raises(ValueError, match="inner dims"):
        jf.block_mm_forward(a, b)
    with pytest.raises(ValueError, match="does not match"):
        jf.block_mm_forward(a, a, cfg=jf.TileConfig.default_for(16))


def test_gemm_qcd_mode(jf):
    rng = np.random.default_rng(4)
    a = bqt(jf, *_rand_q(rng, (64, 96)))
    w = bqt(jf, *_rand_q(rng, (128, 96)))
    r = jf.block_mm_forward(a, w, mode=jf.ExecMode.QCD_EMULATION)
    assert isinstance(r, jf.DenseResult) and r.scale == 1.0
    assert torch.equal(r.values, jf.block_mm_forward(a, w, quantize=False))


# ── K6-K11 fused elementwise ────────────────────────────────────────────


def test_add_stats_golden(jf, golden):
    g = golden("nonlinear")
    a, b = bqt(jf, g["a_q"], g["a_s"]), bqt(jf, g["b_q"], g["b_s"])
    for w in (32, 64, 128, 256):
        y, st = jf.add_forward(a, b, stats_width=w)
        assert same(y.values, g[f"add{w}_q"]) and same(y.scales, g[f"add{w}_s"]), w
        assert same(st.mean, g[f"add{w}_mean"]) and same(st.sumsq, g[f"add{w}_sumsq"]), w
    for second in (None, jf.zeros_like(a)):
        y, st = jf.add_forward(a, second, 64)
        assert same(y.values, g["addz_q"]) and same(st.mean, g["addz_mean"]) and same(st.sumsq, g["addz_sumsq"])


@pytest.mark.parametrize("n,c,w", [(64, 1024, 64), (96, 1280, 64), (32, 96, 32), (128, 4096, 64), (64, 576, 192)])
def test_add_stats_random(jf, n, c, w):
    rng = np.random.default_rng(c)
    aq, as_ = _rand_q(rng, (n, c))
    bq, bs = _rand_q(rng, (n, c), 0.3)
    rq, rs, rm, rss = O.add_forward(aq, as_, bq, bs, w)
    y, st = jf.add_forward(bqt(jf, aq, as_), bqt(jf, bq, bs), w)
    assert same(y.values, rq) and same(y.scales, rs)
    assert same(st.mean, rm) and same(st.sumsq, rss)


def test_layernorm_golden(jf, golden):
    g = golden("nonlinear")
    x = bqt(jf, g["ln_x_q"], g["ln_x_s"])
    st = jf.RowStats(cu(g["ln_mean"]), cu(g["ln_sumsq"]), 64)
    params = jf.NormParams(g["ln_gamma"], g["ln_beta"])
    y, ctx = jf.layernorm_forward(x, st, params)
    assert same(y.values, g["ln_q"]) and same(y.scales, g["ln_s"])
    assert same(ctx.mu, g["ln_mu"]) and same(ctx.inv_std, g["ln_inv_std"])
    dy = bqt(jf, g["lnb_dy_q"], g["lnb_dy_s"])
    dx, dg, db = jf.layernorm_backward(ctx, dy, params)
    assert same(dx.values, g["lnb_q"]) and same(dx.scales, g["lnb_s"])
    np.testing.assert_allclose(npy(dg), g["lnb_dgamma"], rtol=1e-5, atol=1e-5)
    np.testing.assert_allclose(npy(db), g["lnb_dbeta"], rtol=1e-5, atol=1e-5)
    for cc, w in ((1280, 64), (96, 32)):
        p = f"ln{cc}_"
        y, st = jf.add_forward(bqt(jf, g[p + "x1_q"], g[p + "x1_s"]), bqt(jf, g[p + "x2_q"], g[p + "x2_s"]), w)
        assert same(y.values, g[p + "add_q"]) and same(st.mean, g[p + "mean"]) and same(st.sumsq, g[p + "sumsq"])
        prm = jf.NormParams(np.ones(cc, np.float32), np.zeros(cc, np.float32))
        l, ctx = jf.layernorm_forward(y, st, prm)
        assert same(l.values, g[p + "q"]) and same(l.scales, g[p + "s"])
        assert same(ctx.mu, g[p + "mu"]) and same(ctx.inv_std, g[p + "inv_std"])
        dx, dgm, dbt = jf.layernorm_backward(ctx, bqt(jf, g[p + "dy_q"], g[p + "dy_s"]), prm)
        assert same(dx.values, g[p + "dq"]) and same(dx.scales, g[p + "ds"]), cc
        np.testing.assert_allclose(npy(dgm), g[p + "dgamma"], rtol=1e-4, atol=1e-4)


@pytest.mark.parametrize("n,c", [(64, 1024), (128, 4096), (32, 1280), (64, 768), (32, 5120)])
def test_layernorm_random(jf, n, c):
    rng = np.random.default_rng(n * c)
    aq, as_ = _rand_q(rng, (n, c), 2.0)
    bq, bs = _rand_q(rng, (n, c))
    w = 64 if c % 64 == 0 else 32
    hq, hs, m, ss = O.add_forward(aq, as_, bq, bs, w)
    gamma = (1 + 0.1 * rng.standard_normal(c)).astype(np.float32)
    beta = (0.1 * rng.standard_normal(c)).astype(np.float32)
    rq, rs, mu, inv = O.layernorm_forward(hq, hs, m, ss, w, gamma, beta)
    H = bqt(jf, hq, hs)
    y, ctx = jf.layernorm_forward(H, jf.RowStats(cu(m), cu(ss), w), jf.NormParams(gamma, beta))
    assert same(y.values, rq) and same(y.scales, rs)
    assert same(ctx.mu, mu) and same(ctx.inv_std, inv)
    dq, ds = _rand_q(rng, (n, c), 0.1)
    rdq, rds, rdg, rdb = O.layernorm_backward(hq, hs, mu, inv, dq, ds, gamma)
    dx, dg, db = jf.layernorm_backward(ctx, bqt(jf, dq, ds), jf.NormParams(gamma, beta))
    assert same(dx.values, rdq) and same(dx.scales, rds)
    for got, ref in ((dg, rdg), (db, rdb)):   # strip-wise axis-0 sums: tolerance
        np.testing.assert_allclose(npy(got), ref, rtol=1e-3, atol=1e-4 * np.abs(ref).max())


def test_gelu_golden(jf, golden):
    g = golden("nonlinear")
    x = bqt(jf, g["gelu_x_q"], g["gelu_x_s"])
    y = jf.gelu_forward(x)
    assert same(y.values, g["gelu_q"]) and same(y.scales, g["gelu_s"])
    dx = jf.gelu_backward(x, bqt(jf, g["gelub_dy_q"], g["gelub_dy_s"]))
    diff = np.abs(npy(dx.values).astype(int) - g["gelub_q"].astype(int))
    assert diff.max() <= 1 and (diff > 0).mean() <= 1e-3
    np.testing.assert_allclose(npy(dx.scales), g["gelub_s"], rtol=2e-3)


@pytest.mark.parametrize("n,c", [(64, 4096), (256, 16384)])
def test_gelu_random(jf, n, c):
    rng = np.random.default_rng(c)
    xq, xs = _rand_q(rng, (n, c), 2.5)
    rq, rs = O.gelu_forward(xq, xs)
    y = jf.gelu_forward(bqt(jf, xq, xs))
    assert same(y.values, rq) and same(y.scales, rs)
    dq, ds = _rand_q(rng, (n, c), 0.1)
    f32 = O.dequantize(dq, ds) * O.gelu_grad_f32(O.dequantize(xq, xs))
    dx = jf.gelu_backward(bqt(jf, xq, xs), bqt(jf, dq, ds))
    got = npy(dx.dequantize())
    rel = np.abs(got - f32).max() / np.abs(f32).max()
    assert rel <= 1e-2  # one quantization step of the output (|err| <= s/2)
    rq, rs = O.quantize(f32)
    diff = np.abs(npy(dx.values).astype(int) - rq.astype(int))
    assert diff.max() <= 1 and (diff > 0).mean() <= 1e-3


def test_colsum(jf):
    rng = np.random.default_rng(8)
    q, s = _rand_q(rng, (2048, 1024), 0.1)
    ref = O.column_sum(q, s)
    got = npy(jf.column_sum(bqt(jf, q, s)))
    np.testing.assert_allclose(got, ref, rtol=1e-4, atol=1e-5 * np.abs(ref).max())


def test_dropout_mask_and_scales(jf):
    rng = np.random.default_rng(10)
    q, s = _rand_q(rng, (64, 64))
    t = bqt(jf, q, s)
    st = jf.DropoutState.generate(0.5, 10, (64, 64))
    mask = npy(st.mask)
    # drawn on the device, bit-identical to the reference's numpy Philox draw
    assert np.array_equal(mask, np.random.Generator(np.random.Philox(key=10)).random((64, 64)) >= 0.5)
    y = jf.dropout_forward(t, st)
    assert same(y.values, np.where(mask, q, np.int8(0)))
    assert same(y.scales, O.f16_snap(s * np.float32(2.0)))
    same0 = jf.dropout_forward(t, jf.DropoutState.generate(0.0, 1, (64, 64)))
    assert same0 is t


@pytest.mark.parametrize("p,seed,shape", [(0.1, (3, 1), (4096, 1024)), (0.37, 2**70 + 5, (96, 160)),
                                          (0.9, 0, (32, 32)), (0.5, (2**64 - 1, 7), (2048, 4096))])
def test_dropout_mask_device_philox_vs_numpy(jf, p, seed, shape):
    """jf_philox_keep == Generator(Philox(key=seed)).random(shape) >= p (qnonlinear.py:190-200)
    for int, 128-bit and pair seeds, including masks past 2^22 elements."""
    st = jf.DropoutState.generate(p, seed, shape)
    want = np.random.Generator(np.random.Philox(key=seed)).random(shape) >= p
    assert np.array_equal(npy(st.mask), want)


# ── layers ──────────────────────────────────────────────────────────────


def test_quantlinear_golden(jf, golden):
    g = golden("layers")
    lin = jf.QuantLinear(g["lin_w"], g["lin_b"])
    assert same(lin.weight_q.values, g["lin_wq"]) and same(lin.weight_q.scales, g["lin_ws"])
    x = bqt(jf, g["lin_x_q"], g["lin_x_s"])
    y = lin.forward(x)
    assert same(y.values, g["lin_y_q"]) and same(y.scales, g["lin_y_s"])
    dx, dw, db = lin.backward(bqt(jf, g["lin_dy_q"], g["lin_dy_s"]))
    assert same(dx.values, g["lin_dx_q"]) and same(dx.scales, g["lin_dx_s"])
    assert same(dw, g["lin_dw"])
    np.testing.assert_allclose(npy(db), g["lin_db"], rtol=1e-5, atol=1e-6)
    with pytest.raises(RuntimeError):
        jf.QuantLinear(g["lin_w"]).backward(bqt(jf, g["lin_dy_q"], g["lin_dy_s"]))


@pytest.mark.parametrize("attn_dtype", [torch.float32, torch.bfloat16])
def test_transformer_block_vs_reference(jf, golden, attn_dtype):
    g = golden("layers")
    c, heads, hidden, batch, seq = (int(v) for v in g["blk_cfg"])
    cfg = jf.BlockConfig(c_model=c, heads=heads, hidden=hidden, block=32, dropout_p=0.0)
    params = {k[6:]: g[k] for k in g.files if k.startswith("blk_p_")}
    blk = jf.TransformerBlock.from_parameters(cfg, params, attn_dtype=attn_dtype)
    x = bqt(jf, g["blk_x_q"], g["blk_x_s"])
    out = blk.forward(x, batch, seq)
    ref = O.dequantize(g["blk_out_q"], g["blk_out_s"])
    got = npy(out.dequantize())
    assert np.abs(got - ref).max() / np.abs(ref).max() <= (0.02 if attn_dtype == torch.float32 else 0.04)
    # the reference's own tolerance against the FP32 twin (test_qlayers.py:257-273)
    twin = g["blk_ref_out"]
    assert np.abs(got - twin).max() / np.abs(twin).max() <= 0.06
    dx, grads = blk.backward(bqt(jf, g["blk_dy_q"], g["blk_dy_s"]))
    rdx = O.dequantize(g["blk_dx_q"], g["blk_dx_s"])
    assert np.abs(npy(dx.dequantize()) - rdx).max() / np.abs(rdx).max() <= 0.08
    for k, gv in grads.items():
        r = g["blk_g_" + k]
        denom = max(float(np.abs(r).max()), 1e-8)
        assert np.abs(npy(gv) - r).max() / denom <= 0.12, k
    ratio = blk.saved_activation_bytes() / blk.fp16_baseline_bytes()
    assert ratio == (1 + 2 / 32 ** 2) / 2


def test_block_counters_closed_form(jf):
    rng = np.random.default_rng(0)
    cfg = jf.BlockConfig(c_model=64, heads=4, hidden=128, block=32)
    blk = jf.TransformerBlock.initialize(rng, cfg)
    batch, seq = 2, 16
    x = jf.quantize_per_block(cu(rng.standard_normal((batch * seq, 64)).astype(np.float32)))
    ctr = jf.AccessCounters()
    out = blk.forward(x, batch, seq, counters=ctr)
    dy = jf.quantize_per_block(cu(rng.standard_normal(out.shape).astype(np.float32)))
    blk.backward(dy, ctr)
    n, c, h = batch * seq, 64, 128
    assert ctr.int_mac == 3 * n * (3 * c * c + c * c + h * c + c * h)
    assert ctr.fp16_load_store == 0


def test_attention_boundary_kernels(jf):
    """jf_dequantize_qkv_heads / jf_quantize_heads_bf16 == dequantize + view / quantize_per_block."""
    from paper_2403_12422_b200 import qlayers

    rng = np.random.default_rng(11)
    b, s, h, d = 2, 64, 4, 32
    c = h * d
    QKV = bqt(jf, *_rand_q(rng, (b * s, 3 * c)))
    core = jf.AttentionCore(h, d, dtype=torch.bfloat16)
    out = core.forward_q(QKV, b, s)
    q, k, v, o = core._saved
    dense = jf.dequantize(QKV, torch.bfloat16)
    for i, t in enumerate((q, k, v)):
        want = dense[:, i * c:(i + 1) * c].reshape(b, s, h, d).transpose(1, 2)
        assert torch.equal(t.detach(), want)
    ref = jf.quantize_per_block(o.detach().transpose(1, 2).reshape(b * s, c).float())
    assert torch.equal(out.values, ref.values) and torch.equal(out.scales, ref.scales)
    # slice writes: three strided sources into one [N, 3C] tensor
    dq = jf.BlockQuantTensor(torch.zeros(b * s, 3 * c, dtype=torch.int8, device="cuda"),
                             torch.ones(b * s // 32, 3 * c // 32, device="cuda"))
    srcs = [torch.randn(b, h, s, d, device="cuda").to(torch.bfloat16) for _ in range(3)]
    for i, t in enumerate(srcs):
        qlayers._quantize_heads(t, dq, i * c)
    full = torch.cat([t.transpose(1, 2).reshape(b * s, c) for t in srcs], dim=1).float()
    ref = jf.quantize_per_block(full)
    assert torch.equal(dq.values, ref.values) and torch.equal(dq.scales, ref.scales)
    # backward path runs and matches the dense island within bf16 attention noise
    dattn = jf.quantize_per_block(0.1 * torch.randn(b * s, c, device="cuda"))
    dqkv = core.backward_q(dattn, b, s)
    core2 = jf.AttentionCore(h, d, dtype=torch.bfloat16)
    core2.forward(dense, b, s)
    g = core2.backward(jf.dequantize(dattn, torch.bfloat16), b, s).float()
    got = dqkv.dequantize()
    assert (got - g).abs().max() <= 0.05 * g.abs().max()


def test_jqt1_matches_reference_blob(jf):
    """JQT1 BlockQuantTensor bytes (qtensor.py:152-181) equal to the reference's for the same input."""
    import os

    gold = os.path.join(os.path.dirname(__file__), "golden")
    x = np.load(os.path.join(gold, "jqt1_ref_input.npy"))
    with open(os.path.join(gold, "jqt1_ref.bin"), "rb") as fh:
        ref = fh.read()
    xq = jf.quantize_per_block(cu(x))
    assert xq.to_bytes() == ref
    back = jf.BlockQuantTensor.from_bytes(ref)
    assert torch.equal(back.values, xq.values) and torch.equal(back.scales, xq.scales)


def test_nvtx_ranges_on_gpu(jf):
    """With NVTX ranges on, a QuantLinear fwd+bwd runs and gives identical bits."""
    rng = np.random.default_rng(12)
    x = cu(rng.standard_normal((64, 96)).astype(np.float32))
    w = (rng.standard_normal((128, 96)) / 10).astype(np.float32)
    outs = []
    for on in (False, True):
        jf.runtime.set_nvtx(on)
        try:
            lin = jf.QuantLinear(w, np.zeros(128, np.float32))
            y = lin.forward(jf.quantize_per_block(x))
            dx, dw, db = lin.backward(y)
            outs.append((y.values.clone(), dx.values.clone(), dw.clone()))
        finally:
            jf.runtime.set_nvtx(False)
    for a, b in zip(*outs):
        assert torch.equal(a, b)
