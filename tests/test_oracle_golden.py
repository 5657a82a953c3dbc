"""Pin the CPU oracle against the real reference (CPU only, no GPU).

Fixtures in tests/golden were produced by running the unmodified reference
(``tests/golden/make_golden.py``); the frozen literals below are the
reference's own golden vectors (pkg/tests/test_qtensor.py:105-140,505-509,
test_qgemm.py:102-106, test_qnonlinear.py:70-72).
"""

import numpy as np
import pytest

from oracle import int8flow_oracle as O


def eq(a, b):
    return np.asarray(a).tobytes() == np.asarray(b).tobytes() and np.asarray(a).shape == np.asarray(b).shape


# ── frozen literals from the reference tests, embedded in 32x32 blocks ──


def _embed(vals):
    x = np.zeros((32, 32), np.float32)
    v = np.asarray(vals, np.float32)
    x[: v.shape[0], : v.shape[1]] = v
    return x


def test_frozen_example():
    q, s = O.quantize(_embed([[0.5, -1.0], [0.75, 0.25]]))
    assert s[0, 0] == np.float32(0.00787353515625)
    assert q[:2, :2].tolist() == [[64, -127], [95, 32]]


def test_frozen_half_even():
    q, s = O.quantize(_embed([[15.875, 0.1875], [0.3125, -0.3125]]))
    assert s[0, 0] == np.float32(0.125)
    assert q[:2, :2].tolist() == [[127, 2], [2, -2]]


def test_tiny_block_scale():
    q, s = O.quantize(np.full((32, 32), 1.0e-40, np.float32))
    assert s[0, 0] == np.float32(2.0 ** -24)


def test_zero_block_scale_one():
    q, s = O.quantize(np.zeros((32, 64), np.float32))
    assert (s == 1.0).all() and (q == 0).all()


def test_errors():
    x = np.ones((32, 32), np.float32)
    x[3, 3] = np.nan
    with pytest.raises(ValueError, match="finite"):
        O.quantize(x)
    with pytest.raises(ValueError, match="overflow"):
        O.quantize(np.full((32, 32), 1.0e7, np.float32))
    with pytest.raises(ValueError, match="multiple"):
        O.quantize(np.zeros((30, 32), np.float32))
    with pytest.raises(ValueError, match="2-D"):
        O.quantize(np.zeros(32, np.float32))


def test_f16_snap():
    assert O.f16_snap(0.1) == np.float32(0.0999755859375)


def test_micro_closed_form():
    a = np.full((16, 32), 127, np.int8)
    b = np.full((32, 16), 127, np.int8)
    assert (O.int32_partials(a[:, :32], b, 0)[:, :] == 32 * 127 * 127).all()
    assert 16 * 127 ** 2 == 258064


def test_gelu_at_one():
    assert abs(float(O.gelu_f32(np.float32(1.0))) - 0.8413447) < 1e-6


def test_pairwise_model_matches_numpy():
    rng = np.random.default_rng(0)
    for n in (5, 8, 20, 64, 128, 129, 264, 1024, 1280, 4096):
        a = rng.standard_normal(n).astype(np.float32)
        assert eq(O.pairwise_sum(a), np.add.reduce(a)), n


# ── golden fixtures from the real reference ────────────────────────────


def test_quant_golden(golden):
    g = golden("quant")
    for name in g["names"]:
        q, s = O.quantize(g[f"{name}_x"])
        assert eq(q, g[f"{name}_q"]), name
        assert eq(s, g[f"{name}_s"]), name
        assert eq(O.dequantize(q, s), g[f"{name}_deq"]), name
    q, s = O.quantize(g["bf16_x"])
    assert eq(q, g["bf16_q"]) and eq(s, g["bf16_s"])
    with pytest.raises(ValueError, match="finite"):
        O.quantize(g["err_nan_x"])
    with pytest.raises(ValueError, match="overflow"):
        O.quantize(g["err_overflow_x"])


def test_gemm_golden(golden):
    g = golden("gemm")
    for i in range(int(g["nshapes"])):
        p = f"s{i}_"
        x, xs, w, ws = g[p + "x_q"], g[p + "x_s"], g[p + "w_q"], g[p + "w_s"]
        dy, dys = g[p + "dy_q"], g[p + "dy_s"]
        assert eq(O.mm_forward(x, xs, w, ws, quantize_out=False), g[p + "fwd_acc"])
        q, s = O.mm_forward(x, xs, w, ws, bias=g[p + "bias"])
        assert eq(q, g[p + "fwd_q"]) and eq(s, g[p + "fwd_s"])
        assert eq(O.mm_grad_input(dy, dys, w, ws, quantize_out=False), g[p + "dgrad_acc"])
        q, s = O.mm_grad_input(dy, dys, w, ws)
        assert eq(q, g[p + "dgrad_q"]) and eq(s, g[p + "dgrad_s"])
        assert eq(O.mm_grad_weight(dy, dys, x, xs, quantize_out=False), g[p + "wgrad_acc"])
        q, s = O.mm_grad_weight(dy, dys, x, xs)
        assert eq(q, g[p + "wgrad_q"]) and eq(s, g[p + "wgrad_s"])
        assert eq(O.int32_partials(x, w.T, 0).astype(np.int32), g[p + "part0"])


def test_nonlinear_golden(golden):
    g = golden("nonlinear")
    a, as_, b, bs = g["a_q"], g["a_s"], g["b_q"], g["b_s"]
    for w in (32, 64, 128, 256):
        q, s, m, ss = O.add_forward(a, as_, b, bs, w)
        assert eq(q, g[f"add{w}_q"]) and eq(s, g[f"add{w}_s"]), w
        assert eq(m, g[f"add{w}_mean"]) and eq(ss, g[f"add{w}_sumsq"]), w
    q, s, m, ss = O.add_forward(a, as_, np.zeros_like(a), np.ones_like(as_), 64)
    assert eq(q, g["addz_q"]) and eq(m, g["addz_mean"]) and eq(ss, g["addz_sumsq"])
    q, s, mu, inv = O.layernorm_forward(g["ln_x_q"], g["ln_x_s"], g["ln_mean"], g["ln_sumsq"], 64,
                                        g["ln_gamma"], g["ln_beta"])
    assert eq(q, g["ln_q"]) and eq(s, g["ln_s"]) and eq(mu, g["ln_mu"]) and eq(inv, g["ln_inv_std"])
    q, s, dg, db = O.layernorm_backward(g["ln_x_q"], g["ln_x_s"], mu, inv, g["lnb_dy_q"], g["lnb_dy_s"],
                                        g["ln_gamma"])
    assert eq(q, g["lnb_q"]) and eq(s, g["lnb_s"]) and eq(dg, g["lnb_dgamma"]) and eq(db, g["lnb_dbeta"])
    for cc, w in ((1280, 64), (96, 32)):
        p = f"ln{cc}_"
        q, s, m, ss = O.add_forward(g[p + "x1_q"], g[p + "x1_s"], g[p + "x2_q"], g[p + "x2_s"], w)
        assert eq(q, g[p + "add_q"]) and eq(m, g[p + "mean"]) and eq(ss, g[p + "sumsq"])
        one, zero = np.ones(cc, np.float32), np.zeros(cc, np.float32)
        q, s, mu, inv = O.layernorm_forward(q, s, m, ss, w, one, zero)
        assert eq(q, g[p + "q"]) and eq(s, g[p + "s"]) and eq(mu, g[p + "mu"]) and eq(inv, g[p + "inv_std"])
        q, s, dg, db = O.layernorm_backward(g[p + "add_q"], g[p + "add_s"], mu, inv, g[p + "dy_q"],
                                            g[p + "dy_s"], one)
        assert eq(q, g[p + "dq"]) and eq(s, g[p + "ds"]) and eq(dg, g[p + "dgamma"])
    q, s = O.gelu_forward(g["gelu_x_q"], g["gelu_x_s"])
    assert eq(q, g["gelu_q"]) and eq(s, g["gelu_s"])
    # GELU backward: numpy's SIMD float32 exp decides the last bits; bit-exact
    # on the fixture host, tolerance elsewhere.
    f32 = O.dequantize(g["gelub_dy_q"], g["gelub_dy_s"]) * O.gelu_grad_f32(O.dequantize(g["gelu_x_q"], g["gelu_x_s"]))
    np.testing.assert_allclose(f32, g["gelub_f32"], rtol=1e-6, atol=1e-9)
    q, s = O.gelu_backward(g["gelu_x_q"], g["gelu_x_s"], g["gelub_dy_q"], g["gelub_dy_s"])
    assert (np.abs(q.astype(int) - g["gelub_q"].astype(int)) <= 1).all()


def test_layer_golden(golden):
    g = golden("layers")
    q, s = O.linear_forward(g["lin_x_q"], g["lin_x_s"], g["lin_w"], g["lin_b"])
    assert eq(q, g["lin_y_q"]) and eq(s, g["lin_y_s"])
    dq, ds, dw, db = O.linear_backward(g["lin_x_q"], g["lin_x_s"], g["lin_w"], g["lin_dy_q"], g["lin_dy_s"])
    assert eq(dq, g["lin_dx_q"]) and eq(ds, g["lin_dx_s"]) and eq(dw, g["lin_dw"]) and eq(db, g["lin_db"])


def test_block_oracle_matches_reference_golden(golden):
    g = golden("layers")
    c, heads, hidden, batch, seq = (int(v) for v in g["blk_cfg"])
    p = {k[6:]: g[k] for k in g.files if k.startswith("blk_p_")}
    (oq, os_), saved = O.block_forward(p, g["blk_x_q"], g["blk_x_s"], batch, seq, heads)
    # attention is FP32 numpy in both: identical op order -> bit-identical codes
    assert eq(oq, g["blk_out_q"]) and eq(os_, g["blk_out_s"])
    (dq, ds), grads = O.block_backward(p, saved, g["blk_dy_q"], g["blk_dy_s"])
    assert eq(dq, g["blk_dx_q"]) and eq(ds, g["blk_dx_s"])
    for k, v in grads.items():
        np.testing.assert_allclose(v, g["blk_g_" + k], rtol=1e-5, atol=1e-6 * max(1.0, np.abs(v).max()))
