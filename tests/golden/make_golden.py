"""Generate golden fixtures by running the REAL reference (int8flow) here.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py

It imports ``int8flow`` from ``/root/reference/pkg/src`` unmodified, feeds it
seeded inputs and freezes inputs + outputs into ``tests/golden/*.npz``.
Those fixtures travel with the repo; the GPU box never reads
/root/reference.  Regenerating is deterministic (same seeds, same numpy).
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def _load_reference():
    if not os.path.isdir(REF_SRC):
        raise SystemExit(f"reference not found at {REF_SRC}")
    sys.path.insert(0, REF_SRC)
    import int8flow  # noqa: F401
    from int8flow import qgemm, qlayers, qnonlinear, qtensor
    return qtensor, qgemm, qnonlinear, qlayers


def _gauss(rng, shape, scale=1.0):
    return (rng.standard_normal(shape) * scale).astype(np.float32)


def quant_cases(qt):
    rng = np.random.default_rng(1234)
    out = {}
    cases = {
        "g32": _gauss(rng, (32, 32)),
        "g64x96": _gauss(rng, (64, 96), 3.0),
        "g128x256": _gauss(rng, (128, 256), 17.3),
        "wide": _gauss(rng, (64, 1024)) * np.float32(1e-3),
    }
    x = _gauss(rng, (96, 320))
    chans = rng.choice(320, size=4, replace=False)
    x[:, chans] *= np.float32(30.0)
    cases["outlier"] = x
    x = _gauss(rng, (64, 64))
    x[:32, :32] = 0.0
    x[32:, 32:] = np.float32(1.0e-40)          # scale snaps to 0 -> 2**-24
    x[0:32, 32:64] *= np.float32(4.0e6)         # absmax/127 just under 65504 often
    x[0:32, 32:64] = np.clip(x[0:32, 32:64], -8.3e6, 8.3e6)
    cases["edge"] = x
    # reference golden vectors (test_qtensor.py:105-119) embedded in a 32x32 block
    g = np.zeros((32, 64), np.float32)
    g[:2, :2] = [[0.5, -1.0], [0.75, 0.25]]
    g[:2, 32:34] = [[15.875, 0.1875], [0.3125, -0.3125]]
    cases["frozen"] = g
    # exact ties: v * 2**-7 grid with every block attaining 127 plus halves
    v = rng.integers(-127, 128, size=(64, 64)).astype(np.float32)
    v[::32, ::32] = 127
    t = v * np.float32(2.0 ** -7)
    t[5, 5] = np.float32(2.5 * 2.0 ** -7)      # x/s = 2.5 -> 2
    t[6, 6] = np.float32(-3.5 * 2.0 ** -7)     # -3.5 -> -4
    cases["ties"] = t
    for name, x in cases.items():
        q = qt.quantize_per_block(x, 32)
        out[f"{name}_x"] = x
        out[f"{name}_q"] = q.values
        out[f"{name}_s"] = q.scales
        out[f"{name}_deq"] = q.dequantize()
    # bf16-exact input (for the bf16 quantizer entry point)
    xb = _gauss(rng, (64, 128), 2.0)
    xb = (xb.view(np.uint32) & np.uint32(0xFFFF0000)).view(np.float32)
    q = qt.quantize_per_block(xb, 32)
    out["bf16_x"], out["bf16_q"], out["bf16_s"] = xb, q.values, q.scales
    # error cases: inputs only, the expected exception text is fixed
    err = _gauss(rng, (32, 32))
    err[3, 3] = np.nan
    out["err_nan_x"] = err
    out["err_overflow_x"] = np.full((32, 32), 1.0e7, np.float32)
    out["names"] = np.array(sorted(cases))
    return out


def gemm_cases(qt, qg):
    rng = np.random.default_rng(99)
    out = {}
    shapes = [(64, 64, 64), (128, 96, 160), (96, 256, 64), (256, 128, 384), (32, 32, 32)]
    for i, (n, c, d) in enumerate(shapes):
        xq = qt.quantize_per_block(_gauss(rng, (n, c)), 32)
        wq = qt.quantize_per_block(_gauss(rng, (d, c), 1.0 / np.sqrt(c)), 32)
        dyq = qt.quantize_per_block(_gauss(rng, (n, d), 0.1), 32)
        bias = _gauss(rng, (d,), 0.5)
        p = f"s{i}_"
        out[p + "shape"] = np.array([n, c, d])
        for nm, t in (("x", xq), ("w", wq), ("dy", dyq)):
            out[p + nm + "_q"], out[p + nm + "_s"] = t.values, t.scales
        out[p + "bias"] = bias
        out[p + "fwd_acc"] = qg.block_mm_forward(xq, wq, quantize=False)
        y = qg.block_mm_forward(xq, wq, bias=bias)
        out[p + "fwd_q"], out[p + "fwd_s"] = y.values, y.scales
        y = qg.block_mm_forward(xq, wq)
        out[p + "fwdnb_q"], out[p + "fwdnb_s"] = y.values, y.scales
        out[p + "dgrad_acc"] = qg.block_mm_grad_input(dyq, wq, quantize=False)
        y = qg.block_mm_grad_input(dyq, wq)
        out[p + "dgrad_q"], out[p + "dgrad_s"] = y.values, y.scales
        out[p + "wgrad_acc"] = qg.block_mm_grad_weight(dyq, xq, quantize=False)
        y = qg.block_mm_grad_weight(dyq, xq)
        out[p + "wgrad_q"], out[p + "wgrad_s"] = y.values, y.scales
        # int32 partial of K chunk 0 (exact integer product, qgemm.py:225)
        out[p + "part0"] = (xq.values[:, :32].astype(np.int64)
                            @ wq.values.T[:32, :].astype(np.int64)).astype(np.int32)
    out["nshapes"] = np.array(len(shapes))
    return out


def nonlinear_cases(qt, qn):
    rng = np.random.default_rng(7)
    out = {}
    n, c = 64, 256
    a = qt.quantize_per_block(_gauss(rng, (n, c)), 32)
    b = qt.quantize_per_block(_gauss(rng, (n, c), 0.5), 32)
    out["a_q"], out["a_s"], out["b_q"], out["b_s"] = a.values, a.scales, b.values, b.scales
    for w in (32, 64, 128, 256):
        y, st = qn.add_forward(a, b, stats_width=w)
        out[f"add{w}_q"], out[f"add{w}_s"] = y.values, y.scales
        out[f"add{w}_mean"], out[f"add{w}_sumsq"] = st.mean, st.sumsq
    z = qt.zeros_like(a)
    y, st = qn.add_forward(a, z, 64)
    out["addz_q"], out["addz_s"], out["addz_mean"], out["addz_sumsq"] = y.values, y.scales, st.mean, st.sumsq
    # layernorm: stats from the Add, gamma/beta non-trivial
    y, st = qn.add_forward(a, b, 64)
    gamma = (1.0 + 0.1 * rng.standard_normal(c)).astype(np.float32)
    beta = (0.1 * rng.standard_normal(c)).astype(np.float32)
    params = qn.NormParams(gamma, beta)
    ln, ctx = qn.layernorm_forward(y, st, params)
    out["ln_x_q"], out["ln_x_s"] = y.values, y.scales
    out["ln_mean"], out["ln_sumsq"] = st.mean, st.sumsq
    out["ln_gamma"], out["ln_beta"] = gamma, beta
    out["ln_q"], out["ln_s"], out["ln_mu"], out["ln_inv_std"] = ln.values, ln.scales, ctx.mu, ctx.inv_std
    dy = qt.quantize_per_block(_gauss(rng, (n, c), 0.1), 32)
    dx, dg, db = qn.layernorm_backward(ctx, dy, params)
    out["lnb_dy_q"], out["lnb_dy_s"] = dy.values, dy.scales
    out["lnb_q"], out["lnb_s"], out["lnb_dgamma"], out["lnb_dbeta"] = dx.values, dx.scales, dg, db
    # layernorm over C=1280 (20 stat blocks: non power-of-two means) and C=96 (width 32)
    for cc, w in ((1280, 64), (96, 32)):
        x1 = qt.quantize_per_block(_gauss(rng, (32, cc)), 32)
        x2 = qt.quantize_per_block(_gauss(rng, (32, cc)), 32)
        yy, ss = qn.add_forward(x1, x2, w)
        g = np.ones(cc, np.float32)
        bb = np.zeros(cc, np.float32)
        pp = qn.NormParams(g, bb)
        l2, c2 = qn.layernorm_forward(yy, ss, pp)
        dd = qt.quantize_per_block(_gauss(rng, (32, cc), 0.1), 32)
        dx2, dg2, db2 = qn.layernorm_backward(c2, dd, pp)
        p = f"ln{cc}_"
        out[p + "x1_q"], out[p + "x1_s"], out[p + "x2_q"], out[p + "x2_s"] = x1.values, x1.scales, x2.values, x2.scales
        out[p + "add_q"], out[p + "add_s"], out[p + "mean"], out[p + "sumsq"] = yy.values, yy.scales, ss.mean, ss.sumsq
        out[p + "q"], out[p + "s"], out[p + "mu"], out[p + "inv_std"] = l2.values, l2.scales, c2.mu, c2.inv_std
        out[p + "dy_q"], out[p + "dy_s"] = dd.values, dd.scales
        out[p + "dq"], out[p + "ds"], out[p + "dgamma"], out[p + "dbeta"] = dx2.values, dx2.scales, dg2, db2
    # GELU
    g_in = qt.quantize_per_block(_gauss(rng, (64, 512), 2.0), 32)
    gy = qn.gelu_forward(g_in)
    out["gelu_x_q"], out["gelu_x_s"] = g_in.values, g_in.scales
    out["gelu_q"], out["gelu_s"] = gy.values, gy.scales
    gdy = qt.quantize_per_block(_gauss(rng, (64, 512), 0.1), 32)
    gdx = qn.gelu_backward(g_in, gdy)
    out["gelub_dy_q"], out["gelub_dy_s"] = gdy.values, gdy.scales
    out["gelub_q"], out["gelub_s"] = gdx.values, gdx.scales
    out["gelub_f32"] = gdy.dequantize() * qn.gelu_grad_f32(g_in.dequantize())
    return out


def layer_cases(qt, ql, qn):
    rng = np.random.default_rng(2024)
    out = {}
    # QuantLinear fwd/bwd
    n, c, d = 128, 96, 160
    lin = ql.QuantLinear.initialize(rng, d, c)
    lin.bias[:] = _gauss(rng, (d,), 0.2)
    xq = qt.quantize_per_block(_gauss(rng, (n, c)), 32)
    y = lin.forward(xq)
    dyq = qt.quantize_per_block(_gauss(rng, (n, d), 0.1), 32)
    dx, dw, db = lin.backward(dyq)
    out.update(lin_w=lin.master_weight, lin_b=lin.bias, lin_x_q=xq.values, lin_x_s=xq.scales,
               lin_y_q=y.values, lin_y_s=y.scales, lin_dy_q=dyq.values, lin_dy_s=dyq.scales,
               lin_dx_q=dx.values, lin_dx_s=dx.scales, lin_dw=dw, lin_db=db,
               lin_wq=lin.weight_q.values, lin_ws=lin.weight_q.scales)
    # TransformerBlock fwd/bwd (dropout p = 0 like every BASELINE config)
    cfg = ql.BlockConfig(c_model=128, heads=4, hidden=512, block=32, dropout_p=0.0)
    blk = ql.TransformerBlock.initialize(rng, cfg)
    for lin_ in (blk.qkv, blk.proj, blk.mlp1, blk.mlp2):
        lin_.bias[:] = _gauss(rng, lin_.bias.shape, 0.05)
    batch, seq = 2, 64
    x = _gauss(rng, (batch * seq, cfg.c_model))
    xq = qt.quantize_per_block(x, 32)
    outq = blk.forward(xq, batch, seq, dropout_seed=0)
    dyq = qt.quantize_per_block(_gauss(rng, outq.shape, 0.1), 32)
    dxq, grads = blk.backward(dyq)
    for k, v in blk.parameters().items():
        out["blk_p_" + k] = v
    for k, v in grads.items():
        out["blk_g_" + k] = v
    out.update(blk_cfg=np.array([cfg.c_model, cfg.heads, cfg.hidden, batch, seq]),
               blk_x_q=xq.values, blk_x_s=xq.scales, blk_out_q=outq.values, blk_out_s=outq.scales,
               blk_dy_q=dyq.values, blk_dy_s=dyq.scales, blk_dx_q=dxq.values, blk_dx_s=dxq.scales)
    # FP32 twin output for the tolerance-style test (test_qlayers.py:257-273)
    ref = ql.ReferenceBlock.from_block(blk)
    out["blk_ref_out"] = ref.forward(xq.dequantize(), batch, seq, dropout_seed=0)
    return out


def model_cases():
    """ToyModel.loss_and_grads (trainer.py:373-427) of the REAL reference: loss + every grad."""
    from int8flow import trainer

    cfg = trainer.TrainConfig(layers=2, c_model=64, heads=4, mlp_ratio=4, seed=3, batch_size=2,
                              weight_decay=0.1, lr=1e-3)
    vocab, seq = 96, 32
    model = trainer.ToyModel(cfg, vocab)
    rng = np.random.default_rng(77)
    x = rng.integers(0, vocab, size=(cfg.batch_size, seq))
    y = rng.integers(0, vocab, size=(cfg.batch_size, seq))
    mask = np.ones((cfg.batch_size, seq), dtype=np.float32)
    mask[1, -5:] = 0.0
    loss, grads = model.loss_and_grads(x, y, mask, dropout_seed=0)
    out = {"cfg": np.array([cfg.layers, cfg.c_model, cfg.heads, cfg.hidden, vocab, seq, cfg.batch_size]),
           "x": x, "y": y, "mask": mask, "loss": np.float64(loss)}
    for k, v in model.params.items():
        out["p_" + k] = v.copy()  # AdamW.step below updates the arrays in place
    for k, v in grads.items():
        out["g_" + k] = v
    # one AdamW step (trainer.py:247-262) on those grads
    opt = trainer.AdamW(model.params, lr=cfg.lr, weight_decay=cfg.weight_decay, decay_keys=model.decay_keys)
    opt.step(grads)
    for k, v in model.params.items():
        out["p1_" + k] = v.copy()
    out["decay_keys"] = np.array(sorted(model.decay_keys))
    return out


def format_cases(qt, ql):
    """int8flow-checkpoint-v1 files and a JQT1 blob written by the REAL reference."""
    rng = np.random.default_rng(9)
    params = {"b.w": rng.standard_normal((3, 5)).astype(np.float32), "a": rng.standard_normal(4).astype(np.float32),
              "scalar": np.array(1.5, dtype=np.float32)}
    ql.save_params(os.path.join(HERE, "ckpt_ref"), params, {"step": 7, "opt_t": 7, "scheme": "per-block"})
    x = (rng.standard_normal((32, 64)) * 3).astype(np.float32)
    with open(os.path.join(HERE, "jqt1_ref.bin"), "wb") as fh:
        fh.write(qt.quantize_per_block(x, 32).to_bytes())
    np.save(os.path.join(HERE, "jqt1_ref_input.npy"), x)


def main():
    qt, qg, qn, ql = _load_reference()
    np.savez_compressed(os.path.join(HERE, "quant.npz"), **quant_cases(qt))
    np.savez_compressed(os.path.join(HERE, "gemm.npz"), **gemm_cases(qt, qg))
    np.savez_compressed(os.path.join(HERE, "nonlinear.npz"), **nonlinear_cases(qt, qn))
    np.savez_compressed(os.path.join(HERE, "layers.npz"), **layer_cases(qt, ql, qn))
    np.savez_compressed(os.path.join(HERE, "model.npz"), **model_cases())
    format_cases(qt, ql)
    meta = {"numpy": np.__version__}
    import scipy
    meta["scipy"] = scipy.__version__
    with open(os.path.join(HERE, "GENERATED_WITH.txt"), "w") as fh:
        for k, v in meta.items():
            fh.write(f"{k}={v}\n")
        fh.write("reference=/root/reference/pkg/src/int8flow (unmodified)\n")
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
