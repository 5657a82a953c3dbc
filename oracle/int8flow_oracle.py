"""CPU oracle for the Jetfire INT8 data-flow hot path (TEST INFRASTRUCTURE ONLY).

This module is the *checker*, never the product.  Only ``tests/``,
``__graft_entry__.smoke()`` and the ``cpu_baseline`` / ``--impl reference``
legs of ``bench.py`` may import it.  The CUDA library must never route
through it (the product raises if ``libjetfire.so`` is missing).

It is a numpy restatement of the reference package ``int8flow``
(``/root/reference/pkg/src/int8flow``), written independently but
following the reference arithmetic operation-for-operation so that its
outputs are bit-identical to the reference on the same host.  Each function
cites the reference lines it restates.

Parity pinning: ``tests/golden/make_golden.py`` runs the real reference
(imported from ``/root/reference`` in the build container) on seeded inputs
and freezes inputs + outputs into ``tests/golden/*.npz``;
``tests/test_oracle_golden.py`` checks this oracle bit-for-bit against those
fixtures and against the reference's own frozen golden vectors
(``pkg/tests/test_qtensor.py:105-140,505-509``, ``test_qgemm.py:102-106``).
The single unpinnable bit source is numpy's SIMD float32 ``exp`` inside the
GELU backward: fixtures for it are compared under a
tolerance when the host's numpy dispatch differs.

Numerics notes (verified in this container, numpy 2.3.5 / scipy 1.18.1):
* contiguous float32 ``add.reduce`` = numpy's 8-accumulator pairwise sum
  (``pairwise_sum`` below reproduces it bit-exactly; used only as the
  documented model the CUDA kernels mirror);
* ``mean`` = float64 division of that float32 sum by an intp count, cast
  back to float32 (innocuous double rounding: equal to float32 division);
* axis-0 sums are sequential in row order;
* ``scipy.special.erf`` on float32 equals ``float(erf_double(double(x)))``.
"""

from __future__ import annotations

import numpy as np
from scipy.special import erf as _erf

BLOCK = 32
QMAX = 127
F16_TINY = np.float32(2.0 ** -24)        # qtensor.py:195
INV_SQRT2 = np.float32(0.7071067811865476)  # qnonlinear.py:27
INV_SQRT_2PI = np.float32(0.3989422804014327)  # qnonlinear.py:28


class OracleError(ValueError):
    """Raised with the reference's own ValueError texts."""


# ── numeric format (qtensor.py) ─────────────────────────────────────────


def f16_snap(v):
    """Round to the binary16 grid, keep float32 (qtensor.py:26-28)."""
    return np.asarray(v, dtype=np.float16).astype(np.float32)


def block_scales(absmax: np.ndarray) -> np.ndarray:
    """Scale rule of qtensor.py:198-211, restated per element.

    s = f16_RNE(fl32(absmax / 127)); absmax == 0 -> 1.0; a positive absmax
    whose scale snaps to 0 -> 2**-24; an infinite snapped scale raises.
    """
    am = absmax.astype(np.float32)
    with np.errstate(over="ignore"):
        raw = am / np.float32(QMAX)
        raw = np.where(am == 0, np.float32(1.0), raw)
        s = f16_snap(raw)
    if not np.isfinite(s).all():
        raise OracleError("scale overflows the binary16 range; input magnitude too large")
    return np.where((am > 0) & (s == 0), F16_TINY, s).astype(np.float32)


def quantize(x: np.ndarray, block: int = BLOCK):
    """Per-block absmax quantizer (qtensor.py:219-246) -> (int8 codes, f32 scales)."""
    x = np.asarray(x)
    if x.ndim != 2:
        raise OracleError(f"expected a 2-D matrix, got shape {x.shape}")
    x = np.ascontiguousarray(x, dtype=np.float32)
    n, c = x.shape
    if n % block or c % block:
        raise OracleError(f"shape {n}x{c} is not a multiple of block size {block}")
    tiles = x.reshape(n // block, block, c // block, block)
    absmax = np.abs(tiles).max(axis=(1, 3))
    if not np.isfinite(absmax).all():
        raise OracleError("input contains non-finite values")
    s = block_scales(absmax)
    q = tiles / s[:, None, :, None]            # true IEEE float32 division
    q = np.clip(np.rint(q), -QMAX, QMAX)        # round half to even
    return q.reshape(n, c).astype(np.int8), s


def dequantize(q: np.ndarray, s: np.ndarray, block: int = BLOCK) -> np.ndarray:
    """codes * block scale in float32 (qtensor.py:249-255); always exact."""
    n, c = q.shape
    out = q.astype(np.float32).reshape(n // block, block, c // block, block)
    out = out * s[:, None, :, None]
    return out.reshape(n, c).astype(np.float32)


# ── block GEMM core (qgemm.py) ──────────────────────────────────────────


def int32_partials(a: np.ndarray, b: np.ndarray, kblk: int, block: int = BLOCK) -> np.ndarray:
    """Exact integer product of one K chunk (qgemm.py:225, micro_mm_16 :168-180)."""
    k0 = kblk * block
    return a[:, k0:k0 + block].astype(np.int64) @ b[k0:k0 + block, :].astype(np.int64)


def gemm_accumulate(a, sa, b, sb, block: int = BLOCK) -> np.ndarray:
    """FP32 accumulator of (a*sa) @ (b*sb), reference order (qgemm.py:193-229).

    a: [M, K] int8 with scale grid sa [M/B, K/B]; b: [K, N] int8 with grid
    sb [K/B, N/B].  For K chunks ascending: P exact, t = fl(P*sa_row),
    t = fl(t*sb_col), acc = fl(acc + t).  No FMA contraction anywhere.
    """
    m, k = a.shape
    n = b.shape[1]
    af = a.astype(np.float32)
    bf = b.astype(np.float32)
    acc = np.zeros((m, n), dtype=np.float32)
    for ci in range(k // block):
        k0 = ci * block
        prod = af[:, k0:k0 + block] @ bf[k0:k0 + block, :]   # exact integers < 2**24
        prod = prod * np.repeat(sa[:, ci], block)[:, None]
        prod = prod * np.repeat(sb[ci, :], block)[None, :]
        acc = acc + prod
    return acc


def finish(acc: np.ndarray, bias=None, quantize_out: bool = True, block: int = BLOCK):
    """Bias add then requantization (qgemm.py:266-279)."""
    if bias is not None:
        acc = acc + np.asarray(bias, dtype=np.float32)[None, :]
    if not quantize_out:
        return acc
    return quantize(acc, block)


def mm_forward(xq, xs, wq, ws, bias=None, quantize_out=True):
    """Y = X W^T (qgemm.py:282-309)."""
    acc = gemm_accumulate(xq, xs, wq.T, ws.T)
    return finish(acc, bias, quantize_out)


def mm_grad_input(dyq, dys, wq, ws, quantize_out=True):
    """dX = dY W (qgemm.py:312-333)."""
    return finish(gemm_accumulate(dyq, dys, wq, ws), None, quantize_out)


def mm_grad_weight(dyq, dys, xq, xs, quantize_out=True):
    """dW = dY^T X (qgemm.py:336-357)."""
    return finish(gemm_accumulate(dyq.T, dys.T, xq, xs), None, quantize_out)


# ── fused non-linear operators (qnonlinear.py) ──────────────────────────


def pairwise_sum(a: np.ndarray) -> np.float32:
    """numpy's float32 contiguous add.reduce order (documentation model).

    n < 8: sequential from 0; n <= 128: 8 strided accumulators, tree
    ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), then the tail sequentially;
    n > 128: split at n2 = n//2 - (n//2)%8 and add the two halves.
    The CUDA kernels implement exactly this tree.
    """
    a = np.asarray(a, dtype=np.float32)
    n = a.shape[0]
    f = np.float32
    if n < 8:
        r = f(0.0)
        for i in range(n):
            r = f(r + a[i])
        return r
    if n <= 128:
        acc = [f(a[j]) for j in range(8)]
        i = 8
        while i < n - n % 8:
            for j in range(8):
                acc[j] = f(acc[j] + a[i + j])
            i += 8
        r = f(f(f(acc[0] + acc[1]) + f(acc[2] + acc[3])) + f(f(acc[4] + acc[5]) + f(acc[6] + acc[7])))
        for t in range(i, n):
            r = f(r + a[t])
        return r
    n2 = n // 2
    n2 -= n2 % 8
    return f(pairwise_sum(a[:n2]) + pairwise_sum(a[n2:]))


def norm_cdf(x):
    """0.5 * (1 + erf(x/sqrt2)) in float32 with a double erf (qnonlinear.py:34-36)."""
    return np.float32(0.5) * (np.float32(1.0) + _erf(x * INV_SQRT2))


def gelu_f32(x):
    return x * norm_cdf(x)                     # qnonlinear.py:39-40


def gelu_grad_f32(x):
    pdf = INV_SQRT_2PI * np.exp(np.float32(-0.5) * x * x)   # qnonlinear.py:43-46
    return x * pdf + norm_cdf(x)


def gelu_forward(xq, xs):
    """qnonlinear.py:150-158."""
    return quantize(gelu_f32(dequantize(xq, xs)))


def gelu_backward(xq, xs, dyq, dys):
    """qnonlinear.py:161-175."""
    dx = dequantize(dyq, dys) * gelu_grad_f32(dequantize(xq, xs))
    return quantize(dx)


def row_stats(y: np.ndarray, width: int):
    """Blockwise mean and sum of squares (qnonlinear.py:134-144)."""
    n, c = y.shape
    if c % width:
        raise OracleError(f"stats width {width} does not divide {c} columns")
    t = y.reshape(n, c // width, width)
    return t.mean(axis=2).astype(np.float32), (t * t).sum(axis=2).astype(np.float32)


def add_forward(aq, as_, bq, bs, width: int = 64):
    """y = deq(a)+deq(b) requantized, plus stats of the FP32 y (qnonlinear.py:246-267)."""
    y = dequantize(aq, as_) + dequantize(bq, bs)
    q, s = quantize(y)
    mean, sumsq = row_stats(y, width)
    return q, s, mean, sumsq


def stats_row_mean(mean):
    return mean.mean(axis=1)                    # qnonlinear.py:124-126


def stats_row_var(mean, sumsq, width):
    cols = mean.shape[1] * width                # qnonlinear.py:128-131
    mu = stats_row_mean(mean)
    var = sumsq.sum(axis=1) / np.float32(cols) - mu * mu
    return np.maximum(var, 0.0)


def layernorm_forward(xq, xs, mean, sumsq, width, gamma, beta, eps=1e-5):
    """LayerNorm from Add statistics (qnonlinear.py:300-330) -> (q, s, mu, inv_std)."""
    gamma = np.asarray(gamma, np.float32)
    beta = np.asarray(beta, np.float32)
    mu = stats_row_mean(mean)
    inv_std = (1.0 / np.sqrt(stats_row_var(mean, sumsq, width) + np.float32(eps))).astype(np.float32)
    x = dequantize(xq, xs)
    xhat = (x - mu[:, None]) * inv_std[:, None]
    y = gamma * xhat + beta
    q, s = quantize(y)
    return q, s, mu, inv_std


def layernorm_backward(xq, xs, mu, inv_std, dyq, dys, gamma):
    """Three-term LayerNorm gradient (qnonlinear.py:333-355) -> (q, s, dgamma, dbeta)."""
    gamma = np.asarray(gamma, np.float32)
    dy = dequantize(dyq, dys)
    xhat = (dequantize(xq, xs) - mu[:, None]) * inv_std[:, None]
    dxhat = dy * gamma
    m1 = dxhat.mean(axis=1, keepdims=True)
    m2 = (dxhat * xhat).mean(axis=1, keepdims=True)
    dx = inv_std[:, None] * (dxhat - m1 - xhat * m2)
    dgamma = (dy * xhat).sum(axis=0)
    dbeta = dy.sum(axis=0)
    q, s = quantize(dx.astype(np.float32))
    return q, s, dgamma, dbeta


def column_sum(q, s):
    """dbias = sum over rows of deq(dY), sequential (qlayers.py:180)."""
    return dequantize(q, s).sum(axis=0)


# ── layer orchestration (qlayers.py) ────────────────────────────────────


def _weight_codes(w):
    """QuantLinear.weight_q (qlayers.py:139-143): a cached (codes, scales) pair or a master to quantize."""
    return w if isinstance(w, tuple) else quantize(w)


def linear_forward(xq, xs, w_master, bias):
    """QuantLinear.forward (qlayers.py:149-163): INT8 weight, GEMM fwd + bias + requant."""
    wq, ws = _weight_codes(w_master)
    return mm_forward(xq, xs, wq, ws, bias)


def linear_backward(xq, xs, w_master, dyq, dys, has_bias=True):
    """QuantLinear.backward (qlayers.py:165-181) -> (dxq, dxs, dW fp32, dbias)."""
    wq, ws = _weight_codes(w_master)
    dxq, dxs = mm_grad_input(dyq, dys, wq, ws)
    dwq, dws = mm_grad_weight(dyq, dys, xq, xs)
    dbias = column_sum(dyq, dys) if has_bias else None
    return dxq, dxs, dequantize(dwq, dws), dbias


def attention_f32(qkv, batch, seq, heads):
    """Causal multi-head attention in float32 (qlayers.py:204-220)."""
    c = qkv.shape[1] // 3
    hd = c // heads

    def split(t):
        return t.reshape(batch, seq, heads, hd).transpose(0, 2, 1, 3)

    q, k, v = split(qkv[:, :c]), split(qkv[:, c:2 * c]), split(qkv[:, 2 * c:])
    sc = (q @ k.transpose(0, 1, 3, 2)) * np.float32(1.0 / np.sqrt(hd))
    mask = np.triu(np.ones((seq, seq), dtype=bool), k=1)
    sc = np.where(mask, np.float32(-np.inf), sc)
    sc = sc - sc.max(axis=-1, keepdims=True)
    e = np.exp(sc, dtype=np.float32)
    p = e / e.sum(axis=-1, keepdims=True)
    o = p @ v
    return o.transpose(0, 2, 1, 3).reshape(batch * seq, c).astype(np.float32), (q, k, v, p)


def attention_f32_backward(dout, saved, batch, seq, heads):
    """qlayers.py:222-236."""
    q, k, v, p = saved
    c = dout.shape[1]
    hd = c // heads

    def split(t):
        return t.reshape(batch, seq, heads, hd).transpose(0, 2, 1, 3)

    def merge(t):
        return t.transpose(0, 2, 1, 3).reshape(batch * seq, c)

    d = split(dout)
    dv = p.transpose(0, 1, 3, 2) @ d
    dp = d @ v.transpose(0, 1, 3, 2)
    ds = p * (dp - (dp * p).sum(axis=-1, keepdims=True))
    ds = ds * np.float32(1.0 / np.sqrt(hd))
    dq = ds @ k
    dk = ds.transpose(0, 1, 3, 2) @ q
    return np.concatenate([merge(dq), merge(dk), merge(dv)], axis=1).astype(np.float32)


# ── TransformerBlock orchestration (qlayers.py:329-427), dropout p = 0 ───


def block_init(rng, c, hidden):
    """Parameters drawn exactly like TransformerBlock.initialize (qlayers.py:287-303)."""
    def lin(d, cc):
        return (rng.standard_normal((d, cc)) / np.sqrt(cc)).astype(np.float32), np.zeros(d, np.float32)

    p = {}
    p["qkv.w"], p["qkv.b"] = lin(3 * c, c)
    p["proj.w"], p["proj.b"] = lin(c, c)
    p["mlp1.w"], p["mlp1.b"] = lin(hidden, c)
    p["mlp2.w"], p["mlp2.b"] = lin(c, hidden)
    for k in ("ln1", "ln2"):
        p[k + ".gamma"], p[k + ".beta"] = np.ones(c, np.float32), np.zeros(c, np.float32)
    return p


def block_weight_cache(p):
    """Quantize the four master weights once (the reference caches weight_q per layer)."""
    q = dict(p)
    for k in ("qkv.w", "proj.w", "mlp1.w", "mlp2.w"):
        q[k] = quantize(p[k])
    return q


def block_forward(p, xq, xs, batch, seq, heads, eps=1e-5):
    """INT8 data-flow forward; returns ((out_q, out_s), saved) (qlayers.py:329-383).

    ``p`` holds FP32 masters or, via block_weight_cache, cached (codes, scales) weights.
    """
    c = xq.shape[1]
    width = 64 if c % 64 == 0 else BLOCK
    a1q, a1s, m1_, ss1 = add_forward(xq, xs, np.zeros_like(xq), np.ones_like(xs), width)
    l1q, l1s, mu1, inv1 = layernorm_forward(a1q, a1s, m1_, ss1, width, p["ln1.gamma"], p["ln1.beta"], eps)
    qkvq, qkvs = linear_forward(l1q, l1s, p["qkv.w"], p["qkv.b"])
    att, asave = attention_f32(dequantize(qkvq, qkvs), batch, seq, heads)
    atq, ats = quantize(att)
    prq, prs = linear_forward(atq, ats, p["proj.w"], p["proj.b"])
    hq, hs, m2_, ss2 = add_forward(a1q, a1s, prq, prs, width)
    l2q, l2s, mu2, inv2 = layernorm_forward(hq, hs, m2_, ss2, width, p["ln2.gamma"], p["ln2.beta"], eps)
    g1q, g1s = linear_forward(l2q, l2s, p["mlp1.w"], p["mlp1.b"])
    gq, gs = gelu_forward(g1q, g1s)
    g2q, g2s = linear_forward(gq, gs, p["mlp2.w"], p["mlp2.b"])
    oq, os_, _, _ = add_forward(hq, hs, g2q, g2s, width)
    saved = dict(a1=(a1q, a1s, mu1, inv1), l1=(l1q, l1s), asave=asave, at=(atq, ats), h=(hq, hs, mu2, inv2),
                 l2=(l2q, l2s), g1=(g1q, g1s), g=(gq, gs), width=width, batch=batch, seq=seq, heads=heads)
    return (oq, os_), saved


def block_backward(p, saved, dyq, dys):
    """INT8 data-flow backward (qlayers.py:385-427) -> ((dx_q, dx_s), grads)."""
    w = saved["width"]
    gq, gs = saved["g"]
    dgq, dgs, dw_m2, db_m2 = linear_backward(gq, gs, p["mlp2.w"], dyq, dys)
    g1q, g1s = saved["g1"]
    dm1q, dm1s = gelu_backward(g1q, g1s, dgq, dgs)
    l2q, l2s = saved["l2"]
    dl2q, dl2s, dw_m1, db_m1 = linear_backward(l2q, l2s, p["mlp1.w"], dm1q, dm1s)
    hq, hs, mu2, inv2 = saved["h"]
    dhbq, dhbs, dg2, db2 = layernorm_backward(hq, hs, mu2, inv2, dl2q, dl2s, p["ln2.gamma"])
    dhq, dhs, _, _ = add_forward(dhbq, dhbs, dyq, dys, w)
    atq, ats = saved["at"]
    daq, das, dw_pr, db_pr = linear_backward(atq, ats, p["proj.w"], dhq, dhs)
    dqkv = attention_f32_backward(dequantize(daq, das), saved["asave"], saved["batch"], saved["seq"],
                                  saved["heads"])
    dqq, dqs = quantize(dqkv)
    l1q, l1s = saved["l1"]
    dl1q, dl1s, dw_qkv, db_qkv = linear_backward(l1q, l1s, p["qkv.w"], dqq, dqs)
    a1q, a1s, mu1, inv1 = saved["a1"]
    dabq, dabs, dg1, db1 = layernorm_backward(a1q, a1s, mu1, inv1, dl1q, dl1s, p["ln1.gamma"])
    dxq, dxs, _, _ = add_forward(dabq, dabs, dhq, dhs, w)
    grads = {"qkv.w": dw_qkv, "qkv.b": db_qkv, "proj.w": dw_pr, "proj.b": db_pr, "mlp1.w": dw_m1,
             "mlp1.b": db_m1, "mlp2.w": dw_m2, "mlp2.b": db_m2, "ln1.gamma": dg1, "ln1.beta": db1,
             "ln2.gamma": dg2, "ln2.beta": db2}
    return (dxq, dxs), grads


# ── DropoutState.generate's random stream (qnonlinear.py:190-200) ──────
# numpy's Generator(Philox(key=seed)).random(n), restated (the algorithm the CUDA
# kernel jf_philox_keep runs): Philox4x64-10 (Random123), counter incremented before
# each block of four 64-bit outputs (the first block uses counter 1), doubles =
# (u64 >> 11) * 2^-53.  Pure-Python integers: for small n only.
_M64 = (1 << 64) - 1


def philox4x64_10(ctr, key):
    c0, c1, c2, c3 = ctr
    k0, k1 = key
    for r in range(10):
        if r:
            k0 = (k0 + 0x9E3779B97F4A7C15) & _M64
            k1 = (k1 + 0xBB67AE8584CAA73B) & _M64
        p0 = 0xD2E7470EE14C6C93 * c0
        p1 = 0xCA5A826395121157 * c2
        c0, c1, c2, c3 = ((p1 >> 64) ^ c1 ^ k0, p1 & _M64, (p0 >> 64) ^ c3 ^ k1, p0 & _M64)
    return c0, c1, c2, c3


def philox_random(key, n):
    out = np.empty(n, dtype=np.float64)
    for g in range((n + 3) // 4):
        words = philox4x64_10((g + 1, 0, 0, 0), key)
        for e in range(4):
            if 4 * g + e < n:
                out[4 * g + e] = (words[e] >> 11) * (1.0 / 9007199254740992.0)
    return out
