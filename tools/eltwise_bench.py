"""Memory-bound kernel timing at the config-4 block shapes (4096 tokens).

Reports GB/s of ALGORITHMIC bytes (s = 4/1024 B of scale per
element) against the measured 6553 GB/s copy bandwidth.
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_12422_b200 as jf  # noqa: E402

HBM = 6553.0
S = 4.0 / 1024


def timed(fn, iters=20):
    """Device time per call: the calls are captured in a CUDA graph and replayed, so
    Python / launch overhead (tens of us per call) cannot hide the kernel time."""
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(iters):
            fn()
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters


def report(name, n, c, bpe, ms, extra=0):
    gb = (n * c * bpe + extra) / 1e9
    print(json.dumps({"kernel": name, "shape": [n, c], "us": round(ms * 1e3, 2), "GB/s": round(gb / (ms / 1e3), 1),
                      "frac_hbm": round(gb / (ms / 1e3) / HBM, 3)}), flush=True)


def main():
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="config4", choices=["config4", "gpt2"],
                    help="config4: 4096 tokens x 4096 (GELU 16384); gpt2: 8192 tokens x 1024 (GELU 4096)")
    a = ap.parse_args()
    jf.require_cuda()
    jf.set_error_check("deferred")
    n, c, h = (4096, 4096, 16384) if a.shape == "config4" else (8192, 1024, 4096)
    x32 = torch.randn(n, c, device="cuda")
    xb = x32.to(torch.bfloat16)
    a = jf.quantize_per_block(x32)
    b = jf.quantize_per_block(torch.randn(n, c, device="cuda"))
    g = jf.quantize_per_block(torch.randn(n, h, device="cuda"))
    dg = jf.quantize_per_block(torch.randn(n, h, device="cuda") * 0.1)
    report("quantize_f32", n, c, 5 + S, timed(lambda: jf.quantize_per_block(x32)))
    report("quantize_bf16", n, c, 3 + S, timed(lambda: jf.quantize_per_block(xb)))
    report("dequantize_f32", n, c, 5 + S, timed(lambda: jf.dequantize(a)))
    report("dequantize_bf16", n, c, 3 + S, timed(lambda: jf.dequantize(a, torch.bfloat16)))
    report("add_stats", n, c, 3 + 3 * S + 0.125, timed(lambda: jf.add_forward(a, b, 64)))
    report("add_stats_zero", n, c, 2 + 2 * S + 0.125, timed(lambda: jf.add_forward(a, None, 64)))
    y, st = jf.add_forward(a, b, 64)
    prm = jf.NormParams(torch.ones(c, device="cuda"), torch.zeros(c, device="cuda"))
    report("ln_fwd", n, c, 2 + 2 * S + 0.125, timed(lambda: jf.layernorm_forward(y, st, prm)), extra=8 * n)
    _, ctx = jf.layernorm_forward(y, st, prm)
    report("ln_bwd", n, c, 3 + 3 * S, timed(lambda: jf.layernorm_backward(ctx, b, prm)), extra=8 * n)
    report("gelu_fwd", n, h, 2 + 2 * S, timed(lambda: jf.gelu_forward(g)))
    report("gelu_bwd", n, h, 3 + 3 * S, timed(lambda: jf.gelu_backward(g, dg)))
    report("colsum", n, h, 1 + S, timed(lambda: jf.column_sum(dg)))
    report("transpose_codes", n, h, 2, timed(lambda: dg.transposed()))
    # attention-island boundary at the config-4 shape (batch 2, seq 2048, 32 heads x 128):
    # QKV codes -> three bf16 [b, h, s, d] tensors, and a bf16 [b, h, s, d] -> codes
    from paper_2403_12422_b200 import _lib
    from paper_2403_12422_b200.qlayers import _quantize_heads
    from paper_2403_12422_b200.qtensor import empty_like_shape
    bt, sq, hh, hd = (2, 2048, 32, 128) if a.shape == "config4" else (8, 1024, 16, 64)
    qkv = jf.quantize_per_block(torch.randn(bt * sq, 3 * hh * hd, device="cuda"))
    heads = [torch.empty((bt, hh, sq, hd), dtype=torch.bfloat16, device="cuda") for _ in range(3)]
    L = _lib.lib()
    deq = lambda: L.jf_dequantize_qkv_heads(qkv.values.data_ptr(), qkv.scales.data_ptr(), bt, sq, hh, hd,  # noqa: E731
                                            heads[0].data_ptr(), heads[1].data_ptr(), heads[2].data_ptr(),
                                            _lib.stream_handle())
    report("dequant_qkv_heads", bt * sq, 3 * hh * hd, 3 + S, timed(deq))
    out = empty_like_shape(bt * sq, hh * hd, "cuda")
    report("quantize_heads", bt * sq, hh * hd, 3 + S, timed(lambda: _quantize_heads(heads[0], out, 0)))
    jf.check_errors()


if __name__ == "__main__":
    main()
