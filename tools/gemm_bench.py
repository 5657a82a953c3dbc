"""GEMM-only timing of the tcgen05 INT8 block GEMM at the BASELINE block shapes.

python tools/gemm_bench.py [--iters 20] [--shapes fwd,dgrad,wgrad] [--mode exact,fast]
Prints one JSON line per (shape, op, mode): TOPS and fraction of the 4.5 POPS INT8 peak.
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_12422_b200 as jf  # noqa: E402
from paper_2403_12422_b200.qgemm import transpose_codes  # noqa: E402

SHAPES = {  # (N tokens, C in, D out) of the config-4 block at 4096 tokens
    "qkv": (4096, 4096, 12288), "proj": (4096, 4096, 4096), "mlp1": (4096, 4096, 16384),
    "mlp2": (4096, 16384, 4096),
    # GPT-2 medium at 8192 tokens
    "g2qkv": (8192, 1024, 3072), "g2proj": (8192, 1024, 1024), "g2mlp1": (8192, 1024, 4096),
    "g2mlp2": (8192, 4096, 1024),
}


def rq(shape, scale=1.0):
    return jf.quantize_per_block(torch.randn(shape, device="cuda") * scale)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--ops", default="fwd,dgrad,wgrad")
    ap.add_argument("--modes", default="exact,fast")
    ap.add_argument("--shapes", default="mlp1,proj")
    ap.add_argument("--lib", default=None, help="alternative libjetfire build (A/B experiments)")
    ap.add_argument("--operands", default="int8", choices=["auto", "int8", "f16"])
    a = ap.parse_args()
    if a.lib:
        from paper_2403_12422_b200 import _lib
        _lib.load_library(a.lib)
    jf.require_cuda()
    jf.set_error_check("deferred")
    jf.runtime.set_gemm_operands(a.operands)
    for name in a.shapes.split(","):
        n, c, d = SHAPES[name]
        x, w, dy = rq((n, c)), rq((d, c), c ** -0.5), rq((n, d), 0.1)
        wt = w.transposed()
        for op in a.ops.split(","):
            for mode in a.modes.split(","):
                if op == "fwd":
                    fn = lambda: jf.block_mm_forward(x, w, promotion=mode)  # noqa: E731
                elif op == "dgrad":
                    fn = lambda: jf.block_mm_grad_input(dy, w, promotion=mode, wt=wt)  # noqa: E731
                else:
                    dyt, xt = transpose_codes(dy.values), transpose_codes(x.values)
                    fn = lambda: jf.block_mm_grad_weight(dy, x, promotion=mode)  # noqa: E731
                for _ in range(3):
                    fn()
                torch.cuda.synchronize()
                from paper_2403_12422_b200.qgemm import GemmTimer
                with GemmTimer() as gt:
                    for _ in range(a.iters):
                        fn()
                s = gt.summary()
                tops = s["ops"] / (s["ms"] / 1e3) / 1e12
                print(json.dumps({"shape": name, "op": op, "mode": mode, "M_N_K": [n, c, d],
                                  "us_per_launch": round(1e3 * s["ms"] / s["launches"], 1),
                                  "tops": round(tops, 1), "frac_int8_peak": round(tops / 4500, 4)}), flush=True)
    try:
        jf.check_errors()
    except ValueError as e:
        print(json.dumps({"error_flag": str(e)}))


if __name__ == "__main__":
    main()
