"""Interleaved A/B timing of GEMM launch options in ONE process (diagnostics).

python tools/gemm_ab.py --shape mlp1 --mode exact \
    --configs "tma_scales=1" "tma_scales=0" "operands=f16" --rounds 5
Each round times every config once (CUDA events, 10 launches after 2 warm-up);
prints the median us/launch per config.  Options: jf_gemm_set_option keys (ctl_kind /
ctl_ns only act in JF_CTL_RUNTIME builds), plus operands=int8|auto|f16.  --base is applied
before every config so keys do not leak from one config into the next.
"""
import argparse
import json
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_12422_b200 as jf  # noqa: E402

SHAPES = {"qkv": (4096, 4096, 12288), "proj": (4096, 4096, 4096), "mlp1": (4096, 4096, 16384),
          "mlp2": (4096, 16384, 4096)}


def apply(cfg: str):
    for kv in filter(None, cfg.split(",")):
        k, v = kv.split("=")
        if k == "operands":
            jf.runtime.set_gemm_operands(v)
        else:
            jf.runtime.set_gemm_option(k, int(v))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="mlp1")
    ap.add_argument("--mode", default="exact")
    ap.add_argument("--configs", nargs="+", required=True)
    ap.add_argument("--base", default="", help="options applied before every config (reset keys)")
    ap.add_argument("--rounds", type=int, default=5)
    ap.add_argument("--iters", type=int, default=10)
    a = ap.parse_args()
    jf.require_cuda()
    jf.set_error_check("deferred")
    n, c, d = SHAPES[a.shape]
    x = jf.quantize_per_block(torch.randn(n, c, device="cuda"))
    w = jf.quantize_per_block(torch.randn(d, c, device="cuda") * c ** -0.5)
    times = {cfg: [] for cfg in a.configs}
    for _ in range(a.rounds):
        for cfg in a.configs:
            apply(a.base)
            apply(cfg)
            for _ in range(2):
                jf.block_mm_forward(x, w, promotion=a.mode)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            for _ in range(a.iters):
                jf.block_mm_forward(x, w, promotion=a.mode)
            e1.record()
            torch.cuda.synchronize()
            times[cfg].append(1e3 * e0.elapsed_time(e1) / a.iters)
    for cfg, t in times.items():
        print(json.dumps({"shape": a.shape, "mode": a.mode, "config": cfg, "us_median": round(statistics.median(t), 1),
                          "us_all": [round(v, 1) for v in t]}), flush=True)


if __name__ == "__main__":
    main()
