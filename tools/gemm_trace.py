"""CTA-0 event timeline of the f16-path GEMM (JF_GEMM_IMPL=h16; diagnostics; needs `make trace`).

python tools/gemm_trace.py [--shape proj] [--mode fast]
Loads libjetfire_trace.so in place of libjetfire.so, runs one GEMM, and
prints per-stage clock deltas: converter (stage start -> int8 ready ->
f16 slot free -> converted), MMA issuer (hfull wait, tempty wait) and the
epilogue's tfull arrival.
"""
import argparse
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2403_12422_b200 import _lib  # noqa: E402

SHAPES = {"proj": (4096, 4096, 4096), "mlp1": (4096, 4096, 16384)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="proj")
    ap.add_argument("--mode", default="fast")
    ap.add_argument("--impl", default="h16", choices=["h16"])
    a = ap.parse_args()
    os.environ["JF_GEMM_IMPL"] = a.impl
    _lib.load_library(os.path.join(ROOT, "paper_2403_12422_b200", "libjetfire_trace.so"))
    import paper_2403_12422_b200 as jf

    n, c, d = SHAPES[a.shape]
    x = jf.quantize_per_block(torch.randn(n, c, device="cuda"))
    w = jf.quantize_per_block(torch.randn(d, c, device="cuda") * c ** -0.5)
    for _ in range(2):
        jf.block_mm_forward(x, w, promotion=a.mode)
    torch.cuda.synchronize()
    buf = np.zeros(8 * 512, dtype=np.int64)
    rc = _lib.lib().jf_gemm_trace_read(ctypes.c_void_p(buf.ctypes.data))
    assert rc == 0, rc
    t = buf.reshape(8, 512).astype(np.float64)
    t0 = t[t > 0].min()
    names = ["conv_start", "int8_ready", "f16_free", "converted", "iss_start", "hfull_ok", "tempty_ok", "epi_tfull"]
    print("stage " + " ".join(f"{n:>10}" for n in names))
    for g in list(range(0, 12)) + list(range(100, 112)):
        print(f"{g:5d} " + " ".join(f"{(t[e, g] - t0) if t[e, g] else float('nan'):10.0f}" for e in range(8)))
    # steady-state averages over stages 50..400
    rng = slice(50, 400)

    def avg(e1, e0):
        v = t[e1, rng] - t[e0, rng]
        v = v[(t[e1, rng] > 0) & (t[e0, rng] > 0)]
        return float(v.mean()) if v.size else float("nan")

    per = np.diff(t[7, rng][t[7, rng] > 0])
    print(f"period per stage (epilogue tfull-to-tfull): {per.mean():.0f} clk")
    print(f"converter: wait int8 {avg(1, 0):.0f}, wait f16 slot {avg(2, 1):.0f}, convert {avg(3, 2):.0f}")
    print(f"issuer: wait hfull {avg(5, 4):.0f}, wait tempty {avg(6, 5):.0f}")

if __name__ == "__main__":
    main()
