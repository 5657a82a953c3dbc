"""CTA-0 event timeline of gemm_tc_kernel (diagnostics; needs `make trace`).

python tools/gemm_trace.py [--shape mlp1] [--mode fast] [--operands int8|f16]
Loads libjetfire_trace.so in place of libjetfire.so, runs one GEMM and prints, per
chunk, clock64 deltas of the pipeline events: MMA issuer (tempty wait, issue) and
promotion warp 2 (tfull wait, TMEM load, promotion) plus warp 17's promotion end,
and the steady-state averages.
"""
import argparse
import ctypes
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2403_12422_b200 import _lib  # noqa: E402

SHAPES = {"proj": (4096, 4096, 4096), "mlp1": (4096, 4096, 16384), "g2mlp1": (8192, 1024, 4096)}
NAMES = ["iss_wait", "iss_free", "iss_done", "w2_wait", "w2_full", "w2_data", "w2_done", "w17_done"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="mlp1")
    ap.add_argument("--mode", default="fast")
    ap.add_argument("--operands", default="int8")
    ap.add_argument("--dump", action="store_true", help="per-chunk periods and per-stage-position breakdown")
    a = ap.parse_args()
    _lib.load_library(os.path.join(ROOT, "paper_2403_12422_b200", "libjetfire_trace.so"))
    import paper_2403_12422_b200 as jf

    jf.runtime.set_gemm_operands(a.operands)
    n, c, d = SHAPES[a.shape]
    x = jf.quantize_per_block(torch.randn(n, c, device="cuda"))
    w = jf.quantize_per_block(torch.randn(d, c, device="cuda") * c ** -0.5)
    for _ in range(2):
        jf.block_mm_forward(x, w, promotion=a.mode)
    torch.cuda.synchronize()
    buf = np.zeros(32 * 256, dtype=np.int64)
    rc = _lib.lib().jf_gemm_trace_read(ctypes.c_void_p(buf.ctypes.data))
    assert rc == 0, rc
    t = buf.reshape(32, 256).astype(np.float64)
    rng = slice(32, 240)
    done = t[8:24, rng]                       # promotion end per warp (16) per chunk
    ok = (done > 0).all(axis=0)
    done = done[:, ok]
    period = float(np.diff(done.mean(axis=0)).mean())
    # lag of each promotion warp behind the earliest one, per chunk (clk), averaged
    lag = (done - done.min(axis=0)).mean(axis=1)
    iss = t[0:3, rng]
    oki = (iss > 0).all(axis=0)
    sp = [(w + 2) % 4 for w in range(16)]  # promotion warp w is CTA warp w + 2
    by_sp = {f"sp{q}": round(float(np.mean([lag[w] for w in range(16) if sp[w] == q])), 1) for q in range(4)}
    out = {"shape": a.shape, "mode": a.mode, "operands": a.operands, "period_clk": round(period, 1),
           "lag_by_subpartition": by_sp, "lag_by_warp": [round(float(v), 1) for v in lag],
           "iss_wait_tempty": round(float((iss[1] - iss[0])[oki].mean()), 1),
           "iss_issue_to_commit": round(float((iss[2] - iss[1])[oki].mean()), 1),
           "iss_fence": round(float((t[6, rng] - t[1, rng])[(t[6, rng] > 0) & (t[1, rng] > 0)].mean()), 1),
           "iss_mma": round(float((t[7, rng] - t[6, rng])[(t[7, rng] > 0) & (t[6, rng] > 0)].mean()), 1),
           "iss_commit": round(float((t[2, rng] - t[7, rng])[(t[2, rng] > 0) & (t[7, rng] > 0)].mean()), 1),
           "iss_between_chunks": round(float((t[0, rng.start + 1:rng.stop + 1] - t[2, rng])[(t[2, rng] > 0)].mean()), 1),
           "w2_wait_tfull": round(float((t[4, rng] - t[3, rng])[(t[4, rng] > 0) & (t[3, rng] > 0)].mean()), 1),
           "w2_ld": round(float((t[5, rng] - t[4, rng])[(t[5, rng] > 0) & (t[4, rng] > 0)].mean()), 1)}
    if a.dump:
        # per chunk: mean promotion end over the 16 warps, delta to the previous chunk
        d = t[8:24, :]
        okc = (d > 0).all(axis=0)
        m = d.mean(axis=0)
        out["chunk_period_clk"] = [round(float(m[i] - m[i - 1]), 0) if okc[i] and okc[i - 1] else None
                                   for i in range(1, 256)]
        # warp 2 per position in the 4-chunk stage (medians over chunks 8..239):
        # [previous promotion end -> tfull wait start, tfull wait, TMEM load, promotion]
        w2d = t[8, :]
        pos = {}
        for i in range(8, 240):
            if min(t[3, i], t[4, i], t[5, i], w2d[i], w2d[i - 1]) <= 0:
                continue
            pos.setdefault(i % 4, []).append((t[3, i] - w2d[i - 1], t[4, i] - t[3, i], t[5, i] - t[4, i],
                                              w2d[i] - t[5, i]))
        out["w2_by_stage_pos"] = {k: [round(float(x), 0) for x in np.median(np.array(v), axis=0)]
                                  for k, v in sorted(pos.items())}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
