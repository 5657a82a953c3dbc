"""Per-chunk event timeline of one GEMM launch (CTA 0, clock64 cycles).

Needs the trace build: nvcc ... -DJF_GEMM_TRACE -o paper_2403_12422_b200/libjetfire_trace.so
(see tools/build_trace.sh).  Slots: 0 MMA-thread tempty wait done, 1 promotion
warp saw tfull, 2 first promotion warp released the buffer, 3 last promotion
warp released it, 4 MMA-thread wait start, 5 MMA issued, 6 committed,
7 stage-full seen (indexed by first chunk of the stage).
"""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2403_12422_b200 import _lib  # noqa: E402

_lib.load_library(os.path.join(ROOT, "paper_2403_12422_b200", "libjetfire_trace.so"))
import paper_2403_12422_b200 as jf  # noqa: E402

jf.require_cuda()
jf.set_error_check("deferred")
L = _lib.load_library()
L.jf_gemm_debug_timestamps.argtypes = [ctypes.c_void_p]
n, c, d = 4096, 4096, 16384
x = jf.quantize_per_block(torch.randn(n, c, device="cuda"))
w = jf.quantize_per_block(torch.randn(d, c, device="cuda") * c ** -0.5)
for mode in sys.argv[1:] or ["exact"]:
    for _ in range(2):
        jf.block_mm_forward(x, w, promotion=mode)
    torch.cuda.synchronize()
    buf = (ctypes.c_longlong * 2048)()
    L.jf_gemm_debug_timestamps(ctypes.addressof(buf))
    ts = np.array(buf[:], dtype=np.int64).reshape(8, 256)
    t0 = ts[0, 0]
    print(f"mode={mode}  (cycles relative to chunk 0's MMA)")
    print(" chunk  waitbeg  waitdone  mma_iss  commit  tfull_seen  rel_first  rel_last")
    for g in list(range(0, 12)) + list(range(120, 132)):
        print(f"{g:5d} {ts[4,g]-t0:8d} {ts[0,g]-t0:8d} {ts[5,g]-t0:8d} {ts[6,g]-t0:8d} {ts[1,g]-t0:9d} "
              f"{ts[2,g]-t0:9d} {ts[3,g]-t0:9d}")
    s = slice(8, 120)
    med = lambda a: float(np.median(a))  # noqa: E731
    print("period (MMA issue to issue):", med(np.diff(ts[5, 8:121])))
    print("MMA issue -> tfull seen:", med(ts[1, s] - ts[5, s]), "| tfull -> first release:", med(ts[2, s] - ts[1, s]),
          "| first -> last release:", med(ts[3, s] - ts[2, s]))
    print("MMA thread: wait(tempty) duration:", med(ts[0, s] - ts[4, s]), "| wait done -> mma issued:",
          med(ts[5, s] - ts[0, s]), "| mma -> commit:", med(ts[6, s] - ts[5, s]),
          "| commit -> next wait start:", med(ts[4, 9:121] - ts[6, s]))
    print("last release (g) -> MMA (g+4) issued:", med(ts[5, 12:124] - ts[3, s]))
