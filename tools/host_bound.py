"""Host vs device time of the bench step (diagnostics): is the step launch-bound?

python tools/host_bound.py --workload gpt2_medium [--steps 10]
Prints host enqueue time per step (time until the Python loop returns, no sync) and the
device time per step (CUDA events).  Host >= device means the GPU waits for launches.
"""
import argparse
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2403_12422_b200 as jf  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="gpt2_medium")
    ap.add_argument("--steps", type=int, default=10)
    a = ap.parse_args()
    args = bench.parse(["--workload", a.workload, "--no-cpu", "--no-bf16"])
    jf.require_cuda()
    jf.set_error_check("deferred")
    jf.runtime.set_gemm_operands(args.operands)
    w = dict(bench.WORKLOADS[a.workload])
    wl = (bench.ModelWorkload if "model" in w else bench.BlockWorkload)(jf, w, args, 1, 0)
    for _ in range(4):
        wl.step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(a.steps):
        wl.step()
    e1.record()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    dev = e0.elapsed_time(e1) / a.steps
    print(f"{a.workload}: host enqueue {1e3 * (t1 - t0) / a.steps:.2f} ms/step, device {dev:.2f} ms/step, "
          f"wall {1e3 * (t2 - t0) / a.steps:.2f} ms/step")


if __name__ == "__main__":
    main()
