"""cProfile of the host side of a bench step (diagnostics).

python tools/prof_host.py [--workload gpt2_medium] [--steps 5]
"""
import argparse
import cProfile
import os
import pstats
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2403_12422_b200 as jf  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="gpt2_medium")
    ap.add_argument("--steps", type=int, default=5)
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
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(a.steps):
        wl.step()
    pr.disable()
    torch.cuda.synchronize()
    pstats.Stats(pr).sort_stats("tottime").print_stats(25)


if __name__ == "__main__":
    main()
