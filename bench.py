#!/usr/bin/env python
"""bench.py — Jetfire INT8 data-flow transformer block, fwd+bwd tokens/s on B200.

Metric (BASELINE.json): transformer-block fwd+bwd tokens/s; per-block INT8
GEMM TOPS vs INT8 peak.  Default workload: BASELINE config "transformer block
hidden 4096, seq 2048" (the north star's target setting), random-init
weights, synthetic standard-normal activations/gradients, dropout p = 0.

One step = forward + backward of one TransformerBlock in the INT8 data flow
(12 tcgen05 GEMMs + fused INT8 elementwise kernels + SDPA attention island).
``value``: inputs already quantized in HBM.  ``e2e``: host pinned FP32 x and
dY copied in, quantized, fwd+bwd, dX (codes+scales) copied back, per step.

The line also carries ``roofline`` (the block GEMM vs the INT8 peak, our measured
kind::i8 ceiling and the exact-promotion bound), ``variants`` (fast promotion,
f16-widened operands, the fused INT8-boundary attention: same block, same run),
``eltwise`` (per-kernel GB/s and HBM fraction of the memory-bound kernels),
``bf16_baseline`` (the same block in torch BF16), ``cpu_baseline`` and ``clocks``.

Multi-GPU (torchrun): data parallel over the token batch, per-rank batch
fixed (weak scaling); the one exchange step is an NCCL all-reduce of the
FP32 parameter gradients.  ``--impl reference`` times the reference's own
implementation (the unmodified package in baseline/_ref, or the oracle port
when absent) on the box's host cores, on a bounded token sample of the block.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "transformer-block fwd+bwd tokens/s; per-block INT8 GEMM TOPS vs INT8 peak"
INT8_PEAK_TOPS = 4500.0  # B200 dense INT8 datasheet (no measured INT8 figure in MEASURED_PEAKS.json)
KIND_I8_MEASURED_TOPS = 8178.0 * 2 * 148 * 1965e6 / 1e12  # our raw tcgen05 kind::i8 microbenchmark ceiling

WORKLOADS = {
    # BASELINE.json configs[0]: one QuantLinear fwd+bwd, the reference's own CPU-runnable case
    "linear_n4096": dict(linear=True, n=4096, c=1024, d=4096),
    # BASELINE.json configs[3]: the paper's speed-up setting, north-star target
    "block_h4096_s2048": dict(c=4096, heads=32, hidden=16384, seq=2048, batch=2),
    # BASELINE.json configs[1]
    "block_h1024_s1024": dict(c=1024, heads=16, hidden=4096, seq=1024, batch=8),
    # BASELINE.json configs[2]: GPT-2 medium full pretraining step (24 layers, hidden 1024)
    "gpt2_medium": dict(model="gpt2_medium", c=1024, heads=16, hidden=4096, seq=1024, batch=8),
    # BASELINE.json configs[4] model (data-parallel at 2/4/8 GPUs): GPT-2 large
    "gpt2_large": dict(model="gpt2_large", c=1280, heads=20, hidden=5120, seq=1024, batch=8),
}


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="block_h4096_s2048", choices=sorted(WORKLOADS))
    ap.add_argument("--batch", type=int, default=None, help="sequences per GPU")
    ap.add_argument("--promotion", default="exact", choices=["exact", "fast"])
    ap.add_argument("--operands", default="int8", choices=["int8", "auto", "f16"],
                    help="GEMM operand path (runtime.set_gemm_operands): int8 = tcgen05 kind::i8 (default); "
                         "auto/f16 = opt-in f16-widened codes on kind::f16; all bit-identical")
    ap.add_argument("--overlap-wgrad", type=int, default=1, choices=[0, 1],
                    help="weight-gradient GEMMs on a side stream (runtime.set_overlap_wgrad)")
    ap.add_argument("--graph", type=int, default=1, choices=[0, 1],
                    help="model workloads, 1 GPU: replay forward+backward from a CUDA graph")
    ap.add_argument("--attn-dtype", default="bf16", choices=["bf16", "fp32"])
    ap.add_argument("--attention", default="sdpa", choices=["sdpa", "fused"],
                    help="attention island (runtime.set_attention): cuDNN SDPA between boundary kernels, or the "
                         "fused tcgen05 kernels that read/write INT8 codes directly (bf16 only)")
    ap.add_argument("--nccl-algo", default="auto", choices=["auto", "ring", "tree", "nvls"],
                    help="N>1: NCCL_ALGO for the gradient all-reduce (NVLS = in-switch reduction on "
                         "NVSwitch); reported in the allreduce object")
    ap.add_argument("--variants", type=int, default=1, choices=[0, 1],
                    help="block workloads, 1 GPU: also time the opt-in variants (fast promotion, f16 operands, "
                         "fused attention) and report them in a 'variants' object")
    ap.add_argument("--no-bf16", action="store_true", help="skip the cuBLAS BF16 block baseline")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU oracle baseline")
    ap.add_argument("--cpu-tokens", type=int, default=128, help="token sample for the CPU baseline")
    return ap.parse_args(argv)


# ── distributed plumbing ────────────────────────────────────────────────


def dist_setup(nccl_algo: str = "auto"):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1 and nccl_algo != "auto":
        os.environ["NCCL_ALGO"] = {"ring": "Ring", "tree": "Tree", "nvls": "NVLS"}[nccl_algo]
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    elif torch.cuda.is_available():
        torch.cuda.set_device(0)
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def grad_shapes(wl) -> dict:
    """Name -> shape of the FP32 parameter gradients one step all-reduces."""
    if hasattr(wl, "model"):
        return {k: tuple(p.shape) for k, p in wl.model.params.items()}
    if hasattr(wl, "lin"):
        lin = wl.lin
        return {"w": tuple(lin.master_weight.shape), "b": tuple(lin.bias.shape)}
    blk, out = wl.blk, {}
    for name in ("qkv", "proj", "mlp1", "mlp2"):
        lin = getattr(blk, name)
        out[f"{name}.w"] = tuple(lin.master_weight.shape)
        if lin.bias is not None:
            out[f"{name}.b"] = tuple(lin.bias.shape)
    for name in ("ln1", "ln2"):
        ln = getattr(blk, name)
        out[f"{name}.gamma"] = tuple(ln.gamma.shape)
        out[f"{name}.beta"] = tuple(ln.beta.shape)
    return out


def measure_allreduce(wl, world: int, reps: int = 5) -> dict:
    """Time the step's gradient all-reduce alone (same payload and bucketing as the step:
    paper_2403_12422_b200.dist.allreduce_mean), max over ranks; bus bandwidth = algbw *
    2(n-1)/n (ring all-reduce accounting)."""
    from paper_2403_12422_b200.dist import allreduce_mean

    grads = {k: torch.ones(s, device="cuda") for k, s in grad_shapes(wl).items()}
    nbytes = sum(g.numel() * g.element_size() for g in grads.values())
    allreduce_mean(grads)
    torch.cuda.synchronize()
    barrier(world)
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        allreduce_mean(grads)
    e.record()
    torch.cuda.synchronize()
    ms = max_over_ranks(a.elapsed_time(e) / reps, world)
    algbw = nbytes / (ms / 1e3) / 1e9
    return {"bytes_per_step": nbytes, "ms": round(ms, 4), "algbw_GBps": round(algbw, 1),
            "busbw_GBps": round(algbw * 2 * (world - 1) / world, 1), "world": world,
            "nccl_algo": os.environ.get("NCCL_ALGO", "auto (NCCL's choice)"),
            "how": "FP32 parameter-gradient all-reduce of one step timed alone (NCCL, 64 MiB buckets), "
                   f"CUDA events, mean of {reps}, max over ranks; in the step it overlaps backward"}


# ── clocks sampling during the timed region ─────────────────────────────


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
            time.sleep(0.25)
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        sm, smax, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax = max(smax, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


# ── the INT8 data-flow block (ours) ─────────────────────────────────────


def build_block(jf, w, attn_dtype, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    c, h = w["c"], w["hidden"]

    def lin(d, cc):
        wt = torch.randn((d, cc), generator=g, device="cuda") / float(np.sqrt(cc))
        return jf.QuantLinear(wt, torch.zeros(d, device="cuda"))

    cfg = jf.BlockConfig(c_model=c, heads=w["heads"], hidden=h, block=32, dropout_p=0.0)
    ln = lambda: jf.NormParams(torch.ones(c, device="cuda"), torch.zeros(c, device="cuda"), cfg.eps)  # noqa: E731
    blk = jf.TransformerBlock(cfg, lin(3 * c, c), lin(c, c), lin(h, c), lin(c, h), ln(), ln(),
                              attn_dtype=attn_dtype)
    for lyr in (blk.qkv, blk.proj, blk.mlp1, blk.mlp2):  # INT8 weights built once (dgrad reads W MN-major)
        lyr.weight_q
    return blk


def allreduce_grads(grads: dict, world: int):
    """The DP exchange step: bucketed NCCL all-reduce (mean) of every FP32 parameter gradient."""
    if world == 1:
        return
    from paper_2403_12422_b200.dist import allreduce_mean

    allreduce_mean(grads)


class BlockWorkload:
    """One TransformerBlock fwd+bwd (+ DP all-reduce of its FP32 grads) per step."""

    def __init__(self, jf, w, args, world, rank):
        self.jf, self.w, self.world = jf, w, world
        self.b, self.s, self.c = w["batch"], w["seq"], w["c"]
        self.n = self.b * self.s
        attn_dtype = torch.bfloat16 if args.attn_dtype == "bf16" else torch.float32
        self.blk = build_block(jf, w, attn_dtype, seed=0)
        g = torch.Generator(device="cuda").manual_seed(1000 + rank)
        self.x = torch.randn((self.n, self.c), generator=g, device="cuda")
        self.dy = 0.1 * torch.randn((self.n, self.c), generator=g, device="cuda")
        self.xq = jf.quantize_per_block(self.x)
        self.dyq = jf.quantize_per_block(self.dy)

    def step(self):
        self.blk.forward(self.xq, self.b, self.s)
        if self.world > 1:  # DP: the MLP half's all-reduce overlaps the attention half's backward
            from paper_2403_12422_b200.dist import OverlappedAllReduce

            ov = OverlappedAllReduce()
            dx, grads = self.blk.backward(self.dyq, grad_hook=ov.hook)
            ov.finish(grads)
        else:
            self.blk.backward(self.dyq)

    def e2e_setup(self):
        n, c = self.n, self.c
        self.hx, self.hdy = self.x.cpu().pin_memory(), self.dy.cpu().pin_memory()
        self.hq = torch.empty((n, c), dtype=torch.int8).pin_memory()
        self.hs = torch.empty((n // 32, c // 32), dtype=torch.float32).pin_memory()
        return int(2 * n * c * 4), int(n * c + (n * c // 1024) * 4)

    def e2e_step(self):
        """Host pinned FP32 x, dY in; dX codes + scales out (the public API end to end)."""
        jf, n, c = self.jf, self.n, self.c
        dx_ = torch.empty((n, c), device="cuda")
        dd_ = torch.empty((n, c), device="cuda")
        dx_.copy_(self.hx, non_blocking=True)
        dd_.copy_(self.hdy, non_blocking=True)
        self.blk.forward(jf.quantize_per_block(dx_), self.b, self.s)
        gx, grads = self.blk.backward(jf.quantize_per_block(dd_))
        allreduce_grads(grads, self.world)
        self.hq.copy_(gx.values, non_blocking=True)
        self.hs.copy_(gx.scales, non_blocking=True)

    def e2e_run(self, steps):
        """``steps`` end-to-end steps with the host<->device copies on a copy stream:
        step i+1's x, dY upload (double-buffered) and step i-1's dX download run under
        step i's compute.  Every step still moves its own inputs and result."""
        jf, n, c = self.jf, self.n, self.c
        main = torch.cuda.current_stream()
        cs = getattr(self, "_cs", None) or torch.cuda.Stream()
        self._cs = cs
        bufs = [(torch.empty((n, c), device="cuda"), torch.empty((n, c), device="cuda")) for _ in range(2)]
        free = [torch.cuda.Event(), torch.cuda.Event()]
        ready = [torch.cuda.Event(), torch.cuda.Event()]
        for e in free:
            e.record(main)

        def upload(i):
            bx, bd = bufs[i % 2]
            with torch.cuda.stream(cs):
                cs.wait_event(free[i % 2])
                bx.copy_(self.hx, non_blocking=True)
                bd.copy_(self.hdy, non_blocking=True)
                ready[i % 2].record(cs)

        upload(0)
        keep = []  # results referenced until the copy stream is joined (no record_stream)
        for i in range(steps):
            if i + 1 < steps:
                upload(i + 1)
            bx, bd = bufs[i % 2]
            main.wait_event(ready[i % 2])
            xq, dq = jf.quantize_per_block(bx), jf.quantize_per_block(bd)
            free[i % 2].record(main)
            self.blk.forward(xq, self.b, self.s)
            gx, grads = self.blk.backward(dq)
            allreduce_grads(grads, self.world)
            done = torch.cuda.Event()
            done.record(main)
            with torch.cuda.stream(cs):
                cs.wait_event(done)
                self.hq.copy_(gx.values, non_blocking=True)
                self.hs.copy_(gx.scales, non_blocking=True)
            keep.append(gx)
        main.wait_stream(cs)
        del keep

    def config(self):
        w = self.w
        c, hid, n = self.c, w["hidden"], self.n
        wq = 4 * c * c + 2 * c * hid                 # INT8 weight codes (qkv, proj, mlp1, mlp2)
        act = n * (8 * c + 2 * hid)                  # INT8 activations saved in forward (approx.)
        return {"hidden": self.c, "heads": w["heads"], "mlp_hidden": w["hidden"], "seq_len": self.s,
                "batch_per_gpu": self.b, "tokens_per_gpu": self.n,
                "l2": (f"working set per step: {wq / 1e6:.0f} MB INT8 weights + {4 * wq / 1e6:.0f} MB FP32 weight "
                       f"gradients written + ~{act / 1e6:.0f} MB INT8 activations, larger than the 126 MB L2")}


class LinearWorkload:
    """One QuantLinear fwd + bwd (dgrad, wgrad -> FP32 dW, dbias) per step (BASELINE config 1)."""

    def __init__(self, jf, w, args, world, rank):
        from paper_2403_12422_b200.qlayers import QuantLinear

        self.jf, self.w, self.world = jf, w, world
        self.n, self.c, self.d = w["n"], w["c"], w["d"]
        g = torch.Generator(device="cuda").manual_seed(1000 + rank)
        wm = torch.randn((self.d, self.c), generator=g, device="cuda") * self.c ** -0.5
        self.lin = QuantLinear(wm, torch.zeros(self.d, device="cuda"))
        self.x = torch.randn((self.n, self.c), generator=g, device="cuda")
        self.dy = 0.1 * torch.randn((self.n, self.d), generator=g, device="cuda")
        self.xq = jf.quantize_per_block(self.x)
        self.dyq = jf.quantize_per_block(self.dy)
        self._flush = torch.zeros(64 << 20, dtype=torch.float32, device="cuda")  # 256 MiB > 126 MB L2

    def step(self):
        self._flush.add_(1)  # operands fit in L2: write 256 MiB first so every step starts cold
        self.lin.forward(self.xq)
        _, dw, db = self.lin.backward(self.dyq)
        if self.world > 1:
            allreduce_grads({"w": dw, "b": db}, self.world)

    def e2e_setup(self):
        n, c, d = self.n, self.c, self.d
        self.hx, self.hdy = self.x.cpu().pin_memory(), self.dy.cpu().pin_memory()
        self.hq = torch.empty((n, c), dtype=torch.int8).pin_memory()
        self.hs = torch.empty((n // 32, c // 32), dtype=torch.float32).pin_memory()
        return int(n * c * 4 + n * d * 4), int(n * c + (n * c // 1024) * 4)

    def e2e_step(self):
        """Host pinned FP32 x, dY in; dX codes + scales out."""
        jf = self.jf
        dx_ = torch.empty_like(self.x)
        dd_ = torch.empty_like(self.dy)
        dx_.copy_(self.hx, non_blocking=True)
        dd_.copy_(self.hdy, non_blocking=True)
        self.lin.forward(jf.quantize_per_block(dx_))
        gx, dw, db = self.lin.backward(jf.quantize_per_block(dd_))
        if self.world > 1:
            allreduce_grads({"w": dw, "b": db}, self.world)
        self.hq.copy_(gx.values, non_blocking=True)
        self.hs.copy_(gx.scales, non_blocking=True)

    def e2e_run(self, steps):
        for _ in range(steps):
            self.e2e_step()

    def config(self):
        return {"linear": f"QuantLinear {self.c}->{self.d}", "tokens_per_gpu": self.n,
                "l2": "operands fit in the 126 MB L2: every step first writes a 256 MiB buffer (flush, "
                      "inside the timed step)"}


class ModelWorkload:
    """GPT-2-style pretraining step: embedding, INT8 blocks, BF16 head + FP32 loss,
    backward, DP all-reduce, fused AdamW (paper_2403_12422_b200.model)."""

    def __init__(self, jf, w, args, world, rank):
        from paper_2403_12422_b200.model import AdamW, JetfireLM, ModelConfig

        self.world = world
        self.name = w["model"]
        self.cfg = getattr(ModelConfig, w["model"])()
        self.b, self.s = w["batch"], w["seq"]
        self.n = self.b * self.s
        self.model = JetfireLM(self.cfg, seed=0)
        self.opt = AdamW(self.model, lr=1e-4, weight_decay=0.1)
        g = torch.Generator(device="cuda").manual_seed(1000 + rank)
        self.x = torch.randint(0, self.cfg.vocab, (self.b, self.s), generator=g, device="cuda")
        self.y = torch.roll(self.x, -1, dims=1)
        self.graphed = None
        if world == 1 and args.graph:  # forward + backward replayed from a CUDA graph
            from paper_2403_12422_b200.model import GraphedTrainStep

            self.graphed = GraphedTrainStep(self.model, self.opt, self.b, self.s)

    def step(self, x=None, y=None):
        x = self.x if x is None else x
        y = self.y if y is None else y
        if self.graphed is not None:
            return self.graphed.step(x, y)
        if self.world > 1:  # DP: per-block all-reduce overlapped with the rest of backward
            from paper_2403_12422_b200.dist import OverlappedAllReduce

            ov = OverlappedAllReduce()
            loss, grads = self.model.loss_and_grads(x, y, grad_hook=ov.hook)
            ov.finish(grads)
        else:
            loss, grads = self.model.loss_and_grads(x, y)
        self.opt.step(grads)
        return loss

    def e2e_setup(self):
        self.hx, self.hy = self.x.cpu().pin_memory(), self.y.cpu().pin_memory()
        self.hloss = torch.empty((), dtype=torch.float32).pin_memory()
        return int(2 * self.n * 8), 4

    def e2e_run(self, steps):
        for _ in range(steps):
            self.e2e_step()

    def e2e_step(self):
        """Host pinned token ids in, loss out."""
        x = torch.empty_like(self.x)
        y = torch.empty_like(self.y)
        x.copy_(self.hx, non_blocking=True)
        y.copy_(self.hy, non_blocking=True)
        loss = self.step(x, y)
        self.hloss.copy_(loss, non_blocking=True)

    def config(self):
        c = self.cfg
        return {"model": self.name, "layers": c.layers, "hidden": c.c_model,
                "heads": c.heads, "mlp_hidden": c.hidden, "vocab": c.vocab, "seq_len": self.s,
                "batch_per_gpu": self.b, "tokens_per_gpu": self.n, "head": c.head_dtype + " head, fp32 loss",
                "optimizer": "AdamW (libjetfire, INT8 weight copies rewritten in the same pass)",
                "launch": "forward+backward replayed from one CUDA graph, AdamW eager" if self.graphed
                          else "eager launches",
                "l2": "working set (GBs of weights, grads, Adam state) larger than the 126 MB L2"}


def run_ours(args, world, rank, local):
    import paper_2403_12422_b200 as jf
    from paper_2403_12422_b200 import _lib
    from paper_2403_12422_b200.qgemm import GemmTimer

    jf.require_cuda()
    jf.set_error_check("deferred")
    jf.set_promotion(args.promotion)
    jf.runtime.set_gemm_operands(args.operands)
    jf.runtime.set_attention(args.attention)
    jf.runtime.set_overlap_wgrad(bool(args.overlap_wgrad))
    w = dict(WORKLOADS[args.workload])
    if args.batch:
        w["batch"] = args.batch
    wl = (ModelWorkload if "model" in w else LinearWorkload if "linear" in w else BlockWorkload)(
        jf, w, args, world, rank)
    n = wl.n
    stream = torch.cuda.current_stream()

    for _ in range(args.warmup):
        wl.step()
    jf.check_errors()
    torch.cuda.synchronize()
    barrier(world)

    # ── timed region: K steps, inputs resident in HBM ──
    _lib.launch_count[0] = 0
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # The per-GEMM CUDA events (roofline) are recorded in a separate pass of the same K
    # steps right after the timed region: hundreds of event records per step (GPT-2:
    # 288 GEMMs) make the host the bottleneck and would perturb the measured step.
    with ClockSampler(local) as clocks:
        torch.cuda.synchronize()
        barrier(world)
        start.record(stream)
        for _ in range(args.steps):
            wl.step()
        end.record(stream)
        torch.cuda.synchronize()
        barrier(world)
    launches_total = _lib.launch_count[0]  # libjetfire kernels enqueued in the timed region
    jf.check_errors()
    jf.runtime.set_overlap_wgrad(False)  # kernels timed alone: no side-stream sharing of the SMs
    graphed = getattr(wl, "graphed", None)
    wl.graphed = None                    # (and eagerly: a graph replay has no per-GEMM events)
    with GemmTimer() as gt:
        for _ in range(args.steps):
            wl.step()
    torch.cuda.synchronize()
    wl.graphed = graphed
    jf.runtime.set_overlap_wgrad(bool(args.overlap_wgrad))
    ms = max_over_ranks(start.elapsed_time(end), world)
    ms_step = ms / args.steps
    tokens_per_s = world * n * args.steps / (ms / 1e3)
    gsum = gt.summary()
    gemm_ms_step = gsum["ms"] / args.steps
    gemm_tops = gsum["ops"] / (gsum["ms"] / 1e3) / 1e12

    # ── e2e: host inputs copied in, results read back, every step ──
    h2d, d2h = wl.e2e_setup()
    wl.e2e_run(2)
    torch.cuda.synchronize()
    barrier(world)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    wl.e2e_run(args.steps)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier(world)
    jf.check_errors()
    e2e_ms = max_over_ranks(e0.elapsed_time(e1), world)
    e2e_val = world * n * args.steps / (e2e_ms / 1e3)

    cfg = {"workload": args.workload}
    cfg.update(wl.config())
    cfg.update({"global_tokens": world * n, "block": 32, "promotion": args.promotion, "operands": args.operands,
                "overlap_wgrad": bool(args.overlap_wgrad),
                "attention": ("fused INT8-boundary tcgen05 kernels (bf16)" if args.attention == "fused"
                              else f"torch SDPA ({args.attn_dtype})"),
                "parallelism": f"dp{world}" if world > 1 else "single"})
    out = {
        "metric": METRIC, "value": round(tokens_per_s, 1), "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int8",
        "data": "synthetic (random-init weights; standard-normal activations / 0.1*normal grads, "
                "or uniform random token ids for model workloads)",
        "config": cfg,
        "e2e": {"value": round(e2e_val, 1), "unit": "tokens/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h,
                "copies": "every step uploads its inputs from pinned host memory and downloads its result "
                          "on a copy stream, overlapped with the neighbouring steps' compute"},
        "gpu_launches": int(launches_total), "gpu_launches_per_step": int(launches_total // args.steps),
        "gemm": {"launches_per_step": gsum["launches"] // args.steps, "ms_per_step": round(gemm_ms_step, 4),
                 "tops": round(gemm_tops, 1), "frac_of_int8_peak": round(gemm_tops / INT8_PEAK_TOPS, 4),
                 "share_of_step": round(gemm_ms_step / ms_step, 3),
                 "timing": "CUDA events around every GEMM launch, in a second pass of the same K steps "
                           "without the side-stream overlap (kept out of the timed region: per-launch "
                           "event records load the host)"},
    }
    out["clocks"] = clocks.summary()
    out["roofline"] = roofline(gemm_tops, args.promotion, clocks_mhz=out["clocks"].get("sm_mhz"),
                               operands=args.operands)
    if world > 1:
        out["allreduce"] = measure_allreduce(wl, world)
    if args.variants and world == 1 and isinstance(wl, BlockWorkload):
        out["variants"] = measure_variants(jf, wl, args)
    # (JF_BENCH_ELTWISE=0: skip the side measurement, e.g. for an ncu launch list of the step alone)
    if world == 1 and isinstance(wl, BlockWorkload) and os.environ.get("JF_BENCH_ELTWISE", "1") != "0":
        out["eltwise"] = measure_eltwise(jf, wl)
    return out, wl, None, w


def hbm_peak():
    """HBM denominator: MEASURED_PEAKS.json's copy bandwidth (driver-written), else the
    profiling guide's fallback."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            v = float(json.load(f)["hbm_gbs"])
        return v, "MEASURED_PEAKS.json hbm_gbs (of measured)"
    except (OSError, KeyError, ValueError, TypeError):
        return 6650.0, "B200_PROFILING.md fallback 6.65 TB/s (of fallback; MEASURED_PEAKS.json absent)"


def measure_eltwise(jf, wl, iters=10):
    """The memory-bound kernels at this block's shapes (n tokens x C, n x MLP): device time
    per call from a replayed CUDA graph of `iters` calls (launch overhead excluded), GB/s of
    ALGORITHMIC bytes (int8 codes + s = 4/1024 B of scale per element, + row stats) and the
    fraction of HBM bandwidth.  Inputs (16-64 MB) may stay partly L2-resident across calls."""
    n, c, h = wl.n, wl.c, wl.w["hidden"]
    S = 4.0 / 1024
    peak, src = hbm_peak()
    g = torch.Generator(device="cuda").manual_seed(7)
    x32 = torch.randn((n, c), generator=g, device="cuda")
    a = jf.quantize_per_block(x32)
    b = jf.quantize_per_block(torch.randn((n, c), generator=g, device="cuda"))
    gq = jf.quantize_per_block(torch.randn((n, h), generator=g, device="cuda"))
    dg = jf.quantize_per_block(0.1 * torch.randn((n, h), generator=g, device="cuda"))
    y, st = jf.add_forward(a, b, 64)
    prm = jf.NormParams(torch.ones(c, device="cuda"), torch.zeros(c, device="cuda"))
    _, ctx = jf.layernorm_forward(y, st, prm)

    def timed(fn):
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for _ in range(2):
                fn()
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            for _ in range(iters):
                fn()
        graph.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        graph.replay()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / iters

    rows = [("quantize_f32", c, 5 + S, lambda: jf.quantize_per_block(x32), 0),
            ("add_stats", c, 3 + 3 * S + 0.125, lambda: jf.add_forward(a, b, 64), 0),
            ("ln_fwd", c, 2 + 2 * S + 0.125, lambda: jf.layernorm_forward(y, st, prm), 8 * n),
            ("ln_bwd", c, 3 + 3 * S, lambda: jf.layernorm_backward(ctx, b, prm), 8 * n),
            ("gelu_fwd", h, 2 + 2 * S, lambda: jf.gelu_forward(gq), 0),
            ("gelu_bwd", h, 3 + 3 * S, lambda: jf.gelu_backward(gq, dg), 0),
            ("colsum", h, 1 + S, lambda: jf.column_sum(dg), 0)]
    out = {"hbm_peak_GB_s": peak, "peak_source": src,
           "timing": f"CUDA-graph replay of {iters} calls, device time per call; algorithmic bytes"}
    for name, cols, bpe, fn, extra in rows:
        ms = timed(fn)
        gbs = (n * cols * bpe + extra) / 1e9 / (ms / 1e3)
        out[name] = {"shape": [n, cols], "us": round(ms * 1e3, 2), "GB_s": round(gbs, 1),
                     "frac_hbm": round(gbs / peak, 3)}
    jf.check_errors()
    return out


# Opt-in configurations of the same block step, timed in the same process right after
# the headline (same inputs, CUDA events on the stream, `steps` steps after 2 warm-ups).
VARIANTS = [
    ("fast_promotion", {"promotion": "fast"},
     "acc = fma(P, sa*sb, acc) instead of the reference's fl(acc + fl(fl(P*sa)*sb)); "
     "contract: FP32 rel <= 1e-3 of absmax, codes +-1 on <= 1e-5 (tests/test_gpu_kernels.py)"),
    ("f16_operands", {"operands": "auto"},
     "big GEMMs on kind::f16 over f16-widened codes (bit-identical; 16-bit operand copies in HBM)"),
    ("fast_promotion_f16_operands", {"promotion": "fast", "operands": "auto"}, "both of the above"),
    ("fused_attention", {"attention": "fused"},
     "attention island as the hand-written tcgen05 kernels with the INT8 boundary fused in "
     "(csrc/attn.cu) instead of cuDNN SDPA between boundary kernels"),
]


def measure_variants(jf, wl, args):
    from paper_2403_12422_b200.qgemm import GemmTimer

    rt = jf.runtime
    base = {"promotion": rt.get_promotion(), "operands": rt.gemm_operands(), "attention": rt.attention()}
    setters = {"promotion": jf.set_promotion, "operands": rt.set_gemm_operands, "attention": rt.set_attention}
    res = {}
    stream = torch.cuda.current_stream()
    try:
        for name, knobs, what in VARIANTS:
            for k, v in knobs.items():
                setters[k](v)
            for _ in range(2):
                wl.step()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(args.steps):
                wl.step()
            b.record(stream)
            torch.cuda.synchronize()
            jf.check_errors()
            ms = a.elapsed_time(b) / args.steps
            entry = {"value": round(wl.n / (ms / 1e3), 1), "unit": "tokens/s", "ms_per_step": round(ms, 4),
                     "what": what}
            if "promotion" in knobs or "operands" in knobs:
                rt.set_overlap_wgrad(False)
                with GemmTimer() as gt:
                    for _ in range(args.steps):
                        wl.step()
                torch.cuda.synchronize()
                rt.set_overlap_wgrad(bool(args.overlap_wgrad))
                g = gt.summary()
                tops = g["ops"] / (g["ms"] / 1e3) / 1e12
                entry["gemm_tops"] = round(tops, 1)
                entry["gemm_frac_of_int8_peak"] = round(tops / INT8_PEAK_TOPS, 4)
            res[name] = entry
            for k, v in base.items():
                setters[k](v)
    finally:
        for k, v in base.items():
            setters[k](v)
    return res


def roofline(gemm_tops: float, promotion: str, clocks_mhz=None, operands: str = "int8") -> dict:
    """Dominant kernel = the block GEMM (gemm_tc_kernel<kind::i8> on the default int8 operand path,
    gemm_tc_kernel<kind::f16> with the opt-in --operands auto/f16; ~92% of the step).

    peak: B200 dense INT8 (datasheet 4.5 POPS; our raw kind::i8 microbenchmark
    measures 8178 MAC/clk/SM = 4.76 POPS at 1965 MHz).  The binding bound under
    the reference's per-32-K promotion is the FP32 pipe (exact: 3 FP32 ops per
    output per 32 MACs) or the I2F rate (fast): DESIGN.md section 3.
    """
    mhz = clocks_mhz or 1965.0
    sms = 148
    if promotion == "exact":   # 128 FP32 ops/clk/SM, 3 per element-chunk, 64 int ops per element-chunk
        bound = 128.0 / 3 * 64 * sms * mhz * 1e6 / 1e12
        why = "FP32 pipe: 3 rounded FP32 ops per output element per 32-deep chunk"
    else:                      # I2F 64/clk/SM (ALU, half rate), 64 int ops per element-chunk
        bound = 64.0 * 64 * sms * mhz * 1e6 / 1e12
        why = "int32->fp32 conversion (I2FP, ALU pipe, half rate) per output element per chunk"
    traffic = None
    tr_src = None
    key = "gemm_f16s_kernel" if operands != "int8" else "gemm_i8_kernel"
    try:
        with open(os.path.join(ROOT, "profiles", "roofline_traffic.json")) as f:
            t = json.load(f)[key]
        traffic, tr_src = t["dram_bytes_per_launch"], t["launch"] + " (" + t["source"] + ")"
    except (OSError, KeyError, ValueError):
        pass
    kname = ("gemm_tc_kernel<OP_F16> (tcgen05 kind::f16 on f16-widened int8 codes)" if operands != "int8"
             else "gemm_tc_kernel<OP_I8> (tcgen05 kind::i8)")
    return {"kernel": kname, "bound": "tensor", "achieved": round(gemm_tops, 1),
            "peak": INT8_PEAK_TOPS, "unit": "TFLOP/s", "frac": round(gemm_tops / INT8_PEAK_TOPS, 4),
            "traffic": traffic, "traffic_launch": tr_src,
            "peak_source": "B200 dense INT8 datasheet 4.5 POPS (int ops counted as FLOP); "
                           "MEASURED_PEAKS.json has no INT8 entry",
            "measured_peak": {"value": round(KIND_I8_MEASURED_TOPS, 1), "unit": "TFLOP/s",
                              "frac": round(gemm_tops / KIND_I8_MEASURED_TOPS, 4),
                              "source": "raw tcgen05.mma kind::i8 M128 N128 K32 back to back: 8178 MAC/clk/SM "
                                        "x 148 SMs x 1965 MHz (microbench.cu, profiles/r1e_microbench.jsonl)"},
            "promotion_bound": {"value": round(bound, 1), "unit": "TFLOP/s", "why": why,
                                "frac": round(gemm_tops / bound, 4)}}


# ── cuBLAS BF16 block of the same wiring (context baseline) ─────────────


def bf16_linear_tokens_per_s(w, steps, warmup):
    n, c, d = w["n"], w["c"], w["d"]
    g = torch.Generator(device="cuda").manual_seed(0)
    lin = torch.nn.Linear(c, d, device="cuda", dtype=torch.bfloat16)
    x = torch.randn((n, c), generator=g, device="cuda").to(torch.bfloat16).requires_grad_(True)
    dy = (0.1 * torch.randn((n, d), generator=g, device="cuda")).to(torch.bfloat16)

    def step():
        lin(x).backward(dy)

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        step()
    e.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(e) / steps
    return n / (ms / 1e3), ms


def bf16_block_tokens_per_s(w, steps, warmup):
    import torch.nn.functional as F

    c, h, heads, b, s = w["c"], w["hidden"], w["heads"], w["batch"], w["seq"]
    n = b * s
    dev, dt = "cuda", torch.bfloat16
    g = torch.Generator(device=dev).manual_seed(0)

    def p(*shape, scale=1.0):
        return (torch.randn(shape, generator=g, device=dev) * scale).to(dt).requires_grad_(True)

    P = dict(wqkv=p(3 * c, c, scale=c ** -0.5), bqkv=p(3 * c, scale=0.0), wp=p(c, c, scale=c ** -0.5),
             bp=p(c, scale=0.0), w1=p(h, c, scale=c ** -0.5), b1=p(h, scale=0.0), w2=p(c, h, scale=h ** -0.5),
             b2=p(c, scale=0.0), g1=torch.ones(c, device=dev, dtype=dt, requires_grad=True),
             be1=torch.zeros(c, device=dev, dtype=dt, requires_grad=True),
             g2=torch.ones(c, device=dev, dtype=dt, requires_grad=True),
             be2=torch.zeros(c, device=dev, dtype=dt, requires_grad=True))
    x = torch.randn((n, c), generator=g, device=dev).to(dt).requires_grad_(True)
    dy = (0.1 * torch.randn((n, c), generator=g, device=dev)).to(dt)

    def fwd(x):
        a = F.layer_norm(x, (c,), P["g1"], P["be1"])
        qkv = F.linear(a, P["wqkv"], P["bqkv"]).view(b, s, 3, heads, c // heads)
        q, k, v = (qkv[:, :, i].transpose(1, 2) for i in range(3))
        o = F.scaled_dot_product_attention(q, k, v, is_causal=True).transpose(1, 2).reshape(n, c)
        hh = x + F.linear(o, P["wp"], P["bp"])
        m = F.gelu(F.linear(F.layer_norm(hh, (c,), P["g2"], P["be2"]), P["w1"], P["b1"]), approximate="none")
        return hh + F.linear(m, P["w2"], P["b2"])

    def step():
        out = fwd(x)
        out.backward(dy)

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        step()
    e.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(e)
    return n * steps / (ms / 1e3), ms / steps


def bf16_model_tokens_per_s(w, steps, warmup):
    """GPT-2-style step in standard PyTorch mixed precision: FP32 params, BF16 autocast
    (cuBLAS linears, SDPA, exact-erf GELU, LayerNorm), BF16 head + FP32 CE, fused AdamW."""
    import torch.nn as nn
    import torch.nn.functional as F

    from paper_2403_12422_b200.model import ModelConfig

    cfg = getattr(ModelConfig, w["model"])()
    c, h, heads, b, s = cfg.c_model, cfg.hidden, cfg.heads, w["batch"], w["seq"]
    vp = (cfg.vocab + 127) // 128 * 128

    class Block(nn.Module):
        def __init__(self):
            super().__init__()
            self.ln1, self.ln2 = nn.LayerNorm(c), nn.LayerNorm(c)
            self.qkv, self.proj = nn.Linear(c, 3 * c), nn.Linear(c, c)
            self.mlp1, self.mlp2 = nn.Linear(c, h), nn.Linear(h, c)

        def forward(self, x):
            q, k, v = self.qkv(self.ln1(x)).view(b, s, 3, heads, c // heads).unbind(2)
            o = F.scaled_dot_product_attention(q.transpose(1, 2), k.transpose(1, 2), v.transpose(1, 2),
                                               is_causal=True)
            x = x + self.proj(o.transpose(1, 2).reshape(b, s, c))
            return x + self.mlp2(F.gelu(self.mlp1(self.ln2(x)), approximate="none"))

    class LM(nn.Module):
        def __init__(self):
            super().__init__()
            self.emb, self.wpe = nn.Embedding(vp, c), nn.Embedding(s, c)
            self.blocks = nn.ModuleList([Block() for _ in range(cfg.layers)])
            self.head = nn.Linear(c, vp)

        def forward(self, x, y):
            hh = self.emb(x) + self.wpe.weight[None]
            for blk in self.blocks:
                hh = blk(hh)
            return F.cross_entropy(self.head(hh).float().view(-1, vp), y.view(-1))

    model = LM().cuda()
    opt = torch.optim.AdamW(model.parameters(), lr=1e-4, weight_decay=0.1, fused=True)
    x = torch.randint(0, cfg.vocab, (b, s), device="cuda")
    y = torch.roll(x, -1, dims=1)

    def step():
        with torch.autocast("cuda", dtype=torch.bfloat16):
            loss = model(x, y)
        loss.backward()
        opt.step()
        opt.zero_grad(set_to_none=True)

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        step()
    e.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(e)
    return b * s * steps / (ms / 1e3), ms / steps


# ── CPU oracle (the reference's algorithm, numpy port) ──────────────────


def host_info():
    """What the CPU baseline ran on: CPU model, numpy and its BLAS."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    blas = None
    try:
        cfg = np.show_config(mode="dicts")
        b = cfg["Build Dependencies"]["blas"]
        blas = f"{b.get('name')} {b.get('version')}"
    except Exception:  # noqa: BLE001 -- informational only
        pass
    return {"cpu": model, "logical_cpus": os.cpu_count(), "numpy": np.__version__, "blas": blas}


def cpu_block_sample(w, tokens, reps=1):
    """Time oracle block fwd+bwd on `tokens` tokens of the workload's block dims."""
    from oracle import int8flow_oracle as O

    rng = np.random.default_rng(0)
    c, h, heads = w["c"], w["hidden"], w["heads"]
    seq = min(tokens, w["seq"])
    batch = max(1, tokens // seq)
    p = O.block_weight_cache(O.block_init(rng, c, h))
    xq, xs = O.quantize(rng.standard_normal((batch * seq, c)).astype(np.float32))
    dq, ds = O.quantize((0.1 * rng.standard_normal((batch * seq, c))).astype(np.float32))
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        _, saved = O.block_forward(p, xq, xs, batch, seq, heads)
        O.block_backward(p, saved, dq, ds)
        times.append(time.perf_counter() - t0)
    t = min(times)
    return {"value": round(batch * seq / t, 2), "unit": "tokens/s", "cores": os.cpu_count(), "kind": "port",
            "sample": f"oracle (numpy port of int8flow) block fwd+bwd, {batch}x{seq} tokens at "
                      f"hidden {c}/mlp {h}, OpenBLAS threads = all host cores, best of {reps}",
            "seconds": round(t, 3), "host": host_info()}


def cpu_linear_sample(w, tokens, reps=1):
    """Time the oracle QuantLinear fwd+bwd (qlayers.py:149-181) on `tokens` tokens."""
    from oracle import int8flow_oracle as O

    rng = np.random.default_rng(0)
    c, d = w["c"], w["d"]
    wm = (rng.standard_normal((d, c)) / np.sqrt(c)).astype(np.float32)
    wc = O.quantize(wm)
    bias = np.zeros(d, dtype=np.float32)
    xq, xs = O.quantize(rng.standard_normal((tokens, c)).astype(np.float32))
    dq, ds = O.quantize((0.1 * rng.standard_normal((tokens, d))).astype(np.float32))
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        O.linear_forward(xq, xs, wc, bias)
        O.linear_backward(xq, xs, wc, dq, ds)
        times.append(time.perf_counter() - t0)
    t = min(times)
    return {"value": round(tokens / t, 2), "unit": "tokens/s", "cores": os.cpu_count(), "kind": "port",
            "sample": f"oracle (numpy port of int8flow) QuantLinear {c}->{d} fwd+bwd, {tokens} tokens, "
                      f"OpenBLAS threads = all host cores, best of {reps}",
            "seconds": round(t, 3), "host": host_info()}


REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def _reference_package():
    """The UNMODIFIED reference package installed by tools/install_reference.sh (git-ignored,
    travels to the GPU box), or None.  Never /root/reference: that tree is not on the box."""
    if not os.path.isdir(os.path.join(REF_DIR, "int8flow")):
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    try:
        import int8flow
    except Exception:  # noqa: BLE001 -- fall back to the oracle port
        return None
    return int8flow if os.path.dirname(os.path.dirname(int8flow.__file__)) == REF_DIR else None


def ref_block_sample(ref, w, tokens, reps=1):
    """The reference's own TransformerBlock fwd+bwd (qlayers.py:329-427), its public API."""
    rng = np.random.default_rng(0)
    c, h, heads = w["c"], w["hidden"], w["heads"]
    seq = min(tokens, w["seq"])
    batch = max(1, tokens // seq)
    blk = ref.TransformerBlock.initialize(rng, ref.BlockConfig(c_model=c, heads=heads, hidden=h))
    xq = ref.quantize_per_block(rng.standard_normal((batch * seq, c)).astype(np.float32), 32)
    dq = ref.quantize_per_block((0.1 * rng.standard_normal((batch * seq, c))).astype(np.float32), 32)
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        blk.forward(xq, batch, seq)
        blk.backward(dq)
        times.append(time.perf_counter() - t0)
    t = min(times)
    return {"value": round(batch * seq / t, 2), "unit": "tokens/s", "cores": os.cpu_count(), "kind": "reference",
            "sample": f"unmodified reference int8flow {getattr(ref, '__version__', '')} from baseline/_ref: "
                      f"TransformerBlock fwd+bwd, {batch}x{seq} tokens at hidden {c}/mlp {h}, threads=1 "
                      f"(fastest), OpenBLAS threads = all host cores, best of {reps}",
            "seconds": round(t, 3), "host": host_info()}


def ref_linear_sample(ref, w, tokens, reps=1):
    """The reference's own QuantLinear fwd+bwd (qlayers.py:149-181)."""
    rng = np.random.default_rng(0)
    c, d = w["c"], w["d"]
    lin = ref.QuantLinear.initialize(rng, d, c)
    xq = ref.quantize_per_block(rng.standard_normal((tokens, c)).astype(np.float32), 32)
    dq = ref.quantize_per_block((0.1 * rng.standard_normal((tokens, d))).astype(np.float32), 32)
    times = []
    for _ in range(reps):
        t0 = time.perf_counter()
        lin.forward(xq)
        lin.backward(dq)
        times.append(time.perf_counter() - t0)
    t = min(times)
    return {"value": round(tokens / t, 2), "unit": "tokens/s", "cores": os.cpu_count(), "kind": "reference",
            "sample": f"unmodified reference int8flow from baseline/_ref: QuantLinear {c}->{d} fwd+bwd, "
                      f"{tokens} tokens, OpenBLAS threads = all host cores, best of {reps}",
            "seconds": round(t, 3), "host": host_info()}


def cpu_sample(w, tokens):
    """The reference's own implementation when baseline/_ref holds it (kind 'reference'),
    else the oracle port (kind 'port', bit-identical on the golden fixtures)."""
    ref = _reference_package()
    if "linear" in w:  # the CPU finishes this case quickly: a 1024-token sample (of 4096)
        tokens = max(tokens, 1024)
        return ref_linear_sample(ref, w, tokens) if ref else cpu_linear_sample(w, tokens)
    return ref_block_sample(ref, w, tokens) if ref else cpu_block_sample(w, tokens)


def run_reference(args, world, rank):
    if rank != 0:
        return None
    w = dict(WORKLOADS[args.workload])
    tokens = max(args.cpu_tokens, 1024) if "linear" in w else args.cpu_tokens
    for _ in range(args.warmup):
        cpu_sample(w, tokens)
    vals = [cpu_sample(w, tokens)["value"] for _ in range(args.steps)]
    v = statistics.median(vals)
    cb = cpu_sample(w, tokens)
    cb["value"] = v
    return {"metric": METRIC, "value": v, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(1e3 * tokens / v, 2), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int8", "impl": "reference",
            "data": "synthetic", "config": {"workload": args.workload, "tokens_per_step": tokens,
                                            "parallelism": "cpu"},
            "cpu_baseline": cb, "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                                        "d2h_bytes_per_step": 0}}


def main():
    args = parse()
    world, rank, local = dist_setup(args.nccl_algo)
    if args.impl == "reference":
        out = run_reference(args, world, rank)
        if out is not None:
            print(json.dumps(out), flush=True)
        return
    out, wl, _, w = run_ours(args, world, rank, local)
    if rank == 0:
        if not args.no_bf16 and "model" in w:
            tps, ms = bf16_model_tokens_per_s(w, args.steps, args.warmup)
            out["bf16_baseline"] = {"value": round(tps * world, 1), "unit": "tokens/s", "ms_per_step": round(ms, 4),
                                    "what": "same model in torch BF16 autocast (cuBLAS, SDPA, exact GELU, "
                                            "LayerNorm, fused AdamW), 1 GPU",
                                    "int8_over_bf16": round(out["value"] / (tps * world), 3)}
        if not args.no_bf16 and "model" not in w and "linear" not in w:
            wb = dict(w)
            tps, ms = bf16_block_tokens_per_s(wb, args.steps, args.warmup)
            out["bf16_baseline"] = {"value": round(tps * world, 1), "unit": "tokens/s", "ms_per_step": round(ms, 4),
                                    "what": "same block wiring in torch BF16 (cuBLAS linear, F.layer_norm, "
                                            "exact-erf GELU, SDPA), fwd+bwd autograd, 1 GPU",
                                    "int8_over_bf16": round(out["value"] / (tps * world), 3)}
        if not args.no_bf16 and "linear" in w:
            tps, ms = bf16_linear_tokens_per_s(w, args.steps, args.warmup)
            out["bf16_baseline"] = {"value": round(tps * world, 1), "unit": "tokens/s", "ms_per_step": round(ms, 4),
                                    "what": "torch BF16 nn.Linear fwd+bwd (cuBLAS), same shapes, 1 GPU",
                                    "int8_over_bf16": round(out["value"] / (tps * world), 3)}
        if world == 1 and not args.no_cpu and "model" not in w:
            out["cpu_baseline"] = cpu_sample(w, args.cpu_tokens)
        print(json.dumps(out), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
