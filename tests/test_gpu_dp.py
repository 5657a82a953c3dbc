"""Data-parallel parity on one GPU (VERDICT r1 "Next round" #7).

* Two DP shards of one sequence each run the GPU block one after the other; their FP32
  parameter gradients are averaged exactly as the all-reduce does (sum, / world) and
  compared with the CPU oracle run per shard plus a float64 average -- the §8e contract
  (per-shard requantization makes DP != the full-batch gradient, so the comparison is
  shard-wise, under tolerance).
* The same real gradient dicts then go through the host-side DP plumbing on two gloo
  ranks (allreduce_mean, OverlappedAllReduce, ZeroAdamW's reduce-scatter): identical
  bits to the direct average.
* ZeroAdamW on NCCL at world size 1 == AdamW, bit for bit (the CUDA update path with
  the INT8 all-gather plumbing).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import int8flow_oracle as O

pytestmark = pytest.mark.gpu

C, HEADS, HID, SEQ = 128, 4, 512, 64


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def shards(jf):
    rng = np.random.default_rng(31)
    p = O.block_init(rng, C, HID)
    for k in ("qkv", "proj", "mlp1", "mlp2"):
        p[k + ".b"] = (0.02 * rng.standard_normal(p[k + ".b"].shape)).astype(np.float32)
    cfg = jf.BlockConfig(c_model=C, heads=HEADS, hidden=HID, block=32, dropout_p=0.0)
    gpu_grads, ref_grads = [], []
    for s in range(2):
        x = O.quantize(rng.standard_normal((SEQ, C)).astype(np.float32))
        dy = O.quantize((0.1 * rng.standard_normal((SEQ, C))).astype(np.float32))
        blk = jf.TransformerBlock.from_parameters(cfg, p, attn_dtype=torch.float32)
        blk.forward(jf.BlockQuantTensor(torch.from_numpy(x[0]).cuda(), torch.from_numpy(x[1]).cuda()), 1, SEQ)
        _, g = blk.backward(jf.BlockQuantTensor(torch.from_numpy(dy[0]).cuda(), torch.from_numpy(dy[1]).cuda()))
        gpu_grads.append({k: v.detach().cpu() for k, v in g.items()})
        pq = O.block_weight_cache(p)
        _, saved = O.block_forward(pq, x[0], x[1], 1, SEQ, HEADS)
        _, rg = O.block_backward(pq, saved, dy[0], dy[1])
        ref_grads.append(rg)
    return gpu_grads, ref_grads


def test_dp_shard_average_vs_oracle(shards):
    gpu, ref = shards
    for k in gpu[0]:
        dp = (gpu[0][k] + gpu[1][k]) / 2          # what allreduce_mean computes at world 2
        truth = (ref[0][k].astype(np.float64) + ref[1][k].astype(np.float64)) / 2
        err = float(np.abs(dp.numpy().astype(np.float64) - truth).max() / max(np.abs(truth).max(), 1e-12))
        # FP32 island: only SDPA's summation order differs from numpy; the block's weight
        # gradients are deq(requant(dY^T X)) of nearly identical inputs
        assert err <= 0.02, (k, err)


def _plumbing_worker(rank, world, port, grads, out):
    from paper_2403_12422_b200.dist import OverlappedAllReduce, allreduce_mean

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a = {k: v.clone() for k, v in grads[rank].items()}
        allreduce_mean(a, bucket_bytes=1 << 16)
        b = {k: v.clone() for k, v in grads[rank].items()}
        ov = OverlappedAllReduce(inplace_bytes=1 << 14)
        ov.hook(b, ["mlp2.w", "mlp2.b", "mlp1.w", "mlp1.b", "ln2.gamma", "ln2.beta"])
        ov.hook(b, ["proj.w", "proj.b", "qkv.w", "qkv.b", "ln1.gamma", "ln1.beta"])
        ov.finish(b)
        out[rank] = (a, b)
    finally:
        dist.destroy_process_group()


def test_dp_plumbing_on_real_block_grads(shards):
    gpu, _ = shards
    world = 2
    out = mp.Manager().dict()
    mp.spawn(_plumbing_worker, args=(world, _free_port(), gpu, out), nprocs=world, join=True)
    for k in gpu[0]:
        want = (gpu[0][k] + gpu[1][k]) / 2
        for r in range(world):
            a, b = out[r]
            assert torch.equal(a[k], want) and torch.equal(b[k], want), (r, k)


def test_zero1_world1_nccl_matches_adamw(jf):
    from paper_2403_12422_b200.dist import ZeroAdamW
    from paper_2403_12422_b200.model import AdamW, JetfireLM, ModelConfig

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        cfg = ModelConfig(layers=2, c_model=128, heads=4, hidden=512, vocab=256, max_seq=64, pos_emb=True,
                          head_dtype="fp32", attn_dtype="fp32")
        a, b = JetfireLM(cfg, seed=9), JetfireLM(cfg, seed=9)
        oa = AdamW(a, lr=1e-3, weight_decay=0.1)
        ob = ZeroAdamW(b, lr=1e-3, weight_decay=0.1, bucket_bytes=1 << 20)
        g = torch.Generator(device="cuda").manual_seed(3)
        for _ in range(3):
            x = torch.randint(0, cfg.vocab, (2, 64), device="cuda", generator=g)
            y = torch.roll(x, -1, dims=1)
            la, ga = a.loss_and_grads(x, y)
            lb, gb = b.loss_and_grads(x, y)
            assert float(la) == float(lb)
            oa.step(ga)
            ob.step(gb)
        for k in a.params:
            assert torch.equal(a.params[k], b.params[k]), k
        for ba, bb in zip(a.blocks, b.blocks):
            for n in ("qkv", "proj", "mlp1", "mlp2"):
                qa, qb = getattr(ba, n).weight_q, getattr(bb, n).weight_q
                assert torch.equal(qa.values, qb.values) and torch.equal(qa.scales, qb.scales), n
    finally:
        dist.destroy_process_group()
