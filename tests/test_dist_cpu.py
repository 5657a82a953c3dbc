"""Host logic of the data-parallel path on CPU: world size 2 over gloo."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2403_12422_b200.dist import OverlappedAllReduce, allreduce_mean, finish_allreduce, shard_sequences


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _grads(rank):
    g = torch.Generator().manual_seed(100 + rank)
    return {
        "qkv.w": torch.randn(96, 32, generator=g), "qkv.b": torch.randn(96, generator=g),
        "proj.w": torch.randn(32, 32, generator=g), "proj.b": None,
        "ln1.gamma": torch.randn(32, generator=g), "ln1.beta": torch.randn(32, generator=g),
    }


def _worker(rank, world, port, bucket_bytes, use_async, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        grads = _grads(rank)
        if use_async in ("overlap", "overlap_inplace"):  # groups as a model's backward releases them
            ov = OverlappedAllReduce(inplace_bytes=1 if use_async == "overlap_inplace" else 8 << 20)
            ov.hook(grads, ["qkv.w", "qkv.b"])
            ov.hook(grads, ["proj.w", "proj.b"])
            ov.hook(grads, ["ln1.gamma", "ln1.beta"])
            ov.finish(grads)
        elif use_async:
            finish_allreduce(allreduce_mean(grads, bucket_bytes=bucket_bytes, async_op=True), grads)
        else:
            allreduce_mean(grads, bucket_bytes=bucket_bytes)
        out[rank] = {k: (None if v is None else v.clone()) for k, v in grads.items()}
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("bucket_bytes,use_async", [(64 << 20, False), (512, False), (512, True),
                                                    (0, "overlap"), (0, "overlap_inplace")])
def test_allreduce_mean_world2(bucket_bytes, use_async):
    world = 2
    out = mp.Manager().dict()
    mp.spawn(_worker, args=(world, _free_port(), bucket_bytes, use_async, out), nprocs=world, join=True)
    ref = [_grads(r) for r in range(world)]
    for k, v in ref[0].items():
        if v is None:
            assert out[0][k] is None and out[1][k] is None
            continue
        want = (ref[0][k] + ref[1][k]) / 2
        for r in range(world):
            torch.testing.assert_close(out[r][k], want, rtol=0, atol=1e-6)
        assert torch.equal(out[0][k], out[1][k])  # every rank holds identical bits


def test_shard_sequences():
    assert shard_sequences(8, 0, 2) == (0, 4)
    assert shard_sequences(8, 1, 2) == (4, 8)
    assert shard_sequences(8, 3, 4) == (6, 8)
    with pytest.raises(ValueError, match="does not split"):
        shard_sequences(6, 0, 4)


def test_rejects_non_fp32():
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        with pytest.raises(TypeError, match="float32"):
            allreduce_mean({"w": torch.zeros(4, dtype=torch.float16)})
    finally:
        dist.destroy_process_group()


# ── ZeRO-1 (dist.ZeroAdamW): sharded moments, reduce-scatter + all-gather plumbing ──


def _adamw_ref(p, g, m, v, lr, wd, bc1, bc2, b1=0.9, b2=0.999, eps=1e-8):
    """The reference update (trainer.py:247-262) in torch float32, in place."""
    m.mul_(b1).add_(g * (1 - b1))
    v.mul_(b2).add_(g * g * (1 - b2))
    mhat = m / bc1
    vhat = v / bc2
    if wd:
        p.sub_(lr * wd * p)
    p.sub_(lr * mhat / (torch.sqrt(vhat) + eps))


def _fake_quant(p, codes, scales):
    """Any deterministic function of the master rows stands in for jf_adamw_quantize's codes."""
    codes.copy_(torch.clamp(torch.round(p * 8.0), -127, 127).to(torch.int8))
    scales.copy_(p.reshape(p.shape[0] // 32, 32, p.shape[1] // 32, 32).abs().amax(dim=(1, 3)))


class _Lin:
    def __init__(self, w):
        from types import SimpleNamespace

        self.weight_q = SimpleNamespace(values=torch.zeros(w.shape, dtype=torch.int8),
                                        scales=torch.zeros(w.shape[0] // 32, w.shape[1] // 32))

    def drop_derived(self):
        pass


def _zero_model(seed):
    from types import SimpleNamespace

    g = torch.Generator().manual_seed(seed)
    params = {"block0.qkv.w": torch.randn(96, 64, generator=g), "block0.proj.w": torch.randn(64, 64, generator=g),
              "block0.mlp1.w": torch.randn(160, 64, generator=g), "block0.mlp2.w": torch.randn(64, 160, generator=g),
              "block0.qkv.b": torch.randn(96, generator=g), "block0.ln1.gamma": torch.randn(64, generator=g),
              "emb": torch.randn(37, 64, generator=g), "head.b": torch.randn(37, generator=g)}
    blk = SimpleNamespace(**{n: _Lin(params[f"block0.{n}.w"]) for n in ("qkv", "proj", "mlp1", "mlp2")})
    return SimpleNamespace(params=params, blocks=[blk], decay_keys={k for k in params if k.endswith(".w")})


def _zero_grads(rank, step):
    g = torch.Generator().manual_seed(1000 * step + rank)
    return {k: torch.randn(p.shape, generator=g) for k, p in _zero_model(0).params.items()}


def _zero_worker(rank, world, port, bucket_bytes, out):
    from paper_2403_12422_b200.dist import ZeroAdamW

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        model = _zero_model(0)

        def update(key, p, g, m, v, wd, bc1, bc2, codes, scales):
            _adamw_ref(p, g, m, v, 1e-2, wd, bc1, bc2)
            if codes is not None:
                _fake_quant(p, codes, scales)

        opt = ZeroAdamW(model, lr=1e-2, weight_decay=0.1, bucket_bytes=bucket_bytes, update=update)
        for step in range(2):
            opt.step(_zero_grads(rank, step))
        codes = {f"block0.{n}.w": (getattr(model.blocks[0], n).weight_q.values.clone(),
                                   getattr(model.blocks[0], n).weight_q.scales.clone())
                 for n in ("qkv", "proj", "mlp1", "mlp2")}
        opt.gather_masters()
        out[rank] = ({k: p.clone() for k, p in model.params.items()}, codes,
                     sum(m.numel() for m in opt.m.values()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("bucket_bytes", [256 << 20, 20000])
def test_zero1_world2_matches_full_adamw(bucket_bytes):
    """Two ranks with ZeroAdamW == one process averaging the gradients and running AdamW on
    the full tensors: masters (after gather_masters), INT8 codes/scales of the quantized
    weights and every other parameter identical on both ranks; each rank keeps about half
    of the moments."""
    world = 2
    out = mp.Manager().dict()
    mp.spawn(_zero_worker, args=(world, _free_port(), bucket_bytes, out), nprocs=world, join=True)
    ref = _zero_model(0)
    m = {k: torch.zeros_like(p) for k, p in ref.params.items()}
    v = {k: torch.zeros_like(p) for k, p in ref.params.items()}
    for step in range(2):
        gs = [_zero_grads(r, step) for r in range(world)]
        bc1, bc2 = 1 - 0.9 ** (step + 1), 1 - 0.999 ** (step + 1)
        for k, p in ref.params.items():
            g = (gs[0][k] + gs[1][k]) / world
            _adamw_ref(p, g, m[k], v[k], 1e-2, 0.1 if k in ref.decay_keys else 0.0, bc1, bc2)
    total = sum(p.numel() for p in ref.params.values())
    for r in range(world):
        params, codes, nmom = out[r]
        for k, p in ref.params.items():
            assert torch.equal(params[k], p), (r, k)
        for k, (c, s) in codes.items():
            wc, ws = torch.zeros_like(c), torch.zeros_like(s)
            _fake_quant(ref.params[k], wc, ws)
            assert torch.equal(c, wc) and torch.equal(s, ws), (r, k)
        assert nmom <= 0.6 * total  # ~1/world of m, v (32-row alignment of the quantized weights)
