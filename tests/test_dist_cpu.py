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
