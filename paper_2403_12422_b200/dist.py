"""Data parallelism over the token batch.

Sequences are independent, so each rank runs the INT8 block on its own
whole sequences with no data-path collective.  The single exchange step is
the sum of the FP32 parameter gradients — dequantized dW
(``qlayers.py:181``), dbias, dγ/dβ — all-reduced over NCCL (NVLink /
NVSwitch) in flat buckets and scaled by 1/world.  INT8 codes are never
all-reduced: per-rank block scales differ, so the format is not sum-closed.
The functions are backend-agnostic (NCCL on the GPU box, gloo in the CPU
tests).
"""

from __future__ import annotations

import torch
import torch.distributed as dist

DEFAULT_BUCKET_BYTES = 64 << 20


def shard_sequences(batch: int, rank: int, world: int) -> tuple[int, int]:
    """[start, stop) of this rank's sequences; every rank gets whole sequences."""
    if batch % world:
        raise ValueError(f"batch {batch} does not split over {world} ranks")
    per = batch // world
    return rank * per, (rank + 1) * per


def _buckets(keys, grads, bucket_bytes):
    cur, size = [], 0
    for k in keys:
        nb = grads[k].numel() * grads[k].element_size()
        if cur and size + nb > bucket_bytes:
            yield cur
            cur, size = [], 0
        cur.append(k)
        size += nb
    if cur:
        yield cur


def allreduce_mean(grads: dict, group=None, bucket_bytes: int = DEFAULT_BUCKET_BYTES,
                   async_op: bool = False):
    """Average FP32 parameter gradients over the process group, in place.

    Keys are visited in sorted order so every rank packs identical buckets.
    Gradients that are ``None`` (no bias) are skipped.  With ``async_op``
    the collectives are launched and a list of (work, bucket, flat) is
    returned for ``finish_allreduce``; otherwise the call completes.
    """
    world = dist.get_world_size(group)
    keys = sorted(k for k, v in grads.items() if v is not None)
    for k in keys:
        if grads[k].dtype != torch.float32:
            raise TypeError(f"gradient {k!r} must be float32, got {grads[k].dtype}")
    pending = []
    for bucket in _buckets(keys, grads, bucket_bytes):
        flat = torch.cat([grads[k].reshape(-1) for k in bucket])
        work = dist.all_reduce(flat, group=group, async_op=async_op)
        pending.append((work, bucket, flat))
    if async_op:
        return pending
    _unpack(pending, grads, world)
    return None


def finish_allreduce(pending, grads: dict, group=None) -> None:
    for work, _, _ in pending:
        work.wait()
    _unpack(pending, grads, dist.get_world_size(group))


def _unpack(pending, grads, world):
    for _, bucket, flat in pending:
        flat.div_(world)
        off = 0
        for k in bucket:
            n = grads[k].numel()
            grads[k].copy_(flat[off:off + n].view_as(grads[k]))
            off += n


class OverlappedAllReduce:
    """All-reduce gradients group by group while backward continues.

    Pass ``hook`` as ``JetfireLM.loss_and_grads(..., grad_hook=...)``: each call launches
    async all-reduces of the named FP32 gradients (NCCL runs on its own stream, so the
    transfer overlaps the next block's backward kernels); ``finish(grads)`` waits and
    averages.  Weight gradients (>= ``inplace_bytes``) are reduced in place -- no pack /
    unpack copies of the hundreds of MB per block, and on NCCL the 1/world scaling rides
    in the collective (ReduceOp.AVG); the small vectors (bias, gamma, beta) share one
    packed buffer.  Same sums as ``allreduce_mean``.
    """

    def __init__(self, group=None, inplace_bytes: int = 8 << 20):
        self.group = group
        self.inplace_bytes = inplace_bytes
        self.avg = dist.get_backend(group) == "nccl"
        self.pending = []   # packed buckets (work, names, flat)
        self.inplace = []   # (work, tensor) reduced in place

    def hook(self, grads: dict, names) -> None:
        names = [k for k in names if grads.get(k) is not None]
        small = []
        for k in names:
            g = grads[k]
            if g.numel() * g.element_size() >= self.inplace_bytes and g.is_contiguous():
                op = dist.ReduceOp.AVG if self.avg else dist.ReduceOp.SUM
                self.inplace.append((dist.all_reduce(g, op=op, group=self.group, async_op=True), g))
            else:
                small.append(k)
        if small:
            flat = torch.cat([grads[k].reshape(-1) for k in small])
            work = dist.all_reduce(flat, group=self.group, async_op=True)
            self.pending.append((work, small, flat))

    def finish(self, grads: dict) -> None:
        world = dist.get_world_size(self.group)
        for work, g in self.inplace:
            work.wait()
            if not self.avg:
                g.div_(world)
        for work, _, _ in self.pending:
            work.wait()
        _unpack(self.pending, grads, world)
        self.pending, self.inplace = [], []


__all__ = ["OverlappedAllReduce", "allreduce_mean", "finish_allreduce", "shard_sequences"]
