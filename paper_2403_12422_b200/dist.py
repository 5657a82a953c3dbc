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
    unpack copies of the hundreds of MB per block; the small vectors (bias, gamma, beta)
    share one packed buffer.  Every tensor is summed and then divided by the world size
    (not ReduceOp.AVG, which pre-multiplies by fl(1/world) and so rounds differently for
    world sizes that are not powers of two): the same bits as ``allreduce_mean``.
    """

    def __init__(self, group=None, inplace_bytes: int = 8 << 20):
        self.group = group
        self.inplace_bytes = inplace_bytes
        self.pending = []   # packed buckets (work, names, flat)
        self.inplace = []   # (work, tensor) reduced in place

    def hook(self, grads: dict, names) -> None:
        names = [k for k in names if grads.get(k) is not None]
        small = []
        for k in names:
            g = grads[k]
            if g.numel() * g.element_size() >= self.inplace_bytes and g.is_contiguous():
                self.inplace.append((dist.all_reduce(g, group=self.group, async_op=True), g))
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
            g.div_(world)
        for work, _, _ in self.pending:
            work.wait()
        _unpack(self.pending, grads, world)
        self.pending, self.inplace = [], []


# ── ZeRO stage 1: sharded optimizer state, INT8 weight all-gather ──────────


def _shard_rows(rows: int, world: int, align: int) -> list[tuple[int, int]]:
    """Contiguous row ranges [r0, r1) of a tensor's first dimension, one per rank, each a
    multiple of ``align`` rows long (the last ranks may get fewer or none)."""
    per = -(-rows // world)
    per = -(-per // align) * align
    return [(min(r * per, rows), min((r + 1) * per, rows)) for r in range(world)]


def _reduce_scatter_sum(send: torch.Tensor, out: torch.Tensor, group) -> None:
    """out = sum over ranks of send[rank * len(out):(rank+1) * len(out)] (send = [world * S])."""
    if dist.get_backend(group) == "nccl":
        dist.reduce_scatter_tensor(out, send, group=group)
        return
    dist.all_reduce(send, group=group)  # gloo has no reduce-scatter: same sums, more bytes
    r = dist.get_rank(group)
    out.copy_(send[r * out.numel():(r + 1) * out.numel()])


def _all_gather(mine: torch.Tensor, out: torch.Tensor, group) -> None:
    """out = concat over ranks of every rank's ``mine`` (out = [world * S])."""
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, mine, group=group)
        return
    dist.all_gather(list(out.chunk(dist.get_world_size(group))), mine, group=group)


class ZeroAdamW:
    """ZeRO stage 1 for the DP path: AdamW whose FP32 moments m, v
    are sharded over the data-parallel ranks.

    Per step: (1) the FP32 gradients are REDUCE-SCATTERED (summed, then / world -- the
    same per-element sums ``allreduce_mean`` makes), each rank receiving its row shard of
    every parameter; (2) each rank runs the reference AdamW update (trainer.py:247-262)
    on its shards only -- for the block weight matrices the fused ``jf_adamw_quantize``,
    which also writes the shard's INT8 codes + scales; (3) the updated shards are
    ALL-GATHERED: the INT8 codes + scale grid for the quantized weights (1 + 1/256 B per
    element instead of 4 -- the forward only reads the INT8 copy; their FP32 masters stay
    authoritative on the owning rank, ``gather_masters`` collects them for a checkpoint)
    and FP32 values for everything else.  On the wire: 4 B + ~1 B per quantized weight
    element vs 8 B for all-reduce + local AdamW, and each rank keeps 1/world of m, v.
    Row shards of quantized weights are whole 32-row quantization blocks.

    ``update`` (tests only) replaces the CUDA update kernels:
    ``update(key, p, g, m, v, wd, bc1, bc2, codes, scales)`` on the shard views.
    """

    def __init__(self, model, lr: float, weight_decay: float = 0.0, betas=(0.9, 0.999), eps: float = 1e-8,
                 group=None, bucket_bytes: int = 256 << 20, update=None):
        self.model, self.group = model, group
        self.lr, self.weight_decay, self.betas, self.eps = lr, weight_decay, betas, eps
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.bucket_bytes = bucket_bytes
        self._update = update or self._cuda_update
        self.qlin = {}
        for i, blk in enumerate(getattr(model, "blocks", [])):
            for name in ("qkv", "proj", "mlp1", "mlp2"):
                self.qlin[f"block{i}.{name}.w"] = getattr(blk, name)
        self.keys = sorted(model.params)
        self.ranges = {k: _shard_rows(model.params[k].shape[0] if model.params[k].dim() else 1, self.world,
                                      32 if k in self.qlin else 1) for k in self.keys}
        self.m, self.v = {}, {}
        for k in self.keys:
            r0, r1 = self.ranges[k][self.rank]
            p = model.params[k]
            shape = (r1 - r0,) + tuple(p.shape[1:])
            self.m[k] = torch.zeros(shape, dtype=torch.float32, device=p.device)
            self.v[k] = torch.zeros(shape, dtype=torch.float32, device=p.device)
        self.t = 0

    def _row_elems(self, k) -> int:
        p = self.model.params[k]
        return p[0].numel() if p.dim() > 1 else 1

    def _buckets(self):
        cur, size = [], 0
        for k in self.keys:
            nb = self.model.params[k].numel() * 4
            if cur and size + nb > self.bucket_bytes:
                yield cur
                cur, size = [], 0
            cur.append(k)
            size += nb
        if cur:
            yield cur

    def _cuda_update(self, key, p, g, m, v, wd, bc1, bc2, codes, scales):
        from . import _lib
        from . import runtime as _rt

        L = _lib.lib()
        b1, b2 = self.betas
        if codes is not None:
            n, c = p.shape
            _lib.check(L.jf_adamw_quantize(p.data_ptr(), g.data_ptr(), m.data_ptr(), v.data_ptr(), n, c, self.lr,
                                           b1, b2, self.eps, wd, bc1, bc2, codes.data_ptr(), scales.data_ptr(),
                                           _rt.err_ptr(), _lib.stream_handle()), "adamw_quantize")
        else:
            _lib.check(L.jf_adamw(p.data_ptr(), g.data_ptr(), m.data_ptr(), v.data_ptr(), p.numel(), self.lr, b1,
                                  b2, self.eps, wd, bc1, bc2, _lib.stream_handle()), "adamw")

    def step(self, grads: dict) -> None:
        self.t += 1
        b1, b2 = self.betas
        bc1, bc2 = 1.0 - b1 ** self.t, 1.0 - b2 ** self.t
        decay = getattr(self.model, "decay_keys", set())
        params = self.model.params
        world, rank = self.world, self.rank
        for bucket in self._buckets():
            dev = params[bucket[0]].device
            # (1) reduce-scatter the FP32 gradients: send = [world][S], my shard rows per key
            sizes = [[(self.ranges[k][r][1] - self.ranges[k][r][0]) * self._row_elems(k) for k in bucket]
                     for r in range(world)]
            S = max(sum(z) for z in sizes)
            send = torch.zeros(world * S, dtype=torch.float32, device=dev)
            for r in range(world):
                off = r * S
                for k, z in zip(bucket, sizes[r]):
                    if z:
                        r0, r1 = self.ranges[k][r]
                        send[off:off + z].copy_(grads[k].reshape(grads[k].shape[0] if grads[k].dim() else 1,
                                                                 -1)[r0:r1].reshape(-1))
                    off += z
            mine = torch.empty(S, dtype=torch.float32, device=dev)
            _reduce_scatter_sum(send, mine, self.group)
            mine.div_(world)
            del send
            # (2) AdamW on my shards (codes + scales of quantized weights written in the same pass)
            off = 0
            for k, z in zip(bucket, sizes[rank]):
                if not z:
                    continue
                r0, r1 = self.ranges[k][rank]
                p = params[k]
                ps = p[r0:r1] if p.dim() else p.view(1)
                gs = mine[off:off + z].view(ps.shape)
                wd = self.weight_decay if (k in decay and self.weight_decay) else 0.0
                codes = scales = None
                lin = self.qlin.get(k)
                if lin is not None:
                    wq = lin.weight_q
                    codes, scales = wq.values[r0:r1], wq.scales[r0 // 32:r1 // 32]
                self._update(k, ps, gs, self.m[k], self.v[k], wd, bc1, bc2, codes, scales)
                off += z
            # (3) all-gather the updated shards as bytes: INT8 codes + scales, or FP32 rows
            def pieces(k, r):
                r0, r1 = self.ranges[k][r]
                if r1 <= r0:
                    return []
                lin = self.qlin.get(k)
                if lin is not None:
                    wq = lin.weight_q
                    return [wq.values[r0:r1], wq.scales[r0 // 32:r1 // 32]]
                p = params[k]
                return [p[r0:r1] if p.dim() else p.view(1)]

            nbytes = [sum(t.numel() * t.element_size() for k in bucket for t in pieces(k, r)) for r in range(world)]
            B = -(-max(nbytes) // 16) * 16
            mine_b = torch.zeros(B, dtype=torch.uint8, device=dev)
            off = 0
            for k in bucket:
                for t in pieces(k, rank):
                    nb = t.numel() * t.element_size()
                    mine_b[off:off + nb].copy_(t.contiguous().view(-1).view(torch.uint8))
                    off += nb
            allb = torch.empty(world * B, dtype=torch.uint8, device=dev)
            _all_gather(mine_b, allb, self.group)
            for r in range(world):
                if r == rank:
                    continue
                off = r * B
                for k in bucket:
                    for t in pieces(k, r):
                        nb = t.numel() * t.element_size()
                        t.copy_(allb[off:off + nb].view(t.dtype).view(t.shape))
                        off += nb
            if self.qlin:
                for lin in self.qlin.values():
                    lin.drop_derived()

    def gather_masters(self) -> None:
        """Bring every rank's FP32 masters of the quantized weights up to date (the owners'
        rows; e.g. before a checkpoint)."""
        for k in self.qlin:
            p = self.model.params[k]
            S = max(r1 - r0 for r0, r1 in self.ranges[k]) * p.shape[1]
            mine = torch.zeros(S, dtype=torch.float32, device=p.device)
            r0, r1 = self.ranges[k][self.rank]
            mine[:(r1 - r0) * p.shape[1]].copy_(p[r0:r1].reshape(-1))
            allt = torch.empty(self.world * S, dtype=torch.float32, device=p.device)
            _all_gather(mine, allt, self.group)
            for r, (a0, a1) in enumerate(self.ranges[k]):
                if a1 > a0 and r != self.rank:
                    p[a0:a1].copy_(allt[r * S:r * S + (a1 - a0) * p.shape[1]].view(a1 - a0, p.shape[1]))


__all__ = ["OverlappedAllReduce", "ZeroAdamW", "allreduce_mean", "finish_allreduce", "shard_sequences"]
