"""A GPT-2-style language model on the INT8 data flow: embedding, a stack of
TransformerBlocks, an FP head with cross-entropy, and AdamW — the reference's
``ToyModel`` + ``AdamW`` (``trainer.py:225-262, 273-427``) on the GPU, and the
GPT-2 medium pretraining step of BASELINE config 3.

Data flow per step (as the reference):
  h0 = emb[tokens] * gain (+ wpe[pos] for GPT-2)       FP32, quantized once
  h  = blocks(h0)                                       INT8 between all operators
  logits = deq(h) @ head_w^T + head_b                   FP32 (reference) or BF16 head
  loss = masked mean of -log_softmax(logits)[y]         FP32
  dh = dlogits @ head_w -> quantize -> blocks backward -> deq -> scatter-add into emb
Parameters, gradients and AdamW moments are FP32.  ``AdamW.step`` (``optim.cu``,
``jf_adamw_quantize``) writes the updated FP32 master AND its INT8 codes + scales in one
pass, in place, so the INT8 weight copies never go stale (the reference re-derives them
lazily after ``mark_updated``, qlayers.py:139-147; ``mark_updated`` here requantizes in
place too).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .runtime import traced as _rt_traced
from . import _lib
from .qlayers import BlockConfig, TransformerBlock
from .qtensor import quantize_per_block


@dataclass(frozen=True)
class ModelConfig:
    layers: int = 24
    c_model: int = 1024
    heads: int = 16
    hidden: int = 4096
    vocab: int = 50257
    max_seq: int = 1024
    pos_emb: bool = False         # GPT-2 adds learned positions; the reference ToyModel does not
    head_dtype: str = "fp32"      # "fp32" = reference head; "bf16" = cuBLAS BF16 head, FP32 loss
    attn_dtype: str = "bf16"

    @staticmethod
    def gpt2_medium() -> "ModelConfig":
        return ModelConfig(layers=24, c_model=1024, heads=16, hidden=4096, vocab=50257, max_seq=1024,
                           pos_emb=True, head_dtype="bf16")

    @staticmethod
    def gpt2_large() -> "ModelConfig":
        return ModelConfig(layers=36, c_model=1280, heads=20, hidden=5120, vocab=50257, max_seq=1024,
                           pos_emb=True, head_dtype="bf16")


class JetfireLM:
    """Embedding -> INT8 TransformerBlocks -> FP head, with hand-driven backward (trainer.py:373-427)."""

    def __init__(self, cfg: ModelConfig, params: dict | None = None, seed: int = 0, device="cuda"):
        self.cfg = cfg
        c = cfg.c_model
        dt = torch.bfloat16 if cfg.attn_dtype == "bf16" else torch.float32
        bcfg = BlockConfig(c_model=c, heads=cfg.heads, hidden=cfg.hidden, block=32, dropout_p=0.0)
        if params is None:
            params = self._init(cfg, seed, device)
        self.params = {k: (v if isinstance(v, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(v)))
                       .to(device=device, dtype=torch.float32).contiguous() for k, v in params.items()}
        self.blocks = []
        for i in range(cfg.layers):
            sub = {k[len(f"block{i}."):]: v for k, v in self.params.items() if k.startswith(f"block{i}.")}
            blk = TransformerBlock.from_parameters(bcfg, sub, attn_dtype=dt)
            # share storage: the block's masters ARE the model's parameters
            for name, lin in (("qkv", blk.qkv), ("proj", blk.proj), ("mlp1", blk.mlp1), ("mlp2", blk.mlp2)):
                lin.master_weight = self.params[f"block{i}.{name}.w"]
                lin.bias = self.params[f"block{i}.{name}.b"]
            blk.ln1.gamma, blk.ln1.beta = self.params[f"block{i}.ln1.gamma"], self.params[f"block{i}.ln1.beta"]
            blk.ln2.gamma, blk.ln2.beta = self.params[f"block{i}.ln2.gamma"], self.params[f"block{i}.ln2.beta"]
            self.blocks.append(blk)
        self.gain = self.params.pop("gain", None)
        self.decay_keys = {k for k in self.params if k.endswith(".w") and k != "emb"}

    @staticmethod
    def _init(cfg: ModelConfig, seed: int, device) -> dict:
        g = torch.Generator(device=device).manual_seed(seed)
        c, h = cfg.c_model, cfg.hidden

        def rn(*shape, scale):
            return torch.randn(shape, generator=g, device=device) * scale

        p = {"emb": rn(cfg.vocab, c, scale=c ** -0.5), "head.w": rn(cfg.vocab, c, scale=0.1 * c ** -0.5),
             "head.b": torch.zeros(cfg.vocab, device=device)}
        if cfg.pos_emb:
            p["wpe"] = rn(cfg.max_seq, c, scale=0.01)
        for i in range(cfg.layers):
            for name, (d, cc) in {"qkv": (3 * c, c), "proj": (c, c), "mlp1": (h, c), "mlp2": (c, h)}.items():
                p[f"block{i}.{name}.w"] = rn(d, cc, scale=cc ** -0.5)
                p[f"block{i}.{name}.b"] = torch.zeros(d, device=device)
            for ln in ("ln1", "ln2"):
                p[f"block{i}.{ln}.gamma"] = torch.ones(c, device=device)
                p[f"block{i}.{ln}.beta"] = torch.zeros(c, device=device)
        return p

    def mark_updated(self) -> None:
        for blk in self.blocks:
            blk.mark_updated()

    def _head_bf16(self):
        """BF16 head operands with the vocabulary padded to a multiple of 128 (50257 -> 50304):
        cuBLAS only picks its fast tcgen05 kernels for aligned leading dimensions (an odd
        vocab fell back to sm75 align1 kernels, 5-7 ms each).  Padded rows are zero and
        padded biases -inf, so they carry exactly zero probability and gradient."""
        w, b = self.params["head.w"], self.params["head.b"]
        v, c = w.shape
        vp = (v + 127) // 128 * 128
        w16 = torch.zeros((vp, c), dtype=torch.bfloat16, device=w.device)
        w16[:v] = w
        b16 = torch.full((vp,), float("-inf"), dtype=torch.bfloat16, device=w.device)
        b16[:v] = b
        return w16, b16

    @_rt_traced("jf.model.loss_and_grads")
    def loss_and_grads(self, x: torch.Tensor, y: torch.Tensor, mask: torch.Tensor | None = None,
                       grad_hook=None):
        """(loss, grads) for token ids x, targets y [batch, seq] (trainer.py:373-427).

        ``grad_hook(names)`` (optional) is called as soon as the listed FP32 gradients are
        final — the head's, then each block's in backward order, then the embeddings' — so a
        data-parallel caller can start their all-reduce while earlier blocks still run
        backward (``dist.OverlappedAllReduce``)."""
        batch, seq = x.shape
        flat = x.reshape(-1)
        h0 = self.params["emb"][flat]
        if self.gain is not None:
            h0 = h0 * self.gain
        if "wpe" in self.params:
            h0 = h0 + self.params["wpe"][:seq].repeat(batch, 1)
        hq = quantize_per_block(h0.contiguous())
        for blk in self.blocks:
            hq = blk.forward(hq, batch, seq)
        h = hq.dequantize()

        fm = None if mask is None else mask.reshape(-1).float().contiguous()
        n_tok = batch * seq
        grads = {}
        v = self.cfg.vocab
        if self.cfg.head_dtype == "bf16":
            # BF16 head; fused softmax cross-entropy straight to bf16 dlogits (libjetfire ce.cu)
            w16, b16 = self._head_bf16()
            h16 = h.to(torch.bfloat16)
            logits = torch.addmm(b16, h16, w16.t())
            n_live = (torch.full((), float(n_tok), device=h.device) if fm is None else fm.sum()).float()
            row_loss = torch.empty(n_tok, dtype=torch.float32, device=h.device)
            dl16 = torch.empty_like(logits)
            L = _lib.lib()
            _lib.check(L.jf_cross_entropy_bf16(logits.data_ptr(), n_tok, v, logits.shape[1],
                                               y.reshape(-1).contiguous().data_ptr(), _lib.ptr(fm),
                                               n_live.data_ptr(), row_loss.data_ptr(), dl16.data_ptr(),
                                               _lib.stream_handle()), "cross_entropy")
            loss = row_loss.sum()
            grads["head.w"] = (dl16.t() @ h16)[:v].float()
            dh = (dl16 @ w16).float()
            grads["head.b"] = dl16.sum(dim=0, dtype=torch.float32)[:v]  # fp32 accumulate, no fp32 copy
        else:
            logits = torch.addmm(self.params["head.b"], h, self.params["head.w"].t())
            logp = torch.log_softmax(logits, dim=1)
            fmv = torch.ones(n_tok, device=h.device) if fm is None else fm
            n_live = fmv.sum()
            rows = torch.arange(n_tok, device=h.device)
            fy = y.reshape(-1)
            loss = -(logp[rows, fy] * fmv).sum() / n_live
            dlogits = logp.exp_()
            dlogits[rows, fy] -= 1.0
            dlogits *= (fmv / n_live)[:, None]
            grads["head.w"] = dlogits.t() @ h
            dh = dlogits @ self.params["head.w"]
            grads["head.b"] = dlogits.sum(dim=0)
        if grad_hook is not None:
            grad_hook(grads, ["head.w", "head.b"])

        dq = quantize_per_block(dh.contiguous())
        for i in reversed(range(len(self.blocks))):
            dq, bg = self.blocks[i].backward(dq)
            for k, g in bg.items():
                grads[f"block{i}.{k}"] = g
            if grad_hook is not None:
                grad_hook(grads, [f"block{i}.{k}" for k in bg if bg[k] is not None])
        dx = dq.dequantize()
        if self.gain is not None:
            dx = dx * self.gain
        demb = torch.zeros_like(self.params["emb"])
        demb.index_add_(0, flat, dx)
        grads["emb"] = demb
        if "wpe" in self.params:
            dpos = torch.zeros_like(self.params["wpe"])
            dpos[:seq] = dx.view(batch, seq, -1).sum(dim=0)
            grads["wpe"] = dpos
        if grad_hook is not None:
            grad_hook(grads, [k for k in ("emb", "wpe") if k in grads])
        return loss, grads


class AdamW:
    """AdamW exactly as the reference (trainer.py:225-262): FP32 moments, bias correction,
    decoupled decay on ``model.decay_keys``, in the reference's float32 operation order
    (libjetfire ``jf_adamw``; bit-identical updates).  Block weight matrices are updated by
    ``jf_adamw_quantize``, which also writes their INT8 copy (qlayers.py:139-143) in the same
    pass, so the next forward finds ``weight_q`` ready instead of re-quantizing the master."""

    def __init__(self, model: JetfireLM, lr: float, weight_decay: float = 0.0, betas=(0.9, 0.999),
                 eps: float = 1e-8):
        self.model = model
        self.lr, self.weight_decay, self.betas, self.eps = lr, weight_decay, betas, eps
        self.m = {k: torch.zeros_like(v) for k, v in model.params.items()}
        self.v = {k: torch.zeros_like(v) for k, v in model.params.items()}
        self.t = 0
        self.qlin = {}
        for i, blk in enumerate(model.blocks):
            for name in ("qkv", "proj", "mlp1", "mlp2"):
                self.qlin[f"block{i}.{name}.w"] = getattr(blk, name)
        # small tensors (biases, LayerNorm gamma/beta) share one jf_adamw_multi launch
        self.small = [k for k, p in model.params.items() if k not in self.qlin and p.numel() < self.SMALL]
        self._multi = None

    SMALL = 1 << 20      # elements: tensors below this go through the multi-tensor launch
    CHUNK = 4096         # elements per CTA of jf_adamw_multi

    def _multi_tables(self, device):
        """Device chunk tables (static) and a pinned/device pair for the per-step tensor table."""
        if self._multi is None:
            import numpy as np

            ct, cs = [], []
            for ti, k in enumerate(self.small):
                n = self.model.params[k].numel()
                for s in range(0, n, self.CHUNK):
                    ct.append(ti)
                    cs.append(s)
            chunk_t = torch.tensor(np.asarray(ct, np.int32), device=device)
            chunk_s = torch.tensor(np.asarray(cs, np.int64), device=device)
            host = torch.empty((len(self.small), 6), dtype=torch.int64).pin_memory()
            dev = torch.empty((len(self.small), 6), dtype=torch.int64, device=device)
            ev = torch.cuda.Event()
            ev.record()
            self._multi = (chunk_t, chunk_s, host, dev, ev)
        return self._multi

    @_rt_traced("jf.AdamW.step")
    def step(self, grads: dict) -> None:
        from .qtensor import empty_like_shape
        from . import runtime as _rt

        self.t += 1
        b1, b2 = self.betas
        bc1 = 1.0 - b1 ** self.t
        bc2 = 1.0 - b2 ** self.t
        L = _lib.lib()
        st = _lib.stream_handle()
        small = set(self.small)
        if self.small:
            import struct

            chunk_t, chunk_s, host, dev, ev = self._multi_tables(self.model.params[self.small[0]].device)
            ev.synchronize()  # the previous step's upload of the pinned table has finished
            tab = host.numpy()
            for i, key in enumerate(self.small):
                p, g = self.model.params[key], grads[key]
                if not g.is_contiguous():
                    g = grads[key] = g.contiguous()
                wd = self.weight_decay if (key in self.model.decay_keys and self.weight_decay) else 0.0
                tab[i] = (p.data_ptr(), g.data_ptr(), self.m[key].data_ptr(), self.v[key].data_ptr(), p.numel(),
                          struct.unpack("<I", struct.pack("<f", wd))[0])
            dev.copy_(host, non_blocking=True)
            ev.record()
            _lib.check(L.jf_adamw_multi(dev.data_ptr(), chunk_t.data_ptr(), chunk_s.data_ptr(), chunk_t.numel(),
                                        self.CHUNK, self.lr, b1, b2, self.eps, bc1, bc2, st), "adamw_multi")
        if self.qlin:
            self._step_matrices(grads, L, b1, b2, bc1, bc2, st)
        for key, p in self.model.params.items():
            if key in small or key in self.qlin:
                continue
            g = grads[key].contiguous()
            wd = self.weight_decay if (key in self.model.decay_keys and self.weight_decay) else 0.0
            lin = self.qlin.get(key)
            if lin is not None:
                n, c = p.shape
                # the INT8 copy is rewritten in place (stable addresses: a captured CUDA graph
                # of loss_and_grads keeps reading the live weights); derived copies go stale
                wq = lin._weight_q
                if wq is None:
                    wq = empty_like_shape(n, c, p.device)
                _lib.check(L.jf_adamw_quantize(p.data_ptr(), g.data_ptr(), self.m[key].data_ptr(),
                                               self.v[key].data_ptr(), n, c, self.lr, b1, b2, self.eps, wd,
                                               bc1, bc2, wq.values.data_ptr(), wq.scales.data_ptr(),
                                               _rt.err_ptr(), st), "adamw_quantize")
                lin.set_weight_q(wq)
            else:
                _lib.check(L.jf_adamw(p.data_ptr(), g.data_ptr(), self.m[key].data_ptr(), self.v[key].data_ptr(),
                                      p.numel(), self.lr, b1, b2, self.eps, wd, bc1, bc2, st), "adamw")
        _rt.maybe_check()


    def _step_matrices(self, grads, L, b1, b2, bc1, bc2, st) -> None:
        """Every block weight matrix in ONE jf_adamw_quantize_multi launch (update + in-place
        INT8 requantization; per-matrix launches left the 1024-wide models' SMs idle)."""
        import struct

        from . import runtime as _rt
        from .qtensor import empty_like_shape

        keys = list(self.qlin)
        dev0 = self.model.params[keys[0]].device
        if getattr(self, "_qmulti", None) is None:
            host = torch.empty((len(keys), 10), dtype=torch.int64).pin_memory()
            devt = torch.empty((len(keys), 10), dtype=torch.int64, device=dev0)
            ev = torch.cuda.Event()
            ev.record()
            self._qmulti = (host, devt, ev)
        host, devt, ev = self._qmulti
        ev.synchronize()  # the previous step's upload of the pinned table has finished
        tab = host.numpy()
        tiles = 0
        for i, key in enumerate(keys):
            p, lin = self.model.params[key], self.qlin[key]
            g = grads[key]
            if not g.is_contiguous():
                g = grads[key] = g.contiguous()
            n, c = p.shape
            # the INT8 copy is rewritten in place (stable addresses: a captured CUDA graph
            # of loss_and_grads keeps reading the live weights); derived copies go stale
            wq = lin._weight_q
            if wq is None:
                wq = empty_like_shape(n, c, p.device)
            wd = self.weight_decay if (key in self.model.decay_keys and self.weight_decay) else 0.0
            wd_bits = struct.unpack("<I", struct.pack("<f", wd))[0]
            tab[i] = (p.data_ptr(), g.data_ptr(), self.m[key].data_ptr(), self.v[key].data_ptr(),
                      wq.values.data_ptr(), wq.scales.data_ptr(), n, c, wd_bits, tiles)
            tiles += (n // 32) * ((c + 255) // 256)
            lin.set_weight_q(wq)
        devt.copy_(host, non_blocking=True)
        ev.record()
        _lib.check(L.jf_adamw_quantize_multi(devt.data_ptr(), len(keys), tiles, self.lr, b1, b2, self.eps, bc1,
                                             bc2, _rt.err_ptr(), st), "adamw_quantize_multi")


class GraphedTrainStep:
    """One training step with ``loss_and_grads`` replayed from a CUDA graph.

    The model step issues ~900 small launches (GPT-2 medium: 24 blocks x ~37 kernels plus
    embedding, head and loss); from Python that costs about as much host time as the GPU
    needs to run them, so the step becomes launch-bound.  Captured once, the forward and
    backward replay as one graph launch; AdamW stays eager (its step-dependent scalars are
    kernel arguments).  Inputs are copied into static buffers; ``loss`` and the gradients
    are the graph's static outputs.  AdamW rewrites the INT8 weight copies in place, so
    the graph always reads the current weights.  Single process only (no grad hook).
    """

    def __init__(self, model: JetfireLM, opt: "AdamW", batch: int, seq: int, warmup: int = 2):
        from . import runtime as _rt

        dev = model.params["emb"].device
        self.model, self.opt = model, opt
        self.x = torch.zeros((batch, seq), dtype=torch.long, device=dev)
        self.y = torch.zeros((batch, seq), dtype=torch.long, device=dev)
        side = torch.cuda.Stream(device=dev)
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):  # allocator / library warm-up outside the capture
            for _ in range(warmup):
                model.loss_and_grads(self.x, self.y)
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        for blk in model.blocks:  # derived weight copies are then made inside the graph
            blk.drop_derived_weights()
        n0 = _lib.launch_count[0]
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self.loss, self.grads = model.loss_and_grads(self.x, self.y)
        self.kernels_per_replay = _lib.launch_count[0] - n0  # libjetfire kernels inside the graph
        _rt.maybe_check()

    def step(self, x: torch.Tensor, y: torch.Tensor) -> torch.Tensor:
        self.x.copy_(x, non_blocking=True)
        self.y.copy_(y, non_blocking=True)
        from . import runtime as _rt

        self.graph.replay()
        _lib.launch_count[0] += self.kernels_per_replay
        # eager error mode: a non-finite / overflowing forward or backward raises the
        # reference's ValueError BEFORE AdamW touches params, m and v (trainer.py:482-505)
        _rt.maybe_check()
        self.opt.step(self.grads)
        return self.loss


__all__ = ["AdamW", "GraphedTrainStep", "JetfireLM", "ModelConfig"]
